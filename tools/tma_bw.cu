// tma_bw.cu -- TMA read throughput of the Gram's operand pattern without the
// math: 64 columns x 64 rows (32 KB) per stage into a 3-stage mbarrier ring,
// 2 CTAs per SM, consumers only wait and release.  Variants:
//   gather4: 64 x cp.async.bulk.tensor.2d.tile::gather4 (4 columns x 16 rows)
//   tile   : 8 x 2D boxes {16 rows, 32 consecutive columns}
// Answers whether k_gram_tma (2.6 TB/s of G) is bound by TMA request rate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bw tools/tma_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int STAGES = 3, STAGE = 32768;

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity)
{
    asm volatile("{\n .reg .pred p;\nW%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}\n" ::"r"(bar),
                 "r"(parity) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(288, 2) k(const __grid_constant__ CUtensorMap tm, int nslot, int ktiles)
{
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char *x = raw + ((1024 - ((unsigned)__cvta_generic_to_shared(raw) & 1023)) & 1023);
    __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned f0 = (unsigned)__cvta_generic_to_shared(full), e0 = (unsigned)__cvta_generic_to_shared(empty);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(f0 + 8 * s));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(e0 + 8 * s));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned xs = (unsigned)__cvta_generic_to_shared(x);
    // items: (slot, k-tile) in stream-K order
    const int items = nslot * ktiles;
    const int per = (items + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * per, i1 = min(items, i0 + per);
    if (warp == 8) {
        for (int i = i0; i < i1; ++i) {
            const int st = (i - i0) % STAGES;
            const unsigned ph = ((i - i0) / STAGES) & 1;
            if (i - i0 >= STAGES) mbar_wait(e0 + 8 * st, ph ^ 1);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(f0 + 8 * st), "r"(STAGE) : "memory");
            __syncwarp();
            const int slot = i / ktiles, kt = i % ktiles;
            if (MODE == 0) {
                for (int op = lane; op < 64; op += 32) {
                    const int q = op / 16, g = op % 16, c = slot * 64 + 4 * g;
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(xs + st * STAGE + q * 8192 + g * 512),
                        "l"(&tm), "r"(kt * 64 + q * 16), "r"(c), "r"(c + 1), "r"(c + 2), "r"(c + 3), "r"(f0 + 8 * st)
                        : "memory");
                }
            } else if (lane < 8) {
                const int q = lane & 3, h = lane >> 2;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3}], [%4];" ::"r"(xs + st * STAGE + q * 8192 + h * 4096),
                    "l"(&tm), "r"(kt * 64 + q * 16), "r"(slot * 64 + h * 32), "r"(f0 + 8 * st)
                    : "memory");
            }
        }
        return;
    }
    for (int i = i0; i < i1; ++i) {
        const int st = (i - i0) % STAGES;
        const unsigned ph = ((i - i0) / STAGES) & 1;
        mbar_wait(f0 + 8 * st, ph);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(e0 + 8 * st) : "memory");
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main()
{
    const int n = 8192, ncols = 8192;
    double *G;
    cudaMalloc(&G, (size_t)n * ncols * 8);
    cudaMemset(G, 0, (size_t)n * ncols * 8);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const int smem = STAGES * STAGE + 1024;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
        for (int l2 = 0; l2 < 2; ++l2) {
            CUtensorMap tm;
            cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)ncols};
            cuuint64_t strides[1] = {(cuuint64_t)n * 8};
            cuuint32_t box[2] = {16, mode == 0 ? 1u : 32u};
            cuuint32_t es[2] = {1, 1};
            CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, G, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r) { printf("encode failed %d\n", (int)r); continue; }
            for (int grid : {296, 444}) {
                float ms = 0;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a);
                    if (mode == 0) k<0><<<grid, 288, smem>>>(tm, ncols / 64, n / 64);
                    else k<1><<<grid, 288, smem>>>(tm, ncols / 64, n / 64);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    cudaEventElapsedTime(&ms, a, b);
                }
                printf("%s l2promo=%d grid %d: %.1f GB/s (%s)\n", mode ? "tile   " : "gather4", l2, grid,
                       (double)n * ncols * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
