// tma_gather_probe.cu -- checks the TMA gather4 semantics k_gram relies on:
// a 2D tensor map over column-major G (dim0 = rows, dim1 = columns), box
// {16 rows, 1}, 128-byte swizzle; cp.async.bulk.tensor.2d.tile::gather4
// brings 4 arbitrary columns x 16 consecutive rows into shared memory at a
// 512-byte aligned destination inside a 1024-byte swizzle atom.  Prints
// whether every element landed where the swizzled addressing expects it.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_gather_probe tools/tma_gather_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void probe(const __grid_constant__ CUtensorMap tm, int k0, int4 cols, int dst_off, double *out)
{
    __shared__ __align__(1024) double buf[2048];
    __shared__ __align__(8) unsigned long long bar;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = -1.0;
    __syncthreads();
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned s = (unsigned)__cvta_generic_to_shared((char *)buf + dst_off);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(512));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(s),
            "l"(&tm), "r"(k0), "r"(cols.x), "r"(cols.y), "r"(cols.z), "r"(cols.w), "r"(b)
            : "memory");
    }
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(b));
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[i] = buf[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main()
{
    const int n = 256, ncols = 64;
    double *h = (double *)malloc(sizeof(double) * n * ncols);
    for (int c = 0; c < ncols; ++c)
        for (int r = 0; r < n; ++r) h[c * n + r] = c * 1000 + r;
    double *dG, *dout;
    cudaMalloc(&dG, sizeof(double) * n * ncols);
    cudaMalloc(&dout, sizeof(double) * 2048);
    cudaMemcpy(dG, h, sizeof(double) * n * ncols, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    int ok_all = 1;
    for (int variant = 0; variant < 2; ++variant) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)ncols};
        cuuint64_t strides[1] = {(cuuint64_t)n * 8};
        cuuint32_t box[2] = {16, variant == 0 ? 1u : 4u};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dG, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("variant box {16,%u}: encode %d\n", box[1], (int)r);
        if (r) continue;
        int4 cols = make_int4(5, 9, 2, 33);
        for (int dst_off = 0; dst_off <= 512; dst_off += 512) {
            for (int k0 : {32, 248}) {  // 248: rows 256..263 out of bounds
                cudaMemset(dout, 0, sizeof(double) * 2048);
                probe<<<1, 128>>>(tm, k0, cols, dst_off, dout);
                cudaError_t e = cudaDeviceSynchronize();
                double o[2048];
                cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
                int bad = 0;
                const int cc[4] = {cols.x, cols.y, cols.z, cols.w};
                for (int g = 0; g < 4; ++g)
                    for (int k = 0; k < 16; ++k) {
                        // row g of the gather at byte dst_off + g*128, 16B chunk
                        // (k/2) xor (row index within the 1024B atom)
                        const int row = dst_off / 128 + g;
                        const int byte = row * 128 + (((k >> 1) ^ (row & 7)) << 4) + (k & 1) * 8;
                        const double want = k0 + k < n ? cc[g] * 1000.0 + k0 + k : 0.0;
                        if (o[byte / 8] != want) ++bad;
                    }
                printf("  dst_off %d k0 %d: err=%s mismatches=%d\n", dst_off, k0,
                       cudaGetErrorString(e), bad);
                if (bad || e) ok_all = 0;
            }
        }
    }
    printf(ok_all ? "GATHER4 LAYOUT OK\n" : "GATHER4 LAYOUT MISMATCH\n");
    return 0;
}
