// dmma_chain.cu -- what bounds a k-step of k_gram's consumer loop: DMMA
// chains fed by 64-bit shared-memory fragment loads, as in GramRoles, with
// 16 warps per SM (2 CTAs x 8 warps).  Per variant: ns per k-step per warp
// and the SM's DMMA rate (DMMA.8x8x4 per SM-cycle).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_chain tools/dmma_chain.cu
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// NLD fragment loads and NACC DMMAs per k-step (2x2 register tile when
// NLD = NACC = 4; cross class: NLD = 3, NACC = 2); SMEM = 0: register
// operands only
template <int NLD, int NACC, bool SMEM>
__global__ void __launch_bounds__(256, 2) k(double *out, int iters, long long *cyc)
{
    __shared__ double x[64 * 68];
    for (int i = threadIdx.x; i < 64 * 68; i += blockDim.x) x[i] = 1e-3 * (i % 97);
    __syncthreads();
    const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
    double acc[NACC][2];
#pragma unroll
    for (int q = 0; q < NACC; ++q) acc[q][0] = acc[q][1] = 0.0;
    double rf[NLD];
#pragma unroll
    for (int q = 0; q < NLD; ++q) rf[q] = 1e-3 * (q + lane);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 64; kk += 4) {
            double f[NLD];
#pragma unroll
            for (int q = 0; q < NLD; ++q)
                f[q] = SMEM ? x[(16 * (q % 4) + fr) * 68 + kk + fk + 0 * q] : rf[q];
#pragma unroll
            for (int q = 0; q < NACC; ++q) dmma(acc[q][0], acc[q][1], f[q % NLD], f[(q + 1) % NLD]);
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int q = 0; q < NACC; ++q) s += acc[q][0] + acc[q][1];
    if (s == 1234.5) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int NLD, int NACC, bool SMEM>
void run(const char *name, double *out, long long *dcyc)
{
    const int iters = 200, blocks = 296;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<NLD, NACC, SMEM><<<blocks, 256>>>(out, 10, dcyc);
    cudaEventRecord(a);
    k<NLD, NACC, SMEM><<<blocks, 256>>>(out, iters, dcyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long cyc;
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    const double ksteps = (double)iters * 16;
    const double dmmas = ksteps * NACC * 8 * blocks;  // per launch
    printf("%-28s %6.1f cycles/k-step/warp  %6.3f DMMA/SM-cycle  %5.1f TFLOP/s\n", name,
           cyc / ksteps, dmmas / (cyc * 148.0), dmmas * 512 / (ms * 1e-3) / 1e12);
}

int main()
{
    double *out;
    long long *cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    run<4, 4, true>("lds4 dmma4 (2x2 tile)", out, cyc);
    run<5, 5, true>("lds5 dmma5", out, cyc);
    run<3, 2, true>("lds3 dmma2 (cross)", out, cyc);
    run<4, 4, false>("regs dmma4", out, cyc);
    run<3, 2, false>("regs dmma2", out, cyc);
    run<2, 8, true>("lds2 dmma8", out, cyc);
    run<4, 8, true>("lds4 dmma8", out, cyc);
    return 0;
}
