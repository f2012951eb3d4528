// Microbenchmark: FP64 tensor-core (DMMA via mma.sync) vs SIMT DFMA
// throughput on sm_100a.  Informs the block-mode GEMM design.
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_m8n8k4(double *out, int iters)
{
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[ACC][2];
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}

template <int ACC>
__global__ void dmma_m16n8k16(double *out, int iters)
{
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
    double c[ACC][4];
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.0) out[0] = s;
}

template <int ACC>
__global__ void dfma(double *out, int iters)
{
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-9;
    double c[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i) c[i] = fma(c[i], b, a);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i];
    if (s == 12345.0) out[0] = s;
}

template <typename K>
static void run(const char *name, K kern, int blocks, int threads, int iters,
                double flop_per_iter_per_warp)
{
    double *out;
    cudaMalloc(&out, 8);
    kern<<<blocks, threads>>>(out, 10);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double warps = (double)blocks * threads / 32;
    double tf = warps * iters * flop_per_iter_per_warp / (best * 1e-3) / 1e12;
    printf("{\"kernel\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
           name, blocks, threads, best, tf);
    cudaFree(out);
}

int main()
{
    int sms = 148;
    for (int occ : {1, 2, 4, 8}) {
        run("dmma_m8n8k4_acc4", dmma_m8n8k4<4>, sms * occ, 128, 20000, 4 * 2.0 * 8 * 8 * 4);
        run("dmma_m8n8k4_acc8", dmma_m8n8k4<8>, sms * occ, 128, 10000, 8 * 2.0 * 8 * 8 * 4);
        run("dmma_m16n8k16_acc2", dmma_m16n8k16<2>, sms * occ, 128, 5000, 2 * 2.0 * 16 * 8 * 16);
        run("dmma_m16n8k16_acc4", dmma_m16n8k16<4>, sms * occ, 128, 3000, 4 * 2.0 * 16 * 8 * 16);
        run("dfma_acc8", dfma<8>, sms * occ, 256, 20000, 8 * 2.0 * 32);
    }
    return 0;
}
