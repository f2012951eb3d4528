// gather_bw.cu -- HBM read bandwidth of the Gram's access pattern: every
// CTA streams "k-tiles" = CH contiguous bytes from each of 64 columns that
// lie LD*8 bytes apart (column-major G, n = 8192 rows), versus the same
// bytes read as one contiguous range.  Answers whether the Gram (2.6 TB/s
// of G reads, DMMA at 76 %) is limited by DRAM access granularity.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_bw tools/gather_bw.cu
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void gather(const double *__restrict__ G, long ld, int ncols, int rows, int ch_dbl,
                       int ktiles, double *out)
{
    // CTA c: slot = c % (ncols/64); walks its k-tiles; each k-tile reads
    // ch_dbl doubles from each of the slot's 64 columns
    const int nslot = ncols / 64;
    double acc = 0.0;
    for (int item = blockIdx.x; item < nslot * ktiles; item += gridDim.x) {
        const int slot = item % nslot, kt = item / nslot;
        const long k0 = (long)kt * ch_dbl;
        for (int e = threadIdx.x * 2; e < 64 * ch_dbl; e += blockDim.x * 2) {
            const int c = e / ch_dbl, k = e % ch_dbl;
            const double2 v = *(const double2 *)(G + (long)(slot * 64 + c) * ld + k0 + k);
            acc += v.x + v.y;
        }
    }
    if (acc == 12345.678) out[0] = acc;
}

__global__ void contiguous(const double *__restrict__ G, long total, double *out)
{
    double acc = 0.0;
    for (long e = (blockIdx.x * (long)blockDim.x + threadIdx.x) * 2; e < total;
         e += (long)gridDim.x * blockDim.x * 2) {
        const double2 v = *(const double2 *)(G + e);
        acc += v.x + v.y;
    }
    if (acc == 12345.678) out[0] = acc;
}

int main()
{
    const int n = 8192, ncols = 8192;
    const long bytes = (long)n * ncols * 8;
    double *G, *out;
    cudaMalloc(&G, bytes);
    cudaMalloc(&out, 8);
    cudaMemset(G, 0, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        contiguous<<<148 * 8, 256>>>(G, (long)n * ncols, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("contiguous            %7.1f GB/s\n", bytes / ms / 1e6);
    }
    for (int ch : {32, 64, 128, 256, 512}) {
        for (int grid : {296, 592, 1184}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                gather<<<grid, 256>>>(G, n, ncols, n, ch, n / ch, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                if (rep)
                    printf("gather %4d B/column  grid %5d  %7.1f GB/s\n", ch * 8, grid,
                           bytes / ms / 1e6);
            }
        }
    }
    return 0;
}
