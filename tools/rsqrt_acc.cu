// accuracy of fast_rsqrt / fast_rcp / fast_sqrt (hsvd_block_kernels.cuh)
// against the library functions, in ulps, over random operands
#include <cstdio>
#include <cmath>
#include <random>
#include <vector>
#include "hsvd_block_kernels.cuh"
namespace hsvd {
void set_error(const std::string &) {}
int cuda_fail(cudaError_t e, const char *w) { fprintf(stderr, "%s: %s\n", w, cudaGetErrorString(e)); exit(1); }
}
using namespace hsvd;
__global__ void k(const double *x, double *o, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    o[6 * i + 0] = fast_rsqrt(x[i]);
    o[6 * i + 1] = rsqrt(x[i]);
    o[6 * i + 2] = fast_rcp(x[i]);
    o[6 * i + 3] = 1.0 / x[i];
    o[6 * i + 4] = fast_sqrt(x[i]);
    o[6 * i + 5] = sqrt(x[i]);
}
int main()
{
    const int n = 1 << 20;
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(0.5, 4.0);
    std::vector<double> x(n), o(6 * n);
    for (auto &v : x) v = U(rng) * std::pow(2.0, (int)(rng() % 40) - 20);
    double *dx, *dout;
    cudaMalloc(&dx, n * 8); cudaMalloc(&dout, 6 * n * 8);
    cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
    k<<<n / 256, 256>>>(dx, dout, n);
    cudaMemcpy(o.data(), dout, 6 * n * 8, cudaMemcpyDeviceToHost);
    const char *nm[6] = {"fast_rsqrt", "rsqrt", "fast_rcp", "1/x", "fast_sqrt", "sqrt"};
    for (int f = 0; f < 6; ++f) {
        double maxu = 0, sumu = 0; int nz = 0;
        for (int i = 0; i < n; ++i) {
            long double xi = x[i], ref;
            if (f < 2) ref = 1.0L / sqrtl(xi);
            else if (f < 4) ref = 1.0L / xi;
            else ref = sqrtl(xi);
            const double r = (double)ref;
            const double ulp = std::nextafter(std::fabs(r), INFINITY) - std::fabs(r);
            const double u = (double)fabsl((long double)o[6 * i + f] - ref) / ulp;
            maxu = std::fmax(maxu, u); sumu += u; nz += u > 0.5;
        }
        printf("%-11s max %.3f ulp, mean %.3f ulp, %d of %d beyond 0.5 ulp\n", nm[f], maxu, sumu / n, nz, n);
    }
    return 0;
}
