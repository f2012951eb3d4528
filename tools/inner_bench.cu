// Standalone benchmark / trace of the block inner kernel (k_inner) on
// synthetic Gram matrices: nslots slots, one Gram segment each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -Ipaper_1008_1371_b200/csrc tools/inner_bench.cu -o tools/inner_bench
//   tools/inner_bench [nslots] [full] [iters] [jmode]
// It also runs tools/inner_reg_kernel.cuh, an independent register-resident
// implementation of the full-ordering pass (slower: its per-round column
// moves by warp shuffles cost more than k_inner's shared-memory traffic),
// and checks that both produce the same W bit for bit.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "hsvd_block_kernels.cuh"
namespace hsvd {
#include "inner_reg_kernel.cuh"
}

namespace hsvd {
void set_error(const std::string &) {}
int cuda_fail(cudaError_t e, const char *w)
{
    fprintf(stderr, "%s: %s\n", w, cudaGetErrorString(e));
    exit(1);
}
}  // namespace hsvd
using namespace hsvd;

// latency of one rotation_fast / rotation_tc / div / sqrt (dependent chain)
template <int KIND>
__global__ void k_lat(double *out, long long *cyc, double a0)
{
    double x = a0 + threadIdx.x * 1e-3, y = 1.5, z = 0.25;
    const long long t0 = clock64();
    for (int k = 0; k < 256; ++k) {
        double t, c;
        if (KIND == 0) { rotation_fast(x, y, z, -1, t, c); x = 1.0 + t * 0.5 + c; }
        if (KIND == 1) { rotation_fast(x, y, z, 1, t, c); x = 3.0 + t * 0.5 + c; }
        if (KIND == 2) { rotation_tc(x, y, z, -1, t, c); x = 1.0 + t * 0.5 + c; }
        if (KIND == 3) { x = 1.0 + 1.0 / x; }
        if (KIND == 4) { x = 1.0 + sqrt(x); }
        if (KIND == 5) { x = 1.0 + rsqrt(x); }
        if (KIND == 6) { x = fma(x, 0.999, 0.001); }
    }
    const long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = (t1 - t0) / 256;
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main(int argc, char **argv)
{
    constexpr int B2 = 64, b = 32;
    const int nslots = argc > 1 ? atoi(argv[1]) : 128;
    const int full = argc > 2 ? atoi(argv[2]) : 1;
    const int iters = argc > 3 ? atoi(argv[3]) : 20;
    const int jmode = argc > 4 ? atoi(argv[4]) : 0;  // 0: mixed signs, 1: all +1
    const int nseg = argc > 5 ? atoi(argv[5]) : 1;   // Gram segments folded per slot (product: 16)
    const int nb = 2 * nslots, r = nb * b, K = 256;
    std::mt19937_64 rng(1);
    std::normal_distribution<double> N01;
    std::vector<double> A((size_t)nslots * B2 * B2);
    std::vector<double> X((size_t)B2 * K);
    for (int s = 0; s < nslots; ++s) {
        for (auto &v : X) v = N01(rng);
        for (int i = 0; i < B2; ++i)
            for (int j = 0; j < B2; ++j) {
                double acc = 0;
                for (int k = 0; k < K; ++k) acc += X[i * K + k] * X[j * K + k];
                A[(size_t)s * B2 * B2 + i * B2 + j] = acc;
            }
    }
    std::vector<int64_t> js(r), ip(nslots), jp(nslots), ib(nslots), jb(nslots);
    for (int i = 0; i < r; ++i) js[i] = (jmode == 0 && i % 3 == 0) ? -1 : 1;
    for (int k = 0; k < nslots; ++k) { ip[k] = ib[k] = k; jp[k] = jb[k] = nb - 1 - k; }
    double *dA, *dW, *dmaxt;
    int64_t *djs, *dip, *djp, *dib, *djb, *dcur;
    uint8_t *dC, *dts;
    uint32_t *drot, *dskip;
    unsigned long long *derr;
    long long *dtrace;
    CK(cudaMalloc(&dA, A.size() * 8 * nseg));
    CK(cudaMemset(dA, 0, A.size() * 8 * nseg));
    CK(cudaMalloc(&dW, A.size() * 8));
    CK(cudaMalloc(&djs, r * 8));
    CK(cudaMalloc(&dip, nslots * 8)); CK(cudaMalloc(&djp, nslots * 8));
    CK(cudaMalloc(&dib, nslots * 8)); CK(cudaMalloc(&djb, nslots * 8));
    CK(cudaMalloc(&dcur, 2 * nslots * 8));
    CK(cudaMalloc(&dC, nslots)); CK(cudaMalloc(&dts, nslots * kTsetStride));
    CK(cudaMalloc(&drot, nslots * 4)); CK(cudaMalloc(&dskip, nslots * 4));
    CK(cudaMalloc(&dmaxt, nslots * 8));
    CK(cudaMalloc(&derr, 8));
    int64_t *dcolmap, *dcolidx;
    {
        std::vector<int64_t> cm(r);
        for (int i = 0; i < r; ++i) cm[i] = i;
        CK(cudaMalloc(&dcolmap, r * 8));
        CK(cudaMalloc(&dcolidx, (size_t)nslots * B2 * 8));
        CK(cudaMemcpy(dcolmap, cm.data(), r * 8, cudaMemcpyHostToDevice));
    }
    CK(cudaMalloc(&dtrace, 8 * 8 * 64 * 4));
    // slot s's segment 0 holds its Gram, the other segments zeros (same A)
    for (int sl = 0; sl < nslots; ++sl)
        CK(cudaMemcpy(dA + (size_t)sl * nseg * B2 * B2, A.data() + (size_t)sl * B2 * B2,
                      B2 * B2 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(djs, js.data(), r * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(derr, 0xff, 8));
    CK(cudaMemset(dC, 0, nslots)); CK(cudaMemset(drot, 0, nslots * 4));
    CK(cudaMemset(dskip, 0, nslots * 4)); CK(cudaMemset(dmaxt, 0, nslots * 8));
    InnerArgs ia{};
    ia.part.T = 1; ia.part.L = 1; ia.part.NSEG = nseg; ia.part.NS = nslots; ia.part.P = nslots;
    ia.maxseg = nseg; ia.Apart = dA; ia.Wg = dW; ia.jsign = djs;
    ia.ip = dip; ia.jp = djp; ia.iblk = dib; ia.jblk = djb; ia.cur = dcur;
    ia.C = dC; ia.tset = dts; ia.rotk = drot; ia.skipk = dskip; ia.maxt = dmaxt; ia.err = derr;
    ia.nb = nb; ia.slot_base = 0; ia.eps = 0x1p-52; ia.teps = 0x1p-27;
    ia.full = full; ia.use_skip = 1; ia.passes = argc > 6 ? atoi(argv[6]) : 1; ia.trace = nullptr;
    ia.colmap = dcolmap; ia.colidx = dcolidx;
    ia.orig = dcolmap; ia.real_cols = r; ia.skipf = nullptr;
    const size_t smem = sizeof(InnerSmem<B2>), smem_reg = sizeof(InnerRegSmem);
    const size_t smem2 = sizeof(InnerSmem2<B2>);
    CK(cudaFuncSetAttribute(k_inner<B2, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    CK(cudaFuncSetAttribute(k_inner<B2, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    CK(cudaFuncSetAttribute(k_inner_v1<B2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_inner_reg<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_reg));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto reset = [&]() {
        cudaMemcpy(dip, ip.data(), nslots * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(djp, jp.data(), nslots * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dib, ib.data(), nslots * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(djb, jb.data(), nslots * 8, cudaMemcpyHostToDevice);
        cudaMemset(drot, 0, nslots * 4);
        cudaMemset(dskip, 0, nslots * 4);
        cudaMemset(dW, 0, A.size() * 8);
    };
    auto launch = [&](int kind) {
        if (kind == 0 && full) k_inner<B2, true, true><<<nslots, inner2_threads<B2>(), smem2>>>(ia);
        else if (kind == 0) k_inner<B2, true, false><<<nslots, inner2_threads<B2>(), smem2>>>(ia);
        else if (kind == 1) k_inner_v1<B2, true><<<nslots, inner_threads<B2>(), smem>>>(ia);
        else k_inner_reg<true><<<nslots, 256, smem_reg>>>(ia);
    };
    const int rounds = full ? B2 - 1 : b;
    std::vector<double> Wk[3];
    std::vector<uint32_t> rotk[3];
    std::vector<uint8_t> tsk[3];
    for (int kind = 0; kind < (full ? 3 : 2); ++kind) {
        ia.trace = nullptr;
        for (int w = 0; w < 3; ++w) { reset(); launch(kind); }
        CK(cudaDeviceSynchronize());
        float tot = 0;
        for (int i = 0; i < iters; ++i) {
            reset();
            cudaEventRecord(e0);
            launch(kind);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms;
        }
        printf("%s nslots=%d full=%d jmode=%d: %.2f us per launch\n", kind == 2 ? "k_inner_reg" : kind ? "k_inner_v1<64>" : "k_inner<64>",
               nslots, full, jmode, 1e3 * tot / iters);
        Wk[kind].resize(A.size());
        rotk[kind].resize(nslots);
        tsk[kind].resize((size_t)nslots * kTsetStride);
        CK(cudaMemcpy(Wk[kind].data(), dW, A.size() * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(rotk[kind].data(), drot, nslots * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(tsk[kind].data(), dts, tsk[kind].size(), cudaMemcpyDeviceToHost));
        // trace CTA 0: clock64 stamps per round (phase boundaries of each kernel)
        ia.trace = dtrace;
        CK(cudaMemset(dtrace, 0, 8 * 8 * 64 * 4));
        reset();
        launch(kind);
        CK(cudaDeviceSynchronize());
        ia.trace = nullptr;
        std::vector<long long> tr(8 * 64 * 4);
        CK(cudaMemcpy(tr.data(), dtrace, tr.size() * 8, cudaMemcpyDeviceToHost));
        if (kind == 0) {
            // k_inner (leader/bulk): stamps 0 round start, 5 pivots ready,
            // 1 rotation formed, 2 published
            double s05 = 0, s51 = 0, s12 = 0, per = 0;
            for (int it = 0; it < rounds; ++it) {
                long long *t = &tr[8 * it];
                s05 += t[5] - t[0]; s51 += t[1] - t[5]; s12 += t[2] - t[1];
                if (it + 1 < rounds) per += tr[8 * (it + 1)] - t[0];
            }
            printf("  k_inner leader per round: pivots %.0f / rotation %.0f / publish %.0f; period %.0f cycles\n",
                   s05 / rounds, s51 / rounds, s12 / rounds, per / (rounds - 1));
            double s07 = 0, s75 = 0, s26 = 0;
            for (int it = 1; it < rounds; ++it) {
                long long *t = &tr[8 * it];
                s07 += t[7] - t[0]; s75 += t[5] - t[7]; s26 += t[6] - t[2];
            }
            if (ia.passes > 1 && rounds < 64)
                printf("  k_inner pass boundary: round %d start -> pivots %lld cycles (round 1: %lld)\n", rounds,
                       tr[8 * rounds + 5] - tr[8 * rounds], tr[8 * 1 + 5] - tr[8 * 1]);
            printf("  k_inner leader: wait crit %.0f, a_ij + skip test %.0f, after publish %.0f\n",
                   s07 / (rounds - 1), s75 / (rounds - 1), s26 / (rounds - 1));
            double b01 = 0, b12 = 0, b23 = 0, bper = 0;
            for (int it = 1; it < rounds; ++it) {
                long long *t = &tr[1024 + 8 * it];
                b01 += t[1] - t[0]; b12 += t[2] - t[1]; b23 += t[3] - t[2];
                if (it + 1 < rounds) bper += t[8] - t[0];
            }
            printf("  k_inner bulk warp 1 per round: wait R %.0f / wait previous round %.0f / blocks %.0f; period %.0f\n",
                   b01 / (rounds - 1), b12 / (rounds - 1), b23 / (rounds - 1), bper / (rounds - 2));
            printf("  k_inner CTA 0: entry -> prologue done %lld cycles, prologue done -> round 0 %lld\n",
                   tr[8 * 64 + 3] - tr[8 * 64 + 2], tr[0] - tr[8 * 64 + 3]);
            printf("  k_inner CTA 0: leader done %lld cycles after round 0, W replay done %lld, epilogue %lld\n",
                   tr[8 * (rounds - 1) + 2] - tr[0], tr[8 * 64] - tr[0], tr[8 * 64 + 1] - tr[0]);
        } else {
            double sum[4] = {0, 0, 0, 0};
            for (int it = 0; it < rounds; ++it) {
                long long *t = &tr[8 * it];
                sum[0] += t[1] - t[0]; sum[1] += t[2] - t[1]; sum[2] += t[3] - t[2]; sum[3] += t[4] - t[3];
            }
            printf("  avg cycles per round: phases %.0f / %.0f / %.0f / %.0f; total round %.0f\n",
                   sum[0] / rounds, sum[1] / rounds, sum[2] / rounds, sum[3] / rounds,
                   (double)(tr[8 * (rounds - 1) + 4] - tr[0]) / rounds);
        }
    }
    // pairwise comparison of the kernels' W, rotation counts and touched sets
    auto cmp = [&](int x, int y, const char *what) {
        size_t diff = 0, rdiff = 0, tdiff = 0;
        double maxd = 0;
        for (size_t e = 0; e < A.size(); ++e)
            if (Wk[x][e] != Wk[y][e]) {
                ++diff;
                maxd = fmax(maxd, fabs(Wk[x][e] - Wk[y][e]));
            }
        for (int k = 0; k < nslots; ++k) rdiff += rotk[x][k] != rotk[y][k];
        for (size_t e = 0; e < tsk[x].size(); ++e) tdiff += tsk[x][e] != tsk[y][e];
        printf("%s: W entries differing %zu of %zu (max |diff| %.3e), rot counts differing %zu, tset bytes differing %zu\n",
               what, diff, A.size(), maxd, rdiff, tdiff);
    };
    cmp(0, 1, "k_inner vs k_inner_v1");
    if (full) cmp(1, 2, "k_inner_v1 vs k_inner_reg");
    {
        // W J-orthogonality of the new kernel: W^T J_P W = J_P (per slot)
        double worst = 0;
        for (int s = 0; s < nslots; ++s) {
            const double *Wm = &Wk[0][(size_t)s * B2 * B2];  // column-major
            const int64_t I = ib[s] < jb[s] ? ib[s] : jb[s], Jb = ib[s] < jb[s] ? jb[s] : ib[s];
            auto sg = [&](int c) { return (double)js[c < b ? I * b + c : Jb * b + (c - b)]; };
            for (int i = 0; i < B2; ++i)
                for (int j = 0; j < B2; ++j) {
                    double acc = 0;
                    for (int k = 0; k < B2; ++k) acc += Wm[i * B2 + k] * sg(k) * Wm[j * B2 + k];
                    worst = fmax(worst, fabs(acc - (i == j ? sg(i) : 0.0)));
                }
        }
        printf("k_inner: max |W^T J W - J| = %.3e\n", worst);
    }
    {
        double *o; long long *cy, h;
        cudaMalloc(&o, 32 * 8); cudaMalloc(&cy, 8);
        const char *names[] = {"rotation_fast trig", "rotation_fast hyp", "rotation_tc trig", "div", "sqrt", "rsqrt", "dfma"};
#define LAT(K) k_lat<K><<<1, 32>>>(o, cy, 2.0); cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost); printf("latency %-20s %lld cycles\n", names[K], h);
        LAT(0) LAT(1) LAT(2) LAT(3) LAT(4) LAT(5) LAT(6)
    }
    return 0;
}
