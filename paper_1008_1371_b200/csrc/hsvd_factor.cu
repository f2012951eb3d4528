// hsvd_factor.cu -- eigen-pipeline front end on the GPU: the complete-
// pivoting Bunch-Parlett factorization M = G J G^T in double-double
// (hjsvd.factory.bunch_parlett_factor, factory.py:136-282).
//
// Compiled with -fmad=false: every double-double primitive below is the
// reference's (_dd.py:25-93, Dekker's split, no FMA), evaluated with one
// rounding per operation, so the factor, the signs and the permutation are
// bit-identical to the reference's (tests/test_gpu_factor.py).
//
// Layout in HBM (n x n, row-major; M is exactly symmetric, so the storage
// order of the input does not matter):
//   Ah, Al  the trailing matrix (hi, lo): its upper triangle (the matrix
//           stays exactly symmetric, so the lower one is never needed)
//   Lh, Ll  the unit lower factor, rows permuted with the pivots
//   vectors of the current pivot (multipliers and pivot columns), the
//   pivot-search partials, the block records and a device-side state.
//
// One pivot step is two kernels and no host round trip:
//   k_bp_pivot   (one CTA)  reduces the search partials, takes the 1x1 or
//                2x2 decision, swaps rows/columns, forms the multipliers;
//   k_bp_update  (upper-triangle 64x64 tiles) applies the rank-1/2 update
//                and the symmetrization to the new trailing block and
//                searches the updated block for the next pivot (per-tile
//                partial maxima).
// The trailing update is HBM-bound: 16 B read + 16 B written per element of
// the upper triangle (the symmetrized value of (i, j) needs only A_ij = A_ji
// and the pivot vectors).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <stdlib.h>
#include <string.h>

#include "hsvd_internal.cuh"

namespace hsvd {
namespace {

struct dd {
    double h, l;
};

// ---- _dd.py:25-93 ----------------------------------------------------------
__device__ __forceinline__ dd two_sum(double a, double b)
{
    const double s = __dadd_rn(a, b), bb = __dsub_rn(s, a);
    return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b)
{
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ void split(double a, double &hi, double &lo)
{
    const double t = __dmul_rn(134217729.0, a);
    hi = __dsub_rn(t, __dsub_rn(t, a));
    lo = __dsub_rn(a, hi);
}
__device__ __forceinline__ dd two_prod(double a, double b)
{
    const double p = __dmul_rn(a, b);
    double ah, al, bh, bl;
    split(a, ah, al);
    split(b, bh, bl);
    const double e = __dadd_rn(__dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(ah, bh), p), __dmul_rn(ah, bl)),
                                         __dmul_rn(al, bh)),
                               __dmul_rn(al, bl));
    return {p, e};
}
__device__ __forceinline__ dd dd_add(dd x, dd y)
{
    const dd s = two_sum(x.h, y.h);
    return quick_two_sum(s.h, __dadd_rn(s.l, __dadd_rn(x.l, y.l)));
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.h, -x.l}; }
__device__ __forceinline__ dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
__device__ __forceinline__ dd dd_mul(dd x, dd y)
{
    const dd p = two_prod(x.h, y.h);
    return quick_two_sum(p.h, __dadd_rn(p.l, __dadd_rn(__dmul_rn(x.h, y.l), __dmul_rn(x.l, y.h))));
}
// dd_mul with the Dekker splits of x.h and y.h supplied (the same operations:
// the update kernel splits each row's and column's pivot vectors once)
struct sp2 {
    double h, l;
};
__device__ __forceinline__ sp2 split2(double a)
{
    sp2 r;
    split(a, r.h, r.l);
    return r;
}
__device__ __forceinline__ dd dd_mul_s(dd x, sp2 xs, dd y, sp2 ys)
{
    const double p = __dmul_rn(x.h, y.h);
    const double e = __dadd_rn(__dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(xs.h, ys.h), p), __dmul_rn(xs.h, ys.l)),
                                         __dmul_rn(xs.l, ys.h)),
                               __dmul_rn(xs.l, ys.l));
    return quick_two_sum(p, __dadd_rn(e, __dadd_rn(__dmul_rn(x.h, y.l), __dmul_rn(x.l, y.h))));
}
__device__ __forceinline__ dd dd_mul_f(dd x, double f)
{
    const dd p = two_prod(x.h, f);
    return quick_two_sum(p.h, __dadd_rn(p.l, __dmul_rn(x.l, f)));
}
__device__ __forceinline__ dd dd_div(dd x, dd y)
{
    const double q1 = __ddiv_rn(x.h, y.h);
    const dd r = dd_sub(x, dd_mul_f(y, q1));
    const double q2 = __ddiv_rn(__dadd_rn(r.h, r.l), y.h);
    return quick_two_sum(q1, q2);
}
__device__ __forceinline__ dd dd_sqrt(dd x)
{
    const double r = __dsqrt_rn(x.h);
    const dd rr = two_prod(r, r);
    const dd diff = dd_sub(x, rr);
    const double corr = r > 0.0 ? __ddiv_rn(__dadd_rn(diff.h, diff.l), __dmul_rn(2.0, r)) : 0.0;
    return quick_two_sum(r, corr);
}
__device__ __forceinline__ dd dd_abs(dd x) { return x.h < 0.0 ? dd_neg(x) : x; }

// ---- device state and workspace ------------------------------------------
struct BpState {
    int64_t k;       // first row/column of the trailing block
    int64_t nb;      // blocks recorded
    int64_t kind;    // size of the pivot taken by the last k_bp_pivot (0: none)
    int64_t status;  // 0, or 3 = numerical singularity
    int64_t stage;   // k at the singularity
    int64_t p;       // number of +1 signs (after post-processing)
};
struct Cand {
    double v;
    int64_t i;
};
__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi)
{
    return v > bv || (v == bv && i < bi);
}

constexpr int TB = 64;          // update tile
constexpr int UPD_THREADS = 256;
constexpr int PIV_THREADS = 512;

struct BpWs {
    double *Ah, *Al, *Lh, *Ll;
    double *v0h, *v0l, *v1h, *v1l;  // pivot columns c / W0, W1
    double *l0h, *l0l, *l1h, *l1l;  // multipliers l / l0, l1
    Cand *poff, *pdiag;             // per-tile search partials
    int64_t *bcol, *bsz;
    dd *bd;                         // 3 per block
    dd *bp;                         // post-processing parameters, 4 per block
    int8_t *sg;                     // signs in pivot order
    int64_t *ocol;                  // output column of each pivot column
    BpState *st;
};

__host__ __device__ inline int64_t tiles_of(int64_t m) { return (m + TB - 1) / TB; }
__host__ __device__ inline int64_t tri_count(int64_t m)
{
    const int64_t T = tiles_of(m);
    return T * (T + 1) / 2;
}
// linear upper-triangle tile index -> (I, J), I <= J (column-major over J)
__device__ __forceinline__ void tri_tile(int64_t idx, int &I, int &J)
{
    int j = (int)((sqrt(8.0 * (double)idx + 1.0) - 1.0) * 0.5);
    while ((int64_t)(j + 1) * (j + 2) / 2 <= idx) ++j;
    while ((int64_t)j * (j + 1) / 2 > idx) --j;
    J = j;
    I = (int)(idx - (int64_t)j * (j + 1) / 2);
}

template <int NT>
__device__ void block_argmax(double &v, int64_t &i, double &v2, int64_t &i2)
{
    // two independent (value, index) maxima over the CTA; result in thread 0
    __shared__ double sv[NT / 32], sv2[NT / 32];
    __shared__ int64_t si[NT / 32], si2[NT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, v, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, i, o);
        const double ov2 = __shfl_down_sync(0xffffffffu, v2, o);
        const int64_t oi2 = __shfl_down_sync(0xffffffffu, i2, o);
        if (better(ov, oi, v, i)) { v = ov; i = oi; }
        if (better(ov2, oi2, v2, i2)) { v2 = ov2; i2 = oi2; }
    }
    if (lane == 0) { sv[w] = v; si[w] = i; sv2[w] = v2; si2[w] = i2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < NT / 32; ++k) {
            if (better(sv[k], si[k], v, i)) { v = sv[k]; i = si[k]; }
            if (better(sv2[k], si2[k], v2, i2)) { v2 = sv2[k]; i2 = si2[k]; }
        }
    }
    __syncthreads();
}

// ---- setup ---------------------------------------------------------------------
__global__ void k_bp_init(const double *M, const double *Mlo, int64_t ldm, int64_t n, BpWs w)
{
    const int64_t N = n * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e % n;
        w.Ah[e] = M[i * ldm + j];
        w.Al[e] = Mlo ? Mlo[i * ldm + j] : 0.0;
        w.Lh[e] = i == j ? 1.0 : 0.0;
        w.Ll[e] = 0.0;
    }
}
__global__ void k_bp_init_state(int64_t n, BpWs w, int64_t *perm)
{
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
    if (threadIdx.x == 0) *w.st = BpState{0, 0, 0, 0, 0, 0};
}

// pivot search of the whole matrix (step 0); per-tile partials
__global__ void __launch_bounds__(UPD_THREADS) k_bp_search(int64_t n, BpWs w)
{
    const int64_t m = n;
    if (blockIdx.x >= tri_count(m)) return;
    int I, J;
    tri_tile(blockIdx.x, I, J);
    const int tx = threadIdx.x % TB, ty = threadIdx.x / TB;
    double bo = -1.0, bd = -1.0;
    int64_t io = 0, id = 0;
    const int64_t c = (int64_t)J * TB + tx;
    for (int r0 = ty; r0 < TB; r0 += UPD_THREADS / TB) {
        const int64_t r = (int64_t)I * TB + r0;
        if (r >= m || c >= m) continue;
        const double v = fabs(w.Ah[r * n + c]);
        if (r < c) {
            if (better(v, r * m + c, bo, io)) { bo = v; io = r * m + c; }
        } else if (r == c) {
            if (better(v, r, bd, id)) { bd = v; id = r; }
        }
    }
    block_argmax<UPD_THREADS>(bo, io, bd, id);
    if (threadIdx.x == 0) {
        w.poff[blockIdx.x] = Cand{bo, io};
        w.pdiag[blockIdx.x] = Cand{bd, id};
    }
}

// symmetric swap of rows/columns a and b inside the trailing block [k:]
// (_swap_sym, factory.py:117-121) plus the rows of L left of k and perm
// swap X[a-th and b-th elements] of cnt strided pairs, hi and lo: all loads
// of a chunk are issued before its stores (memory-level parallelism)
__device__ __forceinline__ void swap_pairs(double *H, double *Lo, int64_t pa, int64_t pb,
                                           int64_t stride, int64_t cnt)
{
    constexpr int U = 8;
    for (int64_t e0 = threadIdx.x; e0 < cnt; e0 += U * (int64_t)blockDim.x) {
        double xh[U], yh[U], xl[U], yl[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + u * (int64_t)blockDim.x;
            if (e < cnt) {
                xh[u] = H[pa + e * stride]; yh[u] = H[pb + e * stride];
                xl[u] = Lo[pa + e * stride]; yl[u] = Lo[pb + e * stride];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + u * (int64_t)blockDim.x;
            if (e < cnt) {
                H[pa + e * stride] = yh[u]; H[pb + e * stride] = xh[u];
                Lo[pa + e * stride] = yl[u]; Lo[pb + e * stride] = xl[u];
            }
        }
    }
}

// symmetric swap of rows/columns a and b inside the trailing block [k:]
// (_swap_sym, factory.py:117-121) plus the rows of L left of k and perm
__device__ void sym_swap(BpWs &w, int64_t *perm, int64_t n, int64_t k, int64_t a, int64_t b)
{
    // only the upper triangle (row <= column) of the trailing block is kept:
    // P A P with P = (a b), a < b, moves U(r, a) <-> U(r, b) for r != a, b
    // and U(a, a) <-> U(b, b); U(a, b) stays (the reference's row swap then
    // column swap moves the same values)
    constexpr int U = 8;
    const int64_t cnt = n - k;
    for (int64_t e0 = threadIdx.x; e0 < cnt; e0 += U * (int64_t)blockDim.x) {
        int64_t pa[U], pb[U];
        double xh[U], yh[U], xl[U], yl[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = k + e0 + u * (int64_t)blockDim.x;
            pa[u] = -1;
            if (r < n && r != b) {
                if (r == a) {  // the diagonal pair
                    pa[u] = a * n + a;
                    pb[u] = b * n + b;
                } else {
                    pa[u] = r < a ? r * n + a : a * n + r;
                    pb[u] = r < b ? r * n + b : b * n + r;
                }
                xh[u] = w.Ah[pa[u]]; yh[u] = w.Ah[pb[u]];
                xl[u] = w.Al[pa[u]]; yl[u] = w.Al[pb[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (pa[u] < 0) continue;
            w.Ah[pa[u]] = yh[u]; w.Ah[pb[u]] = xh[u];
            w.Al[pa[u]] = yl[u]; w.Al[pb[u]] = xl[u];
        }
    }
    swap_pairs(w.Lh, w.Ll, a * n, b * n, 1, k);  // rows of L left of k
    if (threadIdx.x == 0) {
        const int64_t t = perm[a];
        perm[a] = perm[b];
        perm[b] = t;
    }
    __syncthreads();
}

// ---- one pivot decision (factory.py:153-232 up to the update) -------------
__global__ void __launch_bounds__(PIV_THREADS) k_bp_pivot(int64_t n, double thresh, double alpha,
                                                          BpWs w, int64_t *perm)
{
    __shared__ BpState S;
    __shared__ int64_t sh_i0, sh_off;
    __shared__ double sh_mu0, sh_mu1;
    if (threadIdx.x == 0) S = *w.st;
    __syncthreads();
    if (S.status != 0 || S.k >= n) {
        if (threadIdx.x == 0) w.st->kind = 0;
        return;
    }
    const int64_t k = S.k, m = n - k, cnt = tri_count(m);
    // reduce the search partials of the trailing block
    double bo = -1.0, bd = -1.0;
    int64_t io = 0, id = 0;
    {
        constexpr int U = 8;  // loads of a chunk issued before its comparisons
        for (int64_t e0 = threadIdx.x; e0 < cnt; e0 += U * (int64_t)blockDim.x) {
            Cand o[U], d[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t e = e0 + u * (int64_t)blockDim.x;
                if (e < cnt) {
                    o[u] = w.poff[e];
                    d[u] = w.pdiag[e];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (e0 + u * (int64_t)blockDim.x >= cnt) break;
                if (better(o[u].v, o[u].i, bo, io)) { bo = o[u].v; io = o[u].i; }
                if (better(d[u].v, d[u].i, bd, id)) { bd = d[u].v; id = d[u].i; }
            }
        }
    }
    block_argmax<PIV_THREADS>(bo, io, bd, id);
    if (threadIdx.x == 0) {
        // no off-diagonal candidate (m == 1): mu1 = 0 (numpy: argmax of zeros)
        sh_mu1 = bo < 0.0 ? 0.0 : bo;
        sh_off = bo < 0.0 ? 0 : io;
        sh_mu0 = bd;
        sh_i0 = id;
    }
    __syncthreads();
    const double mu0 = sh_mu0, mu1 = sh_mu1;
    if (!(fmax(mu0, mu1) > thresh)) {
        if (threadIdx.x == 0) {
            w.st->status = 3;
            w.st->stage = k;
            w.st->kind = 0;
        }
        return;
    }
    const bool one = m == 1 || mu0 >= alpha * mu1;
    if (one) {
        if (sh_i0 != 0) sym_swap(w, perm, n, k, k, k + sh_i0);
        const dd d = {w.Ah[k * n + k], w.Al[k * n + k]};
        constexpr int U = 4;
        for (int64_t i0 = k + 1 + threadIdx.x; i0 < n; i0 += U * (int64_t)blockDim.x) {
            dd c[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = i0 + u * (int64_t)blockDim.x;
                if (i < n) c[u] = dd{w.Ah[k * n + i], w.Al[k * n + i]};  // A[i][k] = A[k][i]
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = i0 + u * (int64_t)blockDim.x;
                if (i >= n) continue;
                const dd l = dd_div(c[u], d);
                w.Lh[i * n + k] = l.h;
                w.Ll[i * n + k] = l.l;
                w.v0h[i] = c[u].h; w.v0l[i] = c[u].l;
                w.l0h[i] = l.h; w.l0l[i] = l.l;
            }
        }
        if (threadIdx.x == 0) {
            const int64_t q = S.nb;
            w.bcol[q] = k;
            w.bsz[q] = 1;
            w.bd[3 * q] = d;
            w.st->nb = q + 1;
            w.st->k = k + 1;
            w.st->kind = 1;
        }
    } else {
        // largest off-diagonal entry at (a, b), a < b: the reference's
        // (i1, j1) = (b, a); rows/columns k <- k + j1, then k + 1 <- k + i1
        const int64_t a = sh_off / m, b = sh_off % m;
        if (a != 0) sym_swap(w, perm, n, k, k, k + a);
        if (b != 1) sym_swap(w, perm, n, k, k + 1, k + b);
        const dd ea = {w.Ah[k * n + k], w.Al[k * n + k]};
        const dd eb = {w.Ah[k * n + k + 1], w.Al[k * n + k + 1]};  // upper copy
        const dd ec = {w.Ah[(k + 1) * n + k + 1], w.Al[(k + 1) * n + k + 1]};
        const dd det = dd_sub(dd_mul(ea, ec), dd_mul(eb, eb));
        constexpr int U = 4;
        for (int64_t i0 = k + 2 + threadIdx.x; i0 < n; i0 += U * (int64_t)blockDim.x) {
          dd W0s[U], W1s[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * (int64_t)blockDim.x;
            if (i < n) {
                W0s[u] = dd{w.Ah[k * n + i], w.Al[k * n + i]};
                W1s[u] = dd{w.Ah[(k + 1) * n + i], w.Al[(k + 1) * n + i]};
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * (int64_t)blockDim.x;
            if (i >= n) continue;
            const dd W0 = W0s[u], W1 = W1s[u];
            const dd l0 = dd_div(dd_sub(dd_mul(W0, ec), dd_mul(W1, eb)), det);
            const dd l1 = dd_div(dd_sub(dd_mul(W1, ea), dd_mul(W0, eb)), det);
            w.Lh[i * n + k] = l0.h; w.Ll[i * n + k] = l0.l;
            w.Lh[i * n + k + 1] = l1.h; w.Ll[i * n + k + 1] = l1.l;
            w.v0h[i] = W0.h; w.v0l[i] = W0.l;
            w.v1h[i] = W1.h; w.v1l[i] = W1.l;
            w.l0h[i] = l0.h; w.l0l[i] = l0.l;
            w.l1h[i] = l1.h; w.l1l[i] = l1.l;
          }
        }
        if (threadIdx.x == 0) {
            const int64_t q = S.nb;
            w.bcol[q] = k;
            w.bsz[q] = 2;
            w.bd[3 * q] = ea;
            w.bd[3 * q + 1] = eb;
            w.bd[3 * q + 2] = ec;
            w.st->nb = q + 1;
            w.st->k = k + 2;
            w.st->kind = 2;
        }
    }
}

// ---- trailing update + symmetrization + next search -----------------------
// X = A - upd (both triangles), A <- (X + X^T) / 2 (factory.py:185-193 and
// 213-224 with _symmetrize, 124-128).  A is exactly symmetric, so the new
// (i, j) needs only A_ij and the pivot vectors, and equals the new (j, i)
// bit for bit (two_sum's error term is exact, hence symmetric).
// rows of a tile staged per batch and resident CTAs per SM (n = 8192:
// 16 / 2 1.234 s, 8 / 3 1.158 s, 4 / 4 1.233 s)
#ifndef HSVD_BP_BATCH
#define HSVD_BP_BATCH 8
#define HSVD_BP_OCC 3
#endif
__global__ void __launch_bounds__(UPD_THREADS, HSVD_BP_OCC) k_bp_update(int64_t n, BpWs w)
{
    __shared__ double rl0h[TB], rl0l[TB], rv0h[TB], rv0l[TB], rl1h[TB], rl1l[TB], rv1h[TB], rv1l[TB];
    __shared__ double cl0h[TB], cl0l[TB], cv0h[TB], cv0l[TB], cl1h[TB], cl1l[TB], cv1h[TB], cv1l[TB];
    __shared__ sp2 rsl0[TB], rsv0[TB], csl0[TB], csv0[TB];
    const BpState S = *w.st;
    if (S.kind == 0 || S.status != 0) return;
    const int64_t k = S.k, m = n - k;  // the new trailing block
    if ((int64_t)blockIdx.x >= tri_count(m)) return;
    const bool two = S.kind == 2;
    int I, J;
    tri_tile(blockIdx.x, I, J);
    const int tid = threadIdx.x, tx = tid % TB, ty = tid / TB;
    const int64_t r0 = k + (int64_t)I * TB, c0 = k + (int64_t)J * TB;
    if (tid < TB) {
        const int64_t r = r0 + tid, c = c0 + tid;
        if (r < n) {
            rl0h[tid] = w.l0h[r]; rl0l[tid] = w.l0l[r]; rv0h[tid] = w.v0h[r]; rv0l[tid] = w.v0l[r];
            rsl0[tid] = split2(rl0h[tid]); rsv0[tid] = split2(rv0h[tid]);
            if (two) {
                rl1h[tid] = w.l1h[r]; rl1l[tid] = w.l1l[r]; rv1h[tid] = w.v1h[r]; rv1l[tid] = w.v1l[r];
            }
        }
        if (c < n) {
            cl0h[tid] = w.l0h[c]; cl0l[tid] = w.l0l[c]; cv0h[tid] = w.v0h[c]; cv0l[tid] = w.v0l[c];
            csl0[tid] = split2(cl0h[tid]); csv0[tid] = split2(cv0h[tid]);
            if (two) {
                cl1h[tid] = w.l1h[c]; cl1l[tid] = w.l1l[c]; cv1h[tid] = w.v1h[c]; cv1l[tid] = w.v1l[c];
            }
        }
    }
    __syncthreads();
    double bo = -1.0, bd = -1.0;
    int64_t io = 0, id = 0;
    const int64_t c = c0 + tx;
    constexpr int RPT = TB / (UPD_THREADS / TB);  // rows per thread
    constexpr int BATCH = HSVD_BP_BATCH;           // rows staged at a time
#pragma unroll 1
    for (int u0 = 0; u0 < RPT; u0 += BATCH) {
    double nh[BATCH], nl[BATCH];
    // all loads of the batch first (the stores below may alias them)
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
        const int64_t r = r0 + ty + (u0 + u) * (UPD_THREADS / TB);
        nh[u] = nl[u] = 0.0;
        if (r < n && c < n && r <= c) {
            nh[u] = w.Ah[r * n + c];
            nl[u] = w.Al[r * n + c];
        }
    }
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
        const int rr = ty + (u0 + u) * (UPD_THREADS / TB);
        const int64_t r = r0 + rr;
        if (r >= n || c >= n || r > c) continue;  // upper triangle only
        const dd a = {nh[u], nl[u]};
        const dd li = {rl0h[rr], rl0l[rr]}, ci = {rv0h[rr], rv0l[rr]};
        const dd lj = {cl0h[tx], cl0l[tx]}, cj = {cv0h[tx], cv0l[tx]};
        dd uij, uji;
        if (!two) {
            uij = dd_mul_s(li, rsl0[rr], cj, csv0[tx]);
            uji = dd_mul_s(lj, csl0[tx], ci, rsv0[rr]);
        } else {
            const dd li1 = {rl1h[rr], rl1l[rr]}, ci1 = {rv1h[rr], rv1l[rr]};
            const dd lj1 = {cl1h[tx], cl1l[tx]}, cj1 = {cv1h[tx], cv1l[tx]};
            uij = dd_add(dd_mul_s(li, rsl0[rr], cj, csv0[tx]), dd_mul(li1, cj1));
            uji = dd_add(dd_mul_s(lj, csl0[tx], ci, rsv0[rr]), dd_mul(lj1, ci1));
        }
        const dd xij = dd_sub(a, uij), xji = dd_sub(a, uji);
        const dd s = dd_mul_f(dd_add(xij, xji), 0.5);
        w.Ah[r * n + c] = s.h;
        w.Al[r * n + c] = s.l;
        const double v = fabs(s.h);
        const int64_t ri = r - k, cj_ = c - k;
        if (ri < cj_) {
            if (better(v, ri * m + cj_, bo, io)) { bo = v; io = ri * m + cj_; }
        } else if (ri == cj_) {
            if (better(v, ri, bd, id)) { bd = v; id = ri; }
        }
    }
    }
    block_argmax<UPD_THREADS>(bo, io, bd, id);
    if (tid == 0) {
        w.poff[blockIdx.x] = Cand{bo, io};
        w.pdiag[blockIdx.x] = Cand{bd, id};
    }
}

// ---- post-processing: D's 2x2 blocks diagonalized (factory.py:234-255) ------
__global__ void k_bp_blocks(BpWs w, int64_t n)
{
    const int64_t nb = w.st->nb;
    const dd one = {1.0, 0.0};
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nb;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t col = w.bcol[q];
        if (w.bsz[q] == 1) {
            const dd d = w.bd[3 * q];
            w.bp[4 * q] = dd_sqrt(dd_abs(d));
            w.sg[col] = d.h > 0.0 ? 1 : -1;
        } else {
            const dd ea = w.bd[3 * q], eb = w.bd[3 * q + 1], ec = w.bd[3 * q + 2];
            const dd zeta = dd_div(dd_sub(ec, ea), dd_mul_f(eb, 2.0));
            const double sgn = zeta.h >= 0.0 ? 1.0 : -1.0;
            const dd root = dd_sqrt(dd_add(one, dd_mul(zeta, zeta)));
            const dd t = dd_div(dd{sgn, 0.0}, dd_add(dd_abs(zeta), root));
            const dd cs = dd_div(one, dd_sqrt(dd_add(one, dd_mul(t, t))));
            const dd sn = dd_mul(t, cs);
            const dd lam1 = dd_sub(ea, dd_mul(t, eb));
            const dd lam2 = dd_add(ec, dd_mul(t, eb));
            w.bp[4 * q] = cs;
            w.bp[4 * q + 1] = sn;
            w.bp[4 * q + 2] = dd_sqrt(dd_abs(lam1));
            w.bp[4 * q + 3] = dd_sqrt(dd_abs(lam2));
            w.sg[col] = lam1.h > 0.0 ? 1 : -1;
            w.sg[col + 1] = lam2.h > 0.0 ? 1 : -1;
        }
    }
}
// output column of every pivot column: +1 columns first, each class in pivot
// order (_assemble_factor, factory.py:258-267); signs_out in output order
__global__ void k_bp_order(BpWs w, int64_t n, int8_t *signs_out)
{
    if (threadIdx.x != 0) return;
    int64_t p = 0;
    for (int64_t c = 0; c < n; ++c) p += w.sg[c] == 1;
    int64_t pos = 0, neg = p;
    for (int64_t c = 0; c < n; ++c) {
        const int64_t o = w.sg[c] == 1 ? pos++ : neg++;
        w.ocol[c] = o;
        signs_out[o] = w.sg[c];
    }
    w.st->p = p;
}
// G[perm[i], ocol[col]] = hi + lo of (L Q_D |Lambda_D|^{1/2})[i, col]
__global__ void k_bp_assemble(BpWs w, const int64_t *perm, int64_t n, double *G, int64_t ldg)
{
    const int64_t q = blockIdx.y;
    if (q >= w.st->nb) return;
    const int64_t col = w.bcol[q];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t row = perm[i];
    if (w.bsz[q] == 1) {
        const dd g = dd_mul(dd{w.Lh[i * n + col], w.Ll[i * n + col]}, w.bp[4 * q]);
        G[row + w.ocol[col] * ldg] = __dadd_rn(g.h, g.l);
    } else {
        const dd cs = w.bp[4 * q], sn = w.bp[4 * q + 1], s1 = w.bp[4 * q + 2], s2 = w.bp[4 * q + 3];
        const dd L0 = {w.Lh[i * n + col], w.Ll[i * n + col]};
        const dd L1 = {w.Lh[i * n + col + 1], w.Ll[i * n + col + 1]};
        const dd u1 = dd_sub(dd_mul(L0, cs), dd_mul(L1, sn));
        const dd u2 = dd_add(dd_mul(L0, sn), dd_mul(L1, cs));
        const dd g1 = dd_mul(u1, s1), g2 = dd_mul(u2, s2);
        G[row + w.ocol[col] * ldg] = __dadd_rn(g1.h, g1.l);
        G[row + w.ocol[col + 1] * ldg] = __dadd_rn(g2.h, g2.l);
    }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// carve the workspace (sizes only when base == nullptr)
size_t bp_carve(int64_t n, unsigned char *base, BpWs *w)
{
    size_t off = 0;
    auto take = [&](size_t bytes) {
        unsigned char *p = base ? base + off : nullptr;
        off += align256(bytes);
        return p;
    };
    const size_t N = (size_t)n * n, tc = (size_t)tri_count(n);
    BpWs x;
    x.Ah = (double *)take(N * 8);
    x.Al = (double *)take(N * 8);
    x.Lh = (double *)take(N * 8);
    x.Ll = (double *)take(N * 8);
    x.v0h = (double *)take(n * 8); x.v0l = (double *)take(n * 8);
    x.v1h = (double *)take(n * 8); x.v1l = (double *)take(n * 8);
    x.l0h = (double *)take(n * 8); x.l0l = (double *)take(n * 8);
    x.l1h = (double *)take(n * 8); x.l1l = (double *)take(n * 8);
    x.poff = (Cand *)take(tc * sizeof(Cand));
    x.pdiag = (Cand *)take(tc * sizeof(Cand));
    x.bcol = (int64_t *)take(n * 8);
    x.bsz = (int64_t *)take(n * 8);
    x.bd = (dd *)take(3 * n * sizeof(dd));
    x.bp = (dd *)take(4 * n * sizeof(dd));
    x.sg = (int8_t *)take(n);
    x.ocol = (int64_t *)take(n * 8);
    x.st = (BpState *)take(sizeof(BpState));
    if (w) *w = x;
    return off;
}

}  // namespace
}  // namespace hsvd

using namespace hsvd;

extern "C" {

HSVD_API int hsvd_bp_workspace_size(int64_t n, size_t *bytes)
{
    if (n < 1 || !bytes) {
        set_error("hsvd_bp_workspace_size: bad arguments");
        return HSVD_ERR_ARG;
    }
    *bytes = bp_carve(n, nullptr, nullptr);
    return HSVD_OK;
}

}  // extern "C"

namespace hsvd {
// ||M||_F^2 of an n x n column-major M in a fixed order (deterministic):
// block k sums columns k, k + grid, ... (each column's rows strided over the
// threads, then a fixed tree); one block folds the partials in block order
constexpr int FROB_BLOCKS = 256;
__global__ void k_frob_partials(const double *__restrict__ M, int64_t ldm, int64_t n,
                                double *__restrict__ part)
{
    __shared__ double sh[256];
    double acc = 0.0;
    for (int64_t c = blockIdx.x; c < n; c += gridDim.x)
        for (int64_t e = threadIdx.x; e < n; e += blockDim.x) acc = fma(M[c * ldm + e], M[c * ldm + e], acc);
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_frob_fold(const double *__restrict__ part, int nparts, double *out)
{
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < nparts; ++k) t += part[k];
        *out = t;
    }
}
}  // namespace hsvd

extern "C" {

HSVD_API int hsvd_bp_factor_dd(const double *M, const double *Mlo, int64_t n, int64_t ldm,
                               double thresh, double *G, int64_t ldg, int8_t *signs,
                               int64_t *perm, int64_t *p_out, int64_t *stage_out, void *ws,
                               size_t ws_bytes, void *stream)
{
    if (!M || !G || !signs || !perm || !p_out || n < 1 || ldm < n || ldg < n || !ws) {
        set_error("hsvd_bp_factor: bad arguments");
        return HSVD_ERR_ARG;
    }
    if (ws_bytes < bp_carve(n, nullptr, nullptr)) {
        set_error("hsvd_bp_factor: workspace too small");
        return HSVD_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    BpWs w;
    bp_carve(n, (unsigned char *)ws, &w);
    int dev = 0;
    HSVD_CUDA(cudaGetDevice(&dev));
    int st_ = 0;
    DevCtx *ctx = dev_ctx(dev, &st_);
    if (!ctx) return st_;
    if (ctx->host_reserve(8) != HSVD_OK) return HSVD_ERR_CUDA;
    int64_t *hbuf = ctx->host;  // pinned
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    if (thresh < 0.0) {
        // the reference's singularity threshold n eps ||M||_F (factory.py:
        // 270-282), from M on the device (G's storage as the partial buffer:
        // it is written only after this)
        const int parts = (int)(n < FROB_BLOCKS ? n : FROB_BLOCKS);  // <= n <= n * ldg
        k_frob_partials<<<parts, 256, 0, s>>>(M, ldm, n, G);
        k_frob_fold<<<1, 32, 0, s>>>(G, parts, G);  // total into G[0] (in place)
        HSVD_LAUNCH_CHECK("k_frob");
        HSVD_CUDA(cudaMemcpyAsync(hbuf, G, sizeof(double), cudaMemcpyDeviceToHost, s));
        HSVD_CUDA(cudaStreamSynchronize(s));
        double ss;
        memcpy(&ss, hbuf, sizeof(double));
        thresh = (double)n * 0x1p-52 * sqrt(ss);
    }

    k_bp_init<<<1184, 256, 0, s>>>(M, Mlo, ldm, n, w);
    k_bp_init_state<<<1, 256, 0, s>>>(n, w, perm);
    k_bp_search<<<(unsigned)tri_count(n), UPD_THREADS, 0, s>>>(n, w);
    HSVD_LAUNCH_CHECK("k_bp_search");
    // pivot steps in batches; the state is read back once per batch
    int64_t k = 0;
    for (;;) {
        const int64_t batch = 64;
        for (int64_t j = 0; j < batch; ++j) {
            // after this pivot the trailing block starts at >= k + j + 1
            const int64_t mmax = n - (k + j + 1);
            k_bp_pivot<<<1, PIV_THREADS, 0, s>>>(n, thresh, alpha, w, perm);
            if (mmax > 0) k_bp_update<<<(unsigned)tri_count(mmax), UPD_THREADS, 0, s>>>(n, w);
        }
        HSVD_LAUNCH_CHECK("k_bp_pivot/k_bp_update");
        HSVD_CUDA(cudaMemcpyAsync(hbuf, w.st, sizeof(BpState), cudaMemcpyDeviceToHost, s));
        HSVD_CUDA(cudaStreamSynchronize(s));
        BpState hs;
        memcpy(&hs, hbuf, sizeof(hs));
        if (hs.status != 0) {
            if (stage_out) *stage_out = hs.stage;
            set_error("hsvd_bp_factor: numerical singularity");
            return HSVD_NUMERICAL_SINGULARITY;
        }
        k = hs.k;
        if (k >= n) break;
    }
    k_bp_blocks<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(w, n);
    k_bp_order<<<1, 32, 0, s>>>(w, n, signs);
    HSVD_CUDA(cudaMemcpyAsync(hbuf, w.st, sizeof(BpState), cudaMemcpyDeviceToHost, s));
    HSVD_CUDA(cudaStreamSynchronize(s));
    BpState hs;
    memcpy(&hs, hbuf, sizeof(hs));
    k_bp_assemble<<<dim3((unsigned)((n + 255) / 256), (unsigned)hs.nb), 256, 0, s>>>(w, perm, n, G,
                                                                                  ldg);
    HSVD_LAUNCH_CHECK("k_bp_assemble");
    *p_out = hs.p;
    if (stage_out) *stage_out = -1;
    return HSVD_OK;
}

HSVD_API int hsvd_bp_factor(const double *M, int64_t n, int64_t ldm, double thresh, double *G,
                            int64_t ldg, int8_t *signs, int64_t *perm, int64_t *p_out,
                            int64_t *stage_out, void *ws, size_t ws_bytes, void *stream)
{
    return hsvd_bp_factor_dd(M, nullptr, n, ldm, thresh, G, ldg, signs, perm, p_out, stage_out, ws,
                             ws_bytes, stream);
}

}  // extern "C"

// ===========================================================================
// QR shortening of a tall factor (hjsvd.factory.qr_shorten, factory.py:
// 300-334): Householder QR, G = Q R with R's diagonal made positive.  Plain
// fp64 (the reference's norm and dot products go through numpy's BLAS, so
// this path is checked to the reference's tolerances, not bit for bit).
// One step is two kernels: k_qr_reflector (one CTA: the reflector v, beta
// and column k of R) and k_qr_apply (one CTA per remaining column: its dot
// with v, then its rank-1 update).  Q is formed by applying the reflectors
// to eye(n, r) in reverse order with the same column kernel.
// ===========================================================================
namespace hsvd {
namespace {

constexpr int QR_THREADS = 256;

template <int NT>
__device__ double block_sum(double v)
{
    __shared__ double sh[NT / 32];
    __shared__ double total;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < NT / 32; ++k) s += sh[k];
        total = s;
    }
    __syncthreads();
    const double r = total;
    __syncthreads();
    return r;
}

// A column-major n x r (ld lda); V column-major n x r holds v_k in rows k..;
// beta[k]; status: first dependent column + 1 (0 = none)
__global__ void __launch_bounds__(QR_THREADS) k_qr_reflector(double *A, int64_t lda, int64_t n,
                                                             int64_t k, double *V, double *beta,
                                                             int64_t *status)
{
    if (*status) return;
    double *x = A + k * lda;
    double s = 0.0;
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) s += x[i] * x[i];
    const double normx = sqrt(block_sum<QR_THREADS>(s));
    if (normx == 0.0) {
        if (threadIdx.x == 0) *status = k + 1;
        return;
    }
    const double x0 = x[k];
    const double alpha = -(x0 >= 0.0 ? 1.0 : -1.0) * normx;
    double vv = 0.0;
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) {
        const double vi = i == k ? x0 - alpha : x[i];
        V[k * n + i] = vi;
        vv += vi * vi;
    }
    const double b = 2.0 / block_sum<QR_THREADS>(vv);
    __syncthreads();
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) x[i] = i == k ? alpha : 0.0;
    if (threadIdx.x == 0) beta[k] = b;
}

// for every column j in [j0, j1): M[k:, j] -= beta_k v_k (v_k^T M[k:, j])
__global__ void __launch_bounds__(QR_THREADS) k_qr_apply(double *M, int64_t ldm, int64_t n,
                                                         int64_t k, int64_t j0, const double *V,
                                                         const double *beta,
                                                         const int64_t *status)
{
    if (*status) return;
    const int64_t j = j0 + blockIdx.x;
    double *col = M + j * ldm;
    const double *v = V + k * n;
    double s = 0.0;
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) s += v[i] * col[i];
    const double w = block_sum<QR_THREADS>(s);
    const double bw = beta[k] * w;
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) col[i] -= v[i] * bw;
}

__global__ void k_qr_eye(double *Q, int64_t n, int64_t r)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * r;
         e += (int64_t)gridDim.x * blockDim.x)
        Q[e] = (e % n) == (e / n) ? 1.0 : 0.0;
}

// R = triu(A[:r, :]) (column-major r x r, ldr), flipped rows/columns of
// negative diagonal; status = r + 1 + row of a zero diagonal entry
__global__ void k_qr_finish(const double *A, int64_t lda, int64_t n, int64_t r, double *R,
                            int64_t ldr, double *Q, int64_t ldq, int64_t *status)
{
    if (*status) return;
    const int64_t j = blockIdx.x;  // column
    const double djj = A[j * lda + j];
    for (int64_t i = threadIdx.x; i < r; i += blockDim.x) {
        const double dii = A[i * lda + i];
        const double v = i <= j ? A[j * lda + i] : 0.0;
        R[j * ldr + i] = dii < 0.0 ? -v : v;
    }
    if (djj < 0.0)
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) Q[j * ldq + i] = -Q[j * ldq + i];
    if (threadIdx.x == 0 && djj == 0.0) atomicCAS((unsigned long long *)status, 0ull,
                                                  (unsigned long long)(r + 1 + j));
}

}  // namespace
}  // namespace hsvd

extern "C" {

HSVD_API int hsvd_qr_workspace_size(int64_t n, int64_t r, size_t *bytes)
{
    if (n < 1 || r < 1 || !bytes) {
        set_error("hsvd_qr_workspace_size: bad arguments");
        return HSVD_ERR_ARG;
    }
    *bytes = align256((size_t)n * r * 8) * 2 + align256((size_t)r * 8) + 256;
    return HSVD_OK;
}

HSVD_API int hsvd_qr_shorten(const double *G, int64_t n, int64_t r, int64_t ldg, double *R,
                             int64_t ldr, double *Q, int64_t ldq, int64_t *bad_col, void *ws,
                             size_t ws_bytes, void *stream)
{
    if (!G || !R || !Q || n < 1 || r < 1 || ldg < n || ldr < r || ldq < n || !ws) {
        set_error("hsvd_qr_shorten: bad arguments");
        return HSVD_ERR_ARG;
    }
    if (n <= r) {
        set_error("qr_shorten needs n > r");
        return HSVD_SHAPE_ERROR;
    }
    size_t need = 0;
    hsvd_qr_workspace_size(n, r, &need);
    if (ws_bytes < need) {
        set_error("hsvd_qr_shorten: workspace too small");
        return HSVD_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    unsigned char *b = (unsigned char *)ws;
    double *A = (double *)b;
    double *V = (double *)(b + align256((size_t)n * r * 8));
    double *beta = (double *)(b + 2 * align256((size_t)n * r * 8));
    int64_t *status = (int64_t *)(b + 2 * align256((size_t)n * r * 8) + align256((size_t)r * 8));
    HSVD_CUDA(cudaMemsetAsync(status, 0, 8, s));
    HSVD_CUDA(cudaMemcpy2DAsync(A, n * 8, G, ldg * 8, n * 8, r, cudaMemcpyDeviceToDevice, s));
    for (int64_t k = 0; k < r; ++k) {
        k_qr_reflector<<<1, QR_THREADS, 0, s>>>(A, n, n, k, V, beta, status);
        if (k + 1 < r) k_qr_apply<<<(unsigned)(r - k - 1), QR_THREADS, 0, s>>>(A, n, n, k, k + 1, V, beta, status);
    }
    HSVD_LAUNCH_CHECK("k_qr_apply");
    k_qr_eye<<<1184, 256, 0, s>>>(Q, ldq, r);
    // Q = H_0 ... H_{r-1} eye(n, r): reflector k touches rows k.. of the
    // columns >= k only (the others are zero there)
    for (int64_t k = r - 1; k >= 0; --k)
        k_qr_apply<<<(unsigned)(r - k), QR_THREADS, 0, s>>>(Q, ldq, n, k, k, V, beta, status);
    HSVD_LAUNCH_CHECK("k_qr_apply (Q)");
    k_qr_finish<<<(unsigned)r, 256, 0, s>>>(A, n, n, r, R, ldr, Q, ldq, status);
    int dev = 0;
    HSVD_CUDA(cudaGetDevice(&dev));
    int st_ = 0;
    DevCtx *ctx = dev_ctx(dev, &st_);
    if (!ctx) return st_;
    if (ctx->host_reserve(1) != HSVD_OK) return HSVD_ERR_CUDA;
    HSVD_CUDA(cudaMemcpyAsync(ctx->host, status, 8, cudaMemcpyDeviceToHost, s));
    HSVD_CUDA(cudaStreamSynchronize(s));
    const int64_t st = ctx->host[0];
    if (st) {
        if (bad_col) *bad_col = st <= r ? st - 1 : st - r - 1;
        set_error(st <= r ? "qr_shorten: dependent column" : "qr_shorten: R has a zero diagonal entry");
        return HSVD_RANK_DEFICIENT;
    }
    if (bad_col) *bad_col = -1;
    return HSVD_OK;
}

}  // extern "C"

// ===========================================================================
// Test-matrix generation in double-double (hjsvd.factory._generate_dd,
// factory.py:79-101): M = Q diag(lam) Q^T with Q a product of n - 1 random
// Householder reflectors, every operation the reference's dd primitive, so
// M (hi, lo) is bit-identical.  Per reflector v (drawn by the host from the
// reference's numpy stream):
//   beta  = 2 / tree_sum(two_prod(v, v))            k_gen_scalars (1 CTA)
//   w_i   = tree_sum_j mul_f(M_ij, v_j)             k_gen_matvec (CTA/row)
//   alpha = tree_sum(mul_f(w, v)), gamma = beta^2 alpha   k_gen_scalars
//   M_ij  = (M_ij - (vw + wv)_ij beta) + two_prod(v_i, v_j) gamma
//                                                   k_gen_update
// tree_sum is the reference's pairwise reduction (_dd.py:96-110): pairs
// (0,1), (2,3), ..., an odd last element carried to the end of the level.
// ===========================================================================
namespace hsvd {
namespace {

constexpr int GEN_THREADS = 1024;
constexpr int GEN_MAXP = 8;  // pairs per thread per level: n <= 2 * 16 * 1024

// pairwise tree over (h, l)[0, m) in shared memory (all threads of the CTA)
__device__ dd tree_sum_smem(double *h, double *l, int m)
{
    while (m > 1) {
        const int half = m >> 1;
        dd r[GEN_MAXP];
#pragma unroll
        for (int k = 0; k < GEN_MAXP; ++k) {
            const int t = threadIdx.x + k * GEN_THREADS;
            if (t < half) r[k] = dd_add(dd{h[2 * t], l[2 * t]}, dd{h[2 * t + 1], l[2 * t + 1]});
        }
        dd carry = {0.0, 0.0};
        if ((m & 1) && threadIdx.x == 0) carry = dd{h[m - 1], l[m - 1]};
        __syncthreads();
#pragma unroll
        for (int k = 0; k < GEN_MAXP; ++k) {
            const int t = threadIdx.x + k * GEN_THREADS;
            if (t < half) {
                h[t] = r[k].h;
                l[t] = r[k].l;
            }
        }
        if ((m & 1) && threadIdx.x == 0) {
            h[half] = carry.h;
            l[half] = carry.l;
        }
        __syncthreads();
        m = half + (m & 1);
    }
    return dd{h[0], l[0]};
}

// level 0 of the tree computed while loading: pair t = (x[2t], x[2t+1]);
// returns the length of level 1 (entries in h, l)
template <class F>
__device__ int tree_first_level(double *h, double *l, int m, F term)
{
    const int half = m >> 1;
    for (int t = threadIdx.x; t < half; t += GEN_THREADS) {
        const dd r = dd_add(term(2 * t), term(2 * t + 1));
        h[t] = r.h;
        l[t] = r.l;
    }
    if ((m & 1) && threadIdx.x == 0) {
        const dd c = term(m - 1);
        h[half] = c.h;
        l[half] = c.l;
    }
    __syncthreads();
    return half + (m & 1);
}

struct GenWs {
    double *wh, *wl;  // M v
    dd *sc;           // beta, alpha, gamma
};

__global__ void k_gen_init(const double *lam, int64_t n, double *Mh, double *Ml)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e % n;
        Mh[e] = i == j ? lam[i] : 0.0;
        Ml[e] = 0.0;
    }
}

// which = 0: beta = div(2, tree_sum(two_prod(v, v)));
// which = 1: alpha = tree_sum(mul_f(w, v)), gamma = mul(mul(beta, beta), alpha)
__global__ void __launch_bounds__(GEN_THREADS) k_gen_scalars(const double *v, int64_t n, GenWs g,
                                                             int which)
{
    extern __shared__ double gsm[];
    double *h = gsm, *l = gsm + (n + 1) / 2;
    int m;
    if (which == 0)
        m = tree_first_level(h, l, (int)n, [&](int j) { return two_prod(v[j], v[j]); });
    else
        m = tree_first_level(h, l, (int)n,
                             [&](int j) { return dd_mul_f(dd{g.wh[j], g.wl[j]}, v[j]); });
    const dd s = tree_sum_smem(h, l, m);
    if (threadIdx.x == 0) {
        if (which == 0) {
            g.sc[0] = dd_div(dd{2.0, 0.0}, s);
        } else {
            const dd beta = g.sc[0];
            g.sc[1] = s;
            g.sc[2] = dd_mul(dd_mul(beta, beta), s);
        }
    }
}

// w_i = tree_sum_j mul_f(M_ij, v_j), one CTA per row
__global__ void __launch_bounds__(GEN_THREADS) k_gen_matvec(const double *Mh, const double *Ml,
                                                            const double *v, int64_t n, GenWs g)
{
    extern __shared__ double gsm[];
    double *h = gsm, *l = gsm + (n + 1) / 2;
    const int64_t i = blockIdx.x;
    const double *rh = Mh + i * n, *rl = Ml + i * n;
    const int m = tree_first_level(h, l, (int)n, [&](int j) { return dd_mul_f(dd{rh[j], rl[j]}, v[j]); });
    const dd s = tree_sum_smem(h, l, m);
    if (threadIdx.x == 0) {
        g.wh[i] = s.h;
        g.wl[i] = s.l;
    }
}

// M = add(sub(M, S), T), S = mul(add(vw, wv), beta), T = mul(two_prod(v_i, v_j), gamma)
__global__ void k_gen_update(double *Mh, double *Ml, const double *v, int64_t n, GenWs g)
{
    const dd beta = g.sc[0], gamma = g.sc[2];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e % n;
        const double vi = v[i], vj = v[j];
        const dd wi = {g.wh[i], g.wl[i]}, wj = {g.wh[j], g.wl[j]};
        const dd vw = dd_mul_f(wj, vi), wv = dd_mul_f(wi, vj);
        const dd S = dd_mul(dd_add(vw, wv), beta);
        const dd T = dd_mul(two_prod(vi, vj), gamma);
        const dd r = dd_add(dd_sub(dd{Mh[e], Ml[e]}, S), T);
        Mh[e] = r.h;
        Ml[e] = r.l;
    }
}

// Mh = triu(Mh) + triu(Mh, 1)^T (and Ml): the upper triangle mirrored, + 0.0
__global__ void k_gen_finish(double *Mh, double *Ml, int64_t n)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e % n;
        if (i > j) {
            Mh[e] = __dadd_rn(0.0, Mh[j * n + i]);
            Ml[e] = __dadd_rn(0.0, Ml[j * n + i]);
        }
    }
    // the upper triangle gets + 0.0 in a second pass (after every mirror read)
}
__global__ void k_gen_finish_upper(double *Mh, double *Ml, int64_t n)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e % n;
        if (i <= j) {
            Mh[e] = __dadd_rn(Mh[e], 0.0);
            Ml[e] = __dadd_rn(Ml[e], 0.0);
        }
    }
}

// ---- power-of-two n: the same pairwise trees from warp shuffles ----------
// For n = 2^k every level of tree_sum pairs aligned neighbours and carries
// nothing, so a 64-element aligned segment is a subtree: lane t adds
// elements (2t, 2t + 1) and five shuffle levels finish it; the segment sums
// (n / 64 of them) form the remaining levels the same way.  dd_add is
// commutative bit for bit (two_sum's error term is exact), so which lane
// holds the left operand does not matter.
__device__ __forceinline__ dd shfl_down_dd(dd x, int o)
{
    return dd{__shfl_down_sync(0xffffffffu, x.h, o), __shfl_down_sync(0xffffffffu, x.l, o)};
}
// tree over `cnt` (power of two <= 32) values held by lanes 0..cnt-1; lane 0 gets it
__device__ __forceinline__ dd warp_tree(dd x, int cnt)
{
    for (int o = 1; o < cnt; o <<= 1) {
        const dd y = shfl_down_dd(x, o);
        if (((threadIdx.x & 31) & (2 * o - 1)) == 0) x = dd_add(x, y);
    }
    return x;
}
constexpr int GEN2_THREADS = 256;
// sum over j of term(j), j < n = 2^k >= 64, pairwise tree; all threads of the
// CTA call it; the result is returned to thread 0
template <class F>
__device__ dd tree_pow2(int n, F term, dd *seg)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nseg = n >> 6;
    for (int sg = wid; sg < nseg; sg += GEN2_THREADS / 32) {
        const int e = sg * 64 + 2 * lane;
        dd x = dd_add(term(e), term(e + 1));
        x = warp_tree(x, 32);
        if (lane == 0) seg[sg] = x;
    }
    __syncthreads();
    dd r = {0.0, 0.0};
    if (wid == 0) {
        if (nseg >= 32) {
            // lane t: the subtree of segments [t * per, (t + 1) * per)
            const int per = nseg >> 5;
            dd buf[8];  // per <= 8 (n <= 16384)
            for (int u = 0; u < per; ++u) buf[u] = seg[lane * per + u];
            for (int len = per; len > 1; len >>= 1)
                for (int u = 0; u < len / 2; ++u) buf[u] = dd_add(buf[2 * u], buf[2 * u + 1]);
            r = warp_tree(buf[0], 32);
        } else {
            r = warp_tree(lane < nseg ? seg[lane] : dd{0.0, 0.0}, nseg);
        }
    }
    return r;
}

__global__ void __launch_bounds__(GEN2_THREADS) k_gen_scalars2(const double *v, int n, GenWs g,
                                                                int which)
{
    __shared__ dd seg[256];
    dd s;
    if (which == 0)
        s = tree_pow2(n, [&](int j) { return two_prod(v[j], v[j]); }, seg);
    else
        s = tree_pow2(n, [&](int j) { return dd_mul_f(dd{g.wh[j], g.wl[j]}, v[j]); }, seg);
    if (threadIdx.x == 0) {
        if (which == 0) {
            g.sc[0] = dd_div(dd{2.0, 0.0}, s);
        } else {
            const dd beta = g.sc[0];
            g.sc[1] = s;
            g.sc[2] = dd_mul(dd_mul(beta, beta), s);
        }
    }
}
__global__ void __launch_bounds__(GEN2_THREADS) k_gen_matvec2(const double *Mh, const double *Ml,
                                                               const double *v, int n, GenWs g)
{
    __shared__ dd seg[256];
    const int64_t i = blockIdx.x;
    const double *rh = Mh + i * n, *rl = Ml + i * n;
    const dd s = tree_pow2(n, [&](int j) { return dd_mul_f(dd{rh[j], rl[j]}, v[j]); }, seg);
    if (threadIdx.x == 0) {
        g.wh[i] = s.h;
        g.wl[i] = s.l;
    }
}

// the rank-2 update on the upper triangle in 64x64 tiles, each written with
// its mirror (M stays bitwise symmetric: S and T are, Dekker's two_prod
// being exact), 16 B read + 32 B written per element pair
__global__ void __launch_bounds__(256, 3) k_gen_update_sym(double *Mh, double *Ml,
                                                            const double *v, int64_t n, GenWs g)
{
    extern __shared__ double gus[];  // the tile transposed (hi, lo): 2 x 64 x 65
    double (*th)[65] = reinterpret_cast<double (*)[65]>(gus);
    double (*tl)[65] = reinterpret_cast<double (*)[65]>(gus + 64 * 65);
    const int64_t tiles = (n + 63) / 64;
    const int64_t ntri = tiles * (tiles + 1) / 2;
    const dd beta = g.sc[0], gamma = g.sc[2];
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    for (int64_t t = blockIdx.x; t < ntri; t += gridDim.x) {
        int I, J;
        {
            int j = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
            while ((int64_t)(j + 1) * (j + 2) / 2 <= t) ++j;
            while ((int64_t)j * (j + 1) / 2 > t) --j;
            J = j;
            I = (int)(t - (int64_t)j * (j + 1) / 2);
        }
        const int64_t r0 = (int64_t)I * 64, c0 = (int64_t)J * 64;
        const int64_t c = c0 + tx;
        // 8 rows staged at a time (registers for 3 CTAs per SM); results are
        // kept for the mirror pass in the transposed tile
#pragma unroll 1
        for (int u0 = 0; u0 < 16; u0 += 8) {
            double nh[8], nl[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t r = r0 + ty + 4 * (u0 + u);
                nh[u] = nl[u] = 0.0;
                if (r < n && c < n) {
                    nh[u] = Mh[r * n + c];
                    nl[u] = Ml[r * n + c];
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t r = r0 + ty + 4 * (u0 + u);
                if (r >= n || c >= n) continue;
                const double vi = v[r], vj = v[c];
                const dd wi = {g.wh[r], g.wl[r]}, wj = {g.wh[c], g.wl[c]};
                const dd vw = dd_mul_f(wj, vi), wv = dd_mul_f(wi, vj);
                const dd S = dd_mul(dd_add(vw, wv), beta);
                const dd T = dd_mul(two_prod(vi, vj), gamma);
                const dd res = dd_add(dd_sub(dd{nh[u], nl[u]}, S), T);
                Mh[r * n + c] = res.h;
                Ml[r * n + c] = res.l;
                th[tx][ty + 4 * (u0 + u)] = res.h;
                tl[tx][ty + 4 * (u0 + u)] = res.l;
            }
        }
        if (I != J) {
            __syncthreads();
            const int64_t mc = r0 + tx;
            for (int cc = ty; cc < 64; cc += 4) {
                const int64_t mr = c0 + cc;
                if (mr < n && mc < n) {
                    Mh[mr * n + mc] = th[cc][tx];
                    Ml[mr * n + mc] = tl[cc][tx];
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace
}  // namespace hsvd

extern "C" {

HSVD_API int hsvd_gen_workspace_size(int64_t n, size_t *bytes)
{
    if (n < 2 || !bytes) {
        set_error("hsvd_gen_workspace_size: bad arguments");
        return HSVD_ERR_ARG;
    }
    *bytes = 2 * align256((size_t)n * 8) + align256(3 * sizeof(dd));
    return HSVD_OK;
}

HSVD_API int hsvd_gen_init(const double *lam, int64_t n, double *Mh, double *Ml, void *stream)
{
    if (!lam || !Mh || !Ml || n < 2) {
        set_error("hsvd_gen_init: bad arguments");
        return HSVD_ERR_ARG;
    }
    k_gen_init<<<1184, 256, 0, (cudaStream_t)stream>>>(lam, n, Mh, Ml);
    HSVD_LAUNCH_CHECK("k_gen_init");
    return HSVD_OK;
}

HSVD_API int hsvd_gen_reflect(double *Mh, double *Ml, int64_t n, const double *vs, int64_t count,
                              void *ws, size_t ws_bytes, void *stream)
{
    size_t need = 0;
    if (!Mh || !Ml || !vs || !ws || n < 2 || hsvd_gen_workspace_size(n, &need) != HSVD_OK ||
        ws_bytes < need) {
        set_error("hsvd_gen_reflect: bad arguments");
        return HSVD_ERR_ARG;
    }
    const size_t smem = 2 * (size_t)((n + 1) / 2) * 8;
    if (n > 2 * GEN_MAXP * GEN_THREADS || smem > 200 * 1024) {
        set_error("hsvd_gen_reflect: n too large for the on-chip pairwise tree");
        return HSVD_ERR_UNSUPPORTED;
    }
    // the shared-memory opt-in is per device
    static bool attr[64] = {};
    int dev = 0;
    HSVD_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        HSVD_CUDA(cudaFuncSetAttribute(k_gen_scalars, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       200 * 1024));
        HSVD_CUDA(cudaFuncSetAttribute(k_gen_matvec, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       200 * 1024));
        HSVD_CUDA(cudaFuncSetAttribute(k_gen_update_sym,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(2 * 64 * 65 * sizeof(double))));
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    cudaStream_t s = (cudaStream_t)stream;
    unsigned char *b = (unsigned char *)ws;
    GenWs g;
    g.wh = (double *)b;
    g.wl = (double *)(b + align256((size_t)n * 8));
    g.sc = (dd *)(b + 2 * align256((size_t)n * 8));
    // HSVD_GEN_POW2=0 keeps the generic shared-memory trees (cross-checks)
    static const bool pow2_on = [] {
        const char *e = getenv("HSVD_GEN_POW2");
        return !(e && e[0] == '0');
    }();
    const bool pow2 = pow2_on && n >= 64 && (n & (n - 1)) == 0;
    for (int64_t q = 0; q < count; ++q) {
        const double *v = vs + q * n;
        if (pow2) {  // warp-shuffle trees, upper-triangle update with mirror
            k_gen_scalars2<<<1, GEN2_THREADS, 0, s>>>(v, (int)n, g, 0);
            k_gen_matvec2<<<(unsigned)n, GEN2_THREADS, 0, s>>>(Mh, Ml, v, (int)n, g);
            k_gen_scalars2<<<1, GEN2_THREADS, 0, s>>>(v, (int)n, g, 1);
            k_gen_update_sym<<<1184, 256, 2 * 64 * 65 * sizeof(double), s>>>(Mh, Ml, v, n, g);
        } else {
            k_gen_scalars<<<1, GEN_THREADS, smem, s>>>(v, n, g, 0);
            k_gen_matvec<<<(unsigned)n, GEN_THREADS, smem, s>>>(Mh, Ml, v, n, g);
            k_gen_scalars<<<1, GEN_THREADS, smem, s>>>(v, n, g, 1);
            k_gen_update<<<1184, 256, 0, s>>>(Mh, Ml, v, n, g);
        }
    }
    HSVD_LAUNCH_CHECK("k_gen_update");
    return HSVD_OK;
}

HSVD_API int hsvd_gen_finish(double *Mh, double *Ml, int64_t n, void *stream)
{
    if (!Mh || !Ml || n < 2) {
        set_error("hsvd_gen_finish: bad arguments");
        return HSVD_ERR_ARG;
    }
    k_gen_finish<<<1184, 256, 0, (cudaStream_t)stream>>>(Mh, Ml, n);
    k_gen_finish_upper<<<1184, 256, 0, (cudaStream_t)stream>>>(Mh, Ml, n);
    HSVD_LAUNCH_CHECK("k_gen_finish");
    return HSVD_OK;
}

}  // extern "C"
