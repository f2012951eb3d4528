// hsvd_pointwise.cu -- bit-exact sm_100a kernels of the pointwise
// (reference-parity) one-sided hyperbolic Jacobi method.
//
// Built with -fmad=false (see hsvd_internal.cuh).  The per-pair work of
// _kernels.step_blocks (/root/reference/pkg/src/hjsvd/_kernels.py:188-235)
// runs as ONE CTA PER PIVOT SLOT.  The modulus steps use the streaming
// kernel (k_pointwise_stream): chunk partials straight from global memory,
// only the partials in shared memory, several pairs per SM.  The sequential
// row-cyclic walk (one CTA for all pairs) stages both columns in shared
// memory (process_pair).  HBM traffic per rotated pair = read+write of 2 G
// columns and 2 V columns (the algorithmic 32(n+r) bytes); a skipped pair
// reads its 2 G columns only.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "hsvd_internal.cuh"
#include "hsvd_rotation.cuh"

namespace hsvd {

constexpr int kStepThreads = 256;

// ---- chunked dot pieces: _kernels.py:32-59 ----------------------------
// Chunk b = [b*chunk, min((b+1)*chunk, n)) accumulated sequentially by FMA
// from 0.0, one thread per chunk, operands read from padded smem.
template <int NT>
__device__ __forceinline__ void chunk_partials(const double *sx,
                                               const double *sy, int n,
                                               int chunk, int m, double *part)
{
    for (int b = threadIdx.x; b < m; b += NT) {
        int lo = b * chunk;
        int hi = min(lo + chunk, n);
        double acc = 0.0;
        for (int e = lo; e < hi; ++e) acc = __fma_rn(sx[padx(e)], sy[padx(e)], acc);
        part[b] = acc;
    }
}

// Adjacent-pair tree part[i] = part[2i] + part[2i+1], odd tail carried up,
// ping-ponging between a and b (m entries each).  Returns the root; every
// thread of the CTA must call it (contains __syncthreads).
template <int NT>
__device__ __forceinline__ double tree_sum(double *a, double *b, int m)
{
    __syncthreads();
    int width = m;
    while (width > 1) {
        int half = width >> 1;
        for (int i = threadIdx.x; i < half; i += NT) b[i] = __dadd_rn(a[2 * i], a[2 * i + 1]);
        if ((width & 1) && threadIdx.x == 0) b[half] = a[width - 1];
        __syncthreads();
        double *tmp = a;
        a = b;
        b = tmp;
        width = half + (width & 1);
    }
    return a[0];
}

// Two trees at once (the two norm refreshes of one rotation).
template <int NT>
__device__ __forceinline__ void tree_sum2(double *a0, double *b0, double *a1,
                                          double *b1, int m, double &r0,
                                          double &r1)
{
    __syncthreads();
    int width = m;
    while (width > 1) {
        int half = width >> 1;
        for (int i = threadIdx.x; i < half; i += NT) {
            b0[i] = __dadd_rn(a0[2 * i], a0[2 * i + 1]);
            b1[i] = __dadd_rn(a1[2 * i], a1[2 * i + 1]);
        }
        if ((width & 1) && threadIdx.x == 0) {
            b0[half] = a0[width - 1];
            b1[half] = a1[width - 1];
        }
        __syncthreads();
        double *t0 = a0; a0 = b0; b0 = t0;
        double *t1 = a1; a1 = b1; b1 = t1;
        width = half + (width & 1);
    }
    r0 = a0[0];
    r1 = a1[0];
}

template <int NT>
__device__ __forceinline__ void load_column(double *s, const double *g, int n)
{
    int e = threadIdx.x;
    for (; e + 3 * NT < n; e += 4 * NT) {
        double v0 = g[e], v1 = g[e + NT], v2 = g[e + 2 * NT], v3 = g[e + 3 * NT];
        s[padx(e)] = v0;
        s[padx(e + NT)] = v1;
        s[padx(e + 2 * NT)] = v2;
        s[padx(e + 3 * NT)] = v3;
    }
    for (; e < n; e += NT) s[padx(e)] = g[e];
}

struct StepArgs {
    double *G;
    double *V;
    double *d;
    const int64_t *rho;
    const int64_t *jsign;
    int64_t *ip, *jp, *iblk, *jblk;
    uint8_t *C;
    uint32_t *rotk, *skipk;
    double *maxt;
    unsigned long long *err;
    int64_t ldg, ldv, r, k0;
    double eps, teps;
    int n, rv, chunk, m, npad, use_skip, advance;
};

// One pivot pair (i, j) at slot k, counters at slot `cs`.  Mirrors the body
// of the k-loop of step_blocks (_kernels.py:196-234).  Returns 1 on
// definiteness loss (after recording it), else 0.
template <int NT>
__device__ int process_pair(const StepArgs &a, int64_t k, int64_t i,
                            int64_t j, int64_t cs, double *smem)
{
    __shared__ double s_t, s_c, s_s;
    __shared__ int s_act;
    if (i > j) { int64_t tmp = i; i = j; j = tmp; }
    const int64_t ci = a.rho[i], cj = a.rho[j];
    double *gi = a.G + ci * a.ldg;
    double *gj = a.G + cj * a.ldg;
    double *sx = smem;
    double *sy = smem + a.npad;
    double *p0 = sy + a.npad;
    double *p1 = p0 + a.m;
    double *p2 = p1 + a.m;
    double *p3 = p2 + a.m;
    const int n = a.n;

    load_column<NT>(sx, gi, n);
    load_column<NT>(sy, gj, n);
    __syncthreads();
    chunk_partials<NT>(sx, sy, n, a.chunk, a.m, p0);
    double a_ij = tree_sum<NT>(p0, p1, a.m);
    if (threadIdx.x == 0) {
        double a_ii = a.d[i], a_jj = a.d[j];
        int act;
        if (a_ij == 0.0 ||
            (a.use_skip && fabs(a_ij) < __dmul_rn(a.eps, __dsqrt_rn(__dmul_rn(a_ii, a_jj))))) {
            act = 0;
            a.skipk[cs] += 1u;
        } else {
            int64_t hyp = a.jsign[i] == a.jsign[j] ? -1 : 1;
            double t, c;
            int st = rotation_tc(a_ii, a_jj, a_ij, hyp, t, c);
            if (st != 0) {
                atomicMin(a.err, pack_err(k, i, j));
                act = 2;
            } else {
                act = 1;
                s_t = t;
                s_c = c;
                s_s = hyp < 0 ? -1.0 : 1.0;
            }
        }
        s_act = act;
    }
    __syncthreads();
    const int act = s_act;
    if (act == 2) return 1;
    if (act == 1) {
        const double t = s_t, c = s_c, st = __dmul_rn(s_s, s_t);
        // fused_pair_update (_kernels.py:70-75) on the staged columns
        for (int e = threadIdx.x; e < n; e += NT) {
            const int pe = padx(e);
            double xi = sx[pe], yi = sy[pe];
            double nx = __dmul_rn(__fma_rn(st, yi, xi), c);
            double ny = __dmul_rn(__fma_rn(t, xi, yi), c);
            sx[pe] = nx;
            sy[pe] = ny;
            gi[e] = nx;
            gj[e] = ny;
        }
        if (a.V) {
            double *vi = a.V + ci * a.ldv;
            double *vj = a.V + cj * a.ldv;
            for (int e = threadIdx.x; e < a.rv; e += NT) {
                double xi = vi[e], yi = vj[e];
                vi[e] = __dmul_rn(__fma_rn(st, yi, xi), c);
                vj[e] = __dmul_rn(__fma_rn(t, xi, yi), c);
            }
        }
        __syncthreads();
        chunk_partials<NT>(sx, sx, n, a.chunk, a.m, p0);
        chunk_partials<NT>(sy, sy, n, a.chunk, a.m, p2);
        double di, dj;
        tree_sum2<NT>(p0, p1, p2, p3, a.m, di, dj);
        if (threadIdx.x == 0) {
            a.d[i] = di;
            a.d[j] = dj;
            double at = fabs(t);
            if (at > a.teps) a.C[k] = 3;
            else a.C[k] |= 1;
            a.rotk[cs] += 1u;
            if (at > a.maxt[cs]) a.maxt[cs] = at;
        }
    }
    __syncthreads();  // smem reuse by a following pair (row-cyclic)
    return 0;
}

// ---- streaming step kernel ------------------------------------------------
// The same pair computation without staging the two columns in shared
// memory: thread b owns chunk b of the chunked dot (_kernels.py:44-51) and
// reads it straight from global memory (16-byte loads when aligned), the
// partials go through the same adjacent-pair tree, and the update pass
// rewrites chunk b and accumulates the new squared norms of the chunk in the
// same sequential FMA order as dot_chunked(g, g) (_kernels.py:221-222).
// Only the m chunk partials live in shared memory, so several pairs are
// resident per SM (the staged kernel holds one: two 8192-long columns are
// 135 KB) and one pair's tree / rotation latency hides behind another
// pair's memory traffic.
template <int CH, bool VEC>
__device__ __forceinline__ double chunk_dot(const double *x, const double *y, int lo, int hi)
{
    double acc = 0.0;
    if (CH > 0 && VEC && hi - lo == CH) {
        const double2 *x2 = reinterpret_cast<const double2 *>(x + lo);
        const double2 *y2 = reinterpret_cast<const double2 *>(y + lo);
#pragma unroll
        for (int e = 0; e < CH / 2; ++e) {
            const double2 xv = x2[e], yv = y2[e];
            acc = __fma_rn(xv.x, yv.x, acc);
            acc = __fma_rn(xv.y, yv.y, acc);
        }
        return acc;
    }
    for (int e = lo; e < hi; ++e) acc = __fma_rn(x[e], y[e], acc);
    return acc;
}

// update chunk [lo, hi) of the pair in place, returning the chunk's new
// squared norms (sequential FMA from 0.0)
template <int CH, bool VEC>
__device__ __forceinline__ void chunk_update(double *x, double *y, int lo, int hi, double t,
                                             double c, double st, double &nx2, double &ny2)
{
    double ax = 0.0, ay = 0.0;
    if (CH > 0 && VEC && hi - lo == CH) {
        double2 *x2 = reinterpret_cast<double2 *>(x + lo);
        double2 *y2 = reinterpret_cast<double2 *>(y + lo);
#pragma unroll
        for (int e = 0; e < CH / 2; ++e) {
            const double2 xv = x2[e], yv = y2[e];
            double2 nx, ny;
            nx.x = __dmul_rn(__fma_rn(st, yv.x, xv.x), c);
            ny.x = __dmul_rn(__fma_rn(t, xv.x, yv.x), c);
            nx.y = __dmul_rn(__fma_rn(st, yv.y, xv.y), c);
            ny.y = __dmul_rn(__fma_rn(t, xv.y, yv.y), c);
            x2[e] = nx;
            y2[e] = ny;
            ax = __fma_rn(nx.x, nx.x, ax);
            ax = __fma_rn(nx.y, nx.y, ax);
            ay = __fma_rn(ny.x, ny.x, ay);
            ay = __fma_rn(ny.y, ny.y, ay);
        }
    } else {
        for (int e = lo; e < hi; ++e) {
            const double xi = x[e], yi = y[e];
            const double nx = __dmul_rn(__fma_rn(st, yi, xi), c);
            const double ny = __dmul_rn(__fma_rn(t, xi, yi), c);
            x[e] = nx;
            y[e] = ny;
            ax = __fma_rn(nx, nx, ax);
            ay = __fma_rn(ny, ny, ay);
        }
    }
    nx2 = ax;
    ny2 = ay;
}

// Warp-cooperative coalesced variants for chunk = 32 (lane l owns chunk l of
// the warp's 32 consecutive chunks): the warp loads each 8-element slice of
// its 32 chunks with 64-byte runs per chunk (every sector fully used), a
// shared-memory transpose hands lane l its chunk's slice, and lane l runs
// the chunk's sequential FMA chain in the reference's order.  The direct
// per-lane loads of chunk_dot touch 32 sectors per instruction with half of
// each used, and the second half is refetched once L1 has evicted it.
#ifndef HSVD_PW_VBATCH  // V^{-T} elements per thread with loads in flight together
#define HSVD_PW_VBATCH 16
#endif
#ifndef HSVD_PW_SLICE  // with HSVD_PW_VBATCH 16 (sweep 0 at n = 8192): 16: 3.46 s, 8: 3.76 s, 32: 4.83 s
#define HSVD_PW_SLICE 16
#endif
constexpr int kSlice = HSVD_PW_SLICE, kSliceLd = kSlice + 1;  // padded: conflict-free lane reads
constexpr int kPpc = kSlice / 2;                              // double2 per chunk per slice
struct WarpSlices {
    double x[32][kSliceLd], y[32][kSliceLd];
};
__device__ __forceinline__ void load_slices(WarpSlices &B, const double *gx, const double *gy,
                                            int s, int lane)
{
#pragma unroll
    for (int u = 0; u < kPpc; ++u) {
        const int f = u * 32 + lane, ch = f / kPpc, part = f % kPpc;
        const int off = ch * 32 + s * kSlice + 2 * part;
        const double2 xv = *reinterpret_cast<const double2 *>(gx + off);
        const double2 yv = *reinterpret_cast<const double2 *>(gy + off);
        B.x[ch][2 * part] = xv.x;
        B.x[ch][2 * part + 1] = xv.y;
        B.y[ch][2 * part] = yv.x;
        B.y[ch][2 * part + 1] = yv.y;
    }
    __syncwarp();
}
// dot of the warp's chunks: returns lane l's chunk partial
__device__ __forceinline__ double warp_chunk_dot(WarpSlices &B, const double *gx,
                                                 const double *gy, int lane)
{
    double acc = 0.0;
#pragma unroll 1
    for (int s = 0; s < 32 / kSlice; ++s) {
        load_slices(B, gx, gy, s, lane);
#pragma unroll
        for (int e = 0; e < kSlice; ++e) acc = __fma_rn(B.x[lane][e], B.y[lane][e], acc);
        __syncwarp();
    }
    return acc;
}
// update of the warp's chunks in place; lane l's new squared norms
__device__ __forceinline__ void warp_chunk_update(WarpSlices &B, double *gx, double *gy, int lane,
                                                  double t, double c, double st, double &nx2,
                                                  double &ny2)
{
    double ax = 0.0, ay = 0.0;
#pragma unroll 1
    for (int s = 0; s < 32 / kSlice; ++s) {
        load_slices(B, gx, gy, s, lane);
#pragma unroll
        for (int e = 0; e < kSlice; ++e) {
            const double xi = B.x[lane][e], yi = B.y[lane][e];
            const double nx = __dmul_rn(__fma_rn(st, yi, xi), c);
            const double ny = __dmul_rn(__fma_rn(t, xi, yi), c);
            B.x[lane][e] = nx;
            B.y[lane][e] = ny;
            ax = __fma_rn(nx, nx, ax);
            ay = __fma_rn(ny, ny, ay);
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < kPpc; ++u) {
            const int f = u * 32 + lane, ch = f / kPpc, part = f % kPpc;
            const int off = ch * 32 + s * kSlice + 2 * part;
            *reinterpret_cast<double2 *>(gx + off) = make_double2(B.x[ch][2 * part], B.x[ch][2 * part + 1]);
            *reinterpret_cast<double2 *>(gy + off) = make_double2(B.y[ch][2 * part], B.y[ch][2 * part + 1]);
        }
        __syncwarp();
    }
    nx2 = ax;
    ny2 = ay;
}

template <int NT, int CH, bool VEC>
__global__ void __launch_bounds__(NT) k_pointwise_stream(StepArgs a)
{
    extern __shared__ double smem[];
    __shared__ double s_t, s_c, s_s;
    __shared__ int s_act;
    if (*(volatile unsigned long long *)a.err != kNoError) return;
    const int64_t k = a.k0 + blockIdx.x;
    int64_t i = a.iblk[k], j = a.jblk[k];
    if (i > j) { int64_t tmp = i; i = j; j = tmp; }
    const int64_t ci = a.rho[i], cj = a.rho[j];
    double *gi = a.G + ci * a.ldg;
    double *gj = a.G + cj * a.ldg;
    const int n = a.n, chunk = CH > 0 ? CH : a.chunk, m = a.m;
    double *p0 = smem, *p1 = p0 + m, *p2 = p1 + m, *p3 = p2 + m;

    // coalesced warp path: groups of 32 full chunks (n a multiple of 1024),
    // group g on warp g mod (NT / 32)
    const bool wpath = CH == 32 && VEC && (n & 1023) == 0;
    WarpSlices *WS = reinterpret_cast<WarpSlices *>(p3 + m);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (wpath) {
        for (int g = wid; g < (m >> 5); g += NT / 32)
            p0[g * 32 + lane] = warp_chunk_dot(WS[wid], gi + g * 1024, gj + g * 1024, lane);
    } else {
        for (int bch = threadIdx.x; bch < m; bch += NT) {
            const int lo = bch * chunk, hi = min(lo + chunk, n);
            p0[bch] = chunk_dot<CH, VEC>(gi, gj, lo, hi);
        }
    }
    const double a_ij = tree_sum<NT>(p0, p1, m);
    if (threadIdx.x == 0) {
        const double a_ii = a.d[i], a_jj = a.d[j];
        int act;
        if (a_ij == 0.0 ||
            (a.use_skip && fabs(a_ij) < __dmul_rn(a.eps, __dsqrt_rn(__dmul_rn(a_ii, a_jj))))) {
            act = 0;
            a.skipk[k] += 1u;
        } else {
            const int64_t hyp = a.jsign[i] == a.jsign[j] ? -1 : 1;
            double t, c;
            const int st = rotation_tc(a_ii, a_jj, a_ij, hyp, t, c);
            if (st != 0) {
                atomicMin(a.err, pack_err(k, i, j));
                act = 2;
            } else {
                act = 1;
                s_t = t;
                s_c = c;
                s_s = hyp < 0 ? -1.0 : 1.0;
            }
        }
        s_act = act;
    }
    __syncthreads();
    const int act = s_act;
    if (act == 2) return;
    if (act == 1) {
        const double t = s_t, c = s_c, st = __dmul_rn(s_s, s_t);
        if (wpath) {
            for (int g = wid; g < (m >> 5); g += NT / 32) {
                double nx2, ny2;
                warp_chunk_update(WS[wid], gi + g * 1024, gj + g * 1024, lane, t, c, st, nx2, ny2);
                p0[g * 32 + lane] = nx2;
                p2[g * 32 + lane] = ny2;
            }
        } else {
            for (int bch = threadIdx.x; bch < m; bch += NT) {
                const int lo = bch * chunk, hi = min(lo + chunk, n);
                double nx2, ny2;
                chunk_update<CH, VEC>(gi, gj, lo, hi, t, c, st, nx2, ny2);
                p0[bch] = nx2;
                p2[bch] = ny2;
            }
        }
        if (a.V) {
            // V^{-T} columns: a batch of loads in flight before its stores
            // (one element at a time, each store had to wait for the next
            // load: vi and vj may alias as far as the compiler knows)
            double *vi = a.V + ci * a.ldv;
            double *vj = a.V + cj * a.ldv;
            const int rv = a.rv;
            constexpr int VB = HSVD_PW_VBATCH;
            for (int e0 = threadIdx.x; e0 < rv; e0 += NT * VB) {
                double xs[VB], ys[VB];
#pragma unroll
                for (int u = 0; u < VB; ++u) {
                    const int e = e0 + u * NT;
                    if (e < rv) {
                        xs[u] = vi[e];
                        ys[u] = vj[e];
                    }
                }
#pragma unroll
                for (int u = 0; u < VB; ++u) {
                    const int e = e0 + u * NT;
                    if (e < rv) {
                        vi[e] = __dmul_rn(__fma_rn(st, ys[u], xs[u]), c);
                        vj[e] = __dmul_rn(__fma_rn(t, xs[u], ys[u]), c);
                    }
                }
            }
        }
        double di, dj;
        tree_sum2<NT>(p0, p1, p2, p3, m, di, dj);
        if (threadIdx.x == 0) {
            a.d[i] = di;
            a.d[j] = dj;
            const double at = fabs(t);
            if (at > a.teps) a.C[k] = 3;
            else a.C[k] |= 1;
            a.rotk[k] += 1u;
            if (at > a.maxt[k]) a.maxt[k] = at;
        }
    }
    if (a.advance && threadIdx.x == 0) {
        // advance_stepper (_kernels.py:238-251), this slot only
        const int64_t r = a.r, half = r / 2;
        int64_t ip = a.ip[k], jp = a.jp[k];
        if (ip + jp >= r - 1) {
            ip += 1;
            if (ip == jp) {
                ip -= half;
                jp = ip;
            }
            a.ip[k] = ip;
            a.jp[k] = jp;
            a.iblk[k] = ip;
        } else {
            jp += 1;
            a.jp[k] = jp;
            a.jblk[k] = jp;
        }
    }
}

// Sequential row-cyclic quasi-sweep (solver.py:204-209, 231-243): one CTA
// walks all r(r-1)/2 pairs in order; code per pair, counters at slot 0.
template <int NT>
__global__ void __launch_bounds__(NT) k_rowcyclic_sweep(StepArgs a)
{
    extern __shared__ double smem[];
    if (*(volatile unsigned long long *)a.err != kNoError) return;
    int64_t q = 0;
    for (int64_t i = 0; i < a.r - 1; ++i)
        for (int64_t j = i + 1; j < a.r; ++j, ++q)
            if (process_pair<NT>(a, q, i, j, 0, smem)) return;
}

__global__ void k_advance_stepper(int64_t *ip, int64_t *jp, int64_t *iblk,
                                  int64_t *jblk, int64_t nblk, int64_t r)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nblk) return;
    const int64_t half = r / 2;
    if (ip[k] + jp[k] >= r - 1) {
        ip[k] += 1;
        if (ip[k] == jp[k]) {
            ip[k] -= half;
            jp[k] = ip[k];
        }
        iblk[k] = ip[k];
    } else {
        jp[k] += 1;
        jblk[k] = jp[k];
    }
}

__global__ void k_stepper_init(int64_t *ip, int64_t *jp, int64_t *iblk,
                               int64_t *jblk, int64_t r)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= r / 2) return;
    ip[k] = iblk[k] = k;
    jp[k] = jblk[k] = r - k - 1;
}

// precompute (solver.py:80-94): one CTA per column, chunked dot of g.g.
template <int NT>
__global__ void __launch_bounds__(NT) k_column_norms(
    const double *G, int64_t ldg, int n, int chunk, int m, int npad,
    double *d, unsigned long long *first_zero)
{
    extern __shared__ double smem[];
    const int64_t col = blockIdx.x;
    double *sx = smem;
    double *p0 = smem + npad;
    double *p1 = p0 + m;
    load_column<NT>(sx, G + col * ldg, n);
    __syncthreads();
    chunk_partials<NT>(sx, sx, n, chunk, m, p0);
    double v = tree_sum<NT>(p0, p1, m);
    if (threadIdx.x == 0) {
        d[col] = v;
        if (v == 0.0 && first_zero) atomicMin(first_zero, (unsigned long long)col);
    }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_dot(const double *x, const double *y,
                                            int n, int chunk, int m, int npad,
                                            double *out)
{
    extern __shared__ double smem[];
    double *sx = smem, *sy = smem + npad;
    double *p0 = sy + npad, *p1 = p0 + m;
    load_column<NT>(sx, x, n);
    load_column<NT>(sy, y, n);
    __syncthreads();
    chunk_partials<NT>(sx, sy, n, chunk, m, p0);
    double v = tree_sum<NT>(p0, p1, m);
    if (threadIdx.x == 0) *out = v;
}

__global__ void k_fused_pair_update(double *x, double *y, int64_t n, double t,
                                    double c, double s)
{
    const double st = __dmul_rn(s, t);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        double xi = x[e], yi = y[e];
        x[e] = __dmul_rn(__fma_rn(st, yi, xi), c);
        y[e] = __dmul_rn(__fma_rn(t, xi, yi), c);
    }
}

__global__ void k_rotation_batch(const double *a_ii, const double *a_jj,
                                 const double *a_ij, const int64_t *hyp,
                                 int64_t m, double *t, double *c,
                                 unsigned long long *first_bad)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    double tt, cc;
    int st = rotation_tc(a_ii[k], a_jj[k], a_ij[k], hyp[k], tt, cc);
    if (st) atomicMin(first_bad, (unsigned long long)k);
    t[k] = tt;
    c[k] = cc;
}

// sort_diagonal (solver.py:97-110) as a stable rank sort: the new position
// of package k is its segment start plus the number of segment members that
// precede it (strictly larger d in [0,p), strictly smaller in [p,r), ties
// by original position).  Keys are staged through smem tiles.
constexpr int kSortThreads = 256;
constexpr int kSortTile = 2048;
__global__ void __launch_bounds__(kSortThreads) k_rank_sort(
    const double *d, const int64_t *rho, const int64_t *jsign, int64_t r,
    int64_t p, double *d2, int64_t *rho2, int64_t *js2)
{
    __shared__ double tile[kSortTile];
    const int64_t k = blockIdx.x * (int64_t)kSortThreads + threadIdx.x;
    // A CTA may straddle the segment boundary: scan both segments' tiles
    // but count only members of this thread's own segment.
    const bool valid = k < r;
    const bool pos = k < p;
    const double key = valid ? d[k] : 0.0;
    int64_t cnt = 0;
    const int64_t cta_lo = blockIdx.x * (int64_t)kSortThreads;
    const int64_t cta_hi = min(r, cta_lo + kSortThreads);
    const int64_t scan_lo = cta_lo < p ? 0 : p;
    const int64_t scan_hi = cta_hi > p ? r : p;
    for (int64_t base = scan_lo; base < scan_hi; base += kSortTile) {
        const int64_t len = min((int64_t)kSortTile, scan_hi - base);
        __syncthreads();
        for (int t = threadIdx.x; t < len; t += kSortThreads) tile[t] = d[base + t];
        __syncthreads();
        if (valid) {
            const int64_t seg_lo = pos ? 0 : p, seg_hi = pos ? p : r;
            const int64_t lo = max(base, seg_lo), hi = min(base + len, seg_hi);
            for (int64_t q = lo; q < hi; ++q) {
                const double v = tile[q - base];
                const bool before = pos ? (v > key) : (v < key);
                cnt += (before || (v == key && q < k)) ? 1 : 0;
            }
        }
    }
    if (valid) {
        const int64_t dst = (pos ? 0 : p) + cnt;
        d2[dst] = key;
        rho2[dst] = rho[k];
        js2[dst] = jsign[k];
    }
}

__global__ void k_copy_packages(double *d, int64_t *rho, int64_t *jsign,
                                const double *d2, const int64_t *rho2,
                                const int64_t *js2, int64_t r)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= r) return;
    d[k] = d2[k];
    rho[k] = rho2[k];
    jsign[k] = js2[k];
}

// check_convergence (solver.py:113-121) + the per-sweep stats merge.
__global__ void __launch_bounds__(1024) k_reduce_sweep(
    uint8_t *C, int64_t m, uint32_t *rotk, uint32_t *skipk, double *maxt,
    int64_t nslots, int64_t *out, const unsigned long long *err, int reset)
{
    __shared__ unsigned int s_code;
    __shared__ unsigned long long s_rot, s_skip, s_max;
    if (threadIdx.x == 0) { s_code = 0; s_rot = 0; s_skip = 0; s_max = 0; }
    __syncthreads();
    unsigned int code = 0;
    unsigned long long rot = 0, skip = 0, mx = 0;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) code |= C[k];
    for (int64_t k = threadIdx.x; k < nslots; k += blockDim.x) {
        rot += rotk[k];
        skip += skipk[k];
        // max|t| >= 0: the IEEE bit pattern orders like the value
        unsigned long long b = (unsigned long long)__double_as_longlong(maxt[k]);
        mx = b > mx ? b : mx;
    }
    atomicOr(&s_code, code);
    atomicAdd(&s_rot, rot);
    atomicAdd(&s_skip, skip);
    atomicMax(&s_max, mx);
    __syncthreads();
    if (threadIdx.x == 0) {
        out[0] = (int64_t)s_code;
        out[1] = (int64_t)s_rot;
        out[2] = (int64_t)s_skip;
        out[3] = (int64_t)s_max;
        out[4] = err ? (int64_t)*err : -1;
    }
    if (reset) {
        for (int64_t k = threadIdx.x; k < m; k += blockDim.x) C[k] = 0;
        for (int64_t k = threadIdx.x; k < nslots; k += blockDim.x) {
            rotk[k] = 0;
            skipk[k] = 0;
            maxt[k] = 0.0;
        }
    }
}

__global__ void k_extract_sigma(const double *d, const int64_t *rho,
                                const int64_t *jsign, int64_t r, double *sigma,
                                double *lam)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= r) return;
    const int64_t c = rho[k];
    sigma[c] = __dsqrt_rn(d[k]);
    lam[c] = __dmul_rn(d[k], (double)jsign[k]);
}

__global__ void k_scale_columns(double *G, int64_t n, int64_t ldg,
                                const double *sigma)
{
    const int64_t c = blockIdx.y;
    const double s = sigma[c];
    double *g = G + c * ldg;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        g[e] = __ddiv_rn(g[e], s);
}

__global__ void k_identity(double *V, int64_t r, int64_t ldv)
{
    const int64_t c = blockIdx.y;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < r;
         e += (int64_t)gridDim.x * blockDim.x)
        V[c * ldv + e] = e == c ? 1.0 : 0.0;
}

__global__ void k_init_packages(const int8_t *signs, int64_t r, int64_t *rho,
                                int64_t *jsign)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= r) return;
    rho[k] = k;
    jsign[k] = signs[k];
}

// ======================================================================
// host side
// ======================================================================

static int smem_limit()
{
    static int lim = -1;
    if (lim < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) !=
            cudaSuccess)
            lim = 227 * 1024;
    }
    return lim;
}

int pointwise_smem_bytes(int64_t n, int64_t chunk, size_t *bytes)
{
    if (chunk < 1) {
        set_error("chunk must be >= 1");
        return HSVD_ERR_ARG;
    }
    const int64_t m = (n + chunk - 1) / chunk;
    *bytes = sizeof(double) * (2 * (size_t)padded_len((int)n) + 4 * (size_t)m);
    if ((int64_t)*bytes > smem_limit() || n > (1ll << 30)) {
        set_error("pointwise mode stages both columns in shared memory; n=" +
                  std::to_string(n) + " with chunk=" + std::to_string(chunk) +
                  " needs " + std::to_string(*bytes) +
                  " bytes (> opt-in limit); use block mode");
        return HSVD_ERR_UNSUPPORTED;
    }
    return HSVD_OK;
}

static StepArgs make_args(double *G, int64_t n, int64_t ldg, double *V,
                          int64_t rv, int64_t ldv, double *d,
                          const int64_t *rho, const int64_t *jsign,
                          int64_t *ip, int64_t *jp, int64_t *iblk,
                          int64_t *jblk, int64_t r, uint8_t *C, int64_t k0,
                          double eps, double teps, int use_skip, int64_t chunk,
                          int advance, uint32_t *rotk, uint32_t *skipk,
                          double *maxt, unsigned long long *err)
{
    StepArgs a;
    a.G = G; a.V = V; a.d = d; a.rho = rho; a.jsign = jsign;
    a.ip = ip; a.jp = jp; a.iblk = iblk; a.jblk = jblk; a.C = C;
    a.rotk = rotk; a.skipk = skipk; a.maxt = maxt; a.err = err;
    a.ldg = ldg; a.ldv = ldv; a.r = r; a.k0 = k0; a.eps = eps; a.teps = teps;
    a.n = (int)n; a.rv = (int)rv; a.chunk = (int)chunk;
    a.m = (int)((n + chunk - 1) / chunk);
    a.npad = padded_len((int)n);
    a.use_skip = use_skip; a.advance = advance;
    return a;
}

int launch_pointwise_step(double *G, int64_t n, int64_t ldg, double *V,
                          int64_t rv, int64_t ldv, double *d,
                          const int64_t *rho, const int64_t *jsign,
                          int64_t *ip, int64_t *jp, int64_t *iblk,
                          int64_t *jblk, int64_t r, uint8_t *C, int64_t k0,
                          int64_t k1, double eps, double teps, int use_skip,
                          int64_t chunk, int advance, uint32_t *rotk,
                          uint32_t *skipk, double *maxt,
                          unsigned long long *err, cudaStream_t s)
{
    if (k1 <= k0) return HSVD_OK;
    if (chunk < 1) {
        set_error("chunk must be >= 1");
        return HSVD_ERR_ARG;
    }
    StepArgs a = make_args(G, n, ldg, V, rv, ldv, d, rho, jsign, ip, jp, iblk,
                           jblk, r, C, k0, eps, teps, use_skip, chunk, advance,
                           rotk, skipk, maxt, err);
    // the streaming kernel keeps only the chunk partials in shared memory
    const unsigned grid = (unsigned)(k1 - k0);
    const bool vec = chunk == 32 && ldg % 2 == 0 && ((uintptr_t)G & 15) == 0;
    const size_t smem = sizeof(double) * 4 * (size_t)a.m +
                        (vec && n % 1024 == 0 ? sizeof(WarpSlices) * (kStepThreads / 32) : 0);
    if (vec) {
        HSVD_CUDA(cudaFuncSetAttribute(k_pointwise_stream<kStepThreads, 32, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_pointwise_stream<kStepThreads, 32, true><<<grid, kStepThreads, smem, s>>>(a);
    } else {
        HSVD_CUDA(cudaFuncSetAttribute(k_pointwise_stream<kStepThreads, 0, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_pointwise_stream<kStepThreads, 0, false><<<grid, kStepThreads, smem, s>>>(a);
    }
    HSVD_LAUNCH_CHECK("k_pointwise_stream");
    return HSVD_OK;
}

int launch_rowcyclic_sweep(double *G, int64_t n, int64_t ldg, double *V,
                           int64_t rv, int64_t ldv, double *d,
                           const int64_t *rho, const int64_t *jsign,
                           int64_t r, uint8_t *C, double eps, double teps,
                           int use_skip, int64_t chunk, uint32_t *rotk,
                           uint32_t *skipk, double *maxt,
                           unsigned long long *err, cudaStream_t s)
{
    size_t smem;
    int st = pointwise_smem_bytes(n, chunk, &smem);
    if (st) return st;
    HSVD_CUDA(cudaFuncSetAttribute(k_rowcyclic_sweep<kStepThreads>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    StepArgs a = make_args(G, n, ldg, V, rv, ldv, d, rho, jsign, nullptr,
                           nullptr, nullptr, nullptr, r, C, 0, eps, teps,
                           use_skip, chunk, 0, rotk, skipk, maxt, err);
    k_rowcyclic_sweep<kStepThreads><<<1, kStepThreads, smem, s>>>(a);
    HSVD_LAUNCH_CHECK("k_rowcyclic_sweep");
    return HSVD_OK;
}

}  // namespace hsvd

using namespace hsvd;

static inline unsigned nblocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

extern "C" {

int hsvd_dot_chunked(const double *x, const double *y, int64_t n,
                     int64_t chunk, double *out, void *stream)
{
    if (n < 1) {
        HSVD_CUDA(cudaMemsetAsync(out, 0, sizeof(double), (cudaStream_t)stream));
        return HSVD_OK;
    }
    size_t smem;
    int st = pointwise_smem_bytes(n, chunk, &smem);
    if (st) return st;
    HSVD_CUDA(cudaFuncSetAttribute(k_dot<kStepThreads>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    int m = (int)((n + chunk - 1) / chunk);
    k_dot<kStepThreads><<<1, kStepThreads, smem, (cudaStream_t)stream>>>(
        x, y, (int)n, (int)chunk, m, padded_len((int)n), out);
    HSVD_LAUNCH_CHECK("k_dot");
    return HSVD_OK;
}

int hsvd_fused_pair_update(double *x, double *y, int64_t n, double t, double c,
                           double s, void *stream)
{
    if (n < 1) return HSVD_OK;
    unsigned g = nblocks(n, 256);
    if (g > 4096) g = 4096;
    k_fused_pair_update<<<g, 256, 0, (cudaStream_t)stream>>>(x, y, n, t, c, s);
    HSVD_LAUNCH_CHECK("k_fused_pair_update");
    return HSVD_OK;
}

int hsvd_rotation_batch(const double *a_ii, const double *a_jj,
                        const double *a_ij, const int64_t *hyp, int64_t m,
                        double *t, double *c, int64_t *first_bad, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    HSVD_CUDA(cudaMemsetAsync(first_bad, 0xff, sizeof(int64_t), s));
    if (m < 1) return HSVD_OK;
    k_rotation_batch<<<nblocks(m, 128), 128, 0, s>>>(
        a_ii, a_jj, a_ij, hyp, m, t, c, (unsigned long long *)first_bad);
    HSVD_LAUNCH_CHECK("k_rotation_batch");
    return HSVD_OK;
}

int hsvd_precompute(const double *G, int64_t n, int64_t r, int64_t ldg,
                    int64_t chunk, double *d, int64_t *first_zero,
                    void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (first_zero) HSVD_CUDA(cudaMemsetAsync(first_zero, 0xff, sizeof(int64_t), s));
    if (r < 1 || n < 1) return HSVD_OK;
    const int64_t m = (n + chunk - 1) / chunk;
    size_t smem = sizeof(double) * ((size_t)padded_len((int)n) + 2 * (size_t)m);
    if ((int64_t)smem > smem_limit()) {
        set_error("precompute: column does not fit in shared memory");
        return HSVD_ERR_UNSUPPORTED;
    }
    HSVD_CUDA(cudaFuncSetAttribute(k_column_norms<kStepThreads>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    k_column_norms<kStepThreads><<<(unsigned)r, kStepThreads, smem, s>>>(
        G, ldg, (int)n, (int)chunk, (int)m, padded_len((int)n), d,
        (unsigned long long *)first_zero);
    HSVD_LAUNCH_CHECK("k_column_norms");
    return HSVD_OK;
}

int hsvd_step_blocks(double *G, int64_t n, int64_t ldg, double *V, int64_t rv,
                     int64_t ldv, double *d, const int64_t *rho,
                     const int64_t *jsign, int64_t *ip, int64_t *jp,
                     int64_t *iblk, int64_t *jblk, int64_t r, uint8_t *C,
                     int64_t k0, int64_t k1, double eps, double teps,
                     int32_t use_skip, int64_t chunk, int32_t advance,
                     uint32_t *rotk, uint32_t *skipk, double *maxt,
                     uint64_t *err_packed, void *stream)
{
    if (advance && (!ip || !jp)) {
        set_error("advance requires ip/jp");
        return HSVD_ERR_ARG;
    }
    return launch_pointwise_step(G, n, ldg, V, rv, ldv, d, rho, jsign, ip, jp,
                                 iblk, jblk, r, C, k0, k1, eps, teps, use_skip,
                                 chunk, advance, rotk, skipk, maxt,
                                 (unsigned long long *)err_packed,
                                 (cudaStream_t)stream);
}

int hsvd_advance_stepper(int64_t *ip, int64_t *jp, int64_t *iblk,
                         int64_t *jblk, int64_t nblk, int64_t r, void *stream)
{
    if (nblk < 1) return HSVD_OK;
    k_advance_stepper<<<nblocks(nblk, 256), 256, 0, (cudaStream_t)stream>>>(
        ip, jp, iblk, jblk, nblk, r);
    HSVD_LAUNCH_CHECK("k_advance_stepper");
    return HSVD_OK;
}

int hsvd_stepper_init(int64_t *ip, int64_t *jp, int64_t *iblk, int64_t *jblk,
                      int64_t r, void *stream)
{
    if (r < 2 || r % 2) {
        set_error("r must be even and >= 2");
        return HSVD_SHAPE_ERROR;
    }
    k_stepper_init<<<nblocks(r / 2, 256), 256, 0, (cudaStream_t)stream>>>(
        ip, jp, iblk, jblk, r);
    HSVD_LAUNCH_CHECK("k_stepper_init");
    return HSVD_OK;
}

int hsvd_sort_diagonal(double *d, int64_t *rho, int64_t *jsign, int64_t r,
                       int64_t p, void *ws, void *stream)
{
    if (r < 1) return HSVD_OK;
    cudaStream_t s = (cudaStream_t)stream;
    double *d2 = (double *)ws;
    int64_t *rho2 = (int64_t *)(d2 + r);
    int64_t *js2 = rho2 + r;
    k_rank_sort<<<nblocks(r, kSortThreads), kSortThreads, 0, s>>>(d, rho, jsign, r, p,
                                                               d2, rho2, js2);
    HSVD_LAUNCH_CHECK("k_rank_sort");
    k_copy_packages<<<nblocks(r, 256), 256, 0, s>>>(d, rho, jsign, d2, rho2, js2, r);
    HSVD_LAUNCH_CHECK("k_copy_packages");
    return HSVD_OK;
}

int hsvd_reduce_sweep(uint8_t *C, int64_t m, uint32_t *rotk, uint32_t *skipk,
                      double *maxt, int64_t nslots, int64_t *out,
                      int32_t reset, void *stream)
{
    k_reduce_sweep<<<1, 1024, 0, (cudaStream_t)stream>>>(C, m, rotk, skipk, maxt,
                                                         nslots, out, nullptr, reset);
    HSVD_LAUNCH_CHECK("k_reduce_sweep");
    return HSVD_OK;
}

int hsvd_extract(double *G, int64_t n, int64_t ldg, const double *d,
                 const int64_t *rho, const int64_t *jsign, int64_t r,
                 double *sigma, double *lam, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (r < 1) return HSVD_OK;
    k_extract_sigma<<<nblocks(r, 256), 256, 0, s>>>(d, rho, jsign, r, sigma, lam);
    HSVD_LAUNCH_CHECK("k_extract_sigma");
    unsigned gx = nblocks(n, 256);
    if (gx > 64) gx = 64;
    k_scale_columns<<<dim3(gx, (unsigned)r), 256, 0, s>>>(G, n, ldg, sigma);
    HSVD_LAUNCH_CHECK("k_scale_columns");
    return HSVD_OK;
}

}  // extern "C"

// internal launchers used by the driver
namespace hsvd {
int launch_identity(double *V, int64_t r, int64_t ldv, cudaStream_t s)
{
    unsigned gx = nblocks(r, 256);
    if (gx > 64) gx = 64;
    k_identity<<<dim3(gx, (unsigned)r), 256, 0, s>>>(V, r, ldv);
    HSVD_LAUNCH_CHECK("k_identity");
    return HSVD_OK;
}
int launch_init_packages(const int8_t *signs, int64_t r, int64_t *rho,
                         int64_t *jsign, cudaStream_t s)
{
    k_init_packages<<<nblocks(r, 256), 256, 0, s>>>(signs, r, rho, jsign);
    HSVD_LAUNCH_CHECK("k_init_packages");
    return HSVD_OK;
}
int launch_reduce_sweep(uint8_t *C, int64_t m, uint32_t *rotk, uint32_t *skipk,
                        double *maxt, int64_t nslots, int64_t *out,
                        const unsigned long long *err, int reset, cudaStream_t s)
{
    k_reduce_sweep<<<1, 1024, 0, s>>>(C, m, rotk, skipk, maxt, nslots, out, err, reset);
    HSVD_LAUNCH_CHECK("k_reduce_sweep");
    return HSVD_OK;
}
}  // namespace hsvd
