// hsvd_block_kernels.cuh -- the block-column kernels of one step (Gram,
// inner rotations, update) and their launch wrapper, shared by the one-GPU
// driver (hsvd_block.cu) and the sharded multi-GPU driver (hsvd_sharded.cu).
#pragma once

#include <cuda.h>  // CUtensorMap (the encoder is fetched at run time: no libcuda link)
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "hsvd_internal.cuh"
#include "hsvd_rotation.cuh"

// k_gram tiling: k-tile depth, cp.async stages, resident CTAs per SM
// (64 / 2 / 3 measured 0.5 % faster per solve than 32 / 4 / 3 on the same
// box; 64 / 3 / 2 is 4 % slower on the Gram: occupancy 3 matters)
#ifndef HSVD_GRAM_KT
#define HSVD_GRAM_KT 64
#define HSVD_GRAM_STAGES 2
#define HSVD_GRAM_OCC 3
#endif
// k_gram operand pipeline: 1 = TMA (cp.async.bulk.tensor gather4 through
// rho) + mbarrier ring with a producer warp; 0 = the cp.async kernel
#ifndef HSVD_GRAM_TMA
#define HSVD_GRAM_TMA 1
#endif
#ifndef HSVD_GRAM_NOMATH
#define HSVD_GRAM_NOMATH 0  // diagnostics only (wrong results)
#endif
#ifndef HSVD_GRAM_NOLOAD
#define HSVD_GRAM_NOLOAD 0
#endif
#ifndef HSVD_GRAM_TMA_GMAJOR
#define HSVD_GRAM_TMA_GMAJOR 1
#endif
#ifndef HSVD_GRAM_TMA_STAGES
#define HSVD_GRAM_TMA_STAGES 3
#define HSVD_GRAM_TMA_OCC 2
#endif

namespace hsvd {

// ---------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// mbarrier + TMA (sm_90+ PTX; gather4 is sm_100a)
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "HSVD_MBW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra HSVD_MBW_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// 4 arbitrary columns (dim-1 coordinates c0..c3) x 16 consecutive rows from
// row k0 of the column-major factor, into 4 x 128 swizzled bytes at dst
__device__ __forceinline__ void tma_gather4(unsigned dst, const CUtensorMap *tm, int k0, int c0,
                                            int c1, int c2, int c3, unsigned bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
        "l"(tm), "r"(k0), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

// D(8x8) += A(8x4, row) * B(4x8, col), FP64 tensor core.
// a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
// d = {D[lane>>2][2*(lane&3)], D[lane>>2][2*(lane&3)+1]}.
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

constexpr int kThreads = 256;
#ifndef HSVD_INNER_THREADS
#define HSVD_INNER_THREADS 256
#endif

// position of column c (0..2b) of slot P = (I, J), I < J
__device__ __forceinline__ int64_t slot_pos(int c, int b, int64_t I, int64_t J)
{
    return c < b ? I * b + c : J * b + (c - b);
}

// ---------------------------------------------------------------------
// k_gram: partial Gram matrices over fixed K segments, streamed over CTAs
// ---------------------------------------------------------------------
// A slot's K range (T = ceil(n / KT) k-tiles) is cut into NSEG fixed
// segments of L k-tiles.  L and NSEG depend on n (and KT) only, never on
// how many slots a launch holds, how many SMs the GPU has or how the slots
// are split over streams and shards.  Each segment's partial Gram is one
// DMMA accumulation chain from zero over the segment's k-tiles, and k_inner
// folds a slot's NSEG partials in segment order, so A_P is a function of
// the slot's columns alone: block mode gives the same bits for any
// stream split and any shard count (the reference's worker-count
// invariance, solver.py:127-131).
//
// Who computes which segment is free: the NS = nslots * NSEG segments of a
// launch are dealt to P CTAs in contiguous runs of equal length (stream-K
// at segment granularity: a CTA streams its run through one pipeline and
// flushes its accumulators at every segment end).
struct GramPart {
    int64_t T, L, NSEG, NS, P;
    __host__ __device__ int64_t seg_begin(int64_t c) const { return c * NS / P; }
    // first k-tile item (slot * T + k-tile) of global segment s
    __host__ __device__ int64_t item_of_seg(int64_t s) const
    {
        const int64_t slot = s / NSEG, g = s % NSEG;
        return slot * T + g * L;
    }
    __host__ __device__ int64_t begin(int64_t c) const
    {
        const int64_t s = seg_begin(c);
        return s >= NS ? (NS / NSEG) * T : item_of_seg(s);
    }
};

// ---------------------------------------------------------------------
// Exact reuse of all-skip visits (the late sweeps)
// ---------------------------------------------------------------------
// A slot visit's outcome (rotations, W_P, code, statistics) is a function
// of its 2b columns alone: which columns sit at its positions, their bits
// and J signs, and the inner ordering.  When a visit of the block pair
// (I, J) skipped every pair (no rotation: _kernels.py:210-213 applied to
// every pair of the pass) and since then no column of blocks I and J was
// rewritten and no sort moved another column into them, the next visit of
// (I, J) reads the same bits and must skip every pair again: its Gram,
// inner pass and update are not run, and its statistics are those of the
// recorded visit.  Same bits in, same decision out, so the result is bit
// for bit the one without reuse.
//
// Stamps order events: step k of sweep s is s*(nb+1) + k + 1, the sort at
// the end of sweep s is s*(nb+1) + nb + 1.  blkmod[K] is the stamp of the
// last event that changed block K's columns (a rotation touching one of
// them, written by k_inner, or a sort moving another column in);
// pairstamp[I*nb+J] is the stamp of the last all-skip visit of (I, J)
// (bit 31: it was a full-ordering pass), pairskip its skip count.
struct ReuseWs {
    uint32_t *pairstamp, *pairskip, *blkmod;
    int32_t *dsweep;  // sweeps completed (device)
    // Diagonal-block cache: dcache[K] (b x b) is block K's own Gram
    // G_K^T G_K as folded by the visit at stamp dstamp[K].  While no event
    // has changed block K since (blkmod[K] < dstamp[K]) the same segments
    // would produce the same bits, so a visit whose two blocks are both
    // cached computes only the cross block G_I^T G_J ("cross" class).
    double *dcache;
    uint32_t *dstamp;
    unsigned long long *planstat;  // [full, reused, cross] slot counts of planned steps
};

// slot classes of a planned step (k_plan -> skipf)
constexpr uint8_t kSlotFull = 0, kSlotReused = 1, kSlotCross = 2;

__device__ __forceinline__ uint32_t reuse_stamp(const int32_t *dsweep, int64_t nb, int step)
{
    return (uint32_t)(*(volatile const int32_t *)dsweep) * (uint32_t)(nb + 1) + (uint32_t)step + 1u;
}

template <int B2, int KT, int STAGES>
struct GramSmem {
    static constexpr int LD = KT + 4;  // == 4 mod 16: conflict-free fragments
    static constexpr int MAXSLOTS = 4;  // slots one CTA may touch
    double x[STAGES][B2][LD];
    const double *col[MAXSLOTS][B2];
};

// Per-warp DMMA roles over the upper-triangle 8x8 tiles of the B2 x B2
// output (A is symmetric).  Roles are resolved by warp-uniform branches, so
// no DMMA is ever issued predicated-off (a predicated-off DMMA still
// occupies the tensor pipe).  B2 = 64: 16x16 super-tiles; warps 0-5 own one
// off-diagonal super-tile (4 DMMA per k-step), warps 6-7 two diagonal
// super-tiles (3 DMMA each): 8/8/10/10 DMMA per SM sub-partition.
// B2 = 32: ten 8x8 tiles, warps 0-1 own two, warps 2-7 one.
template <int B2>
struct GramRoles;

// ld(R) returns this lane's fragment element of row R + (lane >> 2) at the
// current k-step (column k + (lane & 3)); R is a multiple of 8.
template <>
struct GramRoles<64> {
    // 36 upper 8x8 tiles over 8 warps, 9 per SM sub-partition (warps w and
    // w + 4) and at most 5 per warp: warps 0-5 own one off-diagonal 16x16
    // super-tile (4 tiles); warps 4 and 5 add one diagonal tile each, (1,1)
    // and (3,3); warps 6 and 7 own the remaining 10 diagonal-block tiles.
    static constexpr int NACC = 5;  // accumulator tiles per warp (max)
    static constexpr int NFRAG = 5;  // fragments per warp and k-step (max)
    // split form for software pipelining: load() the k-step's fragments,
    // compute() its DMMAs (the same operations and order as mma())
    template <class LD>
    __device__ static void load(int warp, LD &&ld, double (&f)[NFRAG])
    {
        if (warp < 6) {
            const int R = warp < 3 ? 0 : (warp < 5 ? 1 : 2);
            const int C = warp < 3 ? warp + 1 : (warp < 5 ? warp - 1 : 3);
            f[0] = ld(16 * R);
            f[1] = ld(16 * R + 8);
            f[2] = ld(16 * C);
            f[3] = ld(16 * C + 8);
            if (warp >= 4) f[4] = ld(8 * (2 * warp - 7));
        } else {
            const int d = warp - 6;
            f[0] = ld(16 * d);
            f[1] = ld(16 * d + 8);
            f[2] = ld(16 * (d + 2));
            f[3] = ld(16 * (d + 2) + 8);
        }
    }
    __device__ static void compute(int warp, const double (&f)[NFRAG], double (&acc)[NACC][2])
    {
        if (warp < 6) {
            dmma(acc[0][0], acc[0][1], f[0], f[2]);
            dmma(acc[1][0], acc[1][1], f[0], f[3]);
            dmma(acc[2][0], acc[2][1], f[1], f[2]);
            dmma(acc[3][0], acc[3][1], f[1], f[3]);
            if (warp >= 4) dmma(acc[4][0], acc[4][1], f[4], f[4]);
        } else {
            dmma(acc[0][0], acc[0][1], f[0], f[0]);
            dmma(acc[1][0], acc[1][1], f[0], f[1]);
            dmma(acc[2][0], acc[2][1], f[2], f[2]);
            dmma(acc[3][0], acc[3][1], f[2], f[3]);
            dmma(acc[4][0], acc[4][1], f[3], f[3]);
        }
    }
    template <class LD>
    __device__ static void mma(int warp, LD &&ld, double (&acc)[NACC][2])
    {
        if (warp < 6) {
            const int R = warp < 3 ? 0 : (warp < 5 ? 1 : 2);
            const int C = warp < 3 ? warp + 1 : (warp < 5 ? warp - 1 : 3);
            const double a0 = ld(16 * R), a1 = ld(16 * R + 8);
            const double b0 = ld(16 * C), b1 = ld(16 * C + 8);
            dmma(acc[0][0], acc[0][1], a0, b0);
            dmma(acc[1][0], acc[1][1], a0, b1);
            dmma(acc[2][0], acc[2][1], a1, b0);
            dmma(acc[3][0], acc[3][1], a1, b1);
            if (warp >= 4) {  // tile (1,1) (warp 4) or (3,3) (warp 5)
                const double e = ld(8 * (2 * warp - 7));
                dmma(acc[4][0], acc[4][1], e, e);
            }
        } else {
            // warp 6: (0,0) (0,1) (4,4) (4,5) (5,5); warp 7: (2,2) (2,3) (6,6) (6,7) (7,7)
            const int d = warp - 6;  // diagonal super-tiles d and d + 2
            const double f0 = ld(16 * d), f1 = ld(16 * d + 8);
            const double g0 = ld(16 * (d + 2)), g1 = ld(16 * (d + 2) + 8);
            dmma(acc[0][0], acc[0][1], f0, f0);
            dmma(acc[1][0], acc[1][1], f0, f1);
            dmma(acc[2][0], acc[2][1], g0, g0);
            dmma(acc[3][0], acc[3][1], g0, g1);
            dmma(acc[4][0], acc[4][1], g1, g1);
        }
    }
    // (row-tile, col-tile) of accumulator q of this warp; -1 if unused
    __device__ static void tile(int warp, int q, int &rt, int &ct)
    {
        rt = ct = -1;
        if (warp < 6) {
            const int R = warp < 3 ? 0 : (warp < 5 ? 1 : 2);
            const int C = warp < 3 ? warp + 1 : (warp < 5 ? warp - 1 : 3);
            if (q < 4) {
                rt = 2 * R + (q >> 1);
                ct = 2 * C + (q & 1);
            } else if (warp >= 4) {
                rt = ct = 2 * warp - 7;  // 1 or 3
            }
        } else {
            const int d = warp - 6;
            if (q == 0) { rt = 2 * d; ct = 2 * d; }
            else if (q == 1) { rt = 2 * d; ct = 2 * d + 1; }
            else if (q == 2) { rt = ct = 2 * (d + 2); }
            else if (q == 3) { rt = 2 * (d + 2); ct = 2 * (d + 2) + 1; }
            else { rt = ct = 2 * (d + 2) + 1; }
        }
    }
};

template <>
struct GramRoles<32> {
    static constexpr int NACC = 2;
    // upper 8x8 tiles of a 4x4 tile grid, in order
    __device__ static void tile(int warp, int q, int &rt, int &ct)
    {
        const int t = q == 0 ? warp : (warp < 2 ? 8 + warp : -1);
        rt = ct = -1;
        if (t < 0) return;
        // nibble t of the packed tables: R = 0,0,0,0,1,1,1,2,2,3  C = 0,1,2,3,1,2,3,2,3,3
        rt = (int)((0x3221110000ull >> (4 * t)) & 0xF);
        ct = (int)((0x3323213210ull >> (4 * t)) & 0xF);
    }
    template <class LD>
    __device__ static void mma(int warp, LD &&ld, double (&acc)[NACC][2])
    {
        int rt, ct;
        tile(warp, 0, rt, ct);
        dmma(acc[0][0], acc[0][1], ld(8 * rt), ld(8 * ct));
        if (warp < 2) {
            tile(warp, 1, rt, ct);
            dmma(acc[1][0], acc[1][1], ld(8 * rt), ld(8 * ct));
        }
    }
    static constexpr int NFRAG = 4;
    template <class LD>
    __device__ static void load(int warp, LD &&ld, double (&f)[NFRAG])
    {
        int rt, ct;
        tile(warp, 0, rt, ct);
        f[0] = ld(8 * rt);
        f[1] = ld(8 * ct);
        if (warp < 2) {
            tile(warp, 1, rt, ct);
            f[2] = ld(8 * rt);
            f[3] = ld(8 * ct);
        }
    }
    __device__ static void compute(int warp, const double (&f)[NFRAG], double (&acc)[NACC][2])
    {
        dmma(acc[0][0], acc[0][1], f[0], f[1]);
        if (warp < 2) dmma(acc[1][0], acc[1][1], f[2], f[3]);
    }
};

// Cross-block roles (kSlotCross): only the b x b block G_I^T G_J (8x8 tile
// rows 0..T-1, columns T..2T-1, T = b / 8).  B2 = 64: 16 tiles, two per
// warp (one A fragment, two B fragments); B2 = 32: 4 tiles on warps 0-3.
template <int B2>
struct GramRolesX {
    static constexpr int TT = B2 / 16;  // tiles per block side
    __device__ static void tile(int warp, int q, int &rt, int &ct)
    {
        rt = ct = -1;
        if (B2 == 64) {
            if (q < 2) {
                rt = warp >> 1;
                ct = TT + 2 * (warp & 1) + q;
            }
        } else if (q == 0 && warp < 4) {
            rt = warp >> 1;
            ct = TT + (warp & 1);
        }
    }
    static constexpr int NFRAG = 3;
    template <class LD>
    __device__ static void load(int warp, LD &&ld, double (&f)[NFRAG])
    {
        if (B2 == 64) {
            const int c0 = TT + 2 * (warp & 1);
            f[0] = ld(8 * (warp >> 1));
            f[1] = ld(8 * c0);
            f[2] = ld(8 * (c0 + 1));
        } else if (warp < 4) {
            f[0] = ld(8 * (warp >> 1));
            f[1] = ld(8 * (TT + (warp & 1)));
        }
    }
    template <int NACC>
    __device__ static void compute(int warp, const double (&f)[NFRAG], double (&acc)[NACC][2])
    {
        if (B2 == 64) {
            dmma(acc[0][0], acc[0][1], f[0], f[1]);
            dmma(acc[1][0], acc[1][1], f[0], f[2]);
        } else if (warp < 4) {
            dmma(acc[0][0], acc[0][1], f[0], f[1]);
        }
    }
    template <class LD, int NACC>
    __device__ static void mma(int warp, LD &&ld, double (&acc)[NACC][2])
    {
        if (B2 == 64) {
            const double a = ld(8 * (warp >> 1));
            const int c0 = TT + 2 * (warp & 1);
            const double b0 = ld(8 * c0), b1 = ld(8 * (c0 + 1));
            dmma(acc[0][0], acc[0][1], a, b0);
            dmma(acc[1][0], acc[1][1], a, b1);
        } else if (warp < 4) {
            dmma(acc[0][0], acc[0][1], ld(8 * (warp >> 1)), ld(8 * (TT + (warp & 1))));
        }
    }
};

template <int B2, int KT, int STAGES>
__global__ void __launch_bounds__(kThreads, HSVD_GRAM_OCC) k_gram(
    const double *__restrict__ G, int64_t ldg, int n, const int64_t *__restrict__ rho,
    const int64_t *__restrict__ iblk, const int64_t *__restrict__ jblk, GramPart part,
    int maxseg, double *__restrict__ Apart, const unsigned long long *err,
    const int32_t *__restrict__ act, const int32_t *__restrict__ nact,
    const uint8_t *__restrict__ skipf)
{
    using Sm = GramSmem<B2, KT, STAGES>;
    using Roles = GramRoles<B2>;
    extern __shared__ __align__(16) unsigned char gsm_raw[];
    auto &S = *reinterpret_cast<Sm *>(gsm_raw);
    if (*(volatile const unsigned long long *)err != kNoError) return;
    constexpr int b = B2 / 2;
    // reuse (k_plan): only the active slots act[0..nact) are computed; the
    // segments of the active slots are re-dealt over the grid in equal runs
    if (act) {
        const int64_t na = *nact;
        part.NS = na * part.NSEG;
        if (part.NS == 0) return;
        const int64_t per = (part.NS + part.P - 1) / part.P;
        part.P = (part.NS + per - 1) / per;
        if ((int64_t)blockIdx.x >= part.P) return;
    }
    const int64_t cta = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t it0 = part.begin(cta), it1 = part.begin(cta + 1);
    if (it1 <= it0) return;
    const int64_t slot0 = it0 / part.T;
    const int nsl = (int)((it1 - 1) / part.T - slot0 + 1);  // <= MAXSLOTS (host-checked)
    for (int q = tid; q < nsl * B2; q += kThreads) {
        const int si = q / B2, c = q % B2;
        const int64_t slot = act ? act[slot0 + si] : slot0 + si;
        int64_t I = iblk[slot], J = jblk[slot];
        if (I > J) { int64_t t = I; I = J; J = t; }
        S.col[si][c] = G + rho[slot_pos(c, b, I, J)] * ldg;
    }
    __syncthreads();

    constexpr int CHUNKS = B2 * (KT / 2);
    constexpr int PER_T = (CHUNKS + kThreads - 1) / kThreads;
    // the item stream (slot, k-tile) is walked with 32-bit counters: no
    // 64-bit division per k-tile
    const int T = (int)part.T, Lseg = (int)part.L;
    auto load_stage = [&](int st, int si, int kt) {
        const int k0 = kt * KT;
#pragma unroll
        for (int u = 0; u < PER_T; ++u) {
            const int q = tid + u * kThreads;
            if (q < CHUNKS) {
                const int c = q / (KT / 2), pp = q % (KT / 2);
                const int k = k0 + 2 * pp;
                const int rem = n - k;
                const int bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
                const double *src = bytes ? S.col[si][c] + k : S.col[si][c];
                cp_async16(&S.x[st][c][2 * pp], src, bytes);
            }
        }
    };

    double acc[Roles::NACC][2];
#pragma unroll
    for (int q = 0; q < Roles::NACC; ++q) acc[q][0] = acc[q][1] = 0.0;
    const int nitems = (int)(it1 - it0);
    const int kt0 = (int)(it0 - slot0 * part.T);
    int ld_si = 0, ld_k = kt0;  // next item to load
    auto ld_next = [&]() {
        if (++ld_k == T) {
            ld_k = 0;
            ++ld_si;
        }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nitems) {
            load_stage(s, ld_si, ld_k);
            ld_next();
        }
        cp_async_commit();
    }
    const int fr = lane >> 2, fk = lane & 3;
    int c_si = 0, c_k = kt0;  // item being computed
    int st_c = 0, st_l = STAGES - 1;
    for (int i = 0; i < nitems; ++i) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        if (i + STAGES - 1 < nitems) {
            load_stage(st_l, ld_si, ld_k);
            ld_next();
        }
        cp_async_commit();
        st_l = st_l + 1 == STAGES ? 0 : st_l + 1;
        const auto X = S.x[st_c];
        st_c = st_c + 1 == STAGES ? 0 : st_c + 1;
        const int64_t cslot = act ? act[slot0 + c_si] : slot0 + c_si;
        const bool cross = act && skipf[cslot] == kSlotCross;
        if (cross) {
#pragma unroll
            for (int kk = 0; kk < KT; kk += 4)
                GramRolesX<B2>::mma(warp, [&](int R) { return X[R + fr][kk + fk]; }, acc);
        } else {
#pragma unroll
            for (int kk = 0; kk < KT; kk += 4)
                Roles::mma(warp, [&](int R) { return X[R + fr][kk + fk]; }, acc);
        }
        // CTA runs start and end on segment boundaries, so every segment
        // is accumulated from zero by exactly one CTA
        const int seg = c_k / Lseg;
        const bool seg_end = c_k == T - 1 || c_k + 1 == (seg + 1) * Lseg;
        const int64_t slot = cslot;
        if (++c_k == T) {
            c_k = 0;
            ++c_si;
        }
        if (seg_end) {
            // flush this segment's partial (upper tiles only)
            double *out = Apart + (slot * maxseg + seg) * (B2 * B2);
#pragma unroll
            for (int q = 0; q < Roles::NACC; ++q) {
                int rt, ct;
                if (cross) GramRolesX<B2>::tile(warp, q, rt, ct);
                else Roles::tile(warp, q, rt, ct);
                if (rt >= 0) {
                    const int row = 8 * rt + fr, col = 8 * ct + 2 * fk;
                    out[row * B2 + col] = acc[q][0];
                    out[row * B2 + col + 1] = acc[q][1];
                }
                acc[q][0] = acc[q][1] = 0.0;
            }
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------
// k_gram_tma: the same partial Grams (same segments, same DMMA sequence,
// hence the same bits), operands brought in by TMA
// ---------------------------------------------------------------------
// A stage is KT rows of the CTA's B2 columns, stored as KT/16 sub-tiles of
// B2 x 128 bytes (16 doubles of one column per 128-byte line) with the
// 128-byte swizzle: the 16-byte chunk j of line L sits at chunk j ^ (L & 7).
// Columns are interleaved within each 8-line atom (consumer comment) so a
// DMMA fragment load is conflict-free without padding.  One producer warp issues the
// gather4 copies (4 columns through rho x 16 rows each; 64 per stage at
// b = 32) into a STAGES-deep ring of full/empty mbarriers; the 8 consumer
// warps keep the cp.async kernel's DMMA roles and accumulation order.
template <int B2, int KT, int STAGES>
struct GramTmaSmem {
    static constexpr int SUB = KT / 16;
    static constexpr int STAGE_BYTES = SUB * B2 * 128;
    static constexpr int MAXSLOTS = 4;
    alignas(1024) unsigned char x[STAGES][STAGE_BYTES];
    unsigned long long full[STAGES], empty[STAGES];
    int cidx[MAXSLOTS][B2];
    int64_t slot[MAXSLOTS];  // the CTA's slots (through the active list)
    int cross[MAXSLOTS];     // their Gram class (kSlotCross or not)
};

// One stage (KT rows) of a warp's DMMAs with the role resolved outside the
// k loop: the loop body is straight-line code, so the next k-step's
// fragment loads can be scheduled under the current k-step's DMMAs.
// NF fragments per k-step at byte offsets fo[] (row base * 128) from the
// lane's swizzled k-chunk; PAIRS lists the DMMAs as (A fragment, B
// fragment) into accumulators 0..ND-1 -- the same operations, in the same
// order, as GramRoles<64>::mma / GramRolesX<64>::mma.
template <int KT, int NF, int ND, class PAIRS, int NACC>
__device__ __forceinline__ void gram_stage(const unsigned char *xs, const unsigned (&off)[4],
                                           const int (&fo)[NF], double (&acc)[NACC][2],
                                           int sub_bytes)
{
    double fa[NF], fb[NF];
    auto load = [&](int kk, double (&f)[NF]) {
        const unsigned char *xq = xs + (kk >> 4) * sub_bytes + off[(kk >> 2) & 3];
#pragma unroll
        for (int j = 0; j < NF; ++j) f[j] = *(const double *)(xq + fo[j]);
    };
    auto comp = [&](const double (&f)[NF]) {
#pragma unroll
        for (int q = 0; q < ND; ++q)
            dmma(acc[q][0], acc[q][1], f[PAIRS::a(q)], f[PAIRS::b(q)]);
    };
    load(0, fa);
#pragma unroll
    for (int kk = 0; kk < KT; kk += 8) {
        load(kk + 4, fb);
        comp(fa);
        if (kk + 8 < KT) load(kk + 8, fa);
        comp(fb);
    }
}
// GramRoles<64> warps 0-5: 2x2 super-tile (a0 a1 b0 b1) [+ diagonal e]
struct PairsSuper {
    __device__ static constexpr int a(int q) { return q < 4 ? (q >> 1) : 4; }
    __device__ static constexpr int b(int q) { return q < 4 ? 2 + (q & 1) : 4; }
};
// GramRoles<64> warps 6-7: f0 f1 g0 g1 -> (f0 f0) (f0 f1) (g0 g0) (g0 g1) (g1 g1)
struct PairsDiag {
    __device__ static constexpr int a(int q) { return q < 2 ? 0 : (q < 4 ? 2 : 3); }
    __device__ static constexpr int b(int q) { return q == 0 ? 0 : (q == 1 ? 1 : (q == 2 ? 2 : 3)); }
};
// GramRolesX<64>: a b0 b1 -> (a b0) (a b1)
struct PairsCross {
    __device__ static constexpr int a(int) { return 0; }
    __device__ static constexpr int b(int q) { return 1 + q; }
};

// fragment row f of an 8-row group <-> line p(f) of the 8-line swizzle atom
__host__ __device__ constexpr int frag_line(int f) { return 2 * (f & 3) + (f >> 2); }

template <int B2, int KT, int STAGES, bool TILE>
__global__ void __launch_bounds__(kThreads + 32, HSVD_GRAM_TMA_OCC) k_gram_tma(
    const __grid_constant__ CUtensorMap gmap, int n, const int64_t *__restrict__ rho,
    const int64_t *__restrict__ iblk, const int64_t *__restrict__ jblk, GramPart part,
    int maxseg, double *__restrict__ Apart, const unsigned long long *err,
    const int32_t *__restrict__ act, const int32_t *__restrict__ nact,
    const uint8_t *__restrict__ skipf)
{
    using Sm = GramTmaSmem<B2, KT, STAGES>;
    using Roles = GramRoles<B2>;
    extern __shared__ __align__(1024) unsigned char gtm_raw[];
    // dynamic shared memory is only 16-byte aligned by contract: align up
    auto &S = *reinterpret_cast<Sm *>(
        gtm_raw + ((1024 - ((unsigned)__cvta_generic_to_shared(gtm_raw) & 1023)) & 1023));
    if (*(volatile const unsigned long long *)err != kNoError) return;
    constexpr int b = B2 / 2;
    if (act) {
        const int64_t na = *nact;
        part.NS = na * part.NSEG;
        if (part.NS == 0) return;
        const int64_t per = (part.NS + part.P - 1) / part.P;
        part.P = (part.NS + per - 1) / per;
        if ((int64_t)blockIdx.x >= part.P) return;
    }
    const int64_t cta = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t it0 = part.begin(cta), it1 = part.begin(cta + 1);
    if (it1 <= it0) return;
    const int64_t slot0 = it0 / part.T;
    const int nsl = (int)((it1 - 1) / part.T - slot0 + 1);  // <= MAXSLOTS (gram_slots_ok)
    for (int q = tid; q < nsl * B2; q += kThreads + 32) {
        const int si = q / B2, c = q % B2;
        const int64_t slot = act ? act[slot0 + si] : slot0 + si;
        int64_t I = iblk[slot], J = jblk[slot];
        if (I > J) { int64_t t = I; I = J; J = t; }
        S.cidx[si][c] = (int)rho[slot_pos(c, b, I, J)];
        if (c == 0) {
            // slot id and Gram class, read once here rather than through
            // two dependent global loads at every stage
            S.slot[si] = slot;
            S.cross[si] = act && skipf[slot] == kSlotCross;
        }
    }
    const unsigned full0 = (unsigned)__cvta_generic_to_shared(&S.full[0]);
    const unsigned empty0 = (unsigned)__cvta_generic_to_shared(&S.empty[0]);
    if (tid == 0) {
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(full0 + 8 * st, 1);
            mbar_init(empty0 + 8 * st, kThreads / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int T = (int)part.T, Lseg = (int)part.L;
    const int nitems = (int)(it1 - it0);
    const int kt0 = (int)(it0 - slot0 * part.T);
    const unsigned x0 = (unsigned)__cvta_generic_to_shared(&S.x[0][0]);

    if (warp == kThreads / 32) {
        // ---- producer warp
        int si = 0, k = kt0;
        for (int i = 0; i < nitems; ++i) {
            const int st = i % STAGES;
            const unsigned ph = (unsigned)(i / STAGES) & 1u;
            if (i >= STAGES) mbar_wait(empty0 + 8 * st, ph ^ 1u);
#if HSVD_GRAM_NOLOAD
            // diagnostic: no operand traffic (the stage is released at once)
            if (lane == 0) mbar_arrive(full0 + 8 * st);
            if (++k == T) {
                k = 0;
                ++si;
            }
            continue;
#endif
            if (lane == 0) mbar_expect_tx(full0 + 8 * st, Sm::STAGE_BYTES);
            __syncwarp();
            if (TILE) {
                // position-ordered storage: block I (J) of the slot is the
                // box {16 rows, b columns} at column I*b (J*b): 2 x SUB boxes
                if (lane < 2 * Sm::SUB) {
                    const int q = lane % Sm::SUB, h = lane / Sm::SUB;
                    const int col0 = S.cidx[si][h * b];
                    const unsigned dst = x0 + st * Sm::STAGE_BYTES + q * (B2 * 128) + h * (b * 128);
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
                        "l"(&gmap), "r"(k * KT + q * 16), "r"(col0), "r"(full0 + 8 * st)
                        : "memory");
                }
                if (++k == T) {
                    k = 0;
                    ++si;
                }
                continue;
            }
            constexpr int GROUPS = B2 / 4, OPS = Sm::SUB * GROUPS;
#pragma unroll
            for (int op = lane; op < OPS; op += 32) {
#if HSVD_GRAM_TMA_GMAJOR
                // consecutive ops walk one column group's k sub-tiles: each
                // column's KT*8 contiguous bytes are requested together
                const int g = op / Sm::SUB, q = op % Sm::SUB;
#else
                const int q = op / GROUPS, g = op % GROUPS;
#endif
                // lines 4h..4h+3 of the 8-line atom of columns 8a..8a+7 hold
                // columns {0,4,1,5} (h = 0) / {2,6,3,7} (h = 1): line 2f + f/4
                // for column f (see the consumer's offsets)
                const int *cc = &S.cidx[si][8 * (g >> 1) + 2 * (g & 1)];
                tma_gather4(x0 + st * Sm::STAGE_BYTES + q * (B2 * 128) + g * 512, &gmap,
                            k * KT + q * 16, cc[0], cc[4], cc[1], cc[5], full0 + 8 * st);
            }
            if (++k == T) {
                k = 0;
                ++si;
            }
        }
        return;
    }

    // ---- consumer warps: fragment offsets of this lane in a sub-tile.
    // Fragment row f of an 8-row group sits on line p = 2 (f & 3) + (f >> 2)
    // of its 1024-byte atom, so the 16 lanes of a half-warp (f = 0..3 or
    // 4..7, two k-chunks each) read 8 distinct swizzled chunks x 2 halves:
    // one wavefront per half-warp, no bank conflict.
    const int fr = lane >> 2, fk = lane & 3;
    const int lp = 2 * (fr & 3) + (fr >> 2);
    unsigned off[4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
        off[a] = (unsigned)(lp * 128 + ((((2 * a) | (fk >> 1)) ^ lp) << 4) + (fk & 1) * 8);
    // fragment row bases (x 128 bytes) of this warp's role (B2 = 64; the
    // same rows GramRoles<64> / GramRolesX<64> read)
    int fo4[4], fo5[5], foX[3];
    {
        const int R = warp < 3 ? 0 : (warp < 5 ? 1 : 2);
        const int C = warp < 3 ? warp + 1 : (warp < 5 ? warp - 1 : 3);
        const int d = warp - 6;
        const bool diag = warp >= 6;
        fo4[0] = (diag ? 16 * d : 16 * R) * 128;
        fo4[1] = (diag ? 16 * d + 8 : 16 * R + 8) * 128;
        fo4[2] = (diag ? 16 * (d + 2) : 16 * C) * 128;
        fo4[3] = (diag ? 16 * (d + 2) + 8 : 16 * C + 8) * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) fo5[j] = fo4[j];
        fo5[4] = (warp >= 4 && warp < 6 ? 8 * (2 * warp - 7) : 0) * 128;
        const int c0 = B2 / 16 + 2 * (warp & 1);
        foX[0] = 8 * (warp >> 1) * 128;
        foX[1] = 8 * c0 * 128;
        foX[2] = 8 * (c0 + 1) * 128;
    }
    double acc[Roles::NACC][2];
#pragma unroll
    for (int q = 0; q < Roles::NACC; ++q) acc[q][0] = acc[q][1] = 0.0;
    int c_si = 0, c_k = kt0;
    int c_seg = kt0 / Lseg, c_in = kt0 % Lseg;  // segment, k-tiles done in it
    for (int i = 0; i < nitems; ++i) {
        const int st = i % STAGES;
        const unsigned ph = (unsigned)(i / STAGES) & 1u;
        const int64_t slot = S.slot[c_si];
        const bool cross = S.cross[c_si] != 0;
        mbar_wait(full0 + 8 * st, ph);
        const unsigned char *xs = S.x[st];
        // fragments of k-step kk + 4 are loaded while k-step kk's DMMAs run
        // (two register sets): the loads no longer wait for the previous
        // DMMAs to release their operand registers
        auto ldk = [&](int kk) {
            const unsigned char *xq = xs + (kk >> 4) * (B2 * 128) + off[(kk >> 2) & 3];
            return [xq](int R) { return *(const double *)(xq + R * 128); };
        };
        if (HSVD_GRAM_NOMATH) {
            // diagnostic: no DMMA (data movement floor)
        } else if (B2 == 64) {
            constexpr int SB = B2 * 128;
            if (cross) {
                gram_stage<KT, 3, 2, PairsCross>(xs, off, foX, acc, SB);
            } else if (warp < 4) {
                gram_stage<KT, 4, 4, PairsSuper>(xs, off, fo4, acc, SB);
            } else if (warp < 6) {
                gram_stage<KT, 5, 5, PairsSuper>(xs, off, fo5, acc, SB);
            } else {
                gram_stage<KT, 4, 5, PairsDiag>(xs, off, fo4, acc, SB);
            }
        } else if (cross) {
            using RX = GramRolesX<B2>;
            double fa[RX::NFRAG], fb[RX::NFRAG];
            RX::load(warp, ldk(0), fa);
#pragma unroll
            for (int kk = 0; kk < KT; kk += 8) {
                RX::load(warp, ldk(kk + 4), fb);
                RX::compute(warp, fa, acc);
                if (kk + 8 < KT) RX::load(warp, ldk(kk + 8), fa);
                RX::compute(warp, fb, acc);
            }
        } else {
            double fa[Roles::NFRAG], fb[Roles::NFRAG];
            Roles::load(warp, ldk(0), fa);
#pragma unroll
            for (int kk = 0; kk < KT; kk += 8) {
                Roles::load(warp, ldk(kk + 4), fb);
                Roles::compute(warp, fa, acc);
                if (kk + 8 < KT) Roles::load(warp, ldk(kk + 8), fa);
                Roles::compute(warp, fb, acc);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * st);
        // segment bookkeeping without a division per stage
        const int seg = c_seg;
        const bool seg_end = c_k == T - 1 || ++c_in == Lseg;
        if (seg_end) {
            c_in = 0;
            ++c_seg;
        }
        if (++c_k == T) {
            c_k = 0;
            c_seg = 0;
            ++c_si;
        }
        if (seg_end) {
            double *out = Apart + (slot * maxseg + seg) * (B2 * B2);
#pragma unroll
            for (int q = 0; q < Roles::NACC; ++q) {
                int rt, ct;
                if (cross) GramRolesX<B2>::tile(warp, q, rt, ct);
                else Roles::tile(warp, q, rt, ct);
                if (rt >= 0) {
                    if (TILE) {
                        // fragment row f read column 8t + p(f) (natural
                        // line order in shared memory)
                        const int row = 8 * rt + frag_line(fr);
                        out[row * B2 + 8 * ct + frag_line(2 * fk)] = acc[q][0];
                        out[row * B2 + 8 * ct + frag_line(2 * fk + 1)] = acc[q][1];
                    } else {
                        const int row = 8 * rt + fr, col = 8 * ct + 2 * fk;
                        out[row * B2 + col] = acc[q][0];
                        out[row * B2 + col + 1] = acc[q][1];
                    }
                }
                acc[q][0] = acc[q][1] = 0.0;
            }
        }
    }
}

// The factor's storage as a 2D tensor for k_gram_tma: dim 0 = rows (n,
// contiguous), dim 1 = storage columns (ld doubles apart); box 16 x 1 with
// the 128-byte swizzle (gather4 takes 4 dim-1 coordinates per copy).
// Rows >= n read as zero.  Returns 0 on success.
int make_gram_tensor_map(CUtensorMap *tm, const double *G, int64_t ld, int64_t n, int64_t ncols,
                         int box_cols = 1);

// ---------------------------------------------------------------------
// k_inner: one pass of 2x2 rotations on the 2b x 2b pivot Gram
// ---------------------------------------------------------------------
struct InnerArgs {
    GramPart part;
    int maxseg;
    const double *Apart;
    double *Wg;
    const int64_t *jsign;
    int64_t *ip, *jp, *iblk, *jblk, *cur;
    uint8_t *C;
    uint32_t *rotk, *skipk;
    uint8_t *tset;  // per slot: [count, touched columns...], kTsetStride bytes
    const int64_t *colmap;  // position -> storage column
    const int64_t *orig;    // position -> original column (padding test)
    int64_t *colidx;        // per slot: storage column of each of its 2b columns
    double *maxt;
    unsigned long long *err;
    int64_t nb, slot_base;
    int64_t real_cols;  // colmap values >= real_cols are inert padding columns
    ReuseWs ru;         // all-skip reuse bookkeeping (pairstamp NULL: off)
    const uint8_t *skipf;  // per slot: 1 = reused all-skip visit (k_plan)
    int step;
    double eps, teps;
    int full, use_skip, passes;
    long long *trace;  // debug: per-round clock64 stamps of CTA 0 (NULL)
};

// Touched-column set of a slot visit: the columns of P that took part in at
// least one rotation.  W_P is the identity outside T x T, so the update only
// has to rewrite the columns in T.
constexpr int kTsetStride = 72;   // count byte + up to 64 column indices
constexpr int kSparseMax = 24;    // |T| <= this: column update without DMMA

template <int B2>
struct InnerSmem {
    static constexpr int LD = B2 + 1;
    double A[B2][LD];
    double W[B2][LD];
    // the round's rotations (written by warp 0, read after the barrier)
    double4 prm[2][B2 / 2];  // (t, c, st, -) of the round, by round parity
    int flag[2];             // bit 0: some pair rotated, bit 1: a pair failed
    int js[B2];
    unsigned int jneg[2], padm[2];  // per-column bit masks (J = -1, padding)
    unsigned int rot, skip, big;
    unsigned long long maxt_bits;
    unsigned long long fail;
    unsigned long long touched;
};

// Plain-double annihilating rotation for block mode (the pointwise mode keeps
// the reference's double-double rotation_tc, hsvd_rotation.cuh).  Same
// branches, sign convention and definiteness test as rotation_tc
// (_kernels.py:128-173), rewritten to one division and one square root:
//   trig (d = a_jj - a_ii, e = 2 a_ij, zeta = d / e):
//     t = sgn(zeta) |e| / (|d| + sqrt(d^2 + e^2)),   c = 1 / sqrt(1 + t^2)
//     (= sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)); for |zeta| > 6.7e7 it is
//     the reference's 1 / (2 zeta) to rounding, and c rounds to 1);
//   hyperbolic (s = a_ii + a_jj, theta = -e / s):
//     t = -e / (s + sqrt((s - |e|)(s + |e|))),       c = 1 / sqrt(1 - t^2)
//     (= theta / (1 + sqrt(1 - theta^2)); |theta| >= 1 -> status 1).
// Operands beyond 1e150 take the reference's quotient form (no overflow).
__device__ __forceinline__ int rotation_fast_wide(double a_ii, double a_jj, double a_ij, int hyp,
                                               double &t_out, double &c_out)
{
    // operands beyond 1e150: the reference's quotient forms (no overflow)
    t_out = 0.0;
    c_out = 1.0;
    const double e = 2.0 * a_ij;
    if (hyp < 0) {
        const double zeta = (a_jj - a_ii) / e;
        if (fabs(zeta) > 6.7e7) {
            t_out = 0.5 / zeta;
            return 0;
        }
        const double az = fabs(zeta);
        double t = 1.0 / (az + sqrt(fma(az, az, 1.0)));
        if (!(zeta >= 0.0)) t = -t;
        t_out = t;
        c_out = rsqrt(fma(t, t, 1.0));
        return 0;
    }
    const double th = -e / (a_ii + a_jj);
    const double D = fma(-th, th, 1.0);
    if (!(D > 0.0)) return 1;
    const double t = th / (1.0 + sqrt(D));
    const double u = fma(-t, t, 1.0);
    if (!(u > 0.0)) return 1;
    t_out = t;
    c_out = rsqrt(u);
    return 0;
}

// Branch-free FP64 reciprocal, reciprocal square root and square root for
// the rotation's critical chain: the hardware approximation (MUFU) refined by
// two Newton steps (error ~2^-20 -> ~2^-80, i.e. within an ulp or so), for
// positive normal operands in [1e-300, 1e300].  The library routines carry a
// slow-path branch each, which keeps the compiler from overlapping them.
#ifndef HSVD_ROT_LIBM  // 1: the library's correctly rounded sqrt / rsqrt / division
#define HSVD_ROT_LIBM 0
#endif
__device__ __forceinline__ double fast_rcp(double x)
{
    if (HSVD_ROT_LIBM) return 1.0 / x;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
// 1/x to ~2^-45 (seed + one Newton step): enough ahead of a quotient's
// correction step, which squares the error
__device__ __forceinline__ double rcp_nr1(double x)
{
    if (HSVD_ROT_LIBM) return 1.0 / x;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return fma(y, fma(-x, y, 1.0), y);
}
__device__ __forceinline__ double fast_rsqrt(double x)
{
    if (HSVD_ROT_LIBM) return rsqrt(x);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);  // 1 - x y^2
    y = fma(0.5 * y, e, y);                 // ~2^-45 from the ~2^-23 seed
    // last step with the residual x y^2 - 1 formed nearly exactly (y^2 and
    // its rounding error by FMA): within ~0.5 ulp, like the library rsqrt
    // (measured, tools/rsqrt_acc.cu; two plain Newton steps: up to 0.99 ulp)
    const double p = y * y, pe = fma(y, y, -p);
    const double r = fma(x, p, -1.0) + x * pe;
    return fma(-0.5 * y, r, y);
}
__device__ __forceinline__ double fast_sqrt(double x)
{
    if (HSVD_ROT_LIBM) return sqrt(x);
    // one Newton step of 1/sqrt(x) (~2^-45) suffices before the correction
    // of x y (the correction squares the error)
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
    const double s = x * y;
    return fma(0.5 * y, fma(-s, s, x), s);  // one correction of x y
}

// c of the rotation.  HSVD_ROT_C_FROM_T=1: c = 1/sqrt(1 +- t^2) from the
// rounded t with the library's reciprocal square root (the round-1 form:
// each (t, c) pair J-orthogonal to the last bits); 0: c = w / sqrt(w^2 +- e^2)
// beside the quotient (one long operation fewer on the chain)
#ifndef HSVD_ROT_C_FROM_T
#define HSVD_ROT_C_FROM_T 1
#endif
__device__ __forceinline__ double rot_c(double t, bool h, double w, double g)
{
    if (HSVD_ROT_C_FROM_T) return fast_rsqrt(fma(h ? -t : t, t, 1.0));
    return w * fast_rsqrt(g);
}

// The trigonometric and hyperbolic forms share one square root, one
// reciprocal and one reciprocal square root, selected per lane: a warp whose
// pairs mix both kinds (every pivot block that straddles the sign boundary)
// runs one dependent chain instead of both branches one after the other.
//   w = base + sqrt(rad),  t = num / w,  c = 1 / sqrt(1 +- t^2) = w / sqrt(w^2 +- e^2)
// so the quotient and c's reciprocal square root run side by side.
__device__ __forceinline__ int rotation_fast(double a_ii, double a_jj, double a_ij, int hyp,
                                             double &t_out, double &c_out)
{
    t_out = 0.0;
    c_out = 1.0;
    if (a_ij == 0.0) return 0;
    const double e = 2.0 * a_ij, ae = fabs(e);
    const bool h = hyp > 0;
    const double d = a_jj - a_ii, ad = fabs(d), sm = a_ii + a_jj;
    const double base = h ? sm : ad;
    const double big = fmax(base, ae);
    // operands beyond 1e150 or below 1e-140: the quotient forms
    if (!(big < 1e150 && big > 1e-140)) return rotation_fast_wide(a_ii, a_jj, a_ij, hyp, t_out, c_out);
    const double sg = (d == 0.0 || (d > 0.0) == (e > 0.0)) ? ae : -ae;
    const double num = h ? -e : sg;
    const double rad = h ? (sm - ae) * (sm + ae) : fma(d, d, e * e);
    if (h && !(rad > 0.0)) return 1;
    const double w = base + fast_sqrt(rad);
    const double g = h ? (w - ae) * (w + ae) : fma(w, w, ae * ae);
    if (h && !(g > 0.0)) return 1;
    const double rw = rcp_nr1(w);
    double t = num * rw;
    t = fma(fma(-w, t, num), rw, t);  // one correction of the quotient
    t_out = t;
    c_out = rot_c(t, h, w, g);
    return 0;
}

// rotation_fast without branches, for a warp none of whose operands needs
// the quotient forms (the caller checks rotation_fast_in_range with a vote):
// the same operations and results as rotation_fast, with the zero,
// definiteness and range exits turned into selects, so the operand-only part
// (d, sm, base) can be scheduled before a_ij arrives
__device__ __forceinline__ bool rotation_fast_in_range(double a_ii, double a_jj, double a_ij, int hyp)
{
    const double ae = fabs(2.0 * a_ij);
    const double base = hyp > 0 ? a_ii + a_jj : fabs(a_jj - a_ii);
    const double big = fmax(base, ae);
    return a_ij == 0.0 || (big < 1e150 && big > 1e-140);
}
__device__ __forceinline__ int rotation_fast_sel(double a_ii, double a_jj, double a_ij, int hyp,
                                                 double &t_out, double &c_out)
{
    const bool h = hyp > 0;
    const double d = a_jj - a_ii, ad = fabs(d), sm = a_ii + a_jj;
    const double base = h ? sm : ad;
    const double e = 2.0 * a_ij, ae = fabs(e);
    const double sg = (d == 0.0 || (d > 0.0) == (e > 0.0)) ? ae : -ae;
    const double num = h ? -e : sg;
    const double rad = h ? (sm - ae) * (sm + ae) : fma(d, d, e * e);
    const bool radok = rad > 0.0;
    const double w = base + fast_sqrt(radok ? rad : 1.0);
    const double g = h ? (w - ae) * (w + ae) : fma(w, w, ae * ae);
    const bool gok = g > 0.0;
    const double rw = rcp_nr1(w);
    double t = num * rw;
    t = fma(fma(-w, t, num), rw, t);  // one correction of the quotient
    const double c = rot_c(t, h, w, gok ? g : 1.0);
    const bool zero = a_ij == 0.0;
    const bool bad = !zero && h && !(radok && gok);
    t_out = zero || bad ? 0.0 : t;
    c_out = zero || bad ? 1.0 : c;
    return bad ? 1 : 0;
}

// k_inner_v1: the round-1 inner pass (both triangles of A and W in shared
// memory, warp 0 forms the rotations, two barriers per round).  The product
// runs k_inner (hsvd_inner.cuh); this kernel stays only as the A/B and
// cross-check reference of tools/inner_bench.cu (it is never instantiated by
// the library).
//
// A round's b pairs are disjoint, so the round is the congruence
// A <- R^T A R with R block-diagonal in 2x2 blocks: every 2x2 block (p, q) of
// A (rows {i_p, j_p}, columns {i_q, j_q}) becomes R_p^T A_pq R_q on its own.
// threads of one k_inner_v1 CTA
constexpr int kInnerThreads = HSVD_INNER_THREADS;
template <int B2>
__host__ __device__ constexpr int inner_threads() { return B2 == 64 ? kInnerThreads : 256; }

// cur = the visited pair; advance_stepper (_kernels.py:238-251) on the
// block indices
__device__ __forceinline__ void inner_advance(const InnerArgs &a, int slot, int64_t I, int64_t J)
{
    a.cur[2 * slot] = I;
    a.cur[2 * slot + 1] = J;
    const int64_t r = a.nb, half = r / 2;
    int64_t ip = a.ip[slot], jp = a.jp[slot];
    if (ip + jp >= r - 1) {
        ip += 1;
        if (ip == jp) {
            ip -= half;
            jp = ip;
        }
        a.ip[slot] = ip;
        a.jp[slot] = jp;
        a.iblk[slot] = ip;
    } else {
        jp += 1;
        a.jp[slot] = jp;
        a.jblk[slot] = jp;
    }
}

// k_plan: which slots of this step replay a recorded all-skip visit, and
// the ordered list of the others (one CTA, one thread per slot: three loads
// decide a slot, then a block-wide ordered compaction)
constexpr int kPlanThreads = 1024;
static __global__ void __launch_bounds__(kPlanThreads) k_plan(const int64_t *__restrict__ iblk,
                                                       const int64_t *__restrict__ jblk,
                                                       int64_t nslots, int64_t nb, ReuseWs ru,
                                                       int step, int full,
                                                       uint8_t *__restrict__ skipf,
                                                       int32_t *__restrict__ act,
                                                       int32_t *__restrict__ nact,
                                                       const unsigned long long *err)
{
    __shared__ int wcnt[kPlanThreads / 32];
    __shared__ int base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t stamp = reuse_stamp(ru.dsweep, nb, step);
    const bool failed = *(volatile const unsigned long long *)err != kNoError;
    if (tid == 0) base = 0;
    for (int64_t s0 = 0; s0 < nslots; s0 += kPlanThreads) {
        const int64_t slot = s0 + tid;
        int sk = 0;
        uint8_t cls = kSlotFull;
        if (slot < nslots && !failed) {
            int64_t I = iblk[slot], J = jblk[slot];
            if (I > J) { int64_t t = I; I = J; J = t; }
            const uint32_t ps = ru.pairstamp[I * nb + J];
            const uint32_t m = max(ru.blkmod[I], ru.blkmod[J]);
            const uint32_t at = ps & 0x7fffffffu;
            sk = ps != 0u && (int)(ps >> 31) >= (full != 0) && m < at && at < stamp;
            if (!sk && ru.dcache) {
                const uint32_t dI = ru.dstamp[I], dJ = ru.dstamp[J];
                cls = dI != 0u && dJ != 0u && ru.blkmod[I] < dI && ru.blkmod[J] < dJ
                          ? kSlotCross : kSlotFull;
            }
        }
        if (slot < nslots) {
            const uint8_t c = sk ? kSlotReused : cls;
            skipf[slot] = c;
            atomicAdd(&ru.planstat[c], 1ull);
        }
        const int live = slot < nslots && !sk;
        const unsigned bal = __ballot_sync(0xffffffffu, live);
        if (lane == 0) wcnt[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {
            // exclusive scan of the warp counts
            const int v = wcnt[lane];
            int x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            wcnt[lane] = x - v;
        }
        __syncthreads();
        if (live) act[base + wcnt[warp] + __popc(bal & ((1u << lane) - 1u))] = (int32_t)slot;
        __syncthreads();
        if (tid == kPlanThreads - 1) base += wcnt[warp] + __popc(bal);
        __syncthreads();
    }
    if (tid == 0) *nact = base;
}

// sweep end: blocks whose positions received another column in the sort
// are stamped, then the sweep counter advances (one CTA per 256 positions)
static __global__ void k_reuse_sweep_end(const int64_t *__restrict__ rho,
                                  const int64_t *__restrict__ rho_prev, int64_t r, int b,
                                  int64_t nb, ReuseWs ru)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const uint32_t stamp = reuse_stamp(ru.dsweep, nb, (int)nb);
    if (k < r && rho[k] != rho_prev[k]) ru.blkmod[k / b] = stamp;
}
static __global__ void k_reuse_next_sweep(int32_t *dsweep) { *dsweep += 1; }

template <int B2, bool FAST>
__global__ void __launch_bounds__(inner_threads<B2>()) k_inner_v1(InnerArgs a)
{
    constexpr int NT = inner_threads<B2>();
    extern __shared__ __align__(16) unsigned char ism_raw[];
    auto &S = *reinterpret_cast<InnerSmem<B2> *>(ism_raw);
    if (*(volatile unsigned long long *)a.err != kNoError) return;
    constexpr int b = B2 / 2;    // pairs per round
    const int slot = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int64_t I = a.iblk[slot], J = a.jblk[slot];
    if (I > J) { int64_t t = I; I = J; J = t; }
    if (a.skipf && a.skipf[slot] == kSlotReused) {
        // reused all-skip visit: the recorded statistics, no rotation, no
        // update (empty touched set), stepper advanced as usual
        if (tid == 0) {
            a.tset[(int64_t)slot * kTsetStride] = 0;
            a.skipk[slot] += a.ru.pairskip[I * a.nb + J];
            inner_advance(a, slot, I, J);
        }
        return;
    }

    // A = sum of the slot's partial segments in segment order (the upper
    // triangle is read coalesced and mirrored); all loads of a batch of
    // segments are issued before the sums
    const double *P0 = a.Apart + (int64_t)slot * a.maxseg * (B2 * B2);
    const int nseg = (int)a.part.NSEG;
    constexpr int PER = B2 * B2 / NT;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int e = tid + k * NT, i = e / B2, j = e % B2;
        S.W[i][j] = i == j ? 1.0 : 0.0;
    }
    {
        // cross class: the two diagonal blocks come from the cache, only the
        // cross block from the partials (the same segment folds as a fresh
        // visit, so the same bits)
        const bool cross = a.skipf && a.skipf[slot] == kSlotCross;
        double v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) v[k] = 0.0;
        constexpr int BATCH = 2;
        for (int s0 = 0; s0 < nseg; s0 += BATCH) {
            double x[BATCH][PER];
#pragma unroll
            for (int u = 0; u < BATCH; ++u)
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const int e = tid + k * NT, i = e / B2, j = e % B2;
                    x[u][k] = (s0 + u < nseg && i <= j && (!cross || (i < b && j >= b)))
                                  ? P0[(int64_t)(s0 + u) * B2 * B2 + e] : 0.0;
                }
#pragma unroll
            for (int u = 0; u < BATCH; ++u)
#pragma unroll
                for (int k = 0; k < PER; ++k)
                    if (s0 + u < nseg) v[k] += x[u][k];
        }
        const bool cache = a.ru.dcache != nullptr;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid + k * NT, i = e / B2, j = e % B2;
            if (i <= j) {
                const bool dI = j < b, dJ = i >= b;  // inside a diagonal block
                if (cross && (dI || dJ)) {
                    v[k] = dI ? a.ru.dcache[(I * b + i) * b + j]
                              : a.ru.dcache[(J * b + (i - b)) * b + (j - b)];
                } else if (cache && !cross && (dI || dJ)) {
                    if (dI) a.ru.dcache[(I * b + i) * b + j] = v[k];
                    else a.ru.dcache[(J * b + (i - b)) * b + (j - b)] = v[k];
                }
                S.A[i][j] = v[k];
                S.A[j][i] = v[k];
            }
        }
    }
    if (tid < B2) {
        const int64_t pos = slot_pos(tid, b, I, J);
        const int neg = a.jsign[pos] < 0;
        const int pad = a.orig[pos] >= a.real_cols;
        S.js[tid] = neg ? -1 : 1;
        const unsigned mneg = __ballot_sync(0xffffffffu, neg);
        const unsigned mpad = __ballot_sync(0xffffffffu, pad);
        if (lane == 0) {
            S.jneg[warp] = mneg;
            S.padm[warp] = mpad;
        }
    }
    if (tid == 0) {
        S.rot = S.skip = S.big = 0;
        S.maxt_bits = 0;
        S.fail = kNoError;
        S.touched = 0;
    }
    __syncthreads();

    const int rounds = a.full ? B2 - 1 : b;
    unsigned int my_rot = 0, my_skip = 0, my_big = 0;
    unsigned long long my_touch = 0;
    double my_max = 0.0;
    static_assert(b == 16 || b == 32, "k_inner: b must be 16 or 32");
    constexpr int PSTRIDE = NT / b;   // row-pair stride of phase U
    constexpr int NBK = b * b / NT;   // A blocks per thread per round
    const int q = lane % b;                 // pair owned by this thread
    const int prow = tid / b;
    long long *tr = (a.trace && blockIdx.x == 0 && tid == 0) ? a.trace : nullptr;
#define HSVD_STAMP(k) \
    if (tr && it < 64) tr[8 * it + (k)] = clock64();
    // negative-sign and padding columns as bit masks (ballots above): hyp
    // without a shared-memory load per pair
    const unsigned long long jneg =
        B2 == 64 ? ((unsigned long long)S.jneg[1] << 32) | S.jneg[0] : S.jneg[0];
    const unsigned long long padm =
        B2 == 64 ? ((unsigned long long)S.padm[1] << 32) | S.padm[0] : S.padm[0];
    // columns of pair x in round rd (circle method on B2 players, or the
    // block-oriented pairing x <-> b + (x + rd) mod b)
    auto pair_cols = [&](int x, int rd, int &ci, int &cj) {
        if (a.full) {
            constexpr int m = B2 - 1;
            if (x == 0) { ci = m; cj = rd; }
            else {
                ci = rd + x;
                if (ci >= m) ci -= m;
                cj = rd - x;
                if (cj < 0) cj += m;
            }
        } else {
            ci = x;
            cj = rd + x;
            if (cj >= b) cj -= b;
            cj += b;
        }
    };
    // W <- W R of round wrd (parameters prm[wpar]) on the W worker rows:
    // warps 1-3 and 5-7 (every SM sub-partition but warp 0's), pair q =
    // lane % b, rows g, g + WG, ...
    constexpr int NWW = (NT / 32) * 3 / 4;  // W worker warps
    constexpr int WG = NWW * 32 / b;
    const int wwarp = (warp & 3) - 1 + 3 * (warp >> 2);  // 0..5 unless warp % 4 == 0
    const int wg = lane / b + (32 / b) * wwarp;
    auto w_update = [&](int wrd, int wpar) {
        const double4 r4 = S.prm[wpar][q];
        const double tw = r4.x, cw = r4.y, sw = r4.z;
        if (tw == 0.0) return;
        int wi, wj;
        pair_cols(q, wrd, wi, wj);
        constexpr int NR = (B2 + WG - 1) / WG;
        double wx[NR], wy[NR];
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const int row = wg + k * WG;
            if (row < B2) {
                wx[k] = S.W[row][wi];
                wy[k] = S.W[row][wj];
            }
        }
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const int row = wg + k * WG;
            if (row < B2) {
                S.W[row][wi] = fma(sw, wy[k], wx[k]) * cw;
                S.W[row][wj] = fma(tw, wx[k], wy[k]) * cw;
            }
        }
    };
    const bool w_worker = (warp & 3) != 0;
    int rd = 0, prev_rd = 0;
    bool prev_act = false, failed = false;
    for (int it = 0; it < rounds * a.passes; ++it, rd = rd + 1 == rounds ? 0 : rd + 1) {
        HSVD_STAMP(0)
        const int par = it & 1;
        if (warp == 0) {
            // ---- phase R: warp 0 forms the round's b rotations.  The pair
            // is rotated in its schedule orientation (i, j), not sorted: lane
            // q then walks consecutive columns (no bank conflicts), and the
            // closed forms are odd (trig: t -> -t when the roles swap) or
            // symmetric (hyperbolic) in the roles, so this is the sorted
            // form's transformation bit for bit except at exactly zeta = 0;
            // the upper copy of a_ij is read, as in the sorted form
            int i, j;
            pair_cols(q, rd, i, j);
            const int lo = i < j ? i : j, hi = i < j ? j : i;
            const double a_ii = S.A[i][i], a_jj = S.A[j][j], a_ij = S.A[lo][hi];
            double t = 0.0, c = 1.0, st = 0.0;
            int act = 0, bad = 0;
            // relative-orthogonality skip |a_ij| < eps sqrt(a_ii a_jj)
            // (_kernels.py:211), squared: no square root on the critical path
            if (!(a_ij == 0.0 ||
                  (a.use_skip && a_ij * a_ij < (a.eps * a.eps) * (a_ii * a_jj)))) {
                const int hyp = (((jneg >> i) ^ (jneg >> j)) & 1) ? 1 : -1;
                const int status = FAST ? rotation_fast(a_ii, a_jj, a_ij, hyp, t, c)
                                        : rotation_tc(a_ii, a_jj, a_ij, hyp, t, c);
                if (status != 0) {
                    bad = 1;
                    t = 0.0;
                    c = 1.0;
                } else {
                    act = 1;
                    st = hyp < 0 ? -t : t;
                }
            }
            if (lane < b) S.prm[par][q] = make_double4(t, c, st, 0.0);
            const unsigned va = __ballot_sync(0xffffffffu, act), vb = __ballot_sync(0xffffffffu, bad);
            if (lane == 0) S.flag[par] = (va ? 1 : 0) | (vb ? 2 : 0);
            // statistics after the publication (off the round's critical path)
            if (lane < b) {
                if (bad) atomicMin(&S.fail, pack_err(a.slot_base + slot, slot_pos(lo, b, I, J),
                                                     slot_pos(hi, b, I, J)));
                else if (act) {
                    ++my_rot;
                    my_touch |= (1ull << i) | (1ull << j);
                    const double at = fabs(t);
                    my_big |= at > a.teps;
                    my_max = fmax(my_max, at);
                } else if (!(((padm >> i) | (padm >> j)) & 1)) {
                    ++my_skip;  // pairs with a padding column are not visits
                }
            }
        } else if (w_worker && prev_act) {
            // the previous round's W update runs beside this round's rotations
            w_update(prev_rd, par ^ 1);
        }
        HSVD_STAMP(1)
        __syncthreads();  // the round's rotations are published
        HSVD_STAMP(2)
        const int f = S.flag[par];
        if (f & 2) { failed = true; break; }
        prev_act = f & 1;
        prev_rd = rd;
        if (!prev_act) continue;
        // ---- phase U (A only).  This thread owns pair q as the column pair
        // of blocks (p, q), p = prow + k * PSTRIDE.
        {
            int i, j;
            pair_cols(q, rd, i, j);
            const double4 rq = S.prm[par][q];
            const double t = rq.x, c = rq.y, st = rq.z;
            double x[NBK][4], tp[NBK], cp[NBK], sp[NBK];
            int ip[NBK], jp[NBK];
#pragma unroll
            for (int k = 0; k < NBK; ++k) {
                const int p = prow + k * PSTRIDE;
                const double4 r4 = S.prm[par][p];
                tp[k] = r4.x;
                cp[k] = r4.y;
                sp[k] = r4.z;
                pair_cols(p, rd, ip[k], jp[k]);
                x[k][0] = S.A[ip[k]][i];
                x[k][1] = S.A[ip[k]][j];
                x[k][2] = S.A[jp[k]][i];
                x[k][3] = S.A[jp[k]][j];
            }
#pragma unroll
            for (int k = 0; k < NBK; ++k) {
                if (t == 0.0 && tp[k] == 0.0) continue;
                // Y = X R_q (columns), X' = R_p^T Y (rows)
                const double y00 = fma(st, x[k][1], x[k][0]) * c;
                const double y01 = fma(t, x[k][0], x[k][1]) * c;
                const double y10 = fma(st, x[k][3], x[k][2]) * c;
                const double y11 = fma(t, x[k][2], x[k][3]) * c;
                S.A[ip[k]][i] = fma(sp[k], y10, y00) * cp[k];
                S.A[jp[k]][j] = fma(tp[k], y01, y11) * cp[k];
                if (prow + k * PSTRIDE == q) {  // the pair itself: annihilated
                    S.A[ip[k]][j] = 0.0;
                    S.A[jp[k]][i] = 0.0;
                } else {
                    S.A[ip[k]][j] = fma(sp[k], y11, y01) * cp[k];
                    S.A[jp[k]][i] = fma(tp[k], y00, y10) * cp[k];
                }
            }
        }
        HSVD_STAMP(3)
        __syncthreads();  // the round's updates are visible
        HSVD_STAMP(4)
    }
    // the last active round's W update
    if (!failed && prev_act && w_worker) w_update(prev_rd, ((rounds * a.passes) - 1) & 1);
#undef HSVD_STAMP
    if (warp == 0) {
        atomicAdd(&S.rot, my_rot);
        atomicAdd(&S.skip, my_skip);
        atomicOr(&S.big, my_big);
        atomicMax(&S.maxt_bits, (unsigned long long)__double_as_longlong(my_max));
        atomicOr(&S.touched, my_touch);
    }
    __syncthreads();
    if (S.fail != kNoError) {
        if (tid == 0) atomicMin(a.err, S.fail);
        return;
    }
    // storage columns of the slot's 2b columns, for the update's prologue
    if (tid < B2) a.colidx[(int64_t)slot * B2 + tid] = a.colmap[slot_pos(tid, b, I, J)];
    // W column-major: Wg[slot][c * B2 + k] = W[k][c]
    double *Wout = a.Wg + (int64_t)slot * B2 * B2;
    for (int e = tid; e < B2 * B2; e += NT) Wout[e] = S.W[e % B2][e / B2];
    if (tid == 0) {
        // touched columns (W == I outside T x T; T empty: k_update skips)
        uint8_t *ts = a.tset + (int64_t)slot * kTsetStride;
        unsigned long long m = S.touched;
        int cnt = 0;
        while (m) {
            const int c = __ffsll((long long)m) - 1;
            m &= m - 1;
            ts[1 + cnt++] = (uint8_t)c;
        }
        ts[0] = (uint8_t)cnt;
        // convergence code (_kernels.py:227-231 semantics per slot)
        if (S.big) a.C[slot] = 3;
        else if (S.rot) a.C[slot] |= 1;
        a.rotk[slot] += S.rot;
        a.skipk[slot] += S.skip;
        const double mt = __longlong_as_double((long long)S.maxt_bits);
        if (mt > a.maxt[slot]) a.maxt[slot] = mt;
        if (a.ru.pairstamp) {
            const uint32_t stamp = reuse_stamp(a.ru.dsweep, a.nb, a.step);
            if (a.ru.dcache && !(a.skipf && a.skipf[slot] == kSlotCross)) {
                // this visit folded both diagonal blocks fresh: cached as of now
                a.ru.dstamp[I] = stamp;
                a.ru.dstamp[J] = stamp;
            }
            if (S.touched) {
                // the blocks' columns are rewritten by this step's update
                a.ru.blkmod[I] = stamp;
                a.ru.blkmod[J] = stamp;
            } else if (!S.rot) {
                // an all-skip visit: recorded for reuse
                a.ru.pairstamp[I * a.nb + J] = stamp | ((uint32_t)(a.full != 0) << 31);
                a.ru.pairskip[I * a.nb + J] = S.skip;
            }
        }
        inner_advance(a, slot, I, J);
    }
}

#include "hsvd_inner.cuh"

// ---------------------------------------------------------------------
// k_update: [G_P; V_P] <- [G_P; V_P] W_P in place, FP64 tensor cores
// ---------------------------------------------------------------------
template <int B2, int MT>
struct UpdSmem {
    static constexpr int LDX = MT + 4;  // == 4 mod 16
    static constexpr int LDW = B2 + 4;
    double w[B2][LDW];  // w[c][k] = W[k][c]
    double x[B2][LDX];  // x[k][row]
    double *col[B2];
};

template <int B2, int MT>
__global__ void __launch_bounds__(kThreads, 2) k_update(
    double *__restrict__ G, int64_t ldg, int n, double *__restrict__ V, int64_t ldv, int rv,
    const int64_t *__restrict__ colidx, const double *__restrict__ Wg,
    const uint8_t *__restrict__ tset, int tiles_g, int slot0, const unsigned long long *err)
{
    extern __shared__ __align__(16) unsigned char usm_raw[];
    auto &S = *reinterpret_cast<UpdSmem<B2, MT> *>(usm_raw);
    const int slot = blockIdx.y + slot0, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // the error word and the touched count are independent loads (no
    // dependent chain in front of the tile loads)
    const unsigned long long e0 = *err;
    const uint8_t *ts = tset + (int64_t)slot * kTsetStride;
    const int nt = ts[0];
    if (e0 != kNoError || nt == 0) return;  // failed run, or W == I
    const bool isV = (int)blockIdx.x >= tiles_g;
    const int tile = isV ? blockIdx.x - tiles_g : blockIdx.x;
    const int nrows = isV ? rv : n;
    const int64_t ld = isV ? ldv : ldg;
    double *M = isV ? V : G;
    const int row0 = tile * MT;
    const int64_t *cix = colidx + (int64_t)slot * B2;
    if (nt <= kSparseMax) {
        // few touched columns: out[:, T] = X[:, T] W[T, T] on the FMA pipe,
        // reading and writing only the |T| columns of this row tile
        if (tid < nt) S.col[tid] = M + cix[ts[1 + tid]] * ld;
        const double *Wsl = Wg + (int64_t)slot * B2 * B2;
        for (int e = tid; e < nt * nt; e += kThreads) {
            const int c = e / nt, k = e % nt;
            S.w[c][k] = Wsl[ts[1 + c] * B2 + ts[1 + k]];  // W[T_k][T_c]
        }
        __syncthreads();
        for (int e = tid; e < nt * MT; e += kThreads) {
            const int k = e / MT, rr = e % MT;
            S.x[k][rr] = row0 + rr < nrows ? S.col[k][row0 + rr] : 0.0;
        }
        __syncthreads();
        for (int e = tid; e < nt * MT; e += kThreads) {
            const int c = e / MT, rr = e % MT;
            if (row0 + rr >= nrows) continue;
            double acc = 0.0;
            for (int k = 0; k < nt; ++k) acc = fma(S.x[k][rr], S.w[c][k], acc);
            S.col[c][row0 + rr] = acc;
        }
        return;
    }
    // W (column-major in global) -> w[c][k]: issued before the column bases
    const double *Wsrc = Wg + (int64_t)slot * B2 * B2;
    for (int q = tid; q < B2 * B2 / 2; q += kThreads) {
        const int c = (2 * q) / B2, k = (2 * q) % B2;
        cp_async16(&S.w[c][k], Wsrc + 2 * q, 16);
    }
    if (tid < B2) S.col[tid] = M + cix[tid] * ld;
    __syncthreads();
    // X tile in two commit groups (K halves) so the first half's DMMAs
    // overlap the second half's loads
    constexpr int CPC = MT / 2;  // 16-byte chunks per column
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        for (int q = tid; q < (B2 / 2) * CPC; q += kThreads) {
            const int k = h * (B2 / 2) + q / CPC, part = q % CPC;
            const int row = row0 + 2 * part;
            const int rem = nrows - row;
            const int bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
            cp_async16(&S.x[k][2 * part], bytes ? S.col[k] + row : S.col[k], bytes);
        }
        cp_async_commit();
    }

    constexpr int WM = MT / 4, WN = B2 / 2, MI = WM / 8, NI = WN / 8;
    const int wm = warp >> 1, wn = warp & 1;
    const int m0 = wm * WM, n0 = wn * WN;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (h == 0) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncthreads();
#pragma unroll 4
        for (int kk = h * (B2 / 2); kk < (h + 1) * (B2 / 2); kk += 4) {
            double a[MI], bb[NI];
#pragma unroll
            for (int i = 0; i < MI; ++i) a[i] = S.x[kk + fk][m0 + 8 * i + fr];
#pragma unroll
            for (int j = 0; j < NI; ++j) bb[j] = S.w[n0 + 8 * j + fr][kk + fk];
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
        }
    }
    // results straight from the accumulators: a warp store covers 8
    // consecutive rows of 4 columns (full 32-byte sectors); the tile's rows
    // belong to this CTA alone, and its input is already in shared memory
#pragma unroll
    for (int i = 0; i < MI; ++i) {
        const int row = row0 + m0 + 8 * i + fr;
        if (row < nrows)
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const int col = n0 + 8 * j + 2 * fk;
                S.col[col][row] = acc[i][j][0];
                S.col[col + 1][row] = acc[i][j][1];
            }
    }
}

// d[k] = ||G[:, rho[k]]||^2 for k < r; first_zero (may be NULL) = min rho of
// a zero column (defined in hsvd_block.cu)
int launch_block_norms(const double *G, int64_t ldg, int64_t n, const int64_t *rho, int64_t r,
                       double *d, unsigned long long *first_zero, cudaStream_t s);

// ---------------------------------------------------------------------
// host-side helpers
// ---------------------------------------------------------------------
struct Carve2 {
    char *base;
    int64_t off;
    template <typename T>
    T *take(int64_t count)
    {
        off = (off + 255) & ~(int64_t)255;
        T *p = (T *)(base + off);
        off += count * (int64_t)sizeof(T);
        return p;
    }
};

inline int num_sms()
{
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
    }
    return sms;
}

constexpr int kGramKT = HSVD_GRAM_KT, kGramStages = HSVD_GRAM_STAGES,
              kGramOcc = HSVD_GRAM_TMA ? HSVD_GRAM_TMA_OCC : HSVD_GRAM_OCC;

// Target number of K segments per slot (a function of nothing but this
// constant and n: see GramPart).  More segments balance the CTAs better
// and cost k_inner more partials to fold.
#ifndef HSVD_GRAM_NSEG
#define HSVD_GRAM_NSEG 16
#endif

// Gram partition of a launch of nslots slots.  The segmentation (L, NSEG)
// depends on n only.  The NS segments are dealt in equal runs of
// ceil(NS / capacity) segments, capacity = #SMs x resident CTAs, so every
// CTA has the same work and, when the runs do not fill the GPU, the spare
// CTA slots go to the other stream's kernels.  A CTA spans at most
// GramSmem::MAXSLOTS slots (checked by the caller through gram_slots_ok).
inline GramPart gram_partition(int64_t n, int64_t nslots)
{
    GramPart g;
    g.T = (n + kGramKT - 1) / kGramKT;
    if (g.T < 1) g.T = 1;
    g.L = (g.T + HSVD_GRAM_NSEG - 1) / HSVD_GRAM_NSEG;
    g.NSEG = (g.T + g.L - 1) / g.L;
    g.NS = nslots * g.NSEG;
    const int64_t cap = (int64_t)num_sms() * kGramOcc;
    const int64_t per = (g.NS + cap - 1) / cap;
    g.P = (g.NS + per - 1) / per;
    return g;
}

inline int gram_maxseg(const GramPart &g, int64_t) { return (int)g.NSEG; }

// every CTA's run of segments touches at most MAXSLOTS slots
inline bool gram_slots_ok(const GramPart &g)
{
    const int64_t per = (g.NS + g.P - 1) / g.P;
    return (per + g.NSEG - 1) / g.NSEG + 1 <= 4;
}

// Per-slot state of one step's kernels: the whole problem on one GPU, or
// one shard's slots when sharded.  colmap maps a column POSITION to its
// column in the G/V storage (rho on one GPU; the shard's area map when
// sharded); js maps a position to its J sign.
struct SlotWs {
    const int64_t *colmap, *js;
    const int64_t *orig;  // position -> original column (NULL: colmap)
    int64_t *ip, *jp, *iblk, *jblk, *cur;
    uint8_t *C, *tset;
    uint32_t *rotk, *skipk;
    double *maxt;
    unsigned long long *err;
    double *Apart, *Wg;
    int64_t *colidx;
    int64_t nslots, nb, slot_base;
    int64_t real_cols;  // colmap values >= this are padding (INT64_MAX: none)
    GramPart gp;
    int maxseg;
    // all-skip reuse (ru.pairstamp NULL: off): per-slot flags, the active
    // slot list of the launch and its length
    ReuseWs ru;
    uint8_t *skipf;
    int32_t *act, *nact;
    // k_gram_tma: tensor map of the storage colmap indexes (NULL: cp.async
    // k_gram); tile: the storage is in position order (block K = columns
    // [K b, K b + b)), so a block's k-tile is one TMA box instead of
    // gather4 copies through colmap
    const CUtensorMap *gmap;
    bool tile;
};

// Carve the per-slot arrays for nslots slots of a problem with nb blocks
// (with the all-skip reuse bookkeeping when reuse is set).
inline void carve_slots(Carve2 &c, int64_t n, int64_t nslots, int64_t nb, int b, SlotWs *w,
                        bool reuse = false)
{
    const int64_t B2 = 2 * b;
    const GramPart gp = gram_partition(n, nslots);
    const int ks = gram_maxseg(gp, nslots);
    SlotWs t;
    t.colmap = t.js = t.orig = nullptr;
    t.tile = false;
    t.ip = c.take<int64_t>(nslots);
    t.jp = c.take<int64_t>(nslots);
    t.iblk = c.take<int64_t>(nslots);
    t.jblk = c.take<int64_t>(nslots);
    t.cur = c.take<int64_t>(2 * nslots);
    t.C = c.take<uint8_t>(nslots);
    t.tset = c.take<uint8_t>(nslots * kTsetStride);
    t.rotk = c.take<uint32_t>(nslots);
    t.skipk = c.take<uint32_t>(nslots);
    t.maxt = c.take<double>(nslots);
    t.err = c.take<unsigned long long>(1);
    t.Apart = c.take<double>(nslots * ks * B2 * B2);
    t.Wg = c.take<double>(nslots * B2 * B2);
    t.colidx = c.take<int64_t>(nslots * B2);
    t.skipf = c.take<uint8_t>(nslots);
    t.act = c.take<int32_t>(nslots);
    t.nact = c.take<int32_t>(4);
    t.gmap = nullptr;
    t.ru.pairstamp = t.ru.pairskip = t.ru.blkmod = nullptr;
    t.ru.dsweep = nullptr;
    t.ru.dcache = nullptr;
    t.ru.dstamp = nullptr;
    t.ru.planstat = nullptr;
    if (reuse) {
        t.ru.pairstamp = c.take<uint32_t>(nb * nb);
        t.ru.pairskip = c.take<uint32_t>(nb * nb);
        t.ru.blkmod = c.take<uint32_t>(nb);
        t.ru.dsweep = c.take<int32_t>(1);
        t.ru.dcache = c.take<double>(nb * b * b);
        t.ru.dstamp = c.take<uint32_t>(nb);
        t.ru.planstat = c.take<unsigned long long>(4);
    }
    t.nslots = nslots;
    t.nb = nb;
    t.slot_base = 0;
    t.real_cols = INT64_MAX;
    t.gp = gp;
    t.maxseg = ks;
    if (w) *w = t;
}

inline int inner_priority()
{
    static int prio = 1;
    if (prio == 1) {
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) hi = 0;
        prio = hi;  // numerically lowest = highest priority
    }
    return prio;
}

// Inner passes per step, shared by the one-GPU and the sharded drivers.
// cfg->inner_passes >= 1 fixes the count for every sweep; 0 ("auto", the
// default) runs 2 passes in the dense sweeps and 1 in the late ones for the
// fast rotation and at least 32 block columns (r >= 1024 at b = 32), else 1
// (small problems: block residual ratios up to 1.00 with 2 passes, and the
// dd cross-check's VtJV 2.6x; they take milliseconds either way).  A
// sweep is dense until a sweep rotates fewer than 5 % of its visits (the
// rule that also ends the split schedule), so every schedule, stream split
// and shard count switches at the same sweep and the results stay
// bit-identical across them.  Measured at n = 8192: 13 -> 11 sweeps,
// 2.01 -> 1.90 s, residual ratios 0.87 / 0.16 / 0.17.
// HSVD_DENSE_PASSES=k overrides the dense count (measurements).
struct PassPolicy {
    hsvd_config dense, late;
    bool dense_now = true;
    void init(const hsvd_config *cfg, int64_t nblocks)
    {
        dense = late = *cfg;
        if (cfg->inner_passes < 1) {
            const bool two = cfg->block_rotation == HSVD_ROTATION_FAST && nblocks >= 32;
            dense.inner_passes = two ? 2 : 1;
            late.inner_passes = 1;
        }
        if (const char *e = getenv("HSVD_DENSE_PASSES")) dense.inner_passes = atoi(e) > 1 ? atoi(e) : 1;
        if (const char *e = getenv("HSVD_DENSE_DIV")) div = atoi(e) > 1 ? atoi(e) : 20;
    }
    int64_t div = 20;  // dense while a sweep rotates >= 1/div of its visits
    const hsvd_config *now() const { return dense_now ? &dense : &late; }
    void after_sweep(int64_t rot, int64_t skip)
    {
        if (dense_now && rot < (rot + skip) / div) dense_now = false;
    }
};

template <int B2>
struct BlockKernels {
    static constexpr int KT = kGramKT, STAGES = kGramStages, MT = 128;
    static constexpr int TSTAGES = HSVD_GRAM_TMA_STAGES;
    static size_t gram_smem() { return sizeof(GramSmem<B2, KT, STAGES>); }
    static size_t gram_tma_smem() { return sizeof(GramTmaSmem<B2, KT, TSTAGES>) + 1024; }
    static size_t inner_smem() { return sizeof(InnerSmem2<B2>); }
    static size_t upd_smem() { return sizeof(UpdSmem<B2, MT>); }
    static int setup()
    {
        HSVD_CUDA(cudaFuncSetAttribute(k_gram<B2, KT, STAGES>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)gram_smem()));
        HSVD_CUDA(cudaFuncSetAttribute(k_gram_tma<B2, KT, TSTAGES, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)gram_tma_smem()));
        HSVD_CUDA(cudaFuncSetAttribute(k_gram_tma<B2, KT, TSTAGES, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)gram_tma_smem()));
        HSVD_CUDA(cudaFuncSetAttribute(k_inner<B2, true, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)inner_smem()));
        HSVD_CUDA(cudaFuncSetAttribute(k_inner<B2, true, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)inner_smem()));
        HSVD_CUDA(cudaFuncSetAttribute(k_inner<B2, false, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)inner_smem()));
        HSVD_CUDA(cudaFuncSetAttribute(k_inner<B2, false, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)inner_smem()));
        HSVD_CUDA(cudaFuncSetAttribute(k_update<B2, MT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)upd_smem()));
        return HSVD_OK;
    }
    // Gram -> inner pass of one step
    // Gram -> inner pass of step `step`; plan: replay recorded all-skip
    // visits (k_plan) instead of recomputing them
    static int gram_inner(double *G, int64_t ldg, int n, const SlotWs &w, int full,
                          const hsvd_config *cfg, cudaStream_t s, KernelTimer &T, int step,
                          bool plan)
    {
        const int64_t nslots = w.nslots;
        const GramPart &gp = w.gp;
        if (!gram_slots_ok(gp)) {
            set_error("block mode: too many slots per Gram CTA (r too large for this GPU)");
            return HSVD_ERR_UNSUPPORTED;
        }
        plan = plan && w.ru.pairstamp != nullptr;
        T.begin(0, s);
        if (plan) {
            k_plan<<<1, kPlanThreads, 0, s>>>(w.iblk, w.jblk, nslots, w.nb, w.ru, step, full,
                                              w.skipf, w.act, w.nact, w.err);
            HSVD_LAUNCH_CHECK("k_plan");
        }
        {
            // Gram and inner pass are the critical path of a step: highest
            // priority (split mode runs a bulk update on another stream)
            cudaLaunchConfig_t lc = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributePriority;
            at[0].val.priority = inner_priority();
            lc.attrs = at;
            lc.numAttrs = 1;
            lc.stream = s;
            const int32_t *actp = plan ? w.act : nullptr;
            if (w.gmap) {
                lc.gridDim = dim3((unsigned)gp.P);
                lc.blockDim = dim3(kThreads + 32);
                lc.dynamicSmemBytes = gram_tma_smem();
                if (w.tile) {
                    HSVD_CUDA(cudaLaunchKernelEx(&lc, k_gram_tma<B2, KT, TSTAGES, true>, *w.gmap,
                                                 n, w.colmap, (const int64_t *)w.iblk,
                                                 (const int64_t *)w.jblk, gp, w.maxseg, w.Apart,
                                                 (const unsigned long long *)w.err, actp,
                                                 (const int32_t *)w.nact,
                                                 (const uint8_t *)w.skipf));
                } else {
                    HSVD_CUDA(cudaLaunchKernelEx(&lc, k_gram_tma<B2, KT, TSTAGES, false>, *w.gmap,
                                                 n, w.colmap, (const int64_t *)w.iblk,
                                                 (const int64_t *)w.jblk, gp, w.maxseg, w.Apart,
                                                 (const unsigned long long *)w.err, actp,
                                                 (const int32_t *)w.nact,
                                                 (const uint8_t *)w.skipf));
                }
            } else {
                lc.gridDim = dim3((unsigned)gp.P);
                lc.blockDim = dim3(kThreads);
                lc.dynamicSmemBytes = gram_smem();
                HSVD_CUDA(cudaLaunchKernelEx(&lc, k_gram<B2, KT, STAGES>, G, ldg, n, w.colmap,
                                             (const int64_t *)w.iblk, (const int64_t *)w.jblk,
                                             gp, w.maxseg, w.Apart,
                                             (const unsigned long long *)w.err, actp,
                                             (const int32_t *)w.nact,
                                             (const uint8_t *)w.skipf));
            }
        }
        T.end(s);
        HSVD_LAUNCH_CHECK("k_gram");
        InnerArgs ia;
        ia.part = gp; ia.maxseg = w.maxseg;
        ia.Apart = w.Apart; ia.Wg = w.Wg; ia.jsign = w.js;
        ia.ip = w.ip; ia.jp = w.jp; ia.iblk = w.iblk; ia.jblk = w.jblk; ia.cur = w.cur;
        ia.C = w.C; ia.tset = w.tset; ia.colmap = w.colmap; ia.orig = w.orig ? w.orig : w.colmap; ia.colidx = w.colidx; ia.rotk = w.rotk; ia.skipk = w.skipk; ia.maxt = w.maxt; ia.err = w.err;
        ia.nb = w.nb; ia.slot_base = w.slot_base; ia.real_cols = w.real_cols; ia.eps = cfg->eps; ia.teps = cfg->teps;
        ia.full = full; ia.use_skip = cfg->use_skip;
        ia.passes = cfg->inner_passes > 1 ? cfg->inner_passes : 1;
        ia.trace = nullptr;
        ia.ru = w.ru;
        ia.skipf = plan ? w.skipf : nullptr;
        ia.step = step;
        T.begin(1, s);
        {
            // the inner pass is latency bound on few SMs: launched at the
            // highest priority, its CTAs take SMs ahead of queued GEMM CTAs
            // of a concurrent stream (split mode)
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)nslots);
            lc.blockDim = dim3(inner2_threads<B2>());
            lc.dynamicSmemBytes = inner_smem();
            lc.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributePriority;
            at[0].val.priority = inner_priority();
            lc.attrs = at;
            lc.numAttrs = 1;
            const bool fast = cfg->block_rotation == HSVD_ROTATION_FAST;
            if (fast && full) {
                HSVD_CUDA(cudaLaunchKernelEx(&lc, k_inner<B2, true, true>, ia));
            } else if (fast) {
                HSVD_CUDA(cudaLaunchKernelEx(&lc, k_inner<B2, true, false>, ia));
            } else if (full) {
                HSVD_CUDA(cudaLaunchKernelEx(&lc, k_inner<B2, false, true>, ia));
            } else {
                HSVD_CUDA(cudaLaunchKernelEx(&lc, k_inner<B2, false, false>, ia));
            }
        }
        T.end(s);
        HSVD_LAUNCH_CHECK("k_inner");
        return HSVD_OK;
    }
    // update of the slots [lo, hi) of w
    static int update(double *G, int64_t ldg, int n, double *V, int64_t ldv, int rv,
                      const SlotWs &w, int64_t lo, int64_t hi, cudaStream_t s, KernelTimer &T,
                      bool urgent = false)
    {
        if (hi <= lo) return HSVD_OK;
        const int tiles_g = (n + MT - 1) / MT;
        const int tiles_v = V ? (rv + MT - 1) / MT : 0;
        T.begin(2, s);
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(tiles_g + tiles_v, (unsigned)(hi - lo));
        lc.blockDim = dim3(kThreads);
        lc.dynamicSmemBytes = upd_smem();
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributePriority;
        at[0].val.priority = urgent ? inner_priority() : 0;
        lc.attrs = at;
        lc.numAttrs = 1;
        HSVD_CUDA(cudaLaunchKernelEx(&lc, k_update<B2, MT>, G, ldg, n, V, ldv, rv,
                                     (const int64_t *)w.colidx, (const double *)w.Wg,
                                     (const uint8_t *)w.tset, tiles_g, (int)lo,
                                     (const unsigned long long *)w.err));
        T.end(s);
        HSVD_LAUNCH_CHECK("k_update");
        return HSVD_OK;
    }
    // one step: Gram -> inner pass -> update
    static int step(double *G, int64_t ldg, int n, double *V, int64_t ldv, int rv,
                    const SlotWs &w, int full, const hsvd_config *cfg, cudaStream_t s,
                    KernelTimer &T, int stepno, bool plan)
    {
        int e = gram_inner(G, ldg, n, w, full, cfg, s, T, stepno, plan);
        if (e) return e;
        return update(G, ldg, n, V, ldv, rv, w, 0, w.nslots, s, T);
    }
};


}  // namespace hsvd
