// hsvd_block.cu -- block-column one-sided hyperbolic Jacobi on sm_100a.
//
// The pivot unit is a pair of block columns P = [B_I B_J] (b columns each,
// positions [I*b, I*b+b) and [J*b, J*b+b) of the sorted package order,
// gathered through rho as the reference addresses columns, solver.py:26-43).
// One step of the modified-modulus schedule on the r/b block indices
// (strategies.py:41-72) processes all r/(2b) slots with three kernels
// (hsvd_block_kernels.cuh):
//
//   k_gram    A_P = G_P^T G_P (2b x 2b), FP64 tensor cores (mma.sync
//             m8n8k4 -> SASS DMMA.8x8x4); each slot's K range is cut into
//             fixed segments (a function of n only) streamed over the CTAs,
//             upper-triangle tiles only.
//   k_inner   one CTA per slot (hsvd_inner.cuh): folds the segment partials
//             in order, runs one pass of 2x2 rotations on (A_P, J_P) in
//             shared memory -- a leader warp forms each round's rotations
//             (trig or hyperbolic from the signs, relative-orthogonality skip
//             _kernels.py:211; "fast" plain-fp64 closed forms by default, the
//             reference's double-double rotation_tc _kernels.py:128-173 with
//             block_rotation="dd") while bulk warps apply the previous round
//             to the upper triangle of A and W warps accumulate the
//             J-orthogonal W_P in registers; writes convergence codes and
//             statistics, advances the stepper.
//   k_update  [G_P; V_P] <- [G_P; V_P] W_P, FP64 tensor cores, in place.
//
// The inner ordering is "full" by default (every pair of the pivot block,
// circle method, at every step); inner_ordering="oriented" is the paper's
// block-oriented scheme (the full triangle at the first
// step of a sweep, only the cross pairs I x J at the other steps).
//
// r not a multiple of 2b: the driver appends inert zero columns (J = -1) in
// a workspace copy and strips them afterwards (block_drive_padded): a zero
// column has a_ij = 0 with every column, so it is never rotated, and pairs
// that include one are not counted as visits.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "hsvd_block_kernels.cuh"

namespace hsvd {

// ---------------------------------------------------------------------
// column norms by position: d[k] = ||G[:, rho[k]]||^2 (one warp per column)
// ---------------------------------------------------------------------
__global__ void k_block_norms(const double *__restrict__ G, int64_t ldg, int n,
                              const int64_t *__restrict__ rho, int64_t r, double *d,
                              unsigned long long *first_zero)
{
    const int64_t k = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (k >= r) return;
    const double *g = G + rho[k] * ldg;
    double s0 = 0.0, s1 = 0.0;
    int e = lane;
    for (; e + 32 < n; e += 64) {
        const double x = g[e], y = g[e + 32];
        s0 = fma(x, x, s0);
        s1 = fma(y, y, s1);
    }
    for (; e < n; e += 32) s0 = fma(g[e], g[e], s0);
    double s = s0 + s1;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        d[k] = s;
        if (s == 0.0 && first_zero) atomicMin(first_zero, (unsigned long long)rho[k]);
    }
}

typedef CUresult (*TensorMapEncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                      const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                      const cuuint32_t *, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

int make_gram_tensor_map(CUtensorMap *tm, const double *G, int64_t ld, int64_t n, int64_t ncols,
                         int box_cols)
{
    static TensorMapEncodeFn enc = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return (TensorMapEncodeFn)fn;
    }();
    if (!enc || (ld * 8) % 16 || ((uintptr_t)G & 15)) return 1;
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)ncols};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    const cuuint32_t box[2] = {16, (cuuint32_t)box_cols};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)G, dims, strides, box,
                           es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : 1;
}

int launch_block_norms(const double *G, int64_t ldg, int64_t n, const int64_t *rho, int64_t r,
                       double *d, unsigned long long *first_zero, cudaStream_t s)
{
    k_block_norms<<<(unsigned)((r + 7) / 8), 256, 0, s>>>(G, ldg, (int)n, rho, r, d, first_zero);
    HSVD_LAUNCH_CHECK("k_block_norms");
    return HSVD_OK;
}

// ---------------------------------------------------------------------
// position-ordered storage (one GPU): column moves
// ---------------------------------------------------------------------
// The one-GPU driver keeps G and V^{-T} with storage column = POSITION of
// the sorted package order, so block K is the contiguous columns
// [K b, K b + b) and the Gram reads a block's k-tile as one TMA box.  After
// each sort the columns move to their new positions: position q takes the
// column of original index tgt[q], which sat at position inv_old[tgt[q]].
// Two passes through a scratch buffer, touching only moved columns.

__global__ void k_iota(int64_t *x, int64_t r)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < r) x[k] = k;
}

__global__ void k_inverse(const int64_t *__restrict__ rho, int64_t *__restrict__ inv, int64_t r)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < r) inv[rho[k]] = k;
}

// phase 0: S[:, q] = W[:, src(q)]; phase 1: W[:, q] = S[:, q] (moved q only)
__global__ void k_move_cols(double *__restrict__ W, int64_t ldw, double *__restrict__ S,
                            int64_t lds, int64_t rows, const int64_t *__restrict__ tgt,
                            const int64_t *__restrict__ inv_old, int phase)
{
    const int64_t q = blockIdx.y;
    const int64_t src = inv_old[tgt[q]];
    if (src == q) return;
    const double2 *from = (const double2 *)(phase ? S + q * lds : W + src * ldw);
    double2 *to = (double2 *)(phase ? W + q * ldw : S + q * lds);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows / 2;
         e += (int64_t)gridDim.x * blockDim.x)
        to[e] = from[e];
    if ((rows & 1) && blockIdx.x == 0 && threadIdx.x == 0)
        (phase ? W + q * ldw : S + q * lds)[rows - 1] = (phase ? S + q * lds : W + src * ldw)[rows - 1];
}

static int move_cols(double *W, int64_t ldw, double *S, int64_t lds, int64_t rows, int64_t r,
                     const int64_t *tgt, const int64_t *inv_old, cudaStream_t s)
{
    unsigned gx = (unsigned)((rows / 2 + 255) / 256);
    if (gx > 16) gx = 16;
    for (int ph = 0; ph < 2; ++ph) {
        k_move_cols<<<dim3(gx, (unsigned)r), 256, 0, s>>>(W, ldw, S, lds, rows, tgt, inv_old, ph);
        HSVD_LAUNCH_CHECK("k_move_cols");
    }
    return HSVD_OK;
}

// ---------------------------------------------------------------------
// one-GPU driver
// ---------------------------------------------------------------------
struct BlockWs {
    double *d;
    int64_t *rho, *js;
    unsigned long long *first_zero;
    void *sortws;
    int64_t *out;
    int8_t *signs;
    int64_t *rho_prev;  // rho before the sweep-end sort (all-skip reuse)
    int64_t *ident;     // 0..r-1 (storage = position)
    int64_t *inv;       // original column -> position (before a sort)
    double *Gs, *Vs;    // scratch columns for the moves (ld lds / r)
    int64_t lds;
    SlotWs sl;
    // split mode: the two half-slot views (shared arrays, own Gram partial
    // buffers and partitions)
    SlotWs half[2];
};

// The slot halves [0, S/2) and [S/2, S) of the step (split mode).
static void half_range(int64_t nslots, int h, int64_t &lo, int64_t &hi)
{
    lo = h ? nslots / 2 : 0;
    hi = h ? nslots : nslots / 2;
}

// profile mode times the kernels of this sweep (HSVD_PROFILE_SWEEP, default 0)
static int64_t profile_sweep()
{
    static const int64_t v = [] {
        const char *e = getenv("HSVD_PROFILE_SWEEP");
        return e ? (int64_t)atoll(e) : (int64_t)0;
    }();
    return v;
}

static int64_t carve_block(Carve2 &c, int64_t n, int64_t r, int b, BlockWs *w, bool withV = true)
{
    const int64_t nb = r / b, nslots = nb / 2 > 0 ? nb / 2 : 1;
    BlockWs t;
    t.d = c.take<double>(r);
    t.rho = c.take<int64_t>(r);
    t.js = c.take<int64_t>(r);
    t.first_zero = c.take<unsigned long long>(1);
    t.sortws = c.take<char>(24 * r);
    t.out = c.take<int64_t>(8);
    t.signs = c.take<int8_t>(r);
    t.rho_prev = c.take<int64_t>(r);
    t.ident = c.take<int64_t>(r);
    t.inv = c.take<int64_t>(r);
    t.lds = n + (n & 1);
    t.Gs = c.take<double>(t.lds * r);
    t.Vs = withV ? c.take<double>(r * r) : nullptr;
    carve_slots(c, n, nslots, nb, b, &t.sl, true);
    t.sl.colmap = t.ident;  // storage column = position
    t.sl.orig = t.rho;
    t.sl.js = t.js;
    const int64_t B2 = 2 * b;
    for (int h = 0; h < 2; ++h) {
        int64_t lo, hi;
        half_range(nslots, h, lo, hi);
        SlotWs v = t.sl;
        const int64_t m = hi > lo ? hi - lo : 1;
        v.ip = t.sl.ip + lo;
        v.jp = t.sl.jp + lo;
        v.iblk = t.sl.iblk + lo;
        v.jblk = t.sl.jblk + lo;
        v.cur = t.sl.cur + 2 * lo;
        v.C = t.sl.C + lo;
        v.tset = t.sl.tset + lo * kTsetStride;
        v.rotk = t.sl.rotk + lo;
        v.skipk = t.sl.skipk + lo;
        v.maxt = t.sl.maxt + lo;
        v.Wg = t.sl.Wg + lo * B2 * B2;
        v.colidx = t.sl.colidx + lo * B2;
        v.skipf = t.sl.skipf + lo;
        v.act = t.sl.act + lo;
        v.nact = t.sl.nact + 1 + h;
        v.nslots = hi - lo;
        v.slot_base = lo;
        v.gp = gram_partition(n, m);
        v.maxseg = gram_maxseg(v.gp, m);
        v.Apart = c.take<double>(m * v.maxseg * B2 * B2);
        t.half[h] = v;
    }
    if (w) *w = t;
    return c.off + 256;
}

// Padding to a multiple of 2b: the padded copy of G (ld even), V^{-T},
// sigma and lam live at the front of the workspace.
struct PadWs {
    double *G, *V, *sigma, *lam;
    int64_t ld, rp;
};

static int64_t pad_cols(int64_t r, int b)
{
    const int64_t m = 2 * (int64_t)b;
    return (r + m - 1) / m * m - r;
}

static int64_t carve_pad(Carve2 &c, int64_t n, int64_t r, int b, bool withV, PadWs *w)
{
    PadWs t;
    t.rp = r + pad_cols(r, b);
    t.ld = n + (n & 1);
    t.G = c.take<double>(t.rp * t.ld);
    t.V = withV ? c.take<double>(t.rp * t.rp) : nullptr;
    t.sigma = c.take<double>(t.rp);
    t.lam = c.take<double>(t.rp);
    if (w) *w = t;
    c.off = (c.off + 255) & ~(int64_t)255;
    return c.off;
}

int64_t block_workspace_size(int64_t n, int64_t r, const hsvd_config *cfg)
{
    // unsupported widths (block_drive rejects them) must not reach the
    // carve's r / b
    const int b = cfg->block_cols;
    if (b != 16 && b != 32) return 256;
    Carve2 c{nullptr, 0};
    int64_t pre = 0;
    if (pad_cols(r, b)) pre = carve_pad(c, n, r, b, cfg->accumulate_v != 0, nullptr);
    Carve2 c2{nullptr, 0};
    return pre + carve_block(c2, n, r + pad_cols(r, b), b, nullptr, cfg->accumulate_v != 0);
}

int launch_reduce_sweep(uint8_t *C, int64_t m, uint32_t *rotk, uint32_t *skipk,
                        double *maxt, int64_t nslots, int64_t *out,
                        const unsigned long long *err, int reset, cudaStream_t s);
int launch_init_packages(const int8_t *signs, int64_t r, int64_t *rho,
                         int64_t *jsign, cudaStream_t s);
int launch_identity(double *V, int64_t r, int64_t ldv, cudaStream_t s);

// d[k] = ||G[:, map[k]]||^2 (map = the identity once storage is in
// position order)
static int block_norms(double *G, int64_t ldg, int64_t n, const BlockWs &w, int64_t r,
                       unsigned long long *first_zero, cudaStream_t s, const int64_t *map)
{
    k_block_norms<<<(unsigned)((r + 7) / 8), 256, 0, s>>>(G, ldg, (int)n, map, r, w.d,
                                                          first_zero);
    HSVD_LAUNCH_CHECK("k_block_norms");
    return HSVD_OK;
}

template <int B2>
static int block_drive_t(double *G, int64_t n, int64_t r, int64_t ldg, double *V, int64_t ldv,
                         const int8_t *signs_host, int64_t p, const hsvd_config *cfg,
                         double *sigma, double *lam, void *ws, int64_t ws_bytes,
                         hsvd_result *res, hsvd_telemetry *tele, DevCtx &ctx,
                         int64_t r_real)
{
    cudaStream_t s = ctx.s;
    using K = BlockKernels<B2>;
    constexpr int b = B2 / 2;
    const int64_t nb = r / b, nslots = nb / 2;
    Carve2 c{(char *)ws, 0};
    BlockWs w;
    if (carve_block(c, n, r, b, &w, V != nullptr) > ws_bytes) {
        set_error("workspace too small");
        return HSVD_ERR_ARG;
    }
    // columns with rho >= r_real are padding (block_drive_padded)
    w.sl.real_cols = w.half[0].real_cols = w.half[1].real_cols = r_real;
    // the Gram's TMA view of G (HSVD_GRAM_TMA=0 in the environment: cp.async)
    alignas(64) CUtensorMap gmap;
    const char *tma_env = getenv("HSVD_GRAM_TMA");
    if (HSVD_GRAM_TMA && !(tma_env && tma_env[0] == '0') &&
        make_gram_tensor_map(&gmap, G, ldg, n, r, b) == 0) {
        w.sl.gmap = w.half[0].gmap = w.half[1].gmap = &gmap;
        w.sl.tile = w.half[0].tile = w.half[1].tile = true;
    }
    int st = K::setup();
    if (st) return st;

    int64_t *host = ctx.host;
    cudaEvent_t t0 = ctx.t0, t1 = ctx.t1;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    struct Cleanup {
        cudaGraph_t &g;
        cudaGraphExec_t &e;
        ~Cleanup()
        {
            if (e) cudaGraphExecDestroy(e);
            if (g) cudaGraphDestroy(g);
        }
    } cleanup{graph, exec};

    if (V) {
        st = launch_identity(V, r, ldv, s);
        if (st) return st;
    }
    HSVD_CUDA(cudaMemcpyAsync(w.signs, signs_host, (size_t)r, cudaMemcpyHostToDevice, s));
    st = launch_init_packages(w.signs, r, w.rho, w.js, s);
    if (st) return st;
    k_iota<<<(unsigned)((r + 255) / 256), 256, 0, s>>>(w.ident, r);
    HSVD_LAUNCH_CHECK("k_iota");
    HSVD_CUDA(cudaMemsetAsync(w.first_zero, 0xff, sizeof(unsigned long long), s));
    st = block_norms(G, ldg, n, w, r, w.first_zero, s, w.ident);
    if (st) return st;
    HSVD_CUDA(cudaMemcpyAsync(host, w.first_zero, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    HSVD_CUDA(cudaStreamSynchronize(s));
    // the smallest zero column; padding columns (>= r_real) are zero by design
    if ((unsigned long long)host[0] < (unsigned long long)r_real) {
        res->err[0] = host[0];
        res->err[1] = res->err[2] = -1;
        set_error("column " + std::to_string(host[0]) + " has zero norm");
        return HSVD_RANK_DEFICIENT;
    }
    if (cfg->sort) {
        st = hsvd_sort_diagonal(w.d, w.rho, w.js, r, p, w.sortws, s);
        if (st) return st;
    }
    // storage into position order (it is in original order: inv = identity)
    st = move_cols(G, ldg, w.Gs, w.lds, n, r, w.rho, w.ident, s);
    if (!st && V) st = move_cols(V, ldv, w.Vs, r, r, r, w.rho, w.ident, s);
    if (st) return st;
    st = hsvd_stepper_init(w.sl.ip, w.sl.jp, w.sl.iblk, w.sl.jblk, nb, s);
    if (st) return st;
    HSVD_CUDA(cudaMemsetAsync(w.sl.C, 0, (size_t)nslots, s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.rotk, 0, sizeof(uint32_t) * nslots, s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.skipk, 0, sizeof(uint32_t) * nslots, s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.maxt, 0, sizeof(double) * nslots, s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.err, 0xff, sizeof(unsigned long long), s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.ru.pairstamp, 0, sizeof(uint32_t) * nb * nb, s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.ru.pairskip, 0, sizeof(uint32_t) * nb * nb, s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.ru.blkmod, 0, sizeof(uint32_t) * nb, s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.ru.dsweep, 0, sizeof(int32_t), s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.ru.dstamp, 0, sizeof(uint32_t) * nb, s));
    HSVD_CUDA(cudaMemsetAsync(w.sl.ru.planstat, 0, sizeof(unsigned long long) * 4, s));

    KernelTimer T;
    // Split mode: the two slot halves run on two streams.  A block only
    // crosses between the halves at their edge slots (the stepper is a ring:
    // a slot trades blocks with slot k +- 1 or the wrap-around), so half h's
    // Gram at step t waits for the other half's EDGE-slot update of step
    // t - 1 only; each half updates its edge slots first.  One half's inner
    // pass then runs beside the other half's GEMMs.
    const bool split = cfg->block_streams >= 2 && !cfg->profile && nslots >= 4;
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev_edge[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}}, ev_fork = nullptr,
                ev_join = nullptr, ev_stagger = nullptr;
    if (split) {
        st = ctx.extra(1);
        if (st) return st;
        st = ctx.events(7);
        if (st) return st;
        s2 = ctx.xs[0];
        ev_edge[0][0] = ctx.evs[0];
        ev_edge[0][1] = ctx.evs[1];
        ev_edge[1][0] = ctx.evs[2];
        ev_edge[1][1] = ctx.evs[3];
        ev_fork = ctx.evs[4];
        ev_join = ctx.evs[5];
        ev_stagger = ctx.evs[6];
    }
    // debug timeline (HSVD_TIMELINE=1, ungraphed first sweep): events after
    // each phase of the first steps, printed relative to the sweep start
    const bool tl_on = getenv("HSVD_TIMELINE") != nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> tl;
    cudaEvent_t tl0 = nullptr;
    auto mark = [&](const std::string &what, cudaStream_t st) -> int {
        if (!tl_on || tl.size() > 200) return HSVD_OK;
        cudaEvent_t e;
        HSVD_CUDA(cudaEventCreate(&e));
        HSVD_CUDA(cudaEventRecord(e, st));
        tl.push_back({what, e});
        return HSVD_OK;
    };
    // replay recorded all-skip visits (k_plan) in the graphed late sweeps;
    // the eager split sweeps only record them (HSVD_REUSE=0: never)
    const bool reuse_ok = [] {
        const char *e = getenv("HSVD_REUSE");
        return !(e && e[0] == '0');
    }();
    bool plan_now = false;
    // inner passes: 2 in the dense sweeps, 1 in the late ones by default
    // (PassPolicy); the late-sweep graph is captured with the late count
    PassPolicy passes;
    passes.init(cfg, nb);
    bool capturing = false;
    auto scfg_now = [&]() { return capturing ? &passes.late : passes.now(); };
    // the graphed late sweeps may use the oriented inner ordering (the full
    // triangle only at a sweep's first step): HSVD_LATE_ORIENTED=1
    const bool late_oriented = [] {
        const char *e = getenv("HSVD_LATE_ORIENTED");
        return e && e[0] == '1';
    }();
    auto inner_full = [&](int64_t step) {
        return (cfg->inner_full && !(capturing && late_oriented)) || step == 0;
    };
    auto enqueue_steps_split = [&]() -> int {
        const hsvd_config *scfg = scfg_now();
        cudaStream_t ss[2] = {s, s2};
        if (tl_on) {
            HSVD_CUDA(cudaEventCreate(&tl0));
            HSVD_CUDA(cudaEventRecord(tl0, s));
        }
        HSVD_CUDA(cudaEventRecord(ev_fork, s));
        HSVD_CUDA(cudaStreamWaitEvent(s2, ev_fork, 0));
        for (int64_t step = 0; step < nb; ++step) {
            const int full = inner_full(step);
            for (int h = 0; h < 2; ++h) {
                const SlotWs &hw = w.half[h];
                const int64_t m = hw.nslots;
                if (step > 0)
                    HSVD_CUDA(cudaStreamWaitEvent(ss[h], ev_edge[h ^ 1][(step - 1) & 1], 0));
                // stagger: the second half starts its sweep after the first
                // half's first inner pass, so the halves stay half a step
                // apart (one's inner pass beside the other's update)
                if (step == 0 && h == 1) HSVD_CUDA(cudaStreamWaitEvent(ss[h], ev_stagger, 0));
                const std::string tag = std::string(h ? "B" : "A") + std::to_string(step);
                int e = mark(tag + " start", ss[h]);
                if (e) return e;
                e = K::gram_inner(G, ldg, (int)n, hw, full, scfg, ss[h], T, (int)step, plan_now);
                if (e) return e;
                if (step == 0 && h == 0) HSVD_CUDA(cudaEventRecord(ev_stagger, ss[h]));
                if ((e = mark(tag + " gram+inner done", ss[h]))) return e;
                // edge slots first, then the rest
                e = K::update(G, ldg, (int)n, V, ldv, (int)r, hw, 0, 1, ss[h], T, true);
                if (e) return e;
                e = K::update(G, ldg, (int)n, V, ldv, (int)r, hw, m - 1, m, ss[h], T, true);
                if (e) return e;
                HSVD_CUDA(cudaEventRecord(ev_edge[h][step & 1], ss[h]));
                if ((e = mark(tag + " edges done", ss[h]))) return e;
                e = K::update(G, ldg, (int)n, V, ldv, (int)r, hw, 1, m - 1, ss[h], T);
                if (e) return e;
                if ((e = mark(tag + " update done", ss[h]))) return e;
            }
        }
        HSVD_CUDA(cudaEventRecord(ev_join, s2));
        HSVD_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
        return HSVD_OK;
    };
    bool split_now = split;  // this sweep's mode (see the sweep loop)
    auto enqueue_sweep = [&]() -> int {
        if (split_now) {
            int e = enqueue_steps_split();
            if (e) return e;
        } else {
            for (int64_t step = 0; step < nb; ++step) {
                const int full = inner_full(step);
                // profile mode plans its eager steps too, so the profiled
                // sweep sees the Gram classes of a graphed sweep
                int e = K::step(G, ldg, (int)n, V, ldv, (int)r, w.sl, full, scfg_now(), s, T,
                                (int)step, plan_now || (cfg->profile && reuse_ok));
                if (e) return e;
            }
        }
        T.begin(3, s);
        int e = block_norms(G, ldg, n, w, r, nullptr, s, w.ident);
        if (e) return e;
        e = launch_reduce_sweep(w.sl.C, nslots, w.sl.rotk, w.sl.skipk, w.sl.maxt, nslots, w.out,
                                w.sl.err, 1, s);
        if (e) return e;
        if (cfg->sort) {
            HSVD_CUDA(cudaMemcpyAsync(w.rho_prev, w.rho, sizeof(int64_t) * r,
                                      cudaMemcpyDeviceToDevice, s));
            e = hsvd_sort_diagonal(w.d, w.rho, w.js, r, p, w.sortws, s);
            if (e) return e;
            k_reuse_sweep_end<<<(unsigned)((r + 255) / 256), 256, 0, s>>>(w.rho, w.rho_prev, r, b,
                                                                         nb, w.sl.ru);
            HSVD_LAUNCH_CHECK("k_reuse_sweep_end");
            // the columns follow their packages to the new positions
            k_inverse<<<(unsigned)((r + 255) / 256), 256, 0, s>>>(w.rho_prev, w.inv, r);
            HSVD_LAUNCH_CHECK("k_inverse");
            e = move_cols(G, ldg, w.Gs, w.lds, n, r, w.rho, w.inv, s);
            if (!e && V) e = move_cols(V, ldv, w.Vs, r, r, r, w.rho, w.inv, s);
            if (e) return e;
        }
        k_reuse_next_sweep<<<1, 1, 0, s>>>(w.sl.ru.dsweep);
        HSVD_LAUNCH_CHECK("k_reuse_next_sweep");
        T.end(s);
        HSVD_CUDA(cudaMemcpyAsync(host, w.out, 5 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        return HSVD_OK;
    };
    // Split mode is launched eagerly: replayed graphs do not honour the
    // kernel priorities that keep the critical path ahead of the bulk update
    // (measured at n = 8192: 227 vs 218 ms per dense sweep).  Once a sweep
    // rotates few pairs (most updates are skipped and launch overhead
    // dominates) the remaining sweeps run as one-stream graph replays.
    const bool graphs = cfg->use_graph && !cfg->profile && !tl_on;
    // the late-sweep graph keeps the two-half schedule (one half's inner pass
    // beside the other half's Gram) unless HSVD_LATE_SPLIT=0
    const bool late_split = split && [] {
        const char *e = getenv("HSVD_LATE_SPLIT");
        return !(e && e[0] == '0');
    }();
    auto capture = [&]() -> int {
        const bool keep = split_now;
        split_now = late_split;
        plan_now = reuse_ok;
        capturing = true;
        HSVD_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        int e = enqueue_sweep();
        cudaError_t ce = cudaStreamEndCapture(s, &graph);
        split_now = keep;
        plan_now = false;
        capturing = false;
        if (e) return e;
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
        HSVD_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        return HSVD_OK;
    };

    const int64_t mv = V ? 4 : 2;  // k_move_cols launches per column move
    int64_t launches = (V ? 1 : 0) + 1 + 1 + 1 + (cfg->sort ? 2 : 0) + 1 + 2 + mv + 1 + mv;
    int64_t sweeps_used = 0, total_rot = 0, total_skip = 0;
    int stop = 2;
    const double t_loop0 = wall_ms();
    res->setup_ms = t_loop0;  // absolute for now; hsvd_drive makes it relative
    for (int64_t sweep = 0; sweep < cfg->max_sweeps; ++sweep) {
        HSVD_CUDA(cudaEventRecord(t0, s));
        {
            // kernels per step: split = 2 x (gram, inner, 3 updates), one
            // stream = gram, inner, update; graphed sweeps add k_plan per launch
            const bool graphed = graphs && !split_now && !passes.dense_now;
            const int64_t per_step = (split_now || (graphed && late_split)) ? 10 : 3;
            const int64_t plans = graphed && reuse_ok ? (late_split ? 2 : 1) : 0;
            launches += (per_step + plans) * nb + 1 + 1 + (cfg->sort ? 4 + mv : 0) + 1;
        }
        // the dense sweeps run eagerly (their inner passes differ from the
        // late sweeps'); the late sweeps replay a graph
        if (split_now || !graphs || passes.dense_now) {
            T.on = cfg->profile && sweep == profile_sweep();
            st = enqueue_sweep();
            if (st) return st;
            // capture the graph for the late sweeps while the device works
            // through this sweep
            if (graphs && !exec) {
                st = capture();
                if (st) return st;
            }
        } else {
            if (!exec) {
                st = capture();
                if (st) return st;
            }
            HSVD_CUDA(cudaGraphLaunch(exec, s));
        }
        HSVD_CUDA(cudaEventRecord(t1, s));
        HSVD_CUDA(cudaStreamSynchronize(s));
        if (T.on) T.collect(res);
        if (tl_on && tl0) {
            for (auto &x : tl) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, tl0, x.second);
                fprintf(stderr, "timeline %9.1f us  %s\n", 1e3 * ms, x.first.c_str());
                cudaEventDestroy(x.second);
            }
            tl.clear();
            cudaEventDestroy(tl0);
            tl0 = nullptr;
        }
        float ms = 0.f;
        HSVD_CUDA(cudaEventElapsedTime(&ms, t0, t1));
        if ((unsigned long long)host[4] != kNoError) {
            unpack_err((unsigned long long)host[4], res->err);
            set_error("definiteness lost at block " + std::to_string(res->err[0]) +
                      ", pivot pair (" + std::to_string(res->err[1]) + ", " +
                      std::to_string(res->err[2]) + ")");
            return HSVD_DEFINITENESS_LOST;
        }
        const int code = (int)host[0];
        double max_t;
        memcpy(&max_t, &host[3], sizeof(double));
        sweeps_used = sweep + 1;
        total_rot += host[1];
        total_skip += host[2];
        // few rotations left: the remaining sweeps skip most updates
        if (split_now && host[1] < (host[1] + host[2]) / 20) split_now = false;
        passes.after_sweep(host[1], host[2]);
        if (tele) {
            tele[sweep].sweep = sweep;
            tele[sweep].rotations = host[1];
            tele[sweep].skips = host[2];
            tele[sweep].max_t = max_t;
            tele[sweep].gpu_ms = ms;
        }
        if (code == 0) { stop = 0; break; }
        if (code == 1) { stop = 1; break; }
    }
    res->sweeps_ms = wall_ms() - t_loop0;
    if (getenv("HSVD_PLAN_STATS")) {
        unsigned long long ps[3] = {0, 0, 0};
        cudaMemcpy(ps, w.sl.ru.planstat, sizeof(ps), cudaMemcpyDeviceToHost);
        fprintf(stderr, "plan stats: full %llu reused %llu cross %llu (planned slot visits)\n",
                ps[0], ps[1], ps[2]);
    }
    // storage back to the original column order, then the extraction
    // (d was refreshed from G at the end of the last sweep, then sorted)
    k_inverse<<<(unsigned)((r + 255) / 256), 256, 0, s>>>(w.rho, w.inv, r);
    HSVD_LAUNCH_CHECK("k_inverse");
    st = move_cols(G, ldg, w.Gs, w.lds, n, r, w.ident, w.inv, s);
    if (!st && V) st = move_cols(V, ldv, w.Vs, r, r, r, w.ident, w.inv, s);
    if (st) return st;
    st = hsvd_extract(G, n, ldg, w.d, w.rho, w.js, r, sigma, lam, s);
    if (st) return st;
    res->sweeps_used = sweeps_used;
    res->stop_reason = stop;
    res->rotations = total_rot;
    res->skips = total_skip;
    res->launches = launches;
    return HSVD_OK;
}

// r not a multiple of 2b: solve the padded factor [G 0] with J = [J, -1...]
// in a workspace copy, then copy U, V^{-T}, sigma and lam back.  The zero
// columns are inert (never rotated, never counted), so the result is the
// solve of G itself; sigma/lam/U of the original columns are unaffected by
// where the padding sits in the sorted order.
static int block_drive_padded(double *G, int64_t n, int64_t r, int64_t ldg, double *V,
                              int64_t ldv, const int8_t *signs_host, int64_t p,
                              const hsvd_config *cfg, double *sigma, double *lam, void *ws,
                              int64_t ws_bytes, hsvd_result *res, hsvd_telemetry *tele,
                              DevCtx &ctx)
{
    const int b = cfg->block_cols;
    Carve2 c{(char *)ws, 0};
    PadWs pw;
    const int64_t pre = carve_pad(c, n, r, b, V != nullptr, &pw);
    if (pre >= ws_bytes) {
        set_error("workspace too small");
        return HSVD_ERR_ARG;
    }
    cudaStream_t s = ctx.s;
    const int64_t rp = pw.rp;
    HSVD_CUDA(cudaMemcpy2DAsync(pw.G, pw.ld * sizeof(double), G, ldg * sizeof(double),
                                n * sizeof(double), r, cudaMemcpyDeviceToDevice, s));
    HSVD_CUDA(cudaMemsetAsync(pw.G + r * pw.ld, 0, (rp - r) * pw.ld * sizeof(double), s));
    std::vector<int8_t> sg(signs_host, signs_host + r);
    sg.resize(rp, (int8_t)-1);
    int st;
    if (b == 16)
        st = block_drive_t<32>(pw.G, n, rp, pw.ld, pw.V, rp, sg.data(), p, cfg, pw.sigma,
                               pw.lam, (char *)ws + pre, ws_bytes - pre, res, tele, ctx, r);
    else
        st = block_drive_t<64>(pw.G, n, rp, pw.ld, pw.V, rp, sg.data(), p, cfg, pw.sigma,
                               pw.lam, (char *)ws + pre, ws_bytes - pre, res, tele, ctx, r);
    if (st) return st;
    HSVD_CUDA(cudaMemcpy2DAsync(G, ldg * sizeof(double), pw.G, pw.ld * sizeof(double),
                                n * sizeof(double), r, cudaMemcpyDeviceToDevice, s));
    if (V)
        HSVD_CUDA(cudaMemcpy2DAsync(V, ldv * sizeof(double), pw.V, rp * sizeof(double),
                                    r * sizeof(double), r, cudaMemcpyDeviceToDevice, s));
    HSVD_CUDA(cudaMemcpyAsync(sigma, pw.sigma, r * sizeof(double), cudaMemcpyDeviceToDevice, s));
    HSVD_CUDA(cudaMemcpyAsync(lam, pw.lam, r * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return HSVD_OK;
}

int block_drive(double *G, int64_t n, int64_t r, int64_t ldg, double *V, int64_t ldv,
                const int8_t *signs_host, int64_t p, const hsvd_config *cfg, double *sigma,
                double *lam, void *ws, int64_t ws_bytes, hsvd_result *res,
                hsvd_telemetry *tele, DevCtx &ctx)
{
    const int b = cfg->block_cols;
    if (b != 16 && b != 32) {
        set_error("block mode supports block_cols 16 or 32");
        return HSVD_ERR_UNSUPPORTED;
    }
    if (r % (2 * b) != 0)
        return block_drive_padded(G, n, r, ldg, V, ldv, signs_host, p, cfg, sigma, lam, ws,
                                  ws_bytes, res, tele, ctx);
    if (ldg % 2 || (V && ldv % 2) || ((uintptr_t)G & 15) || (V && ((uintptr_t)V & 15))) {
        set_error("block mode needs 16-byte aligned columns (even leading dimensions)");
        return HSVD_ERR_UNSUPPORTED;
    }
    if (b == 16)
        return block_drive_t<32>(G, n, r, ldg, V, ldv, signs_host, p, cfg, sigma, lam, ws,
                                 ws_bytes, res, tele, ctx, r);
    return block_drive_t<64>(G, n, r, ldg, V, ldv, signs_host, p, cfg, sigma, lam, ws,
                             ws_bytes, res, tele, ctx, r);
}

}  // namespace hsvd
