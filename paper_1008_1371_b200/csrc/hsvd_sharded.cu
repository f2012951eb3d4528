// hsvd_sharded.cu -- block-column HSVD sharded over GPUs.
//
// The r/(2b) block-pair slots of a step are independent (solver.py:124-131),
// so the slots are split contiguously over N shards and each shard keeps the
// block columns of its slots (G: n x b, V^{-T}: r x b each) resident in its
// own HBM.  The modified-modulus stepper (strategies.py:41-72 on the block
// indices) is a ring: after every step each slot holds one new block that
// came from slot k-1 or k+1 (or the wrap-around).  With contiguous shards a
// shard therefore sends exactly one block column to one ring neighbour and
// receives one per step -- (n + r) * b * 8 bytes by NCCL send/recv over
// NVLink, received into a spare area so sends and receives never alias.
// At the end of a sweep the shards all-gather the column norms, every shard
// runs the identical stable sort (solver.py:97-110), and the columns are
// redistributed to the canonical placement of the next sweep by one grouped
// all-to-all.  The stop decision is an all-reduce of the per-shard
// convergence words, so every rank takes the same branch.
//
// Two transports drive the same plan:
//  * NCCL: one process per GPU (torchrun), one shard per process;
//  * local: one process drives all N shards (streams on one or several
//    devices, copies by cudaMemcpyPeerAsync).  It exists so the sharded path
//    -- plan, exchanges, redistribution, kernels on shard-local storage --
//    runs and is checked on a single GPU.
//
// NCCL is loaded at run time (dlopen), so the library has no link-time NCCL
// dependency for single-GPU users.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include <nccl.h>

#include "hsvd_block_kernels.cuh"

namespace hsvd {

int launch_reduce_sweep(uint8_t *C, int64_t m, uint32_t *rotk, uint32_t *skipk,
                        double *maxt, int64_t nslots, int64_t *out,
                        const unsigned long long *err, int reset, cudaStream_t s);
int launch_init_packages(const int8_t *signs, int64_t r, int64_t *rho,
                         int64_t *jsign, cudaStream_t s);

// ---------------------------------------------------------------------
// NCCL, resolved at run time
// ---------------------------------------------------------------------
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t);
    const char *(*GetErrorString)(ncclResult_t);
};

static NcclApi *nccl()
{
    static NcclApi api;
    static bool tried = false;
    if (tried) return api.ok ? &api : nullptr;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        set_error(std::string("cannot load NCCL: ") + dlerror());
        return nullptr;
    }
#define HSVD_SYM(f)                                                   \
    api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f));   \
    if (!api.f) {                                                     \
        set_error("NCCL symbol missing: nccl" #f);                    \
        return nullptr;                                               \
    }
    HSVD_SYM(GetUniqueId)
    HSVD_SYM(CommInitRank)
    HSVD_SYM(CommDestroy)
    HSVD_SYM(GroupStart)
    HSVD_SYM(GroupEnd)
    HSVD_SYM(Send)
    HSVD_SYM(Recv)
    HSVD_SYM(AllGather)
    HSVD_SYM(AllReduce)
    HSVD_SYM(GetErrorString)
#undef HSVD_SYM
    api.ok = true;
    return &api;
}

struct Comm {
    ncclComm_t comm;
    int nranks, rank;
};

#define HSVD_NCCL(call)                                                              \
    do {                                                                             \
        ncclResult_t _r = (call);                                                    \
        if (_r != ncclSuccess) {                                                     \
            set_error(std::string(#call) + ": " + nccl()->GetErrorString(_r));       \
            return HSVD_ERR_CUDA;                                                    \
        }                                                                            \
    } while (0)

#define HSVD_CUDA_OK(call)          \
    do {                            \
        int _s = (call);            \
        if (_s) return _s;          \
    } while (0)

// ---------------------------------------------------------------------
// the shard plan (host, identical on every rank)
// ---------------------------------------------------------------------
struct Move {
    int64_t P;        // block index
    int from, from_area, to, to_area;
};

struct ShardPlan {
    int64_t nb = 0, S = 0;
    int N = 0;
    std::vector<int64_t> s0;                  // shard g owns slots [s0[g], s0[g+1])
    std::vector<int64_t> ip, jp, iblk, jblk;  // the stepper of all S slots
    std::vector<int> owner, area;             // per block
    std::vector<int> spare;                   // per shard

    int64_t m(int g) const { return s0[g + 1] - s0[g]; }
    int64_t areas(int g) const { return 2 * m(g) + 1; }
    int64_t max_areas() const
    {
        int64_t a = 0;
        for (int g = 0; g < N; ++g) a = std::max(a, areas(g));
        return a;
    }
    int shard_of(int64_t k) const
    {
        return (int)(std::upper_bound(s0.begin(), s0.end(), k) - s0.begin()) - 1;
    }
    int init(int64_t nblocks, int nshards)
    {
        nb = nblocks;
        S = nb / 2;
        N = nshards;
        if (N < 1 || S < N || nb % 2) {
            set_error("sharded: need r/(2b) >= number of shards");
            return HSVD_ERR_UNSUPPORTED;
        }
        s0.resize(N + 1);
        for (int g = 0; g <= N; ++g) s0[g] = (int64_t)g * S / N;
        ip.resize(S), jp.resize(S), iblk.resize(S), jblk.resize(S);
        for (int64_t k = 0; k < S; ++k) {  // stepper_init (strategies.py:41-47)
            ip[k] = iblk[k] = k;
            jp[k] = jblk[k] = nb - k - 1;
        }
        owner.assign(nb, -1);
        area.assign(nb, -1);
        spare.assign(N, 0);
        place();
        return HSVD_OK;
    }
    // canonical placement of the current pairs: slot k's iblk in area
    // 2(k - s0), its jblk in 2(k - s0) + 1, the spare last
    void place()
    {
        for (int64_t k = 0; k < S; ++k) {
            const int g = shard_of(k);
            const int a = (int)(2 * (k - s0[g]));
            owner[iblk[k]] = g;
            area[iblk[k]] = a;
            owner[jblk[k]] = g;
            area[jblk[k]] = a + 1;
        }
        for (int g = 0; g < N; ++g) spare[g] = (int)(2 * m(g));
    }
    // advance_stepper (_kernels.py:238-251) on every slot, then the
    // cross-shard block moves that make the next pairs resident
    int advance(std::vector<Move> &mv)
    {
        mv.clear();
        const int64_t r = nb, half = nb / 2;
        std::vector<int> in(N, 0), out(N, 0);
        for (int64_t k = 0; k < S; ++k) {
            int64_t P;
            if (ip[k] + jp[k] >= r - 1) {
                ip[k] += 1;
                if (ip[k] == jp[k]) {
                    ip[k] -= half;
                    jp[k] = ip[k];
                }
                iblk[k] = ip[k];
                P = iblk[k];
            } else {
                jp[k] += 1;
                jblk[k] = jp[k];
                P = jblk[k];
            }
            const int to = shard_of(k);
            if (owner[P] != to) {
                mv.push_back(Move{P, owner[P], area[P], to, -1});
                in[to]++;
                out[owner[P]]++;
            }
        }
        for (int g = 0; g < N; ++g)
            if (in[g] > 1 || in[g] != out[g]) {
                set_error("sharded: plan needs more than one block exchange per shard and step");
                return HSVD_ERR_UNSUPPORTED;
            }
        // receive into the spare; the departing block's area is the new spare
        for (auto &x : mv) x.to_area = spare[x.to];
        for (auto &x : mv) {
            spare[x.from] = x.from_area;
            owner[x.P] = x.to;
            area[x.P] = x.to_area;
        }
        return HSVD_OK;
    }
    // block held in area a of shard g (-1 for the spare)
    std::vector<int64_t> blocks_of(int g) const
    {
        std::vector<int64_t> out(areas(g), -1);
        for (int64_t P = 0; P < nb; ++P)
            if (owner[P] == g) out[area[P]] = P;
        return out;
    }
};

// Redistribution of the columns after the sort: column x moves from its old
// (shard, local column) to the canonical placement of its new position.
// send[g][h] lists the local columns shard g sends to h, recv[h][g] the
// local columns they land in (same order).
struct Redist {
    std::vector<std::vector<std::vector<int64_t>>> send, recv;
};

static void plan_redistribute(const ShardPlan &old_pl, const ShardPlan &new_pl, int64_t b,
                              const std::vector<int64_t> &rho_old,
                              const std::vector<int64_t> &rho_new, Redist &R)
{
    const int N = old_pl.N;
    const int64_t r = (int64_t)rho_old.size();
    std::vector<int64_t> inv(r);
    for (int64_t q = 0; q < r; ++q) inv[rho_old[q]] = q;
    R.send.assign(N, std::vector<std::vector<int64_t>>(N));
    R.recv.assign(N, std::vector<std::vector<int64_t>>(N));
    for (int64_t qn = 0; qn < r; ++qn) {
        const int64_t qo = inv[rho_new[qn]];
        const int64_t Po = qo / b, Pn = qn / b;
        const int go = old_pl.owner[Po], gn = new_pl.owner[Pn];
        R.send[go][gn].push_back(old_pl.area[Po] * b + qo % b);
        R.recv[gn][go].push_back(new_pl.area[Pn] * b + qn % b);
    }
}

// ---------------------------------------------------------------------
// small kernels of the sharded path
// ---------------------------------------------------------------------
// dst[:, k] = src[:, idx[k]] (idx < 0: leave), columns of length len
__global__ void k_gather_cols(double *__restrict__ dst, int64_t ldd,
                              const double *__restrict__ src, int64_t lds,
                              const int64_t *__restrict__ idx, int64_t len)
{
    const int64_t k = blockIdx.y;
    const int64_t c = idx[k];
    if (c < 0) return;
    const double *s = src + c * lds;
    double *d = dst + k * ldd;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
         e += (int64_t)gridDim.x * blockDim.x)
        d[e] = s[e];
}

// dst[:, idx[k]] = src[:, k]
__global__ void k_scatter_cols(double *__restrict__ dst, int64_t ldd,
                               const double *__restrict__ src, int64_t lds,
                               const int64_t *__restrict__ idx, int64_t len)
{
    const int64_t k = blockIdx.y;
    const double *s = src + k * lds;
    double *d = dst + idx[k] * ldd;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
         e += (int64_t)gridDim.x * blockDim.x)
        d[e] = s[e];
}

// V storage column k = e_{idx[k]} (the identity's column), idx < 0: leave
__global__ void k_unit_cols(double *__restrict__ V, int64_t ldv, const int64_t *__restrict__ idx,
                            int64_t r)
{
    const int64_t k = blockIdx.y;
    const int64_t c = idx[k];
    if (c < 0) return;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < r;
         e += (int64_t)gridDim.x * blockDim.x)
        V[k * ldv + e] = e == c ? 1.0 : 0.0;
}

// loc[P*b + c] = a*b + c for one received block
__global__ void k_set_loc(int64_t *loc, int64_t P, int64_t a, int b)
{
    const int c = threadIdx.x;
    if (c < b) loc[P * b + c] = a * b + c;
}

// d[q] = dall[posmap[q]]
__global__ void k_gather_d(double *d, const double *dall, const int64_t *posmap, int64_t r)
{
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < r) d[q] = dall[posmap[q]];
}

// squared norms of the storage columns (one warp per column)
__global__ void k_storage_norms(const double *__restrict__ G, int64_t ldg, int n, int64_t ncols,
                                double *__restrict__ dloc)
{
    const int64_t k = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (k >= ncols) return;
    const double *g = G + k * ldg;
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
    if (lane == 0) dloc[k] = s;
}

// convergence word of one shard -> all-reduce operands:
// mx = {code, max|t| bits, ~err} (max), sm = {rotations, skips} (sum)
__global__ void k_pack_stats(const int64_t *out, unsigned long long *mx, long long *sm)
{
    mx[0] = (unsigned long long)out[0];
    mx[1] = (unsigned long long)out[3];
    mx[2] = ~(unsigned long long)out[4];
    sm[0] = out[1];
    sm[1] = out[2];
}

// extraction on the canonical placement: column k holds position qpos[k]
// (solver.py:261-267): sigma = sqrt(d), lam = d * j, U = G / sigma
__global__ void k_shard_extract(const double *__restrict__ d, const int64_t *__restrict__ js,
                                const int64_t *__restrict__ qpos, int64_t ncols,
                                double *__restrict__ sigma, double *__restrict__ lam)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= ncols) return;
    const int64_t q = qpos[k];
    sigma[k] = __dsqrt_rn(d[q]);
    lam[k] = __dmul_rn(d[q], (double)js[q]);
}

__global__ void k_shard_scale(double *__restrict__ U, int64_t ldu, const double *__restrict__ G,
                              int64_t ldg, int64_t n, const double *__restrict__ sigma)
{
    const int64_t c = blockIdx.y;
    const double s = sigma[c];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        U[c * ldu + e] = __ddiv_rn(G[c * ldg + e], s);
}

static unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
static unsigned colgrid(int64_t len)
{
    unsigned g = nblk(len, 256);
    return g > 64 ? 64 : g;
}

// ---------------------------------------------------------------------
// per-shard state
// ---------------------------------------------------------------------
struct ShardWs {
    double *Gs, *Vs;          // storage: areas*b columns (ld n / r)
    double *sendG, *sendV;    // redistribution buffers: 2m*b columns
    double *recvG, *recvV;
    double *dloc, *dall, *d;  // norms of storage columns, all shards', by position
    int64_t *rho, *js, *loc, *posmap;
    int64_t *idx_a, *idx_b;   // column index lists (send / recv / gather)
    void *sortws;
    int64_t *out;
    unsigned long long *mx;
    long long *sm;
    unsigned long long *first_zero;
    int8_t *signs;
    double *sigma, *lam;
    SlotWs sl;
    SlotWs half[2];  // split mode: the two halves of the shard's slots
};

static int64_t carve_shard(Carve2 &c, const ShardPlan &pl, int g, int64_t n, int64_t r, int b,
                           bool withV, ShardWs *w)
{
    const int64_t m = pl.m(g), A = pl.areas(g), stride = pl.max_areas() * b;
    ShardWs t;
    t.Gs = c.take<double>(A * b * n);
    t.Vs = withV ? c.take<double>(A * b * r) : nullptr;
    t.sendG = c.take<double>(2 * m * b * n);
    t.recvG = c.take<double>(2 * m * b * n);
    t.sendV = withV ? c.take<double>(2 * m * b * r) : nullptr;
    t.recvV = withV ? c.take<double>(2 * m * b * r) : nullptr;
    t.dloc = c.take<double>(stride);
    t.dall = c.take<double>(stride * pl.N);
    t.d = c.take<double>(r);
    t.rho = c.take<int64_t>(r);
    t.js = c.take<int64_t>(r);
    t.loc = c.take<int64_t>(r);
    t.posmap = c.take<int64_t>(r);
    t.idx_a = c.take<int64_t>(std::max<int64_t>(A * b, r));
    t.idx_b = c.take<int64_t>(std::max<int64_t>(A * b, r));
    t.sortws = c.take<char>(24 * r);
    t.out = c.take<int64_t>(8);
    t.mx = c.take<unsigned long long>(4);
    t.sm = c.take<long long>(4);
    t.first_zero = c.take<unsigned long long>(1);
    t.signs = c.take<int8_t>(r);
    t.sigma = c.take<double>(2 * m * b);
    t.lam = c.take<double>(2 * m * b);
    carve_slots(c, n, m, pl.nb, b, &t.sl);
    t.sl.colmap = t.loc;
    t.sl.js = t.js;
    t.sl.slot_base = pl.s0[g];
    const int64_t B2 = 2 * b;
    for (int h = 0; h < 2; ++h) {
        const int64_t lo = h ? m / 2 : 0, hi = h ? m : m / 2;
        const int64_t mh = hi > lo ? hi - lo : 1;
        SlotWs v = t.sl;
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
        v.nslots = hi - lo;
        v.slot_base = pl.s0[g] + lo;
        v.gp = gram_partition(n, mh);
        v.maxseg = gram_maxseg(v.gp, mh);
        v.Apart = c.take<double>(mh * v.maxseg * B2 * B2);
        t.half[h] = v;
    }
    if (w) *w = t;
    return c.off + 256;
}

struct Shard {
    int g = 0, dev = 0;
    cudaStream_t s = nullptr;
    cudaEvent_t ev = nullptr, t0 = nullptr, t1 = nullptr;
    const double *G = nullptr;  // the caller's full factor on this device
    ShardWs w;
    alignas(64) CUtensorMap gmap;  // k_gram_tma's view of the shard's storage
    // split mode: half B's stream, the (high-priority) exchange stream and
    // their events: edge updates per half and step parity, exchange per
    // step parity, sweep fork / join, first-step stagger
    cudaStream_t s2 = nullptr, sc = nullptr;
    cudaEvent_t e_edge[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    cudaEvent_t e_comm[2] = {nullptr, nullptr}, e_fork = nullptr, e_join = nullptr,
                e_join2 = nullptr, e_stag = nullptr;
};

// ---------------------------------------------------------------------
// the driver
// ---------------------------------------------------------------------
template <int B2>
struct ShardedDriver {
    using K = BlockKernels<B2>;
    static constexpr int b = B2 / 2;

    Comm *comm;                      // nullptr: local transport
    std::vector<Shard> sh;           // the shards this process drives
    ShardPlan pl;
    int64_t n, r, ldg, p;
    const hsvd_config *cfg;
    PassPolicy passes;  // inner passes per sweep (the one-GPU driver's policy)
    bool withV;
    // pinned host memory: [0, rho_off) per-shard stats, [rho_off, stage_base)
    // a copy of rho, then the staging of the uploads of one sync epoch
    int64_t *host = nullptr;
    int64_t host_len = 0, rho_off = 0, stage_base = 0, stage_off = 0;
    int64_t launches = 0;
    bool split = false;

    ~ShardedDriver()
    {
        // streams, events and pinned memory belong to the device contexts
        for (auto &x : sh) {
            cudaSetDevice(x.dev);
            if (x.s) cudaStreamSynchronize(x.s);
        }
    }

    int local_index(int g) const
    {
        for (size_t i = 0; i < sh.size(); ++i)
            if (sh[i].g == g) return (int)i;
        return -1;
    }

    // every local stream waits for the work so far on every other one
    int local_barrier()
    {
        if (sh.size() < 2) return HSVD_OK;
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            HSVD_CUDA(cudaEventRecord(x.ev, x.s));
        }
        for (auto &x : sh)
            for (auto &y : sh)
                if (&x != &y) HSVD_CUDA(cudaStreamWaitEvent(x.s, y.ev, 0));
        return HSVD_OK;
    }

    int upload(Shard &x, int64_t *dst, const std::vector<int64_t> &v)
    {
        if (v.empty()) return HSVD_OK;
        // pinned staging per call: the copies are stream ordered, so a
        // fresh region per upload within one sync epoch
        if (stage_off + (int64_t)v.size() > host_len) {
            set_error("sharded: host staging overflow");
            return HSVD_ERR_ARG;
        }
        int64_t *h = host + stage_off;
        memcpy(h, v.data(), v.size() * sizeof(int64_t));
        stage_off += (int64_t)v.size();
        HSVD_CUDA(cudaMemcpyAsync(dst, h, v.size() * sizeof(int64_t), cudaMemcpyHostToDevice, x.s));
        return HSVD_OK;
    }
    int sync_all()
    {
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            HSVD_CUDA(cudaStreamSynchronize(x.s));
        }
        stage_off = stage_base;
        return HSVD_OK;
    }

    // loc of the resident positions of shard g under the current placement
    std::vector<int64_t> loc_table(int g) const
    {
        std::vector<int64_t> loc(r, -1);
        for (int64_t P = 0; P < pl.nb; ++P)
            if (pl.owner[P] == g)
                for (int c = 0; c < b; ++c) loc[P * b + c] = (int64_t)pl.area[P] * b + c;
        return loc;
    }

    // one exchange of blocks after a step
    int exchange(const std::vector<Move> &mv)
    {
        if (mv.empty()) return HSVD_OK;
        if (!comm) {
            HSVD_CUDA_OK(local_barrier());
            for (const auto &x : mv) {
                Shard &src = sh[local_index(x.from)], &dst = sh[local_index(x.to)];
                HSVD_CUDA(cudaSetDevice(dst.dev));
                HSVD_CUDA(cudaMemcpyPeerAsync(dst.w.Gs + (int64_t)x.to_area * b * n, dst.dev,
                                              src.w.Gs + (int64_t)x.from_area * b * n, src.dev,
                                              sizeof(double) * b * n, dst.s));
                if (withV)
                    HSVD_CUDA(cudaMemcpyPeerAsync(dst.w.Vs + (int64_t)x.to_area * b * r, dst.dev,
                                                  src.w.Vs + (int64_t)x.from_area * b * r,
                                                  src.dev, sizeof(double) * b * r, dst.s));
                k_set_loc<<<1, 64, 0, dst.s>>>(dst.w.loc, x.P, x.to_area, b);
                HSVD_LAUNCH_CHECK("k_set_loc");
                ++launches;
            }
            return local_barrier();
        }
        Shard &x = sh[0];
        NcclApi *N = nccl();
        HSVD_NCCL(N->GroupStart());
        for (const auto &m : mv) {
            if (m.from == x.g) {
                HSVD_NCCL(N->Send(x.w.Gs + (int64_t)m.from_area * b * n, (size_t)b * n,
                                  ncclFloat64, m.to, comm->comm, x.s));
                if (withV)
                    HSVD_NCCL(N->Send(x.w.Vs + (int64_t)m.from_area * b * r, (size_t)b * r,
                                      ncclFloat64, m.to, comm->comm, x.s));
            }
            if (m.to == x.g) {
                HSVD_NCCL(N->Recv(x.w.Gs + (int64_t)m.to_area * b * n, (size_t)b * n,
                                  ncclFloat64, m.from, comm->comm, x.s));
                if (withV)
                    HSVD_NCCL(N->Recv(x.w.Vs + (int64_t)m.to_area * b * r, (size_t)b * r,
                                      ncclFloat64, m.from, comm->comm, x.s));
            }
        }
        HSVD_NCCL(N->GroupEnd());
        for (const auto &m : mv)
            if (m.to == x.g) {
                k_set_loc<<<1, 64, 0, x.s>>>(x.w.loc, m.P, m.to_area, b);
                HSVD_LAUNCH_CHECK("k_set_loc");
                ++launches;
            }
        return HSVD_OK;
    }

    // all-gather of the storage norms, then d by position on every shard
    int gather_norms()
    {
        const int64_t stride = pl.max_areas() * b;
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            const int64_t nc = pl.areas(x.g) * b;
            k_storage_norms<<<nblk(nc, 8), 256, 0, x.s>>>(x.w.Gs, n, (int)n, nc, x.w.dloc);
            HSVD_LAUNCH_CHECK("k_storage_norms");
            ++launches;
            // position -> slot of dall
            std::vector<int64_t> pm(r);
            for (int64_t q = 0; q < r; ++q) {
                const int64_t P = q / b;
                pm[q] = pl.owner[P] * stride + (int64_t)pl.area[P] * b + q % b;
            }
            HSVD_CUDA_OK(upload(x, x.w.posmap, pm));
        }
        if (!comm) {
            HSVD_CUDA_OK(local_barrier());
            for (auto &x : sh)
                for (auto &y : sh) {
                    HSVD_CUDA(cudaSetDevice(x.dev));
                    HSVD_CUDA(cudaMemcpyPeerAsync(x.w.dall + (int64_t)y.g * stride, x.dev, y.w.dloc,
                                                  y.dev, sizeof(double) * stride, x.s));
                }
            HSVD_CUDA_OK(local_barrier());
        } else {
            Shard &x = sh[0];
            HSVD_NCCL(nccl()->AllGather(x.w.dloc, x.w.dall, (size_t)stride, ncclFloat64,
                                        comm->comm, x.s));
        }
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            k_gather_d<<<nblk(r, 256), 256, 0, x.s>>>(x.w.d, x.w.dall, x.w.posmap, r);
            HSVD_LAUNCH_CHECK("k_gather_d");
            ++launches;
        }
        return HSVD_OK;
    }

    // convergence word of the sweep, reduced over all shards, to host[0..4]
    int reduce_stats()
    {
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            HSVD_CUDA_OK(launch_reduce_sweep(x.w.sl.C, x.w.sl.nslots, x.w.sl.rotk, x.w.sl.skipk,
                                             x.w.sl.maxt, x.w.sl.nslots, x.w.out, x.w.sl.err, 1,
                                             x.s));
            ++launches;
        }
        if (comm) {
            Shard &x = sh[0];
            k_pack_stats<<<1, 1, 0, x.s>>>(x.w.out, x.w.mx, x.w.sm);
            HSVD_LAUNCH_CHECK("k_pack_stats");
            ++launches;
            HSVD_NCCL(nccl()->AllReduce(x.w.mx, x.w.mx, 3, ncclUint64, ncclMax, comm->comm, x.s));
            HSVD_NCCL(nccl()->AllReduce(x.w.sm, x.w.sm, 2, ncclInt64, ncclSum, comm->comm, x.s));
            HSVD_CUDA(cudaMemcpyAsync(host, x.w.mx, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, x.s));
            HSVD_CUDA(cudaMemcpyAsync(host + 3, x.w.sm, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                      x.s));
        } else {
            for (size_t i = 0; i < sh.size(); ++i) {
                HSVD_CUDA(cudaSetDevice(sh[i].dev));
                HSVD_CUDA(cudaMemcpyAsync(host + 5 * i, sh[i].w.out, 5 * sizeof(int64_t),
                                          cudaMemcpyDeviceToHost, sh[i].s));
            }
        }
        return HSVD_OK;
    }
    // after sync: combine into {code, rot, skip, maxt bits, err}
    void combine_stats(int64_t out[5]) const
    {
        if (comm) {
            out[0] = host[0];
            out[3] = host[1];
            out[4] = (int64_t)~(unsigned long long)host[2];
            out[1] = host[3];
            out[2] = host[4];
            return;
        }
        unsigned long long code = 0, mt = 0, err = ~0ull;
        int64_t rot = 0, skip = 0;
        for (size_t i = 0; i < sh.size(); ++i) {
            const int64_t *o = host + 5 * i;
            code |= (unsigned long long)o[0];
            rot += o[1];
            skip += o[2];
            mt = std::max(mt, (unsigned long long)o[3]);
            err = std::min(err, (unsigned long long)o[4]);
        }
        out[0] = (int64_t)code;
        out[1] = rot;
        out[2] = skip;
        out[3] = (int64_t)mt;
        out[4] = (int64_t)err;
    }

    // columns to their canonical placement under the new rho
    int redistribute(const ShardPlan &old_pl, const std::vector<int64_t> &rho_old,
                     const std::vector<int64_t> &rho_new)
    {
        Redist R;
        plan_redistribute(old_pl, pl, b, rho_old, rho_new, R);
        const int N = pl.N;
        // pack (per destination, in destination order)
        std::vector<std::vector<int64_t>> soff(sh.size()), roff(sh.size());
        for (size_t i = 0; i < sh.size(); ++i) {
            Shard &x = sh[i];
            HSVD_CUDA(cudaSetDevice(x.dev));
            std::vector<int64_t> sl, rl;
            soff[i].assign(N + 1, 0);
            roff[i].assign(N + 1, 0);
            for (int h = 0; h < N; ++h) {
                soff[i][h + 1] = soff[i][h] + (int64_t)R.send[x.g][h].size();
                sl.insert(sl.end(), R.send[x.g][h].begin(), R.send[x.g][h].end());
                roff[i][h + 1] = roff[i][h] + (int64_t)R.recv[x.g][h].size();
                rl.insert(rl.end(), R.recv[x.g][h].begin(), R.recv[x.g][h].end());
            }
            HSVD_CUDA_OK(upload(x, x.w.idx_a, sl));
            HSVD_CUDA_OK(upload(x, x.w.idx_b, rl));
            const int64_t ns = (int64_t)sl.size();
            if (ns) {
                k_gather_cols<<<dim3(colgrid(n), (unsigned)ns), 256, 0, x.s>>>(x.w.sendG, n, x.w.Gs,
                                                                             n, x.w.idx_a, n);
                HSVD_LAUNCH_CHECK("k_gather_cols");
                ++launches;
                if (withV) {
                    k_gather_cols<<<dim3(colgrid(r), (unsigned)ns), 256, 0, x.s>>>(
                        x.w.sendV, r, x.w.Vs, r, x.w.idx_a, r);
                    HSVD_LAUNCH_CHECK("k_gather_cols");
                    ++launches;
                }
            }
        }
        // all-to-all
        if (!comm) {
            HSVD_CUDA_OK(local_barrier());
            for (size_t i = 0; i < sh.size(); ++i) {
                Shard &dst = sh[i];
                HSVD_CUDA(cudaSetDevice(dst.dev));
                for (size_t j = 0; j < sh.size(); ++j) {
                    Shard &src = sh[j];
                    const int64_t cnt = roff[i][src.g + 1] - roff[i][src.g];
                    if (!cnt) continue;
                    const int64_t so = soff[j][dst.g];
                    HSVD_CUDA(cudaMemcpyPeerAsync(dst.w.recvG + roff[i][src.g] * n, dst.dev,
                                                  src.w.sendG + so * n, src.dev,
                                                  sizeof(double) * cnt * n, dst.s));
                    if (withV)
                        HSVD_CUDA(cudaMemcpyPeerAsync(dst.w.recvV + roff[i][src.g] * r, dst.dev,
                                                      src.w.sendV + so * r, src.dev,
                                                      sizeof(double) * cnt * r, dst.s));
                }
            }
            HSVD_CUDA_OK(local_barrier());
        } else {
            Shard &x = sh[0];
            NcclApi *Nc = nccl();
            HSVD_NCCL(Nc->GroupStart());
            for (int h = 0; h < N; ++h) {
                const int64_t cs = soff[0][h + 1] - soff[0][h], cr = roff[0][h + 1] - roff[0][h];
                if (h == x.g) {
                    if (cs)
                        HSVD_CUDA(cudaMemcpyAsync(x.w.recvG + roff[0][h] * n, x.w.sendG + soff[0][h] * n,
                                                  sizeof(double) * cs * n, cudaMemcpyDeviceToDevice,
                                                  x.s));
                    if (cs && withV)
                        HSVD_CUDA(cudaMemcpyAsync(x.w.recvV + roff[0][h] * r, x.w.sendV + soff[0][h] * r,
                                                  sizeof(double) * cs * r, cudaMemcpyDeviceToDevice,
                                                  x.s));
                    continue;
                }
                if (cs) {
                    HSVD_NCCL(Nc->Send(x.w.sendG + soff[0][h] * n, (size_t)(cs * n), ncclFloat64, h,
                                       comm->comm, x.s));
                    if (withV)
                        HSVD_NCCL(Nc->Send(x.w.sendV + soff[0][h] * r, (size_t)(cs * r), ncclFloat64,
                                           h, comm->comm, x.s));
                }
                if (cr) {
                    HSVD_NCCL(Nc->Recv(x.w.recvG + roff[0][h] * n, (size_t)(cr * n), ncclFloat64, h,
                                       comm->comm, x.s));
                    if (withV)
                        HSVD_NCCL(Nc->Recv(x.w.recvV + roff[0][h] * r, (size_t)(cr * r), ncclFloat64,
                                           h, comm->comm, x.s));
                }
            }
            HSVD_NCCL(Nc->GroupEnd());
        }
        // unpack into the canonical areas, rebuild loc
        for (size_t i = 0; i < sh.size(); ++i) {
            Shard &x = sh[i];
            HSVD_CUDA(cudaSetDevice(x.dev));
            const int64_t nr = roff[i][N];
            if (nr) {
                k_scatter_cols<<<dim3(colgrid(n), (unsigned)nr), 256, 0, x.s>>>(x.w.Gs, n, x.w.recvG,
                                                                              n, x.w.idx_b, n);
                HSVD_LAUNCH_CHECK("k_scatter_cols");
                ++launches;
                if (withV) {
                    k_scatter_cols<<<dim3(colgrid(r), (unsigned)nr), 256, 0, x.s>>>(
                        x.w.Vs, r, x.w.recvV, r, x.w.idx_b, r);
                    HSVD_LAUNCH_CHECK("k_scatter_cols");
                    ++launches;
                }
            }
            HSVD_CUDA_OK(upload(x, x.w.loc, loc_table(x.g)));
        }
        return HSVD_OK;
    }

    // One sweep in split mode.  Per shard, the two halves of its slots run
    // on two streams as in the one-GPU driver (Gram, inner pass and edge-slot
    // updates at high priority, the bulk update behind them); half h's step
    // t + 1 waits for the other half's edge updates and for the shard's
    // exchange of step t.  The exchange of step t runs on a high-priority
    // stream as soon as the edge slots (the only ones that can hold an
    // outgoing block) are updated, so it overlaps the bulk updates.
    int sweep_split(std::vector<Move> &mv)
    {
        const int64_t nb = pl.nb;
        KernelTimer Toff;
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            HSVD_CUDA(cudaEventRecord(x.e_fork, x.s));
            HSVD_CUDA(cudaStreamWaitEvent(x.s2, x.e_fork, 0));
            HSVD_CUDA(cudaStreamWaitEvent(x.sc, x.e_fork, 0));
        }
        for (int64_t step = 0; step < nb; ++step) {
            const int full = cfg->inner_full || step == 0;
            const int par = step & 1;
            for (auto &x : sh) {
                HSVD_CUDA(cudaSetDevice(x.dev));
                cudaStream_t ss[2] = {x.s, x.s2};
                for (int h = 0; h < 2; ++h) {
                    const SlotWs &hw = x.w.half[h];
                    const int64_t m = hw.nslots;
                    if (step > 0) {
                        HSVD_CUDA(cudaStreamWaitEvent(ss[h], x.e_edge[h ^ 1][par ^ 1], 0));
                        HSVD_CUDA(cudaStreamWaitEvent(ss[h], x.e_comm[par ^ 1], 0));
                    } else if (h == 1) {
                        HSVD_CUDA(cudaStreamWaitEvent(ss[h], x.e_stag, 0));
                    }
                    double *V = withV ? x.w.Vs : nullptr;
                    HSVD_CUDA_OK(K::gram_inner(x.w.Gs, n, (int)n, hw, full, passes.now(), ss[h], Toff,
                                               (int)step, false));
                    if (step == 0 && h == 0) HSVD_CUDA(cudaEventRecord(x.e_stag, ss[h]));
                    HSVD_CUDA_OK(K::update(x.w.Gs, n, (int)n, V, r, (int)r, hw, 0, 1, ss[h], Toff,
                                           true));
                    HSVD_CUDA_OK(K::update(x.w.Gs, n, (int)n, V, r, (int)r, hw, m - 1, m, ss[h],
                                           Toff, true));
                    HSVD_CUDA(cudaEventRecord(x.e_edge[h][par], ss[h]));
                    HSVD_CUDA_OK(K::update(x.w.Gs, n, (int)n, V, r, (int)r, hw, 1, m - 1, ss[h],
                                           Toff));
                    launches += 5;
                }
            }
            HSVD_CUDA_OK(pl.advance(mv));
            // exchange of step t on each shard's exchange stream
            for (auto &x : sh) {
                HSVD_CUDA(cudaSetDevice(x.dev));
                if (comm) {
                    HSVD_CUDA(cudaStreamWaitEvent(x.sc, x.e_edge[0][par], 0));
                    HSVD_CUDA(cudaStreamWaitEvent(x.sc, x.e_edge[1][par], 0));
                } else {  // local transport: the sources are other shards
                    for (auto &y : sh) {
                        HSVD_CUDA(cudaStreamWaitEvent(x.sc, y.e_edge[0][par], 0));
                        HSVD_CUDA(cudaStreamWaitEvent(x.sc, y.e_edge[1][par], 0));
                        if (step > 0 && &y != &x)
                            HSVD_CUDA(cudaStreamWaitEvent(x.sc, y.e_comm[par ^ 1], 0));
                    }
                }
            }
            if (comm && !mv.empty()) {
                Shard &x = sh[0];
                NcclApi *Nc = nccl();
                HSVD_NCCL(Nc->GroupStart());
                for (const auto &mm : mv) {
                    if (mm.from == x.g) {
                        HSVD_NCCL(Nc->Send(x.w.Gs + (int64_t)mm.from_area * b * n, (size_t)b * n,
                                           ncclFloat64, mm.to, comm->comm, x.sc));
                        if (withV)
                            HSVD_NCCL(Nc->Send(x.w.Vs + (int64_t)mm.from_area * b * r,
                                               (size_t)b * r, ncclFloat64, mm.to, comm->comm, x.sc));
                    }
                    if (mm.to == x.g) {
                        HSVD_NCCL(Nc->Recv(x.w.Gs + (int64_t)mm.to_area * b * n, (size_t)b * n,
                                           ncclFloat64, mm.from, comm->comm, x.sc));
                        if (withV)
                            HSVD_NCCL(Nc->Recv(x.w.Vs + (int64_t)mm.to_area * b * r,
                                               (size_t)b * r, ncclFloat64, mm.from, comm->comm,
                                               x.sc));
                    }
                }
                HSVD_NCCL(Nc->GroupEnd());
            }
            for (const auto &mm : mv) {
                const int li = local_index(mm.to);
                if (li < 0) continue;
                Shard &dst = sh[li];
                HSVD_CUDA(cudaSetDevice(dst.dev));
                if (!comm) {
                    Shard &src = sh[local_index(mm.from)];
                    HSVD_CUDA(cudaMemcpyPeerAsync(dst.w.Gs + (int64_t)mm.to_area * b * n, dst.dev,
                                                  src.w.Gs + (int64_t)mm.from_area * b * n,
                                                  src.dev, sizeof(double) * b * n, dst.sc));
                    if (withV)
                        HSVD_CUDA(cudaMemcpyPeerAsync(dst.w.Vs + (int64_t)mm.to_area * b * r,
                                                      dst.dev,
                                                      src.w.Vs + (int64_t)mm.from_area * b * r,
                                                      src.dev, sizeof(double) * b * r, dst.sc));
                }
                k_set_loc<<<1, 64, 0, dst.sc>>>(dst.w.loc, mm.P, mm.to_area, b);
                HSVD_LAUNCH_CHECK("k_set_loc");
                ++launches;
            }
            for (auto &x : sh) {
                HSVD_CUDA(cudaSetDevice(x.dev));
                HSVD_CUDA(cudaEventRecord(x.e_comm[par], x.sc));
            }
        }
        // join: the sweep-end work runs on the shard's main stream
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            HSVD_CUDA(cudaEventRecord(x.e_join, x.s2));
            HSVD_CUDA(cudaEventRecord(x.e_join2, x.sc));
            HSVD_CUDA(cudaStreamWaitEvent(x.s, x.e_join, 0));
            HSVD_CUDA(cudaStreamWaitEvent(x.s, x.e_join2, 0));
        }
        return HSVD_OK;
    }

    int run(int8_t const *signs_host, double *const *U_out, double *const *V_out,
            int64_t *const *cols_host, double *const *sigma_out, double *const *lam_out,
            hsvd_result *res, hsvd_telemetry *tele)
    {
        const int64_t nb = r / b;
        HSVD_CUDA_OK(pl.init(nb, (int)(comm ? comm->nranks : sh.size())));
        passes.init(cfg, nb);
        split = cfg->block_streams >= 2 && !cfg->profile;
        for (auto &x : sh)
            if (pl.m(x.g) < 4) split = false;
        rho_off = 8 * std::max<int64_t>(2, (int64_t)sh.size());
        stage_base = rho_off + r;
        host_len = stage_base + (int64_t)sh.size() * (8 * r + 4 * pl.max_areas() * b + 1024);
        // borrow streams / events / pinned memory from the device contexts:
        // the k-th shard on a device takes that device's k-th extra stream
        std::vector<int> used_on;
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            HSVD_CUDA_OK(K::setup());
            int cst = 0;
            DevCtx *c = dev_ctx(x.dev, &cst);
            if (!c) return cst;
            if ((int)used_on.size() <= x.dev) used_on.resize(x.dev + 1, 0);
            const int k = used_on[x.dev]++;
            HSVD_CUDA_OK(c->extra(2 * k + 2));
            HSVD_CUDA_OK(c->extra_hi(k + 1));
            HSVD_CUDA_OK(c->events(10 * k + 10));
            x.s = c->xs[2 * k];
            x.ev = c->xev[2 * k];
            x.t0 = c->xt0[2 * k];
            x.t1 = c->xt1[2 * k];
            x.s2 = c->xs[2 * k + 1];
            x.sc = c->xhi[k];
            cudaEvent_t *e = &c->evs[10 * k];
            x.e_edge[0][0] = e[0];
            x.e_edge[0][1] = e[1];
            x.e_edge[1][0] = e[2];
            x.e_edge[1][1] = e[3];
            x.e_comm[0] = e[4];
            x.e_comm[1] = e[5];
            x.e_fork = e[6];
            x.e_join = e[7];
            x.e_join2 = e[8];
            x.e_stag = e[9];
        }
        {
            HSVD_CUDA(cudaSetDevice(sh[0].dev));
            int cst = 0;
            DevCtx *c = dev_ctx(sh[0].dev, &cst);
            if (!c) return cst;
            HSVD_CUDA_OK(c->host_reserve(host_len));
            host = c->host;
        }
        HSVD_CUDA_OK(sync_all());
        // ---- precompute + sort on every shard from the full factor
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            HSVD_CUDA(cudaMemcpyAsync(x.w.signs, signs_host, (size_t)r, cudaMemcpyHostToDevice, x.s));
            HSVD_CUDA_OK(launch_init_packages(x.w.signs, r, x.w.rho, x.w.js, x.s));
            HSVD_CUDA(cudaMemsetAsync(x.w.first_zero, 0xff, sizeof(unsigned long long), x.s));
            HSVD_CUDA_OK(launch_block_norms(x.G, ldg, n, x.w.rho, r, x.w.d, x.w.first_zero, x.s));
            launches += 2;
            if (cfg->sort) {
                HSVD_CUDA_OK(hsvd_sort_diagonal(x.w.d, x.w.rho, x.w.js, r, p, x.w.sortws, x.s));
                launches += 2;
            }
        }
        Shard &x0 = sh[0];
        HSVD_CUDA(cudaSetDevice(x0.dev));
        HSVD_CUDA(cudaMemcpyAsync(host, x0.w.first_zero, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                  x0.s));
        HSVD_CUDA(cudaMemcpyAsync(host + rho_off, x0.w.rho, r * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, x0.s));
        HSVD_CUDA_OK(sync_all());
        if ((unsigned long long)host[0] != kNoError) {
            res->err[0] = host[0];
            res->err[1] = res->err[2] = -1;
            set_error("column " + std::to_string(host[0]) + " has zero norm");
            return HSVD_RANK_DEFICIENT;
        }
        std::vector<int64_t> rho(host + rho_off, host + rho_off + r);
        // ---- initial placement: gather the shard's columns, V = I columns
        for (auto &x : sh) {
            HSVD_CUDA(cudaSetDevice(x.dev));
            const auto blk = pl.blocks_of(x.g);
            std::vector<int64_t> src(pl.areas(x.g) * b, -1);
            for (size_t a = 0; a < blk.size(); ++a)
                if (blk[a] >= 0)
                    for (int c = 0; c < b; ++c) src[a * b + c] = rho[blk[a] * b + c];
            HSVD_CUDA_OK(upload(x, x.w.idx_a, src));
            k_gather_cols<<<dim3(colgrid(n), (unsigned)src.size()), 256, 0, x.s>>>(
                x.w.Gs, n, x.G, ldg, x.w.idx_a, n);
            HSVD_LAUNCH_CHECK("k_gather_cols");
            ++launches;
            if (withV) {
                k_unit_cols<<<dim3(colgrid(r), (unsigned)src.size()), 256, 0, x.s>>>(x.w.Vs, r,
                                                                                   x.w.idx_a, r);
                HSVD_LAUNCH_CHECK("k_unit_cols");
                ++launches;
            }
            HSVD_CUDA_OK(upload(x, x.w.loc, loc_table(x.g)));
            const int64_t a0 = pl.s0[x.g], m = pl.m(x.g);
            std::vector<int64_t> st(4 * m);
            for (int64_t k = 0; k < m; ++k) {
                st[k] = pl.ip[a0 + k];
                st[m + k] = pl.jp[a0 + k];
                st[2 * m + k] = pl.iblk[a0 + k];
                st[3 * m + k] = pl.jblk[a0 + k];
            }
            HSVD_CUDA_OK(upload(x, x.w.sl.ip, std::vector<int64_t>(st.begin(), st.begin() + m)));
            HSVD_CUDA_OK(upload(x, x.w.sl.jp, std::vector<int64_t>(st.begin() + m, st.begin() + 2 * m)));
            HSVD_CUDA_OK(upload(x, x.w.sl.iblk,
                                std::vector<int64_t>(st.begin() + 2 * m, st.begin() + 3 * m)));
            HSVD_CUDA_OK(upload(x, x.w.sl.jblk, std::vector<int64_t>(st.begin() + 3 * m, st.end())));
            HSVD_CUDA(cudaMemsetAsync(x.w.sl.C, 0, (size_t)m, x.s));
            HSVD_CUDA(cudaMemsetAsync(x.w.sl.rotk, 0, sizeof(uint32_t) * m, x.s));
            HSVD_CUDA(cudaMemsetAsync(x.w.sl.skipk, 0, sizeof(uint32_t) * m, x.s));
            HSVD_CUDA(cudaMemsetAsync(x.w.sl.maxt, 0, sizeof(double) * m, x.s));
            HSVD_CUDA(cudaMemsetAsync(x.w.sl.err, 0xff, sizeof(unsigned long long), x.s));
        }
        HSVD_CUDA_OK(sync_all());

        // profile mode: CUDA events around shard 0's kernels of sweep 0
        KernelTimer T, Toff;
        std::vector<Move> mv;
        int64_t sweeps_used = 0, total_rot = 0, total_skip = 0;
        int stop = 2;
        const double t_loop0 = wall_ms();
        res->setup_ms = t_loop0;
        for (int64_t sweep = 0; sweep < cfg->max_sweeps; ++sweep) {
            HSVD_CUDA(cudaSetDevice(x0.dev));
            HSVD_CUDA(cudaEventRecord(x0.t0, x0.s));
            T.on = cfg->profile && sweep == 0;
            if (split && !T.on) {
                HSVD_CUDA_OK(sweep_split(mv));
            } else {
                for (int64_t step = 0; step < nb; ++step) {
                    const int full = cfg->inner_full || step == 0;
                    for (auto &x : sh) {
                        HSVD_CUDA(cudaSetDevice(x.dev));
                        HSVD_CUDA_OK(K::step(x.w.Gs, n, (int)n, withV ? x.w.Vs : nullptr, r,
                                             (int)r, x.w.sl, full, passes.now(), x.s,
                                             &x == &sh[0] ? T : Toff, (int)step, false));
                        launches += 3;
                    }
                    HSVD_CUDA_OK(pl.advance(mv));
                    HSVD_CUDA_OK(exchange(mv));
                }
            }
            // ---- sweep end: norms, convergence word, sort, redistribution
            HSVD_CUDA_OK(gather_norms());
            HSVD_CUDA_OK(reduce_stats());
            for (auto &x : sh) {
                HSVD_CUDA(cudaSetDevice(x.dev));
                if (cfg->sort) {
                    HSVD_CUDA_OK(hsvd_sort_diagonal(x.w.d, x.w.rho, x.w.js, r, p, x.w.sortws, x.s));
                    launches += 2;
                }
            }
            HSVD_CUDA(cudaSetDevice(x0.dev));
            HSVD_CUDA(cudaMemcpyAsync(host + rho_off, x0.w.rho, r * sizeof(int64_t),
                                      cudaMemcpyDeviceToHost, x0.s));
            HSVD_CUDA(cudaEventRecord(x0.t1, x0.s));
            HSVD_CUDA_OK(sync_all());
            if (T.on) T.collect(res);
            float ms = 0.f;
            HSVD_CUDA(cudaEventElapsedTime(&ms, x0.t0, x0.t1));
            int64_t o[5];
            combine_stats(o);
            if ((unsigned long long)o[4] != kNoError) {
                unpack_err((unsigned long long)o[4], res->err);
                set_error("definiteness lost at block " + std::to_string(res->err[0]) +
                          ", pivot pair (" + std::to_string(res->err[1]) + ", " +
                          std::to_string(res->err[2]) + ")");
                return HSVD_DEFINITENESS_LOST;
            }
            std::vector<int64_t> rho_new(host + rho_off, host + rho_off + r);
            ShardPlan old_pl = pl;
            pl.place();
            HSVD_CUDA_OK(redistribute(old_pl, rho, rho_new));
            rho.swap(rho_new);
            const int code = (int)o[0];
            double max_t;
            memcpy(&max_t, &o[3], sizeof(double));
            sweeps_used = sweep + 1;
            total_rot += o[1];
            total_skip += o[2];
            passes.after_sweep(o[1], o[2]);
            if (tele) {
                tele[sweep].sweep = sweep;
                tele[sweep].rotations = o[1];
                tele[sweep].skips = o[2];
                tele[sweep].max_t = max_t;
                tele[sweep].gpu_ms = ms;
            }
            if (code == 0) { stop = 0; break; }
            if (code == 1) { stop = 1; break; }
        }
        res->sweeps_ms = wall_ms() - t_loop0;
        // ---- extraction on the canonical placement
        for (size_t i = 0; i < sh.size(); ++i) {
            Shard &x = sh[i];
            HSVD_CUDA(cudaSetDevice(x.dev));
            const auto blk = pl.blocks_of(x.g);
            const int64_t nc = 2 * pl.m(x.g) * b;
            std::vector<int64_t> qpos(nc);
            for (int64_t k = 0; k < nc; ++k) {
                qpos[k] = blk[k / b] * b + k % b;
                cols_host[i][k] = rho[qpos[k]];
            }
            HSVD_CUDA_OK(upload(x, x.w.idx_a, qpos));
            k_shard_extract<<<nblk(nc, 256), 256, 0, x.s>>>(x.w.d, x.w.js, x.w.idx_a, nc,
                                                             sigma_out[i], lam_out[i]);
            HSVD_LAUNCH_CHECK("k_shard_extract");
            k_shard_scale<<<dim3(colgrid(n), (unsigned)nc), 256, 0, x.s>>>(U_out[i], n, x.w.Gs, n, n,
                                                                          sigma_out[i]);
            HSVD_LAUNCH_CHECK("k_shard_scale");
            launches += 2;
            if (withV && V_out[i])
                HSVD_CUDA(cudaMemcpyAsync(V_out[i], x.w.Vs, sizeof(double) * nc * r,
                                          cudaMemcpyDeviceToDevice, x.s));
        }
        HSVD_CUDA_OK(sync_all());
        res->sweeps_used = sweeps_used;
        res->stop_reason = stop;
        res->rotations = total_rot;
        res->skips = total_skip;
        res->launches = launches;
        return HSVD_OK;
    }
};

static int64_t shard_ws_size(int64_t n, int64_t r, int nshards, int g, const hsvd_config *cfg)
{
    ShardPlan pl;
    if (cfg->block_cols != 16 && cfg->block_cols != 32) return -1;
    if (pl.init(r / cfg->block_cols, nshards)) return -1;
    Carve2 c{nullptr, 0};
    return carve_shard(c, pl, g, n, r, cfg->block_cols, cfg->accumulate_v != 0, nullptr);
}

template <int B2>
static int sharded_drive_t(Comm *comm, int nshards, int nlocal, const int *shard_ids,
                           const int *devices, const double *const *G, int64_t n, int64_t r,
                           int64_t ldg, const int8_t *signs_host, int64_t p,
                           const hsvd_config *cfg, double *const *U_out, double *const *V_out,
                           int64_t *const *cols_host, double *const *sigma_out,
                           double *const *lam_out, void *const *ws, const int64_t *ws_bytes,
                           hsvd_result *res, hsvd_telemetry *tele)
{
    ShardedDriver<B2> D;
    D.comm = comm;
    D.n = n;
    D.r = r;
    D.ldg = ldg;
    D.p = p;
    D.cfg = cfg;
    D.withV = cfg->accumulate_v != 0;
    D.sh.resize(nlocal);
    ShardPlan pl;
    int st = pl.init(r / (B2 / 2), nshards);
    if (st) return st;
    for (int i = 0; i < nlocal; ++i) {
        Shard &x = D.sh[i];
        x.g = shard_ids[i];
        x.dev = devices[i];
        x.G = G[i];
        if (x.g < 0 || x.g >= nshards) {
            set_error("sharded: bad shard id");
            return HSVD_ERR_ARG;
        }
        Carve2 c{(char *)ws[i], 0};
        if (carve_shard(c, pl, x.g, n, r, B2 / 2, D.withV, &x.w) > ws_bytes[i]) {
            set_error("sharded: workspace too small");
            return HSVD_ERR_ARG;
        }
        const char *tma_env = getenv("HSVD_GRAM_TMA");
        if (HSVD_GRAM_TMA && !(tma_env && tma_env[0] == '0') &&
            make_gram_tensor_map(&x.gmap, x.w.Gs, n, n, pl.areas(x.g) * (B2 / 2)) == 0)
            x.w.sl.gmap = x.w.half[0].gmap = x.w.half[1].gmap = &x.gmap;
    }
    return D.run(signs_host, U_out, V_out, cols_host, sigma_out, lam_out, res, tele);
}

}  // namespace hsvd

using namespace hsvd;

extern "C" {

int hsvd_comm_unique_id(uint8_t *id_out)
{
    NcclApi *N = nccl();
    if (!N) return HSVD_ERR_UNSUPPORTED;
    ncclUniqueId id;
    HSVD_NCCL(N->GetUniqueId(&id));
    memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return HSVD_OK;
}

int hsvd_comm_init(const uint8_t *id_in, int nranks, int rank, void **comm_out)
{
    NcclApi *N = nccl();
    if (!N) return HSVD_ERR_UNSUPPORTED;
    ncclUniqueId id;
    memcpy(id.internal, id_in, NCCL_UNIQUE_ID_BYTES);
    Comm *c = new Comm();
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t e = N->CommInitRank(&c->comm, nranks, id, rank);
    if (e != ncclSuccess) {
        set_error(std::string("ncclCommInitRank: ") + N->GetErrorString(e));
        delete c;
        return HSVD_ERR_CUDA;
    }
    *comm_out = c;
    return HSVD_OK;
}

int hsvd_comm_destroy(void *comm)
{
    if (!comm) return HSVD_OK;
    Comm *c = (Comm *)comm;
    NcclApi *N = nccl();
    if (N) N->CommDestroy(c->comm);
    delete c;
    return HSVD_OK;
}

int64_t hsvd_shard_columns(int64_t r, int32_t block_cols, int32_t nshards, int32_t shard)
{
    ShardPlan pl;
    if (block_cols < 1 || r % block_cols || pl.init(r / block_cols, nshards)) return -1;
    if (shard < 0 || shard >= nshards) return -1;
    return 2 * pl.m(shard) * block_cols;
}

int64_t hsvd_sharded_workspace_size(int64_t n, int64_t r, int32_t nshards, int32_t shard,
                                    const hsvd_config *cfg)
{
    return shard_ws_size(n, r, nshards, shard, cfg);
}

int hsvd_drive_sharded(void *comm, int32_t nshards, int32_t nlocal, const int32_t *shard_ids,
                       const int32_t *devices, const double *const *G, int64_t n, int64_t r,
                       int64_t ldg, const int8_t *signs_host, int64_t p, const hsvd_config *cfg,
                       double *const *U_out, double *const *V_out, int64_t *const *cols_host,
                       double *const *sigma_out, double *const *lam_out, void *const *ws,
                       const int64_t *ws_bytes, hsvd_result *res_host,
                       hsvd_telemetry *tele_host)
{
    const double t_entry = wall_ms();
    memset(res_host, 0, sizeof(*res_host));
    res_host->err[0] = res_host->err[1] = res_host->err[2] = -1;
    const int b = cfg->block_cols;
    if (cfg->mode != HSVD_MODE_BLOCK) {
        set_error("sharded solve runs block mode only");
        return res_host->status = HSVD_ERR_UNSUPPORTED;
    }
    if (r % 2 || n < r) {
        set_error(r % 2 ? "r must be even; use border() first" : "G must have n >= r");
        return res_host->status = HSVD_SHAPE_ERROR;
    }
    if ((b != 16 && b != 32) || r % (2 * b) || n % 2 || ldg % 2) {
        set_error("sharded: block_cols 16 or 32, r a multiple of 2*block_cols, even n and ldg");
        return res_host->status = HSVD_ERR_UNSUPPORTED;
    }
    if (comm && (nlocal != 1 || ((Comm *)comm)->nranks != nshards ||
                 shard_ids[0] != ((Comm *)comm)->rank)) {
        set_error("sharded: with a communicator, one local shard = this rank");
        return res_host->status = HSVD_ERR_ARG;
    }
    if (!comm && nlocal != nshards) {
        set_error("sharded: without a communicator every shard is local");
        return res_host->status = HSVD_ERR_ARG;
    }
    int st;
    if (b == 16)
        st = sharded_drive_t<32>((Comm *)comm, nshards, nlocal, shard_ids, devices, G, n, r, ldg,
                                 signs_host, p, cfg, U_out, V_out, cols_host, sigma_out, lam_out,
                                 ws, ws_bytes, res_host, tele_host);
    else
        st = sharded_drive_t<64>((Comm *)comm, nshards, nlocal, shard_ids, devices, G, n, r, ldg,
                                 signs_host, p, cfg, U_out, V_out, cols_host, sigma_out, lam_out,
                                 ws, ws_bytes, res_host, tele_host);
    res_host->status = st;
    if (st == HSVD_OK) {
        const double t_loop0 = res_host->setup_ms;
        res_host->setup_ms = t_loop0 - t_entry;
        res_host->finish_ms = wall_ms() - t_loop0 - res_host->sweeps_ms;
    }
    return st;
}

// ---- the plan alone (host only; for CPU tests of the exchange protocol) ----
void *hsvd_plan_create(int64_t nblocks, int32_t nshards)
{
    ShardPlan *pl = new ShardPlan();
    if (pl->init(nblocks, nshards)) {
        delete pl;
        return nullptr;
    }
    return pl;
}

void hsvd_plan_destroy(void *plan) { delete (ShardPlan *)plan; }

int64_t hsvd_plan_advance(void *plan, int64_t *moves, int64_t max_moves)
{
    ShardPlan *pl = (ShardPlan *)plan;
    std::vector<Move> mv;
    if (pl->advance(mv)) return -1;
    if ((int64_t)mv.size() > max_moves) return -1;
    for (size_t i = 0; i < mv.size(); ++i) {
        moves[5 * i + 0] = mv[i].P;
        moves[5 * i + 1] = mv[i].from;
        moves[5 * i + 2] = mv[i].from_area;
        moves[5 * i + 3] = mv[i].to;
        moves[5 * i + 4] = mv[i].to_area;
    }
    return (int64_t)mv.size();
}

int hsvd_plan_state(void *plan, int64_t *iblk, int64_t *jblk, int32_t *owner, int32_t *area,
                    int64_t *slot_begin)
{
    ShardPlan *pl = (ShardPlan *)plan;
    for (int64_t k = 0; k < pl->S; ++k) {
        iblk[k] = pl->iblk[k];
        jblk[k] = pl->jblk[k];
    }
    for (int64_t P = 0; P < pl->nb; ++P) {
        owner[P] = pl->owner[P];
        area[P] = pl->area[P];
    }
    for (int g = 0; g <= pl->N; ++g) slot_begin[g] = pl->s0[g];
    return HSVD_OK;
}

// Redistribution lists of shard g after a sort: columns g sends to each
// peer (send, grouped by peer in peer order, counts in send_count[N]) and
// the local columns it receives from each peer (recv / recv_count).  The
// plan is re-placed canonically for the current pairs.
int hsvd_plan_redistribute(void *plan, int32_t b, const int64_t *rho_old, const int64_t *rho_new,
                           int64_t r, int32_t g, int64_t *send, int64_t *send_count,
                           int64_t *recv, int64_t *recv_count)
{
    ShardPlan *pl = (ShardPlan *)plan;
    ShardPlan old_pl = *pl;
    ShardPlan new_pl = *pl;
    new_pl.place();
    Redist R;
    plan_redistribute(old_pl, new_pl, b, std::vector<int64_t>(rho_old, rho_old + r),
                      std::vector<int64_t>(rho_new, rho_new + r), R);
    int64_t so = 0, ro = 0;
    for (int h = 0; h < pl->N; ++h) {
        send_count[h] = (int64_t)R.send[g][h].size();
        for (auto v : R.send[g][h]) send[so++] = v;
        recv_count[h] = (int64_t)R.recv[g][h].size();
        for (auto v : R.recv[g][h]) recv[ro++] = v;
    }
    return HSVD_OK;
}

void hsvd_plan_place(void *plan) { ((ShardPlan *)plan)->place(); }

}  // extern "C"
