// hsvd_driver.cu -- native sweep driver and C-ABI whole-solver entry points.
//
// hsvd_drive restates solver.drive (/root/reference/pkg/src/hjsvd/
// solver.py:179-269) with every array resident in HBM: precompute, sort,
// quasi-sweeps of r fused step kernels (captured once as a CUDA graph and
// replayed per sweep), the on-device convergence/statistics reduction and the
// sort, then one 40-byte device->host read per sweep to take the stop
// decision -- the only host synchronisation inside the loop, as the paper's
// Check_Convergence.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <string>
#include <vector>

#include "hsvd_internal.cuh"

namespace hsvd {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char *what)
{
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return HSVD_ERR_CUDA;
}

int DevCtx::host_reserve(int64_t len)
{
    if (len <= host_len) return HSVD_OK;
    if (host) cudaFreeHost(host);
    host = nullptr;
    host_len = 0;
    HSVD_CUDA(cudaHostAlloc((void **)&host, len * sizeof(int64_t), cudaHostAllocDefault));
    host_len = len;
    return HSVD_OK;
}

int DevCtx::extra(size_t k)
{
    while (xs.size() < k) {
        cudaStream_t st;
        cudaEvent_t a, b, c;
        HSVD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        HSVD_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        HSVD_CUDA(cudaEventCreate(&b));
        HSVD_CUDA(cudaEventCreate(&c));
        xs.push_back(st);
        xev.push_back(a);
        xt0.push_back(b);
        xt1.push_back(c);
    }
    return HSVD_OK;
}

int DevCtx::extra_hi(size_t k)
{
    int lo = 0, hi = 0;
    HSVD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    while (xhi.size() < k) {
        cudaStream_t st;
        HSVD_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
        xhi.push_back(st);
    }
    return HSVD_OK;
}

int DevCtx::events(size_t k)
{
    while (evs.size() < k) {
        cudaEvent_t e;
        HSVD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs.push_back(e);
    }
    return HSVD_OK;
}

DevCtx::~DevCtx()
{
    // thread exit: the context's device may not be current; best effort
    int cur = -1;
    cudaGetDevice(&cur);
    if (dev >= 0) cudaSetDevice(dev);
    for (auto e : evs) cudaEventDestroy(e);
    for (auto st : xhi) cudaStreamDestroy(st);
    for (size_t i = 0; i < xs.size(); ++i) {
        cudaStreamDestroy(xs[i]);
        cudaEventDestroy(xev[i]);
        cudaEventDestroy(xt0[i]);
        cudaEventDestroy(xt1[i]);
    }
    if (host) cudaFreeHost(host);
    if (ev) cudaEventDestroy(ev);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
    if (s) cudaStreamDestroy(s);
    if (cur >= 0) cudaSetDevice(cur);
}

DevCtx *dev_ctx(int dev, int *status)
{
    static thread_local std::vector<DevCtx *> ctxs;
    *status = HSVD_OK;
    if (dev < 0) {
        *status = HSVD_ERR_ARG;
        return nullptr;
    }
    if ((int)ctxs.size() <= dev) ctxs.resize(dev + 1, nullptr);
    if (ctxs[dev]) return ctxs[dev];
    struct Owner {
        std::vector<DevCtx *> *v;
        ~Owner()
        {
            for (auto c : *v) delete c;
        }
    };
    static thread_local Owner owner{&ctxs};
    (void)owner;
    DevCtx *c = new DevCtx();
    c->dev = dev;
    cudaError_t e = cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreate(&c->t0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->t1);
    if (e == cudaSuccess) e = cudaHostAlloc((void **)&c->host, 64 * sizeof(int64_t),
                                            cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaMalloc((void **)&c->dword, sizeof(unsigned long long));
    if (e != cudaSuccess) {
        *status = cuda_fail(e, "dev_ctx");
        delete c;
        return nullptr;
    }
    c->host_len = 64;
    ctxs[dev] = c;
    return c;
}

int launch_identity(double *V, int64_t r, int64_t ldv, cudaStream_t s);
int launch_init_packages(const int8_t *signs, int64_t r, int64_t *rho,
                         int64_t *jsign, cudaStream_t s);
int launch_reduce_sweep(uint8_t *C, int64_t m, uint32_t *rotk, uint32_t *skipk,
                        double *maxt, int64_t nslots, int64_t *out,
                        const unsigned long long *err, int reset, cudaStream_t s);
int block_drive(double *G, int64_t n, int64_t r, int64_t ldg, double *V,
                int64_t ldv, const int8_t *signs_host, int64_t p,
                const hsvd_config *cfg, double *sigma, double *lam,
                void *ws, int64_t ws_bytes, hsvd_result *res,
                hsvd_telemetry *tele, DevCtx &ctx);
int64_t block_workspace_size(int64_t n, int64_t r, const hsvd_config *cfg);

// Bump allocator over the caller's workspace.
struct Carve {
    char *base;
    int64_t off, cap;
    template <typename T>
    T *take(int64_t count)
    {
        off = (off + 255) & ~(int64_t)255;
        T *p = (T *)(base + off);
        off += count * (int64_t)sizeof(T);
        return p;
    }
};

struct PointwiseWs {
    double *d;
    int64_t *rho, *js, *ip, *jp, *iblk, *jblk;
    uint8_t *C;
    uint32_t *rotk, *skipk;
    double *maxt;
    unsigned long long *err;
    void *sortws;
    int64_t *out;
    unsigned long long *first_zero;
    int8_t *signs;
    int64_t ncodes, nslots;
};

static int64_t carve_pointwise(Carve &c, int64_t r, const hsvd_config *cfg,
                               PointwiseWs *w)
{
    const bool rc = cfg->schedule == HSVD_SCHEDULE_ROW_CYCLIC;
    const int64_t half = r / 2;
    const int64_t ncodes = rc ? r * (r - 1) / 2 : half;
    const int64_t nslots = rc ? 1 : half;
    PointwiseWs t;
    t.d = c.take<double>(r);
    t.rho = c.take<int64_t>(r);
    t.js = c.take<int64_t>(r);
    t.ip = c.take<int64_t>(half);
    t.jp = c.take<int64_t>(half);
    t.iblk = c.take<int64_t>(half);
    t.jblk = c.take<int64_t>(half);
    t.C = c.take<uint8_t>(ncodes);
    t.rotk = c.take<uint32_t>(nslots);
    t.skipk = c.take<uint32_t>(nslots);
    t.maxt = c.take<double>(nslots);
    t.err = c.take<unsigned long long>(1);
    t.sortws = c.take<char>(24 * r);
    t.out = c.take<int64_t>(8);
    t.first_zero = c.take<unsigned long long>(1);
    t.signs = c.take<int8_t>(r);
    t.ncodes = ncodes;
    t.nslots = nslots;
    if (w) *w = t;
    return c.off + 256;
}

// RAII for the per-call graph.
struct DriveRes {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    ~DriveRes()
    {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
    }
};

// One quasi-sweep's device work: r steps (or the row-cyclic walk), the
// convergence reduction, the sort, and the summary copy to pinned memory.
static int enqueue_sweep(double *G, int64_t n, int64_t r, int64_t ldg,
                         double *V, int64_t ldv, int64_t p,
                         const hsvd_config *cfg, const PointwiseWs &w,
                         int64_t *host_out, cudaStream_t s, KernelTimer &T)
{
    int st;
    if (cfg->schedule == HSVD_SCHEDULE_ROW_CYCLIC) {
        T.begin(0, s);
        st = launch_rowcyclic_sweep(G, n, ldg, V, r, ldv, w.d, w.rho, w.js, r,
                                    w.C, cfg->eps, cfg->teps, cfg->use_skip,
                                    cfg->chunk, w.rotk, w.skipk, w.maxt, w.err, s);
        T.end(s);
        if (st) return st;
    } else {
        for (int64_t step = 0; step < r; ++step) {
            T.begin(0, s);
            st = launch_pointwise_step(G, n, ldg, V, r, ldv, w.d, w.rho, w.js,
                                       w.ip, w.jp, w.iblk, w.jblk, r, w.C, 0,
                                       r / 2, cfg->eps, cfg->teps,
                                       cfg->use_skip, cfg->chunk, 1, w.rotk,
                                       w.skipk, w.maxt, w.err, s);
            T.end(s);
            if (st) return st;
        }
    }
    T.begin(3, s);
    st = launch_reduce_sweep(w.C, w.ncodes, w.rotk, w.skipk, w.maxt, w.nslots,
                             w.out, w.err, 1, s);
    if (st) return st;
    if (cfg->sort) {
        st = hsvd_sort_diagonal(w.d, w.rho, w.js, r, p, w.sortws, s);
        if (st) return st;
    }
    T.end(s);
    HSVD_CUDA(cudaMemcpyAsync(host_out, w.out, 5 * sizeof(int64_t),
                              cudaMemcpyDeviceToHost, s));
    return HSVD_OK;
}

static int pointwise_drive(double *G, int64_t n, int64_t r, int64_t ldg,
                           double *V, int64_t ldv, const int8_t *signs_host,
                           int64_t p, const hsvd_config *cfg, double *sigma,
                           double *lam, void *ws, int64_t ws_bytes,
                           hsvd_result *res, hsvd_telemetry *tele,
                           DevCtx &ctx, DriveRes &R)
{
    cudaStream_t s = ctx.s;
    Carve c{(char *)ws, 0, ws_bytes};
    PointwiseWs w;
    if (carve_pointwise(c, r, cfg, &w) > ws_bytes) {
        set_error("workspace too small");
        return HSVD_ERR_ARG;
    }
    // the row-cyclic walk stages both columns in shared memory (the
    // modulus steps stream them and have no size limit)
    size_t smem;
    int st = cfg->schedule == HSVD_SCHEDULE_ROW_CYCLIC ? pointwise_smem_bytes(n, cfg->chunk, &smem)
                                                       : (cfg->chunk < 1 ? HSVD_ERR_ARG : HSVD_OK);
    if (st) {
        if (st == HSVD_ERR_ARG) set_error("chunk must be >= 1");
        return st;
    }
    int64_t *host = ctx.host;

    if (V) {
        st = launch_identity(V, r, ldv, s);
        if (st) return st;
    }
    // precompute (solver.py:80-94)
    st = hsvd_precompute(G, n, r, ldg, cfg->chunk, w.d, (int64_t *)w.first_zero, s);
    if (st) return st;
    HSVD_CUDA(cudaMemcpyAsync(w.signs, signs_host, (size_t)r, cudaMemcpyHostToDevice, s));
    st = launch_init_packages(w.signs, r, w.rho, w.js, s);
    if (st) return st;
    HSVD_CUDA(cudaMemcpyAsync(host, w.first_zero, sizeof(int64_t),
                              cudaMemcpyDeviceToHost, s));
    HSVD_CUDA(cudaStreamSynchronize(s));
    if ((unsigned long long)host[0] != kNoError) {
        res->status = HSVD_RANK_DEFICIENT;
        res->err[0] = host[0];
        res->err[1] = res->err[2] = -1;
        set_error("column " + std::to_string(host[0]) + " has zero norm");
        return HSVD_RANK_DEFICIENT;
    }
    if (cfg->sort) {
        st = hsvd_sort_diagonal(w.d, w.rho, w.js, r, p, w.sortws, s);
        if (st) return st;
    }
    if (cfg->schedule == HSVD_SCHEDULE_MODULUS) {
        st = hsvd_stepper_init(w.ip, w.jp, w.iblk, w.jblk, r, s);
        if (st) return st;
    }
    HSVD_CUDA(cudaMemsetAsync(w.C, 0, (size_t)w.ncodes, s));
    HSVD_CUDA(cudaMemsetAsync(w.rotk, 0, sizeof(uint32_t) * w.nslots, s));
    HSVD_CUDA(cudaMemsetAsync(w.skipk, 0, sizeof(uint32_t) * w.nslots, s));
    HSVD_CUDA(cudaMemsetAsync(w.maxt, 0, sizeof(double) * w.nslots, s));
    HSVD_CUDA(cudaMemsetAsync(w.err, 0xff, sizeof(unsigned long long), s));

    KernelTimer T;
    if (cfg->use_graph && !cfg->profile) {
        HSVD_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        st = enqueue_sweep(G, n, r, ldg, V, ldv, p, cfg, w, host, s, T);
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(s, &g);
        if (st) {
            if (g) cudaGraphDestroy(g);
            return st;
        }
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
        R.graph = g;
        HSVD_CUDA(cudaGraphInstantiate(&R.exec, g, 0));
    }

    const bool rc = cfg->schedule == HSVD_SCHEDULE_ROW_CYCLIC;
    const int64_t per_sweep = (rc ? 1 : r) + 1 + (cfg->sort ? 2 : 0);
    int64_t launches = 1 + (V ? 1 : 0) + 1 + (cfg->sort ? 2 : 0) + (rc ? 0 : 1) + 2;
    int64_t sweeps_used = 0, total_rot = 0, total_skip = 0;
    int stop = 2;
    const double t_loop0 = wall_ms();
    res->setup_ms = t_loop0;  // absolute for now; hsvd_drive makes it relative
    for (int64_t sweep = 0; sweep < cfg->max_sweeps; ++sweep) {
        HSVD_CUDA(cudaEventRecord(ctx.t0, s));
        launches += per_sweep;
        if (R.exec) {
            HSVD_CUDA(cudaGraphLaunch(R.exec, s));
        } else {
            T.on = cfg->profile && sweep == 0;
            st = enqueue_sweep(G, n, r, ldg, V, ldv, p, cfg, w, host, s, T);
            if (st) return st;
        }
        HSVD_CUDA(cudaEventRecord(ctx.t1, s));
        HSVD_CUDA(cudaStreamSynchronize(s));
        if (T.on) T.collect(res);
        float sweep_ms = 0.f;
        HSVD_CUDA(cudaEventElapsedTime(&sweep_ms, ctx.t0, ctx.t1));
        if ((unsigned long long)host[4] != kNoError) {
            unpack_err((unsigned long long)host[4], res->err);
            res->status = HSVD_DEFINITENESS_LOST;
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
        if (tele) {
            tele[sweep].sweep = sweep;
            tele[sweep].rotations = host[1];
            tele[sweep].skips = host[2];
            tele[sweep].max_t = max_t;
            tele[sweep].gpu_ms = sweep_ms;
        }
        if (code == 0) { stop = 0; break; }
        if (code == 1) { stop = 1; break; }
    }
    res->sweeps_ms = wall_ms() - t_loop0;
    st = hsvd_extract(G, n, ldg, w.d, w.rho, w.js, r, sigma, lam, s);
    if (st) return st;
    res->sweeps_used = sweeps_used;
    res->stop_reason = stop;
    res->rotations = total_rot;
    res->skips = total_skip;
    res->launches = launches;
    res->status = HSVD_OK;
    return HSVD_OK;
}

}  // namespace hsvd

using namespace hsvd;

extern "C" {

const char *hsvd_last_error(void) { return g_last_error.c_str(); }

int hsvd_version(void) { return 100; }

void hsvd_abi_sizes(int64_t *out)
{
    out[0] = (int64_t)sizeof(hsvd_config);
    out[1] = (int64_t)sizeof(hsvd_result);
    out[2] = (int64_t)sizeof(hsvd_telemetry);
}

void hsvd_default_config(hsvd_config *cfg)
{
    memset(cfg, 0, sizeof(*cfg));
    cfg->max_sweeps = 30;
    cfg->eps = 0x1p-52;
    cfg->teps = 0x1p-27;
    cfg->accumulate_v = 1;
    cfg->use_skip = 1;
    cfg->chunk = 32;
    cfg->schedule = HSVD_SCHEDULE_MODULUS;
    cfg->sort = 1;
    cfg->mode = HSVD_MODE_POINTWISE;
    cfg->block_cols = 32;
    cfg->inner_full = 1;
    cfg->use_graph = 1;
    cfg->block_rotation = HSVD_ROTATION_FAST;
    cfg->inner_passes = 0;  /* auto: 2 in the dense sweeps, 1 in the late ones */
    cfg->block_streams = 2;
}

}  // extern "C"

namespace hsvd {
// smallest column index holding a NaN or an infinity (block.y = column)
__global__ void k_first_nonfinite(const double *__restrict__ G, int64_t ldg, int64_t n,
                                  unsigned long long *first)
{
    const int64_t c = blockIdx.y;
    const double *g = G + c * ldg;
    bool bad = false;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(g[e]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMin(first, (unsigned long long)c);
}
}  // namespace hsvd

extern "C" {

int64_t hsvd_drive_workspace_size(int64_t n, int64_t r, const hsvd_config *cfg)
{
    if (cfg->mode == HSVD_MODE_BLOCK) return block_workspace_size(n, r, cfg);
    Carve c{nullptr, 0, 0};
    return carve_pointwise(c, r, cfg, nullptr);
}

int hsvd_drive(double *G, int64_t n, int64_t r, int64_t ldg, double *Vinv_t,
               int64_t ldv, const int8_t *signs_host, int64_t p,
               const hsvd_config *cfg, double *sigma, double *lam,
               void *workspace, int64_t workspace_bytes,
               hsvd_result *res_host, hsvd_telemetry *tele_host, void *stream)
{
    const double t_entry = wall_ms();
    memset(res_host, 0, sizeof(*res_host));
    res_host->err[0] = res_host->err[1] = res_host->err[2] = -1;
    if (r % 2 != 0 || r < 2) {
        set_error("r must be even; use border() first");
        return res_host->status = HSVD_SHAPE_ERROR;
    }
    if (n < r) {
        set_error("G must have n >= r");
        return res_host->status = HSVD_SHAPE_ERROR;
    }
    if (ldg < n || (cfg->accumulate_v && (!Vinv_t || ldv < r))) {
        set_error("bad leading dimension or missing V buffer");
        return res_host->status = HSVD_ERR_ARG;
    }
    if (r >= (1ll << 21)) {
        set_error("r too large for the packed error word");
        return res_host->status = HSVD_ERR_UNSUPPORTED;
    }
    DriveRes R;
    cudaStream_t caller = (cudaStream_t)stream;
    int dev = 0, cst = 0;
    HSVD_CUDA(cudaGetDevice(&dev));
    DevCtx *ctx = dev_ctx(dev, &cst);
    if (!ctx) return res_host->status = cst;
    HSVD_CUDA(cudaEventRecord(ctx->ev, caller));
    HSVD_CUDA(cudaStreamWaitEvent(ctx->s, ctx->ev, 0));
    double *V = cfg->accumulate_v ? Vinv_t : nullptr;
    // as_factor's finiteness check (linalg.py:58-65), on the device: one
    // read of G before anything else touches it
    {
        HSVD_CUDA(cudaMemsetAsync(ctx->dword, 0xff, sizeof(unsigned long long), ctx->s));
        const unsigned gx = (unsigned)((n + 255) / 256 < 8 ? (n + 255) / 256 : 8);
        k_first_nonfinite<<<dim3(gx, (unsigned)r), 256, 0, ctx->s>>>(G, ldg, n, ctx->dword);
        HSVD_LAUNCH_CHECK("k_first_nonfinite");
        HSVD_CUDA(cudaMemcpyAsync(ctx->host, ctx->dword, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                  ctx->s));
        HSVD_CUDA(cudaStreamSynchronize(ctx->s));
        if ((unsigned long long)ctx->host[0] != kNoError) {
            set_error("G contains non-finite entries (column " + std::to_string(ctx->host[0]) +
                      ")");
            return res_host->status = HSVD_ERR_ARG;
        }
    }
    int st;
    if (cfg->mode == HSVD_MODE_BLOCK)
        st = block_drive(G, n, r, ldg, V, ldv, signs_host, p, cfg, sigma, lam,
                         workspace, workspace_bytes, res_host, tele_host, *ctx);
    else
        st = pointwise_drive(G, n, r, ldg, V, ldv, signs_host, p, cfg, sigma,
                             lam, workspace, workspace_bytes, res_host,
                             tele_host, *ctx, R);
    res_host->status = st;
    // hand the results back to the caller's stream
    cudaError_t e1 = cudaEventRecord(ctx->ev, ctx->s);
    cudaError_t e2 = cudaStreamWaitEvent(caller, ctx->ev, 0);
    if (st == HSVD_OK && (e1 != cudaSuccess || e2 != cudaSuccess))
        return cuda_fail(e1 != cudaSuccess ? e1 : e2, "stream join");
    cudaStreamSynchronize(ctx->s);
    if (st == HSVD_OK) {
        const double t_loop0 = res_host->setup_ms;
        res_host->setup_ms = t_loop0 - t_entry;
        res_host->finish_ms = wall_ms() - t_loop0 - res_host->sweeps_ms;
    }
    return st;
}

int hsvd_drive_host(const double *G_host, int64_t n, int64_t r,
                    const int8_t *signs_host, int64_t p,
                    const hsvd_config *cfg, double *U_host,
                    double *Vinv_t_host, double *sigma_host, double *lam_host,
                    hsvd_result *res_host, hsvd_telemetry *tele_host)
{
    if (r % 2 != 0 || r < 2 || n < r) {
        memset(res_host, 0, sizeof(*res_host));
        set_error(r % 2 ? "r must be even; use border() first" : "G must have n >= r");
        return res_host->status = HSVD_SHAPE_ERROR;
    }
    const int64_t wsb = hsvd_drive_workspace_size(n, r, cfg);
    double *G = nullptr, *V = nullptr, *sg = nullptr, *lm = nullptr;
    void *ws = nullptr;
    cudaStream_t s = nullptr;
    int st = HSVD_OK;
    auto cleanup = [&]() {
        if (s) cudaStreamSynchronize(s);
        cudaFree(G); cudaFree(V); cudaFree(sg); cudaFree(lm); cudaFree(ws);
        if (s) cudaStreamDestroy(s);
    };
#define HSVD_HCUDA(call)                                         \
    do {                                                         \
        cudaError_t _e = (call);                                 \
        if (_e != cudaSuccess) {                                 \
            st = cuda_fail(_e, #call);                           \
            cleanup();                                           \
            return res_host->status = st;                        \
        }                                                        \
    } while (0)
    HSVD_HCUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    HSVD_HCUDA(cudaMalloc(&G, sizeof(double) * n * r));
    if (cfg->accumulate_v) HSVD_HCUDA(cudaMalloc(&V, sizeof(double) * r * r));
    HSVD_HCUDA(cudaMalloc(&sg, sizeof(double) * r));
    HSVD_HCUDA(cudaMalloc(&lm, sizeof(double) * r));
    HSVD_HCUDA(cudaMalloc(&ws, wsb));
    HSVD_HCUDA(cudaMemcpyAsync(G, G_host, sizeof(double) * n * r, cudaMemcpyHostToDevice, s));
    st = hsvd_drive(G, n, r, n, V, r, signs_host, p, cfg, sg, lm, ws, wsb,
                    res_host, tele_host, s);
    if (st == HSVD_OK) {
        HSVD_HCUDA(cudaMemcpyAsync(U_host, G, sizeof(double) * n * r, cudaMemcpyDeviceToHost, s));
        if (cfg->accumulate_v && Vinv_t_host)
            HSVD_HCUDA(cudaMemcpyAsync(Vinv_t_host, V, sizeof(double) * r * r,
                                       cudaMemcpyDeviceToHost, s));
        HSVD_HCUDA(cudaMemcpyAsync(sigma_host, sg, sizeof(double) * r, cudaMemcpyDeviceToHost, s));
        HSVD_HCUDA(cudaMemcpyAsync(lam_host, lm, sizeof(double) * r, cudaMemcpyDeviceToHost, s));
        HSVD_HCUDA(cudaStreamSynchronize(s));
    }
#undef HSVD_HCUDA
    cleanup();
    return st;
}

}  // extern "C"
