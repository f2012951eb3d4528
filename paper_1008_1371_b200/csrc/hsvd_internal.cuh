// hsvd_internal.cuh -- shared device helpers of the B200 HSVD library.
//
// Compiled into the pointwise (bit-exact) translation unit with
// -fmad=false: every a*b+c that the reference evaluates with two roundings
// stays two roundings, and fma() appears exactly where the reference calls
// its llvm.fma intrinsic (/root/reference/pkg/src/hjsvd/_kernels.py:17-29).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <string>
#include <vector>

#include "../../include/hsvd_b200.h"

namespace hsvd {

// ---- error plumbing (host) ----------------------------------------------
void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define HSVD_CUDA(call)                                   \
    do {                                                  \
        cudaError_t _e = (call);                          \
        if (_e != cudaSuccess) return hsvd::cuda_fail(_e, #call); \
    } while (0)

#define HSVD_LAUNCH_CHECK(what)                                   \
    do {                                                          \
        cudaError_t _e = cudaGetLastError();                      \
        if (_e != cudaSuccess) return hsvd::cuda_fail(_e, what);  \
    } while (0)

constexpr unsigned long long kNoError = ~0ull;

inline double wall_ms()
{
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// Profile-mode kernel timer: CUDA events around each launch of sweep 0,
// summed per kernel class after the sweep's synchronisation.
struct KernelTimer {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<int> cls;
    size_t used = 0;
    ~KernelTimer()
    {
        for (auto e : ev) cudaEventDestroy(e);
    }
    void begin(int c, cudaStream_t s)
    {
        if (!on) return;
        if (used + 2 > ev.size()) {
            for (int i = 0; i < 2; ++i) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                ev.push_back(e);
            }
        }
        cls.push_back(c);
        cudaEventRecord(ev[used++], s);
    }
    void end(cudaStream_t s)
    {
        if (!on) return;
        cudaEventRecord(ev[used++], s);
    }
    // call after synchronising the stream
    void collect(hsvd_result *res)
    {
        for (size_t k = 0; k < cls.size(); ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[2 * k], ev[2 * k + 1]);
            res->kernel_ms[cls[k]] += ms;
            res->kernel_launches[cls[k]] += 1;
        }
        cls.clear();
        used = 0;
        on = false;
    }
};

// Per-thread, per-device resources reused across solves: creating and
// destroying streams, events and pinned buffers per call costs from
// milliseconds to hundreds of milliseconds (measured), so a solve borrows
// them from here.  xs/xev/xt0/xt1 are extra streams for the shards of the
// sharded driver's local transport.
struct DevCtx {
    int dev = -1;
    cudaStream_t s = nullptr;
    cudaEvent_t ev = nullptr, t0 = nullptr, t1 = nullptr;
    int64_t *host = nullptr;  // pinned
    int64_t host_len = 0;
    unsigned long long *dword = nullptr;  // one device word (input checks)
    std::vector<cudaStream_t> xs;
    std::vector<cudaEvent_t> xev, xt0, xt1;
    std::vector<cudaEvent_t> evs;   // plain (non-timing) events
    std::vector<cudaStream_t> xhi;  // extra streams at the highest priority
    int host_reserve(int64_t len);  // grow-only
    int extra(size_t k);            // at least k extra streams
    int events(size_t k);           // at least k plain events
    int extra_hi(size_t k);         // at least k high-priority streams
    ~DevCtx();
};
// the calling thread's context of device dev (created on first use; the
// device must be current)
DevCtx *dev_ctx(int dev, int *status);

// Packed (block, i, j) error word; min over failing slots = first slot.
__host__ __device__ inline unsigned long long pack_err(int64_t k, int64_t i,
                                                       int64_t j)
{
    return ((unsigned long long)k << 42) | ((unsigned long long)i << 21) |
           (unsigned long long)j;
}
inline void unpack_err(unsigned long long w, int64_t *out)
{
    out[0] = (int64_t)(w >> 42);
    out[1] = (int64_t)((w >> 21) & ((1ull << 21) - 1));
    out[2] = (int64_t)(w & ((1ull << 21) - 1));
}

// Smem column layout: one pad double per 32 so that the chunk-sequential
// reads of a warp (lane c reads element 32c+q) are bank-conflict free.
__host__ __device__ inline int padx(int e) { return e + (e >> 5); }
__host__ __device__ inline int padded_len(int n) { return n + (n >> 5) + 1; }

// ---- host-side launch helpers (defined in hsvd_pointwise.cu) -------------
int launch_pointwise_step(double *G, int64_t n, int64_t ldg, double *V,
                          int64_t rv, int64_t ldv, double *d,
                          const int64_t *rho, const int64_t *jsign,
                          int64_t *ip, int64_t *jp, int64_t *iblk,
                          int64_t *jblk, int64_t r, uint8_t *C, int64_t k0,
                          int64_t k1, double eps, double teps, int use_skip,
                          int64_t chunk, int advance, uint32_t *rotk,
                          uint32_t *skipk, double *maxt,
                          unsigned long long *err, cudaStream_t s);
int launch_rowcyclic_sweep(double *G, int64_t n, int64_t ldg, double *V,
                           int64_t rv, int64_t ldv, double *d,
                           const int64_t *rho, const int64_t *jsign,
                           int64_t r, uint8_t *C, double eps, double teps,
                           int use_skip, int64_t chunk, uint32_t *rotk,
                           uint32_t *skipk, double *maxt,
                           unsigned long long *err, cudaStream_t s);
int pointwise_smem_bytes(int64_t n, int64_t chunk, size_t *bytes);

}  // namespace hsvd
