/*
 * hsvd_b200.h -- C ABI of the B200-native one-sided hyperbolic Jacobi HSVD.
 *
 * Plain pointers, sizes and a CUDA stream (passed as void*); no C++ or torch
 * types cross this boundary.  Every matrix is float64 column-major with an
 * explicit leading dimension; every pointer argument is a DEVICE pointer
 * unless its name ends in _host.  Return value: HSVD_OK (0), a positive
 * algorithmic status mirroring the reference's exceptions, or a negative
 * CUDA/usage error with a message in hsvd_last_error().
 *
 * Each entry point replaces one function of the reference package
 * (/root/reference/pkg/src/hjsvd/...), cited per declaration.  The Python
 * host package paper_1008_1371_b200 binds these with ctypes; INTEGRATION.md
 * shows the binding a maintainer would add to the reference itself.
 */
#ifndef HSVD_B200_H
#define HSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HSVD_API __attribute__((visibility("default")))
#else
#define HSVD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-30) ------------------------------------- */
#define HSVD_OK 0
#define HSVD_DEFINITENESS_LOST 1 /* DefinitenessLostError(block, i, j)   */
#define HSVD_RANK_DEFICIENT 2    /* RankDeficiencyError (zero column)     */
#define HSVD_SHAPE_ERROR 3       /* ShapeError                            */
#define HSVD_NUMERICAL_SINGULARITY 4 /* NumericalSingularityError (factor)  */
#define HSVD_ERR_CUDA (-1)
#define HSVD_ERR_ARG (-2)
#define HSVD_ERR_UNSUPPORTED (-3)

/* ---- solver modes ------------------------------------------------------ */
#define HSVD_MODE_POINTWISE 0 /* bit-exact mirror of the reference          */
#define HSVD_MODE_BLOCK 1     /* block-column pairs, FP64 DMMA Gram/update  */

/* ---- block-mode 2x2 rotation formula ----------------------------------- */
#define HSVD_ROTATION_DD 0   /* the reference's double-double rotation_tc  */
#define HSVD_ROTATION_FAST 1 /* plain fp64, same branches and tests         */

/* ---- schedules (solver.py:204-209) ------------------------------------- */
#define HSVD_SCHEDULE_MODULUS 0
#define HSVD_SCHEDULE_ROW_CYCLIC 1

/* Solver knobs: SolverConfig (solver.py:46-64) plus the B200 additions. */
typedef struct hsvd_config {
    int64_t max_sweeps;   /* 30                                           */
    double eps;           /* 2^-52                                        */
    double teps;          /* sqrt(eps)/2                                  */
    int32_t accumulate_v; /* 1                                            */
    int32_t use_skip;     /* use_rel_orth_skip, 1                         */
    int64_t chunk;        /* 32 (DEFAULT_CHUNK, linalg.py:20)             */
    int32_t schedule;     /* HSVD_SCHEDULE_*                              */
    int32_t sort;         /* 1                                            */
    int32_t mode;         /* HSVD_MODE_*                                  */
    int32_t block_cols;   /* block mode: b, columns per block (32 or 64)  */
    int32_t inner_full;   /* block mode: 1 = full inner pass every step (default), 0 = block-oriented */
    int32_t use_graph;    /* capture each sweep as a CUDA graph           */
    int32_t profile;      /* time every kernel of sweep 0 with CUDA events
                             (no graph); fills hsvd_result.kernel_ms     */
    int32_t block_rotation; /* block mode: HSVD_ROTATION_*               */
    int32_t inner_passes;   /* block mode: passes of the inner ordering
                               per step; 0 = auto (default): 2 in the dense
                               sweeps, 1 once a sweep rotates < 5 % of its
                               visits; >= 1: that count in every sweep    */
    int32_t block_streams;  /* block mode, one GPU: 2 = the slots run as two
                               halves on two streams, each half's step
                               waiting only for the other half's edge slots,
                               so one half's inner pass overlaps the other's
                               GEMMs; 1 = one stream */
} hsvd_config;

/* Per-run result record: the scalar part of HsvdResult (solver.py:67-77). */
typedef struct hsvd_result {
    int64_t sweeps_used;
    int32_t stop_reason; /* 0 orthogonal, 1 quadratic, 2 max_sweeps   */
    int32_t status;      /* HSVD_* of the run                          */
    int64_t rotations;
    int64_t skips;
    int64_t err[3];      /* (block, i, j) or (column, -1, -1)          */
    int64_t launches;    /* kernels this library launched for the run   */
    double setup_ms;     /* host wall: entry -> first sweep launched     */
    double sweeps_ms;    /* host wall: all sweeps incl. stop decisions   */
    double finish_ms;    /* host wall: extraction + teardown             */
    /* profile mode, sweep 0: device time and launches per kernel class
       [0] step / gram, [1] inner, [2] update, [3] sweep-end kernels   */
    double kernel_ms[4];
    int64_t kernel_launches[4];
} hsvd_result;

/* Per-sweep telemetry row (solver.py:247): (sweep, rot, skip, max|t|). */
typedef struct hsvd_telemetry {
    int64_t sweep;
    int64_t rotations;
    int64_t skips;
    double max_t;
    double gpu_ms;     /* device time of the sweep (CUDA events on the
                          launching stream): steps + reduction + sort    */
} hsvd_telemetry;

HSVD_API const char *hsvd_last_error(void);
HSVD_API int hsvd_version(void);
/* sizeof(hsvd_config), sizeof(hsvd_result), sizeof(hsvd_telemetry) into
 * out[0..3): lets a binding check its struct layouts against the library. */
HSVD_API void hsvd_abi_sizes(int64_t *out);
HSVD_API void hsvd_default_config(hsvd_config *cfg);

/* ---- reference-kernel mirrors ------------------------------------------ */

/* _kernels.dot_chunked (_kernels.py:32-59): *out (device) = x.y with
 * chunk-sequential FMA partials and the adjacent-pair tree; bit-exact. */
HSVD_API int hsvd_dot_chunked(const double *x, const double *y, int64_t n,
                     int64_t chunk, double *out, void *stream);

/* _kernels.fused_pair_update (_kernels.py:62-75), in place. */
HSVD_API int hsvd_fused_pair_update(double *x, double *y, int64_t n, double t, double c,
                           double s, void *stream);

/* _kernels.rotation_batch (_kernels.py:176-185): t[k], c[k] per entry;
 * *first_bad (device int64) = first failing index or -1. */
HSVD_API int hsvd_rotation_batch(const double *a_ii, const double *a_jj,
                        const double *a_ij, const int64_t *hyp, int64_t m,
                        double *t, double *c, int64_t *first_bad,
                        void *stream);

/* solver.precompute (solver.py:80-94): d[k] = dot_chunked(g_k, g_k);
 * *first_zero (device int64) = first zero column or -1. */
HSVD_API int hsvd_precompute(const double *G, int64_t n, int64_t r, int64_t ldg,
                    int64_t chunk, double *d, int64_t *first_zero,
                    void *stream);

/* _kernels.step_blocks (_kernels.py:188-235) over slots [k0, k1) of one
 * step, all slots concurrently (one CTA per slot).  V may be NULL.
 * rotk/skipk (uint32[k1]) and maxt (double[k1]) are per-slot counters that
 * are incremented / max-ed; *err_packed (device uint64) is atomically
 * min-ed with the packed (block, i, j) of a failing slot and, when not ~0
 * on entry, makes the launch a no-op.  If advance != 0 each slot then
 * advances its stepper quadruple (ip, jp, iblk, jblk), fusing
 * _kernels.advance_stepper (_kernels.py:238-251). */
HSVD_API int hsvd_step_blocks(double *G, int64_t n, int64_t ldg, double *V, int64_t rv,
                     int64_t ldv, double *d, const int64_t *rho,
                     const int64_t *jsign, int64_t *ip, int64_t *jp,
                     int64_t *iblk, int64_t *jblk, int64_t r, uint8_t *C,
                     int64_t k0, int64_t k1, double eps, double teps,
                     int32_t use_skip, int64_t chunk, int32_t advance,
                     uint32_t *rotk, uint32_t *skipk, double *maxt,
                     uint64_t *err_packed, void *stream);

/* _kernels.advance_stepper (_kernels.py:238-251). */
HSVD_API int hsvd_advance_stepper(int64_t *ip, int64_t *jp, int64_t *iblk,
                         int64_t *jblk, int64_t nblk, int64_t r, void *stream);

/* strategies.stepper_init (strategies.py:41-47). */
HSVD_API int hsvd_stepper_init(int64_t *ip, int64_t *jp, int64_t *iblk, int64_t *jblk,
                      int64_t r, void *stream);

/* solver.sort_diagonal (solver.py:97-110): stable, [0,p) descending,
 * [p,r) ascending; rho and jsign travel.  ws: 24*r bytes of device scratch. */
HSVD_API int hsvd_sort_diagonal(double *d, int64_t *rho, int64_t *jsign, int64_t r,
                       int64_t p, void *ws, void *stream);

/* solver.check_convergence (solver.py:113-121) fused with the per-sweep
 * statistics merge of _run_ranges (solver.py:147-156): OR of C[0..m),
 * sums of rotk/skipk and max of maxt over nslots, written to out (device):
 * out = {code, rotations, skips, max_t bits}.  reset != 0 zeroes C and the
 * counters afterwards. */
HSVD_API int hsvd_reduce_sweep(uint8_t *C, int64_t m, uint32_t *rotk, uint32_t *skipk,
                      double *maxt, int64_t nslots, int64_t *out,
                      int32_t reset, void *stream);

/* Result extraction (solver.py:261-267): sigma[rho]=sqrt(d), lam[rho]=d*j,
 * U[:,c] = G[:,c] / sigma[c] (in place on G, true division). */
HSVD_API int hsvd_extract(double *G, int64_t n, int64_t ldg, const double *d,
                 const int64_t *rho, const int64_t *jsign, int64_t r,
                 double *sigma, double *lam, void *stream);

/* ---- whole solver ------------------------------------------------------- */

/* Device scratch bytes hsvd_drive needs for (n, r, cfg). */
HSVD_API int64_t hsvd_drive_workspace_size(int64_t n, int64_t r, const hsvd_config *cfg);

/* solver.drive (solver.py:179-269) entirely on the device: G (n x r, ldg)
 * is overwritten by U; Vinv_t (r x r, ldv) receives V^{-T} if
 * cfg->accumulate_v; sigma/lam receive the results in original column
 * order; res_host / tele_host (max_sweeps rows, may be NULL) are host
 * memory.  signs_host: int8 +-1 with the p +1 entries leading. */
HSVD_API int hsvd_drive(double *G, int64_t n, int64_t r, int64_t ldg, double *Vinv_t,
               int64_t ldv, const int8_t *signs_host, int64_t p,
               const hsvd_config *cfg, double *sigma, double *lam,
               void *workspace, int64_t workspace_bytes,
               hsvd_result *res_host, hsvd_telemetry *tele_host,
               void *stream);

/* Same as hsvd_drive on HOST buffers (G_host is read, not modified):
 * allocates device memory, copies in, solves, copies U, V^{-T}, sigma, lam
 * back.  The e2e entry a ctypes/cffi binding of the reference would call. */
HSVD_API int hsvd_drive_host(const double *G_host, int64_t n, int64_t r,
                    const int8_t *signs_host, int64_t p,
                    const hsvd_config *cfg, double *U_host,
                    double *Vinv_t_host, double *sigma_host, double *lam_host,
                    hsvd_result *res_host, hsvd_telemetry *tele_host);

/* ---- multi-GPU: block mode sharded over N GPUs --------
 *
 * The reference splits the slots of a step into contiguous ranges and runs
 * them on worker threads (_run_ranges, solver.py:124-156); here the ranges
 * are GPUs.  Shard g owns slots [g*S/N, (g+1)*S/N) of the S = r/(2b) block
 * slots and keeps their block columns resident; after every step one block
 * column moves to a ring neighbour (NCCL send/recv), after every sweep the
 * norms are all-gathered, every shard runs the same stable sort, and the
 * columns are redistributed (grouped all-to-all).  Block mode only. */

/* NCCL communicator (NCCL is dlopen-ed; HSVD_ERR_UNSUPPORTED if absent).
 * Rank 0 creates the 128-byte id, the caller broadcasts it (e.g. with
 * torch.distributed), every rank calls hsvd_comm_init with its CUDA device
 * current. */
HSVD_API int hsvd_comm_unique_id(uint8_t *id_out);
HSVD_API int hsvd_comm_init(const uint8_t *id, int nranks, int rank, void **comm_out);
HSVD_API int hsvd_comm_destroy(void *comm);

/* Columns shard `shard` returns (2 * its slots * b), -1 if r, b, nshards
 * do not shard (need r/(2b) >= nshards). */
HSVD_API int64_t hsvd_shard_columns(int64_t r, int32_t block_cols, int32_t nshards,
                                    int32_t shard);
/* Device scratch bytes of one shard. */
HSVD_API int64_t hsvd_sharded_workspace_size(int64_t n, int64_t r, int32_t nshards,
                                             int32_t shard, const hsvd_config *cfg);

/* Sharded solve.  comm != NULL: one process per GPU, nlocal == 1 and
 * shard_ids[0] == rank.  comm == NULL: this process drives all nshards
 * shards (nlocal == nshards; devices[i] may repeat -- the local transport
 * copies with cudaMemcpyPeerAsync).  Per local shard i: G[i] is the FULL
 * n x r factor (ldg) on devices[i] (read only); the outputs hold the
 * shard's hsvd_shard_columns() columns after the final sweep:
 * U_out[i] (n x cols, ld n), V_out[i] (r x cols of V^{-T}, ld r, may be
 * NULL without accumulate_v), sigma_out[i] / lam_out[i] (device) and
 * cols_host[i] (host int64: the ORIGINAL column index of each returned
 * column).  ws[i] / ws_bytes[i]: hsvd_sharded_workspace_size bytes on
 * devices[i].  Statuses as hsvd_drive; every rank returns the same one. */
HSVD_API int hsvd_drive_sharded(void *comm, int32_t nshards, int32_t nlocal,
                                const int32_t *shard_ids, const int32_t *devices,
                                const double *const *G, int64_t n, int64_t r, int64_t ldg,
                                const int8_t *signs_host, int64_t p, const hsvd_config *cfg,
                                double *const *U_out, double *const *V_out,
                                int64_t *const *cols_host, double *const *sigma_out,
                                double *const *lam_out, void *const *ws,
                                const int64_t *ws_bytes, hsvd_result *res_host,
                                hsvd_telemetry *tele_host);

/* ---- eigen-pipeline front end (hjsvd.factory, factory.py:136-282) ------
 * Complete-pivoting Bunch-Parlett factorization M = G J G^T in
 * double-double, bit-identical to bunch_parlett_factor.  M (device, n x n,
 * exactly symmetric, leading dimension ldm), G out (device, column-major,
 * ldg; rows un-permuted, +1 columns first), signs out (device int8, +1
 * first), perm out (device int64: the symmetric pivot permutation), *p_out
 * (host) = number of +1 signs.  thresh = n * eps * ||M||_F (the reference's
 * singularity threshold, computed by the caller).  Returns
 * HSVD_NUMERICAL_SINGULARITY with *stage_out = the pivot stage when every
 * remaining pivot candidate is <= thresh.  ws: device workspace of
 * hsvd_bp_workspace_size bytes (4 n^2 doubles + O(n)). */
HSVD_API int hsvd_bp_workspace_size(int64_t n, size_t *bytes);
/* the same on an unrounded double-double M = (M, Mlo) (generate_factor_pair,
 * factory.py:285-297, factorizes the generator's M before rounding).
 * thresh < 0: the reference's n * eps * ||M||_F, computed from M on the
 * device (G's storage is the scratch; it is written by the factorization
 * afterwards). */
HSVD_API int hsvd_bp_factor_dd(const double *M, const double *Mlo, int64_t n, int64_t ldm,
                               double thresh, double *G, int64_t ldg, int8_t *signs,
                               int64_t *perm, int64_t *p_out, int64_t *stage_out, void *ws,
                               size_t ws_bytes, void *stream);
HSVD_API int hsvd_bp_factor(const double *M, int64_t n, int64_t ldm, double thresh, double *G,
                            int64_t ldg, int8_t *signs, int64_t *perm, int64_t *p_out,
                            int64_t *stage_out, void *ws, size_t ws_bytes, void *stream);

/* QR shortening of a tall factor (factory.py:300-334): G (device, n x r,
 * column-major, n > r) = Q R; R (r x r, ldr) upper triangular with a
 * positive diagonal, Q (n x r, ldq) orthonormal columns.  Plain fp64
 * Householder.  HSVD_RANK_DEFICIENT (+ *bad_col) for a dependent column or a
 * zero diagonal of R; HSVD_SHAPE_ERROR for n <= r. */
HSVD_API int hsvd_qr_workspace_size(int64_t n, int64_t r, size_t *bytes);
HSVD_API int hsvd_qr_shorten(const double *G, int64_t n, int64_t r, int64_t ldg, double *R,
                             int64_t ldr, double *Q, int64_t ldq, int64_t *bad_col, void *ws,
                             size_t ws_bytes, void *stream);

/* Test-matrix generation in double-double (factory.py:79-101), bit-identical
 * to the reference: hsvd_gen_init sets M = diag(lam) (device lam, Mh, Ml
 * n x n row-major), hsvd_gen_reflect applies `count` Householder reflectors
 * (device vs, count x n row-major, the reference's standard_normal draws),
 * hsvd_gen_finish mirrors the upper triangle (np.triu(M) + np.triu(M, 1).T).
 * n <= 16384 (the pairwise tree of a row stays on chip). */
HSVD_API int hsvd_gen_workspace_size(int64_t n, size_t *bytes);
HSVD_API int hsvd_gen_init(const double *lam, int64_t n, double *Mh, double *Ml, void *stream);
HSVD_API int hsvd_gen_reflect(double *Mh, double *Ml, int64_t n, const double *vs, int64_t count,
                              void *ws, size_t ws_bytes, void *stream);
HSVD_API int hsvd_gen_finish(double *Mh, double *Ml, int64_t n, void *stream);

/* The shard plan alone (host only, no GPU): the stepper of all slots, the
 * block placement and the per-step block moves, for tests of the exchange
 * protocol.  hsvd_plan_advance writes (block, from, from_area, to, to_area)
 * per move and returns the count (-1 on error). */
HSVD_API void *hsvd_plan_create(int64_t nblocks, int32_t nshards);
HSVD_API void hsvd_plan_destroy(void *plan);
HSVD_API int64_t hsvd_plan_advance(void *plan, int64_t *moves, int64_t max_moves);
HSVD_API int hsvd_plan_state(void *plan, int64_t *iblk, int64_t *jblk, int32_t *owner,
                             int32_t *area, int64_t *slot_begin);
HSVD_API int hsvd_plan_redistribute(void *plan, int32_t b, const int64_t *rho_old,
                                    const int64_t *rho_new, int64_t r, int32_t shard,
                                    int64_t *send, int64_t *send_count, int64_t *recv,
                                    int64_t *recv_count);
HSVD_API void hsvd_plan_place(void *plan);

#ifdef __cplusplus
}
#endif
#endif /* HSVD_B200_H */
