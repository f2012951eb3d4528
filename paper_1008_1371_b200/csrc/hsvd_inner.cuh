// hsvd_inner.cuh -- k_inner: one pass of 2x2 rotations on the 2b x 2b pivot
// Gram A_P in shared memory, accumulating the J-orthogonal W_P
// (A_P <- W^T A_P W).  Included by hsvd_block_kernels.cuh (namespace hsvd).
//
// The pass is a chain of 2b-1 (full ordering) or b (oriented) rounds of b
// disjoint rotations; each round needs the previous round's A.  The kernel
// is laid out around that chain (round-1 k_inner_v1 moved ~128 KB of shared
// memory per round and ran at ~2.7k cycles per round):
//
// * A holds only its upper triangle: entry (r, c) lives at [min][max].  A
//   round is the congruence A <- R^T A R with R block-diagonal in 2x2
//   blocks, so only the b(b+1)/2 blocks (p, q), q = p + d (mod b),
//   d = 0..b/2, are rewritten: half the shared-memory traffic of updating
//   both triangles, and A stays exactly symmetric.
// * Warp 0 forms the round's b rotations (lane q owns pair q) and publishes
//   them into a per-round log (t, c, st) with an mbarrier per round
//   (release/acquire: the other warps' stores of round k wait for warp 0's
//   loads of round k).  The A warps then update their blocks; one named
//   barrier among the A warps ends an active round.  A round in which no
//   pair rotates costs no barrier.
// * W never touches shared memory: W_P's rows are independent under
//   W <- W R, so each of the 2b rows lives in the registers of one thread of
//   the W warps, which replay the rotation log behind the A chain (off its
//   critical path).  Registers cannot be indexed at run time, so a W row is
//   kept in "position space": under the circle method pair x of round rd is
//   columns (rd + x, rd - x) mod (2b-1) (pair 0: (2b-1, rd)), which in
//   positions pos(c) = (c - rd) mod (2b-1) is the FIXED pairing (x, 2b-1-x),
//   (0, 2b-1); between rounds every position moves down by one.  The move is
//   register renaming inside U unrolled rounds and one cyclic shift of the
//   row per U rounds.  The oriented ordering is the same with the j half
//   cycling.
// The element operations (and their order) are those of k_inner_v1, so a
// W row sees exactly the same FMA sequence; A's upper entries are computed
// by the same formulas (block (p, q) as rows of pair p, columns of pair q).

#ifndef HSVD_INNER_DIAG_NOW
#define HSVD_INNER_DIAG_NOW 0
#endif
#ifndef HSVD_INNER_DIAG_NOUPD
#define HSVD_INNER_DIAG_NOUPD 0
#endif
// HSVD_INNER_COMPACT: half-row W, 3 bulk warps, <= 128 registers per thread
// (32k per CTA, ~99 KB shared): a k_update CTA fits beside the inner CTA
#ifndef HSVD_INNER_COMPACT
#define HSVD_INNER_COMPACT 0
#endif
#if HSVD_INNER_COMPACT
#define HSVD_INNER_WHALF 1
#define HSVD_INNER_BWARPS64H 3
#define HSVD_INNER_MINB 2
#else
#define HSVD_INNER_MINB 1
#endif
#ifndef HSVD_INNER_PRE0  // bulk: the critical slot's entries loaded before the round's rotations
#define HSVD_INNER_PRE0 1  // slots prefetched; 2: 1403, 4: 1455 cycles per round (1: 1392)
#endif
#ifndef HSVD_W_SUSPEND_NS  // W warps' mbarrier wait: suspend-time hint
#define HSVD_W_SUSPEND_NS 1000000
#endif
#ifndef HSVD_INNER_WHALF
#define HSVD_INNER_WHALF 0  // 1: W rows split over two threads (half rows; measured slower: 1600 vs 1470 cycles per round)
#endif
#ifndef HSVD_INNER_BWARPS64H
#define HSVD_INNER_BWARPS64H 7  // bulk warps at b = 32 with half rows (+ leader + 4 W: 12 warps)
#endif
#ifndef HSVD_INNER_BWARPS64
#define HSVD_INNER_BWARPS64 5  // bulk warps at b = 32 (+ leader + 2 W warps: 8 warps, 255 registers)
#endif

template <int B2>
struct InnerCfg {
    static constexpr int b = B2 / 2;
#if HSVD_INNER_WHALF
    static constexpr int NBW = B2 == 64 ? HSVD_INNER_BWARPS64H : 3;  // bulk warps
#else
    static constexpr int NBW = B2 == 64 ? HSVD_INNER_BWARPS64 : 3;  // bulk warps
#endif
    static constexpr int NBT = NBW * 32;                           // bulk threads
    static constexpr int NAW = 1 + NBW;                            // leader + bulk ("A side")
    static constexpr int NA = NAW * 32;
#if HSVD_INNER_WHALF
    static constexpr int NWW = B2 / 16;  // W warps: half a row per thread, two halves per row group
#else
    static constexpr int NWW = B2 / 32;  // W warps: a row per thread
#endif
    static constexpr int NT = NA + NWW * 32;
    static constexpr int LDA = B2;
    // bulk block slots: thread (g, p) of the bulk owns blocks (p, p + d),
    // d = g + G k; d < b/2 for every p, d = b/2 for p < b/2
    static constexpr int G = NBT / b;
    static constexpr int NB = (b / 2 + G) / G;
    static_assert(NBT % b == 0, "k_inner: bulk warp count");
    // bulk warps holding the critical groups 1 and 2 (threads b .. 3b-1)
    static constexpr int CW0 = b / 32, NCW = (3 * b - 1) / 32 - b / 32 + 1;
    // full ordering: 2b-1 rounds, cyclic over M = 2b-1 positions; U rounds
    // are renamed in registers between row shifts (U divides the rounds)
    static constexpr int M = B2 - 1;
    static constexpr int UF = (M % 3 == 0) ? 3 : 1;
    static constexpr int UO = 4;  // oriented: b rounds, b % 4 == 0
};

template <int B2>
struct InnerSmem2 {
    double A[2][B2 * B2];            // two copies (round k reads one, writes the other);
                                     // upper triangle, [min][max], ld B2
    double2 ltc[B2][B2 / 2];         // rotation log of the pass: (t, c) per round and pair
    unsigned long long full[B2];     // mbarrier per round: the log entry is published
    unsigned long long wdone;        // W warps have replayed a whole pass
    int lflag[B2];                   // bit 0: some pair rotated, bit 1: a pair failed
    unsigned int lact[B2];           // per round: the pairs that rotated (bit x: pair x)
    unsigned int lhyp[B2];           // per round: hyperbolic pairs (st = t), else st = -t
    unsigned int jneg[2], padm[2];   // per-column bit masks (J = -1, padding)
    double wx[2][2][B2];             // W half-row exchange: [round parity][half][row]
    unsigned int rot, skip, big;
    unsigned long long maxt_bits;
    unsigned long long fail;
    unsigned long long touched;
};

template <int B2>
__host__ __device__ constexpr int inner2_threads() { return InnerCfg<B2>::NT; }

__device__ __forceinline__ void named_bar_sync(int id, int count)
{
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count)
{
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
// named barriers of k_inner: 0 the whole CTA; leader -> bulk (a round's
// rotations are published); bulk -> leader (the critical blocks of a round
// are written); bulk only (a round is complete).  Hardware barriers park the
// waiting warps without polling, and each is passed once per round by
// construction (no lapping: the bulk reaches round k+1's barriers only after
// the leader consumed round k's)
constexpr int kBarRound = 1, kBarCrit = 2, kBarDone = 3;

// W warps wait for a published round without polling the shared-memory
// pipe: the suspend hint parks the warp until the phase completes
__device__ __forceinline__ void mbar_wait_parked(unsigned bar, unsigned parity)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "HSVD_MBP_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra HSVD_MBP_%=;\n}\n" ::"r"(bar),
        "r"(parity), "r"(HSVD_W_SUSPEND_NS)
        : "memory");
}

// columns of pair x in round rd: circle method on B2 players (FULL), or the
// block-oriented pairing x <-> b + (x + rd) mod b.  Selects, no branches.
template <int B2, bool FULL>
__device__ __forceinline__ void inner_cols(int x, int rd, int &ci, int &cj)
{
    constexpr int b = B2 / 2;
    if (FULL) {
        constexpr int m = B2 - 1;
        int u = rd + x, v = rd - x;
        u = u >= m ? u - m : u;
        v = v < 0 ? v + m : v;
        ci = x == 0 ? m : u;
        cj = v;  // x = 0: v = rd
    } else {
        int v = rd + x;
        v = v >= b ? v - b : v;
        ci = x;
        cj = v + b;
    }
}

// pair of column c in round rd and its role (false: the pair's first
// column ci, true: its second cj); inverse of inner_cols
template <int B2, bool FULL>
__device__ __forceinline__ void inner_pair_of(int c, int rd, int &x, bool &isj)
{
    constexpr int b = B2 / 2;
    if (FULL) {
        constexpr int m = B2 - 1;
        int u = c - rd;
        u = u < 0 ? u + m : u;
        x = c == m ? 0 : (u == 0 ? 0 : (u < b ? u : m - u));
        isj = c != m && (u == 0 || u >= b);
    } else {
        int y = c - b - rd;
        y = y < 0 ? y + b : y;
        x = c < b ? c : y;
        isj = c >= b;
    }
}

// Entries of S_k = R^T S_{k-1} R (round k's congruence, pairing rd) from
// S_{k-1} in Ab, with the bulk's formulas and operation order (so the same
// bits).  Diagonal entry of the pair's column ci (isj false) or cj:
template <int B2, bool FULL>
__device__ __forceinline__ double inner_diag_after(const double *Ab, int P, bool isj, int rd,
                                                   double t, double c, double st)
{
    constexpr int LDA = B2;
    int iP, jP;
    inner_cols<B2, FULL>(P, rd, iP, jP);
    const double a_ii = Ab[iP * (LDA + 1)], a_jj = Ab[jP * (LDA + 1)],
                 a_ij = Ab[min(iP, jP) * LDA + max(iP, jP)];
    const double ya = isj ? fma(t, a_ii, a_ij) * c : fma(st, a_ij, a_ii) * c;  // y01 / y00
    const double yb = isj ? fma(t, a_ij, a_jj) * c : fma(st, a_jj, a_ij) * c;  // y11 / y10
    const double v = isj ? fma(t, ya, yb) * c : fma(st, yb, ya) * c;
    return t == 0.0 ? (isj ? a_jj : a_ii) : v;  // a skipped pair's block is copied
}
// off-diagonal entry of block (p, q) (rows of pair p, columns of pair q): the
// row member of p with role rpj and the column member of q with role rqj
template <int B2, bool FULL>
__device__ __forceinline__ double inner_off_after(const double *Ab, int p, int q, bool rpj, bool rqj,
                                                  int rd, double tp, double cp, double sp,
                                                  double tq, double cq, double sq)
{
    constexpr int LDA = B2;
    int ip, jp, iq, jq;
    inner_cols<B2, FULL>(p, rd, ip, jp);
    inner_cols<B2, FULL>(q, rd, iq, jq);
    const double x0 = Ab[min(ip, iq) * LDA + max(ip, iq)], x1 = Ab[min(ip, jq) * LDA + max(ip, jq)];
    const double x2 = Ab[min(jp, iq) * LDA + max(jp, iq)], x3 = Ab[min(jp, jq) * LDA + max(jp, jq)];
    // column step (R_q) on the needed column, then the row step (R_p)
    const double ya = rqj ? fma(tq, x0, x1) * cq : fma(sq, x1, x0) * cq;  // y01 / y00
    const double yb = rqj ? fma(tq, x2, x3) * cq : fma(sq, x3, x2) * cq;  // y11 / y10
    const double v = rpj ? fma(tp, ya, yb) * cp : fma(sp, yb, ya) * cp;
    const double xo = rpj ? (rqj ? x3 : x2) : (rqj ? x1 : x0);
    return (tp == 0.0 && tq == 0.0) ? xo : v;  // both pairs skipped: copied
}

// ---- position space of the A copies (see the kernel).  FULL: moving
// positions 0..M-1 (M = B2-1) shift down by one per round (0 wraps to M-1),
// position M stays; oriented: the j half (b..2b-1) shifts, the i half stays.
// fixed positions of pair x
template <int B2, bool FULL>
__host__ __device__ constexpr void inner_ppos(int x, int &u, int &v)
{
    if (FULL) {
        u = x == 0 ? B2 - 1 : x;
        v = x == 0 ? 0 : B2 - 1 - x;
    } else {
        u = x;
        v = B2 / 2 + x;
    }
}
// position in round k+1 of the value at position u in round k
template <int B2, bool FULL>
__host__ __device__ constexpr int inner_next(int u)
{
    constexpr int M = B2 - 1, b = B2 / 2;
    return FULL ? (u == M ? M : (u == 0 ? M - 1 : u - 1)) : (u < b ? u : (u == b ? B2 - 1 : u - 1));
}
// position in round k - L of the value at position u in round k; L is
// reduced (0 <= L < the period: M for FULL, b oriented, inner_lag)
template <int B2, bool FULL>
__host__ __device__ inline int inner_prev(int u, int L)
{
    constexpr int M = B2 - 1, b = B2 / 2;
    if (FULL) {
        if (u == M) return M;
        const int w = u + L;
        return w >= M ? w - M : w;
    }
    if (u < b) return u;
    const int w = u - b + L;
    return b + (w >= b ? w - b : w);
}
template <int B2, bool FULL>
__host__ __device__ inline int inner_lag(int rounds_behind)
{
    return rounds_behind % (FULL ? B2 - 1 : B2 / 2);
}
// pair (and role: true = its second position) holding position w
template <int B2, bool FULL>
__host__ __device__ constexpr void inner_pos_pair(int w, int &x, bool &isj)
{
    constexpr int M = B2 - 1, b = B2 / 2;
    if (FULL) {
        x = w == M ? 0 : (w == 0 ? 0 : (w < b ? w : M - w));
        isj = w != M && (w == 0 || w >= b);
    } else {
        x = w < b ? w : w - b;
        isj = w >= b;
    }
}
// canonical offset of the (symmetric) entry at positions (u, v)
template <int B2>
__host__ __device__ constexpr int inner_canon(int u, int v)
{
    return u < v ? u * B2 + v : v * B2 + u;
}
// a per-position bit mask moved to the next round's positions
template <int B2, bool FULL>
__device__ __forceinline__ unsigned long long inner_next_mask(unsigned long long m)
{
    constexpr int M = B2 - 1, b = B2 / 2;
    if (FULL) {
        const unsigned long long moving = (M == 64 ? ~0ull : ((1ull << M) - 1));
        const unsigned long long mv = m & moving;
        return (m & ~moving) | (mv >> 1) | ((mv & 1ull) << (M - 1));
    }
    const unsigned long long jm = ((1ull << b) - 1) << b;
    const unsigned long long mv = m & jm;
    return (m & ~jm) | ((mv >> 1) & jm) | ((mv & (1ull << b)) << (b - 1));
}

// register of position p after S renamed rounds
template <int B2, bool FULL>
__host__ __device__ constexpr int inner_wreg(int p, int S)
{
    return FULL ? (p == B2 - 1 ? p : (p + S) % (B2 - 1))
                : (p < B2 / 2 ? p : B2 / 2 + (p - B2 / 2 + S) % (B2 / 2));
}

// st = t for a hyperbolic pair, -t for a trigonometric one (a sign flip)
__device__ __forceinline__ double inner_st(double t, unsigned hyp)
{
    return __longlong_as_double(__double_as_longlong(t) ^ ((unsigned long long)(hyp ^ 1u) << 63));
}

// per-pass statistics kept by W warp 0 (lane x: pair x), off the A chain
struct InnerStats {
    unsigned int rot = 0, skip = 0, big = 0;
    unsigned long long touch = 0;
    double maxt = 0.0;
};

// one round of the W replay on a register-resident row (sub-round S of U).
// Straight-line: an inactive pair (and every pair of an inactive round) has
// t = st = 0, c = 1, an exact no-op on the row up to the sign of a zero; no
// branch keeps the 2b live doubles out of phi copies at every join.
template <int B2, bool FULL, int S>
__device__ __forceinline__ int inner_w_round(double (&w)[B2], const InnerSmem2<B2> &Sm, int rd,
                                             unsigned bar, unsigned par, bool stats,
                                             InnerStats &st_, unsigned long long padm,
                                             double teps)
{
    constexpr int b = B2 / 2, M = B2 - 1;
    mbar_wait_parked(bar, par);
    const int f = *(volatile const int *)&Sm.lflag[rd];
    const unsigned hm = Sm.lhyp[rd];
#pragma unroll
    for (int x = 0; x < b; ++x) {
        // pair x in position space: full (x, M - x), pair 0 (M, 0);
        // oriented (x, b + x)
        const int pi = FULL ? (x == 0 ? M : x) : x;
        const int pj = FULL ? (x == 0 ? 0 : M - x) : b + x;
        const int ri = inner_wreg<B2, FULL>(pi, S), rj = inner_wreg<B2, FULL>(pj, S);
        const double2 tc = Sm.ltc[rd][x];
        const double t = tc.x, c = tc.y, st = inner_st(t, (hm >> x) & 1u);
        const double wx = w[ri], wy = w[rj];
        w[ri] = fma(st, wy, wx) * c;
        w[rj] = fma(t, wx, wy) * c;
    }
    if (stats) {
        // the reference's per-visit statistics (_kernels.py:218-233): lane x
        // counts pair x of this round
        const unsigned lane = threadIdx.x & 31;
        if (lane < (unsigned)b && !(f & 2)) {
            int i, j;
            inner_cols<B2, FULL>((int)lane, rd, i, j);
            const bool act = (Sm.lact[rd] >> lane) & 1u;
            if (act) {
                const double at = fabs(Sm.ltc[rd][lane].x);
                ++st_.rot;
                st_.touch |= (1ull << i) | (1ull << j);
                st_.big |= at > teps;
                st_.maxt = fmax(st_.maxt, at);
            } else if (!(((padm >> i) | (padm >> j)) & 1)) {
                ++st_.skip;  // pairs with a padding column are not visits
            }
        }
    }
    return f;
}

// W warps: replay the log onto one row of W (registers), U rounds per
// cyclic shift of the row; returns false if the pass failed
template <int B2, bool FULL>
__device__ __forceinline__ bool inner_w_replay(double (&w)[B2], const InnerSmem2<B2> &Sm,
                                               int passes, unsigned full0, unsigned wdone,
                                               bool stats, InnerStats &st_,
                                               unsigned long long padm, double teps)
{
    using C = InnerCfg<B2>;
    constexpr int U = FULL ? C::UF : C::UO;
    constexpr int rounds = FULL ? B2 - 1 : B2 / 2;
    static_assert(U <= 4 && rounds % U == 0, "k_inner: W unroll");
    for (int ps = 0; ps < passes; ++ps) {
        const unsigned par = (unsigned)ps & 1u;
        for (int r0 = 0; r0 < rounds; r0 += U) {
            int f = inner_w_round<B2, FULL, 0>(w, Sm, r0, full0 + 8 * r0, par, stats, st_, padm, teps);
            if (U > 1) f |= inner_w_round<B2, FULL, (U > 1 ? 1 : 0)>(w, Sm, r0 + 1, full0 + 8 * (r0 + 1), par, stats, st_, padm, teps);
            if (U > 2) f |= inner_w_round<B2, FULL, (U > 2 ? 2 : 0)>(w, Sm, r0 + 2, full0 + 8 * (r0 + 2), par, stats, st_, padm, teps);
            if (U > 3) f |= inner_w_round<B2, FULL, (U > 3 ? 3 : 0)>(w, Sm, r0 + 3, full0 + 8 * (r0 + 3), par, stats, st_, padm, teps);
            // a failed round and every later round of the pass are published
            // as failed: stop at the group that failed
            if (f & 2) return false;
            // positions move down by U: new reg[p] = old reg[p + U] (cyclic)
            if (FULL) {
                constexpr int M = B2 - 1;
                double tmp[U];
#pragma unroll
                for (int k = 0; k < U; ++k) tmp[k] = w[k];
#pragma unroll
                for (int p = 0; p < M - U; ++p) w[p] = w[p + U];
#pragma unroll
                for (int k = 0; k < U; ++k) w[M - U + k] = tmp[k];
            } else {
                constexpr int b = B2 / 2;
                double tmp[U];
#pragma unroll
                for (int k = 0; k < U; ++k) tmp[k] = w[b + k];
#pragma unroll
                for (int p = 0; p < b - U; ++p) w[b + p] = w[b + p + U];
#pragma unroll
                for (int k = 0; k < U; ++k) w[B2 - U + k] = tmp[k];
            }
        }
        mbar_arrive(wdone);  // every W lane: this pass's log entries are consumed
    }
    return true;
}

// ---- W rows split in two halves (HSVD_INNER_WHALF): the b pairs of a
// round in position space are split into two fixed halves (pairs 0..b/2-1
// and b/2..b-1); each half's positions form one "arc" of the moving
// positions (plus fixed ones), and between rounds exactly one value leaves
// each arc for the other.  A W row is held by two threads (warps of
// different halves, the same rows), 32 doubles each, exchanging one double
// per round through shared memory: registers fall from ~240 to ~100 per
// thread, so the CTA can carry more bulk warps.
//
// full ordering (M = 2b-1 moving positions + position M fixed):
//   half 0: arc a in [0, b/2-1) = position M-b/2+1+a, a in [b/2-1, b-1) =
//           position a-(b/2-1); fixed: position M.  pair 0 = (fixed, arc
//           b/2-1), pair j = (arc b/2-1+j, arc b/2-1-j)
//   half 1: arc a = position b/2+a (b of them); pair b/2+j = (arc j, arc b-1-j)
// oriented ordering (i side fixed, j side cycling over b positions):
//   half h: fixed f = column h b/2 + f, arc a = position b + h b/2 + a;
//           pair h b/2 + j = (fixed j, arc j)
// Values move from arc index a to a-1; arc 0 leaves for the other half's
// last arc index.  Within U renamed rounds arc a of sub-round s lives in
// register (a + s) mod L.
template <int B2, bool FULL, int HALF>
struct WHalf {
    static constexpr int b = B2 / 2, hb = b / 2, M = B2 - 1;
    static constexpr int L = FULL ? (HALF == 0 ? b - 1 : b) : hb;  // arc length
    static constexpr int NF = FULL ? (HALF == 0 ? 1 : 0) : hb;     // fixed registers
    static constexpr int NFA = NF > 0 ? NF : 1;
    // local pair j: (kind, index) of its ci and cj; kind 1 = fixed, 0 = arc
    __host__ __device__ static constexpr int ci_fixed(int j) { return FULL ? (HALF == 0 && j == 0) : 1; }
    __host__ __device__ static constexpr int ci_idx(int j)
    {
        return FULL ? (HALF == 0 ? (j == 0 ? 0 : hb - 1 + j) : j) : j;
    }
    __host__ __device__ static constexpr int cj_idx(int j)
    {
        return FULL ? (HALF == 0 ? hb - 1 - j : b - 1 - j) : j;
    }
    // column of arc index a / fixed register f (after whole passes)
    __host__ __device__ static constexpr int arc_col(int a)
    {
        return FULL ? (HALF == 0 ? (a <= hb - 2 ? M - hb + 1 + a : a - (hb - 1)) : hb + a)
                    : b + HALF * hb + a;
    }
    __host__ __device__ static constexpr int fix_col(int f) { return FULL ? M : HALF * hb + f; }
};

template <int B2, bool FULL, int HALF, int S>
__device__ __forceinline__ int inner_wh_round(double (&ar)[WHalf<B2, FULL, HALF>::L],
                                              double (&fx)[WHalf<B2, FULL, HALF>::NFA],
                                              InnerSmem2<B2> &Sm, int rd, unsigned bar,
                                              unsigned par, int rnd, int row, int rg, bool stats,
                                              InnerStats &st_, unsigned long long padm, double teps)
{
    using H = WHalf<B2, FULL, HALF>;
    constexpr int L = H::L, hb = H::hb;
    mbar_wait_parked(bar, par);
    const int f = *(volatile const int *)&Sm.lflag[rd];
    const unsigned hm = Sm.lhyp[rd];
#pragma unroll
    for (int j = 0; j < hb; ++j) {
        const int x = HALF * hb + j;
        const double2 tc = Sm.ltc[rd][x];
        const double t = tc.x, c = tc.y, st = inner_st(t, (hm >> x) & 1u);
        const int ra = (H::ci_idx(j) + S) % L, rb = (H::cj_idx(j) + S) % L;
        if (H::ci_fixed(j)) {
            const double wx = fx[H::ci_idx(j) < H::NFA ? H::ci_idx(j) : 0], wy = ar[rb];
            fx[H::ci_idx(j) < H::NFA ? H::ci_idx(j) : 0] = fma(st, wy, wx) * c;
            ar[rb] = fma(t, wx, wy) * c;
        } else {
            const double wx = ar[ra], wy = ar[rb];
            ar[ra] = fma(st, wy, wx) * c;
            ar[rb] = fma(t, wx, wy) * c;
        }
    }
    // one value leaves each arc for the other half (arc 0 -> last arc index)
    Sm.wx[rnd & 1][HALF][row] = ar[S % L];
    named_bar_sync(4 + rg, 64);
    ar[S % L] = Sm.wx[rnd & 1][HALF ^ 1][row];
    if (stats) {
        // the reference's per-visit statistics (_kernels.py:218-233): lane x
        // counts pair x of this round
        const unsigned lane = threadIdx.x & 31;
        constexpr int b = B2 / 2;
        if (lane < (unsigned)b && !(f & 2)) {
            int i, j;
            inner_cols<B2, FULL>((int)lane, rd, i, j);
            const bool act = (Sm.lact[rd] >> lane) & 1u;
            if (act) {
                const double at = fabs(Sm.ltc[rd][lane].x);
                ++st_.rot;
                st_.touch |= (1ull << i) | (1ull << j);
                st_.big |= at > teps;
                st_.maxt = fmax(st_.maxt, at);
            } else if (!(((padm >> i) | (padm >> j)) & 1)) {
                ++st_.skip;  // pairs with a padding column are not visits
            }
        }
    }
    return f;
}

// one half of a W row: replay the pass(es); false if the pass failed.  Writes
// the half's columns of row `row` to Wout (column-major, ld B2) on success.
template <int B2, bool FULL, int HALF>
__device__ __forceinline__ bool inner_wh_replay(InnerSmem2<B2> &Sm, int passes, unsigned full0,
                                                unsigned wdone, int row, int rg, bool stats,
                                                InnerStats &st_, unsigned long long padm,
                                                double teps, double *Wout)
{
    using C = InnerCfg<B2>;
    using H = WHalf<B2, FULL, HALF>;
    constexpr int L = H::L, U = FULL ? C::UF : C::UO;
    constexpr int rounds = FULL ? B2 - 1 : B2 / 2;
    static_assert(U <= 4 && rounds % U == 0, "k_inner: W unroll");
    double ar[L], fx[H::NFA];
#pragma unroll
    for (int a = 0; a < L; ++a) ar[a] = H::arc_col(a) == row ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < H::NFA; ++k) fx[k] = (H::NF > 0 && H::fix_col(k) == row) ? 1.0 : 0.0;
    int rnd = 0;
    for (int ps = 0; ps < passes; ++ps) {
        const unsigned par = (unsigned)ps & 1u;
        for (int r0 = 0; r0 < rounds; r0 += U, rnd += U) {
            int f = inner_wh_round<B2, FULL, HALF, 0>(ar, fx, Sm, r0, full0 + 8 * r0, par, rnd, row, rg, stats, st_, padm, teps);
            if (U > 1) f |= inner_wh_round<B2, FULL, HALF, (U > 1 ? 1 : 0)>(ar, fx, Sm, r0 + 1, full0 + 8 * (r0 + 1), par, rnd + 1, row, rg, stats, st_, padm, teps);
            if (U > 2) f |= inner_wh_round<B2, FULL, HALF, (U > 2 ? 2 : 0)>(ar, fx, Sm, r0 + 2, full0 + 8 * (r0 + 2), par, rnd + 2, row, rg, stats, st_, padm, teps);
            if (U > 3) f |= inner_wh_round<B2, FULL, HALF, (U > 3 ? 3 : 0)>(ar, fx, Sm, r0 + 3, full0 + 8 * (r0 + 3), par, rnd + 3, row, rg, stats, st_, padm, teps);
            if (f & 2) return false;
            // arc a moves to register a: new reg[a] = old reg[(a + U) mod L]
            double tmp[U];
#pragma unroll
            for (int k = 0; k < U; ++k) tmp[k] = ar[k];
#pragma unroll
            for (int a = 0; a < L - U; ++a) ar[a] = ar[a + U];
#pragma unroll
            for (int k = 0; k < U; ++k) ar[L - U + k] = tmp[k];
        }
        mbar_arrive(wdone);  // every W lane: this pass's log entries are consumed
    }
    // W column-major: Wout[c * B2 + row] = W[row][c]; after whole passes
    // every position is its column again
#pragma unroll
    for (int a = 0; a < L; ++a) Wout[H::arc_col(a) * B2 + row] = ar[a];
#pragma unroll
    for (int k = 0; k < H::NF; ++k) Wout[H::fix_col(k) * B2 + row] = fx[k];
    return true;
}

// A_P = sum of the slot's partial Gram segments in segment order (the upper
// triangle; the same additions in the same order as a one-element-per-thread
// fold, so the same bits).  Every thread of the CTA takes part: chunks of two
// adjacent row entries are read 16 bytes at a time, four segments in flight.
template <int B2>
__device__ __forceinline__ void inner_fold(const InnerArgs &a, double *A, int slot, int64_t I,
                                           int64_t J, int tid)
{
    using C = InnerCfg<B2>;
    constexpr int NT = C::NT, LDA = B2, b = B2 / 2;
    constexpr int NCHUNK = B2 * B2 / 2, PER = (NCHUNK + NT - 1) / NT, BATCH = HSVD_INNER_COMPACT ? 1 : 4;
    const double2 *P0 = reinterpret_cast<const double2 *>(a.Apart + (int64_t)slot * a.maxseg * (B2 * B2));
    const int nseg = (int)a.part.NSEG;
    // cross class: the two diagonal blocks come from the cache, only the
    // cross block from the partials (the same segment folds as a fresh
    // visit, so the same bits)
    const bool cross = a.skipf && a.skipf[slot] == kSlotCross;
    bool need[PER];
    double2 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int ch = tid + k * NT, i = ch / (B2 / 2), j0 = 2 * (ch % (B2 / 2));
        need[k] = ch < NCHUNK && j0 + 1 >= i && (!cross || (i < b && j0 >= b));
        v[k] = make_double2(0.0, 0.0);
    }
    for (int s0 = 0; s0 < nseg; s0 += BATCH) {
        double2 x[BATCH][PER];
#pragma unroll
        for (int u = 0; u < BATCH; ++u)
#pragma unroll
            for (int k = 0; k < PER; ++k)
                x[u][k] = (s0 + u < nseg && need[k])
                              ? P0[(int64_t)(s0 + u) * (NCHUNK) + tid + k * NT]
                              : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < BATCH; ++u)
#pragma unroll
            for (int k = 0; k < PER; ++k)
                if (s0 + u < nseg) {
                    v[k].x += x[u][k].x;
                    v[k].y += x[u][k].y;
                }
    }
    const bool cache = a.ru.dcache != nullptr;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int ch = tid + k * NT, i = ch / (B2 / 2), j0 = 2 * (ch % (B2 / 2));
        if (ch >= NCHUNK) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = j0 + h;
            if (i > j) continue;
            double val = h ? v[k].y : v[k].x;
            const bool dI = j < b, dJ = i >= b;  // inside a diagonal block
            if (cross && (dI || dJ)) {
                val = dI ? a.ru.dcache[(I * b + i) * b + j]
                         : a.ru.dcache[(J * b + (i - b)) * b + (j - b)];
            } else if (cache && !cross && (dI || dJ)) {
                if (dI) a.ru.dcache[(I * b + i) * b + j] = val;
                else a.ru.dcache[(J * b + (i - b)) * b + (j - b)] = val;
            }
            A[i * LDA + j] = val;
        }
    }
}

template <int B2, bool FAST, bool FULL>
__global__ void __launch_bounds__(inner2_threads<B2>(), HSVD_INNER_MINB) k_inner(InnerArgs a)
{
    using C = InnerCfg<B2>;
    constexpr int NA = C::NA, NT = C::NT, LDA = C::LDA, b = C::b;
    constexpr int rounds = FULL ? B2 - 1 : b;
    extern __shared__ __align__(16) unsigned char ism_raw[];
    auto &S = *reinterpret_cast<InnerSmem2<B2> *>(ism_raw);
    const long long t_entry = clock64();
    if (*(volatile unsigned long long *)a.err != kNoError) return;
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
    const unsigned full0 = (unsigned)__cvta_generic_to_shared(&S.full[0]);
    const unsigned wdone = (unsigned)__cvta_generic_to_shared(&S.wdone);
    // roles: warp 0 leads, warps 1..NBW bulk, then the W warps (the bulk is
    // spread over all four SM sub-partitions: measured faster than keeping
    // the leader's sub-partition free of bulk warps)
    const bool wwarp = warp >= C::NAW;
    const int arank = warp;  // rank among leader + bulk warps
    const int atid = arank * 32 + lane;

    inner_fold<B2>(a, S.A[0], slot, I, J, tid);

    if (wwarp) {
        // ---- W warps: their own code path (barrier 0 is shared with the A
        // warps by count, so the row's registers never overlap the fold's)
        const int wi = warp - C::NAW;
        named_bar_sync(0, NT);  // the prologue (A, masks, mbarriers) is done
        const unsigned long long padm =
            B2 == 64 ? ((unsigned long long)S.padm[1] << 32) | S.padm[0] : S.padm[0];
        const bool stats = wi == 0;
        InnerStats st_;
#if HSVD_INNER_WHALF
        const int half = wi & 1, rg = wi >> 1, wrow = rg * 32 + lane;
        double *Wout = a.Wg + (int64_t)slot * B2 * B2;
#if !HSVD_INNER_DIAG_NOW  // diagnostics only (wrong W): no replay
        if (half == 0)
            inner_wh_replay<B2, FULL, 0>(S, a.passes, full0, wdone, wrow, rg, stats, st_, padm, a.teps, Wout);
        else
            inner_wh_replay<B2, FULL, 1>(S, a.passes, full0, wdone, wrow, rg, stats, st_, padm, a.teps, Wout);
#endif
#else
        const int wrow = wi * 32 + lane;
        double w[B2];  // row `wrow` of W in position space
#pragma unroll
        for (int p = 0; p < B2; ++p) w[p] = p == wrow ? 1.0 : 0.0;
#if !HSVD_INNER_DIAG_NOW  // diagnostics only (wrong W): no replay
        const bool ok = inner_w_replay<B2, FULL>(w, S, a.passes, full0, wdone, stats, st_, padm, a.teps);
#else
        const bool ok = true;
#endif
        if (ok) {
            // W column-major: Wg[slot][c * B2 + k] = W[k][c]; after whole
            // passes every position is its column again
            double *Wout = a.Wg + (int64_t)slot * B2 * B2 + wrow;
#pragma unroll
            for (int c = 0; c < B2; ++c) Wout[c * B2] = w[c];
        }
#endif
        if (stats) {
            atomicAdd(&S.rot, st_.rot);
            atomicAdd(&S.skip, st_.skip);
            atomicOr(&S.big, st_.big);
            atomicMax(&S.maxt_bits, (unsigned long long)__double_as_longlong(st_.maxt));
            atomicOr(&S.touched, st_.touch);
        }
        named_bar_sync(0, NT);  // statistics and failure word are in
        if (a.trace && blockIdx.x == 0 && wrow == 0) a.trace[8 * 64] = clock64();
        return;
    }

    {
        if (tid < B2) {
            const int64_t pos = slot_pos(tid, b, I, J);
            const int neg = a.jsign[pos] < 0;
            const int pad = a.orig[pos] >= a.real_cols;
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
            for (int k = 0; k < rounds; ++k) mbar_init(full0 + 8 * k, 32);
            mbar_init(wdone, C::NWW * 32);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
    }
    named_bar_sync(0, NT);
    if (a.trace && blockIdx.x == 0 && tid == 0) {
        a.trace[8 * 64 + 2] = t_entry;
        a.trace[8 * 64 + 3] = clock64();
    }

    const int total = rounds * a.passes;
    long long *tr = (a.trace && blockIdx.x == 0 && tid == 0) ? a.trace : nullptr;
#define HSVD_STAMP(k) \
    if (tr && it < 64) tr[8 * it + (k)] = clock64();
    // A lives in "position space": in round k the entry of columns (c, c')
    // is stored at positions (pos_k(c), pos_k(c')) (inner_pos), in which
    // pair x is the FIXED position pair (inner_ppos).  The bulk reads round
    // k's copy and writes S_k at round k+1's positions (every value moves to
    // inner_next of its position), so every block address is loop-invariant
    // and the accesses of a warp walk consecutive positions (no bank
    // conflicts).  A round in which nothing rotates writes nothing: the copy
    // then lags ("epoch" ep < k) and is read through inner_prev^(k - ep).
    if (warp == 0) {
        // ---- leader: forms round it's b rotations while the bulk finishes
        // round it-1.  Lane x keeps the diagonal entries of its pair in
        // registers (it updates them itself with the bulk's formulas and
        // passes them on by shuffles), so the only entry it reads is the
        // pivot a_ij = S_{it-1}(i, j).  That entry lies in one of the bulk's
        // "critical" blocks of round it-1 (d = 1 or 2: the pairs that hand
        // i and j to this round), which the bulk computes first and signals.
        const int q = lane % b;  // pair owned by this lane
        int ux, vx;
        inner_ppos<B2, FULL>(q, ux, vx);
        const int oij = inner_canon<B2>(ux, vx);
        // where this lane's next-round diagonal entries are in this round:
        // the positions inner_prev(ux), inner_prev(vx) and their pairs
        int si, sj;
        bool ri, rj;
        inner_pos_pair<B2, FULL>(inner_prev<B2, FULL>(ux, 1), si, ri);
        inner_pos_pair<B2, FULL>(inner_prev<B2, FULL>(vx, 1), sj, rj);
        // J signs by position (bit u: the column at position u is negative)
        unsigned long long jpos =
            B2 == 64 ? ((unsigned long long)S.jneg[1] << 32) | S.jneg[0] : S.jneg[0];
        int lbuf = 0, ep = 0;  // buffer holding S_{it-1}, and its epoch
        double dci = S.A[0][ux * (LDA + 1)], dcj = S.A[0][vx * (LDA + 1)];
        int rd = 0;
        for (int it = 0; it < total; ++it) {
            HSVD_STAMP(0)
            if (it > 0 && rd == 0) {
                // pass boundary (passes > 1): the W warps must have replayed
                // the previous pass before its log is overwritten
                mbar_wait(wdone, (unsigned)((it / rounds) & 1) ^ 1u);
            }
            const int hyp = (((jpos >> ux) ^ (jpos >> vx)) & 1) ? 1 : -1;
            const unsigned vh = __ballot_sync(0xffffffffu, hyp > 0);
            const double a_ii = dci, a_jj = dcj, thr = (a.eps * a.eps) * (a_ii * a_jj);
            int oa = oij;
            if (it != ep) {  // the copy lags behind inactive rounds (warp-uniform)
                const int lag = inner_lag<B2, FULL>(it - ep);
                oa = inner_canon<B2>(inner_prev<B2, FULL>(ux, lag), inner_prev<B2, FULL>(vx, lag));
            }
            if (it >= 1) named_bar_sync(kBarCrit, 32 + C::NCW * 32);  // round it-1's critical blocks
            HSVD_STAMP(7)
            const double a_ij = S.A[lbuf][oa];
            // relative-orthogonality skip |a_ij| < eps sqrt(a_ii a_jj)
            // (_kernels.py:211), squared: no square root on the chain; the
            // rotation is formed beside the test (a_ij = 0 gives the
            // identity) and selected.  The pair is rotated in its schedule
            // orientation (ci, cj): the closed forms are odd (trig) or
            // symmetric (hyperbolic) in the roles, so this is the sorted
            // form's transformation except at zeta = 0
            const bool skip = a_ij == 0.0 || (a.use_skip && a_ij * a_ij < thr);
            HSVD_STAMP(5)
            double t, c;
            int status;
            if (!FAST) {
                status = rotation_tc(a_ii, a_jj, a_ij, hyp, t, c);
            } else if (__all_sync(0xffffffffu, rotation_fast_in_range(a_ii, a_jj, a_ij, hyp))) {
                status = rotation_fast_sel(a_ii, a_jj, a_ij, hyp, t, c);
            } else {
                status = rotation_fast(a_ii, a_jj, a_ij, hyp, t, c);
            }
            const bool bad = !skip && status != 0, act = !skip && status == 0;
            t = act ? t : 0.0;
            c = act ? c : 1.0;
            HSVD_STAMP(1)
            if (lane < b) S.ltc[rd][q] = make_double2(t, c);
            const unsigned va = __ballot_sync(0xffffffffu, act),
                           vb = __ballot_sync(0xffffffffu, bad);
            if (lane == 0) {
                S.lflag[rd] = (va ? 1 : 0) | (vb ? 2 : 0);
                S.lact[rd] = va;
                S.lhyp[rd] = vh;
            }
            named_bar_arrive(kBarRound, 32 + C::NBT);  // release to the bulk
            if (bad && lane < b) {
                int i, j;
                inner_cols<B2, FULL>(q, rd, i, j);
                const int lo = i < j ? i : j, hi = i < j ? j : i;
                atomicMin(&S.fail, pack_err(a.slot_base + slot, slot_pos(lo, b, I, J),
                                            slot_pos(hi, b, I, J)));
            }
            if (vb) {
                // the other warps wait round by round: publish the rest of
                // the pass as failed so none of them waits forever
                for (int r2 = rd + 1; r2 < rounds; ++r2) {
                    if (lane == 0) S.lflag[r2] = 2;
                    mbar_arrive(full0 + 8 * r2);
                }
            }
            mbar_arrive(full0 + 8 * rd);  // release to the W warps
            HSVD_STAMP(2)
            if (vb) break;
            // this pair's diagonal after the round (the bulk's diagonal-block
            // formulas, so its bits; a skipped pair keeps its entries), then
            // handed to the lanes that hold those positions next round
            const double st = inner_st(t, hyp > 0);
            double nci = a_ii, ncj = a_jj;
            if (act) {
                const double y00 = fma(st, a_ij, a_ii) * c, y10 = fma(st, a_jj, a_ij) * c;
                const double y01 = fma(t, a_ii, a_ij) * c, y11 = fma(t, a_ij, a_jj) * c;
                nci = fma(st, y10, y00) * c;
                ncj = fma(t, y01, y11) * c;
            }
            const double xi = __shfl_sync(0xffffffffu, nci, si), yi = __shfl_sync(0xffffffffu, ncj, si);
            const double xj = __shfl_sync(0xffffffffu, nci, sj), yj = __shfl_sync(0xffffffffu, ncj, sj);
            dci = ri ? yi : xi;
            dcj = rj ? yj : xj;
            jpos = inner_next_mask<B2, FULL>(jpos);
            if (va) {  // the bulk writes S_it into the other buffer, at epoch it+1
                lbuf ^= 1;
                ep = it + 1;
            }
            rd = rd + 1 == rounds ? 0 : rd + 1;
            HSVD_STAMP(6)
            // the last round's critical signal is consumed too (balanced barrier)
            if (it + 1 == total) named_bar_sync(kBarCrit, 32 + C::NCW * 32);
        }
    } else {
        // ---- bulk: round it's congruence on the upper blocks, buffer cb to
        // cb ^ 1.  Thread (group g, pair p) owns blocks (p, p + d), d = g + G k
        // (the rest of the upper triangle's blocks), larger d are dead slots;
        // p is the same in every slot.  Slot 0 of groups 1 and 2 (d = 1, 2)
        // holds the blocks the leader's next pivots come from: it is done
        // first and signalled
        constexpr int G = C::G, NB = C::NB;
        static_assert(G >= 3, "k_inner: the critical blocks need d = 1, 2 in slot 0");
        const int bt = atid - 32;
        const int pk = bt % b, g = bt / b;
        // the warps holding groups 1 and 2 signal as whole warps (a named
        // barrier counts warps): bulk warps CW0 .. CW0 + NCW - 1
        const bool critg = bt / 32 >= C::CW0 && bt / 32 < C::CW0 + C::NCW;
        int qk[NB];
        bool dg[NB], live[NB];
        // positions of the slots' four entries (rows of pair p, columns of
        // pair q; a diagonal block is (up,up) (up,vp) (vp,up) (vp,vp)), their
        // offsets in this round's copy (no lag) and in the next round's
        int up, vp;
        inner_ppos<B2, FULL>(pk, up, vp);
        int orr[NB][4], ow[NB][4];
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const int d = g + G * k;
            live[k] = d < b / 2 || (d == b / 2 && pk < b / 2);
            qk[k] = (pk + (live[k] ? d : 0)) % b;  // dead slots use block (p, p)
            dg[k] = qk[k] == pk;
            int uq, vq;
            inner_ppos<B2, FULL>(qk[k], uq, vq);
            const int rr[4] = {up, up, vp, vp}, cc[4] = {uq, vq, uq, vq};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                orr[k][e] = inner_canon<B2>(rr[e], cc[e]);
                ow[k][e] = inner_canon<B2>(inner_next<B2, FULL>(rr[e]), inner_next<B2, FULL>(cc[e]));
            }
        }
        int cb = 0, ep = 0;  // buffer holding S_{it-1}, and its epoch
        int orl[NB][4];      // read offsets of a lagging copy
        int rd = 0;
        long long *btr = (a.trace && blockIdx.x == 0 && tid == 32) ? a.trace + 1024 : nullptr;
        for (int it = 0; it < total; ++it, rd = rd + 1 == rounds ? 0 : rd + 1) {
            if (btr && it < 64) btr[8 * it] = clock64();
#if HSVD_INNER_PRE0
            // the first HSVD_INNER_PRE0 slots' entries (the critical slot
            // first) do not depend on the round's rotations: loaded before
            // the leader publishes them
            constexpr int NPRE = HSVD_INNER_PRE0 < NB ? HSVD_INNER_PRE0 : NB;
            double xp[NPRE][4];
            {
                const double *Ar = S.A[cb];
                if (it == ep) {
#pragma unroll
                    for (int k = 0; k < NPRE; ++k)
                        if (live[k]) {
#pragma unroll
                            for (int e = 0; e < 4; ++e) xp[k][e] = Ar[orr[k][e]];
                        }
                } else {
                    const int lag = inner_lag<B2, FULL>(it - ep);
#pragma unroll
                    for (int k = 0; k < NPRE; ++k) {
                        int uq, vq;
                        inner_ppos<B2, FULL>(qk[k], uq, vq);
                        const int rr[4] = {up, up, vp, vp}, cc[4] = {uq, vq, uq, vq};
                        if (live[k]) {
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                xp[k][e] = Ar[inner_canon<B2>(inner_prev<B2, FULL>(rr[e], lag),
                                                              inner_prev<B2, FULL>(cc[e], lag))];
                        }
                    }
                }
            }
#endif
            named_bar_sync(kBarRound, 32 + C::NBT);  // the leader published round it
            if (btr && it < 64) btr[8 * it + 1] = clock64();
            if (btr && it < 64) btr[8 * it + 2] = clock64();
            const int f = S.lflag[rd];
            if (f & 2) break;
            if (f & 1) {
                // X' = R_p^T X R_q per block (rows of pair p, columns of pair
                // q); blocks whose two pairs both skipped are copied through
                const double *Ar = S.A[cb];
                double *Aw = S.A[cb ^ 1];
                const bool lagging = it != ep;  // warp-uniform
                if (lagging) {
                    const int lag = inner_lag<B2, FULL>(it - ep);
#pragma unroll
                    for (int k = 0; k < NB; ++k) {
                        int uq, vq;
                        inner_ppos<B2, FULL>(qk[k], uq, vq);
                        const int rr[4] = {up, up, vp, vp}, cc[4] = {uq, vq, uq, vq};
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            orl[k][e] = inner_canon<B2>(inner_prev<B2, FULL>(rr[e], lag),
                                                        inner_prev<B2, FULL>(cc[e], lag));
                    }
                }
                const unsigned hm = S.lhyp[rd];
                const double2 tcp = S.ltc[rd][pk];
                const double tp = tcp.x, cp = tcp.y, sp = inner_st(tp, (hm >> pk) & 1u);
                auto read_off = [&](int k, int e) { return lagging ? orl[k][e] : orr[k][e]; };
                auto slot_apply = [&](int k, const double (&x)[4], double tq, double cq, double sq) {
                    double n0 = x[0], n1 = x[1], n2 = x[2], n3 = x[3];
                    if (!(tp == 0.0 && tq == 0.0)) {
                        const double y00 = fma(sq, x[1], x[0]) * cq;
                        const double y01 = fma(tq, x[0], x[1]) * cq;
                        const double y10 = fma(sq, x[3], x[2]) * cq;
                        const double y11 = fma(tq, x[2], x[3]) * cq;
                        n0 = fma(sp, y10, y00) * cp;
                        n3 = fma(tp, y01, y11) * cp;
                        n1 = dg[k] ? 0.0 : fma(sp, y11, y01) * cp;  // the pair itself: annihilated
                        n2 = fma(tp, y00, y10) * cp;
                    }
                    Aw[ow[k][0]] = n0;
                    Aw[ow[k][3]] = n3;
                    Aw[ow[k][1]] = n1;
                    if (!dg[k]) Aw[ow[k][2]] = n2;
                };
                // slot 0 first (the critical blocks), then the others batched
                {
                    const double2 tcq = S.ltc[rd][qk[0]];
                    const double sq = inner_st(tcq.x, (hm >> qk[0]) & 1u);
#if HSVD_INNER_PRE0
                    if (live[0]) slot_apply(0, xp[0], tcq.x, tcq.y, sq);
#else
                    double x[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) x[u] = Ar[read_off(0, u)];
                    if (live[0]) slot_apply(0, x, tcq.x, tcq.y, sq);
#endif
                }
                if (critg) named_bar_arrive(kBarCrit, 32 + C::NCW * 32);  // release: S_it's critical blocks
                double x[NB][4], tq[NB], cq[NB], sq[NB];
#pragma unroll
                for (int k = 1; k < NB; ++k) {
                    const double2 tcq = S.ltc[rd][qk[k]];
                    tq[k] = tcq.x;
                    cq[k] = tcq.y;
                    sq[k] = inner_st(tcq.x, (hm >> qk[k]) & 1u);
                    if (live[k]) {
#if HSVD_INNER_PRE0
                        if (k < NPRE) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) x[k][u] = xp[k < NPRE ? k : 0][u];
                            continue;
                        }
#endif
#pragma unroll
                        for (int u = 0; u < 4; ++u) x[k][u] = Ar[read_off(k, u)];
                    }
                }
#pragma unroll
                for (int k = 1; k < NB; ++k)
                    if (live[k]) slot_apply(k, x[k], tq[k], cq[k], sq[k]);
                cb ^= 1;
                ep = it + 1;
            } else if (critg) {
                named_bar_arrive(kBarCrit, 32 + C::NCW * 32);  // nothing moved: S_it = S_{it-1}
            }
            if (btr && it < 64) btr[8 * it + 3] = clock64();
            named_bar_sync(kBarDone, C::NBT);  // S_it complete before round it+1 reads it
        }
    }
#undef HSVD_STAMP
    named_bar_sync(0, NT);
    if (S.fail != kNoError) {
        if (tid == 0) atomicMin(a.err, S.fail);
        return;
    }
    // storage columns of the slot's 2b columns, for the update's prologue
    if (tid < B2) a.colidx[(int64_t)slot * B2 + tid] = a.colmap[slot_pos(tid, b, I, J)];
    if (tid == 0) {
        if (a.trace && blockIdx.x == 0) a.trace[8 * 64 + 1] = clock64();
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
                a.ru.pairstamp[I * a.nb + J] = stamp | ((uint32_t)FULL << 31);
                a.ru.pairskip[I * a.nb + J] = S.skip;
            }
        }
        inner_advance(a, slot, I, J);
    }
}
