// Test/benchmark only (tools/inner_bench.cu): an independent register-resident
// implementation of the full-ordering inner pass, used to cross-check k_inner.
// ---------------------------------------------------------------------
// k_inner_reg: the full-ordering inner pass with A_P and W_P in registers
// ---------------------------------------------------------------------
// The two-barrier kernel above moves all of A and W through shared memory
// in every round (128 KB per round at b = 32; its rounds are bound by the
// shared-memory pipe, ~2.2k wavefronts of ~3.3k cycles).  Here the data
// follow the circle schedule instead of the schedule following the data.
//
// Layout of round rd (circle method on 63 + 1 players): column-pair q holds
// the columns a_q = (rd + q) mod 63, b_q = (rd - q) mod 63 (q >= 1) and
// a_0 = 63, b_0 = rd; row-pair p holds the rows a_p, b_p likewise.  Lane q
// of warp w keeps, for its four row-pairs p = 4w + k,
//     X[k][s][u] = A[row(p, s)][col(q, u)]     (s, u: 0 = a side, 1 = b side)
// and, for the W rows 8w + m, Wv[m][u] = W[8w + m][col(q, u)].  The pair of
// round rd is (a_q, b_q): lane q forms its rotation itself, applies it to its
// columns from registers and the row-pair rotations of its warp from a
// four-entry table.  Going from round rd to rd + 1 moves every column one
// step along the 63-cycle a_1 <- a_2 <- ... <- a_31 <- b_31 <- ... <- b_0
// <- a_1 (two shuffles per register pair) and every row the same way (a
// register renaming inside the warp; two rows per warp cross to the
// neighbouring warps through shared memory).  The next round's diagonal
// 2x2 blocks are published by the lanes that hold them: one barrier per
// round, no shared-memory traffic for A or W.
//
// The rotation of pair q is formed on (a_q, b_q) in that orientation: the
// closed forms are odd (trig: t -> -t when the roles swap) or symmetric
// (hyperbolic), so this is the same transformation, bit for bit, as the
// sorted (i < j) form of k_inner, except at exactly zeta = 0, where both
// are exact annihilations with opposite sign conventions.
struct InnerRegSmem {
    double A[64][65];          // the summed Gram; later the W staging area
    double D[2][32][4];        // diagonal blocks of the next round (a-a, a-b, b-a, b-b)
    double up[2][8][32][2];    // row (4w, a) of warp w -> warp w - 1
    double dn[2][8][32][2];    // row (4w + 3, b) of warp w -> warp w + 1
    double R[8][4][4];         // per warp: t, c, st of its four row-pairs
    int js[64];
    unsigned int rot, skip, big;
    unsigned long long maxt_bits;
    unsigned long long fail;
    unsigned long long touched;
};

__device__ __forceinline__ int circle_col(int x, int side, int rd)
{
    if (x == 0) return side ? rd : 63;
    const int v = side ? rd - x : rd + x;
    return v < 0 ? v + 63 : (v >= 63 ? v - 63 : v);
}

// one step along the 63-cycle for the register pair (v0, v1) of lane q
__device__ __forceinline__ void circle_shift(double &v0, double &v1, int q)
{
    const double dn0 = __shfl_down_sync(0xffffffffu, v0, 1);
    const double up1 = __shfl_up_sync(0xffffffffu, v1, 1);
    const double n0 = q == 0 ? v0 : (q == 31 ? v1 : dn0);
    v1 = q == 0 ? dn0 : up1;
    v0 = n0;
}

template <bool FAST>
__global__ void __launch_bounds__(kThreads, 1) k_inner_reg(InnerArgs a)
{
    constexpr int B2 = 64, b = 32;
    extern __shared__ __align__(16) unsigned char ism_raw[];
    auto &S = *reinterpret_cast<InnerRegSmem *>(ism_raw);
    if (*(volatile unsigned long long *)a.err != kNoError) return;
    const int slot = blockIdx.x, tid = threadIdx.x, q = tid & 31, w = tid >> 5;
    int64_t I = a.iblk[slot], J = a.jblk[slot];
    if (I > J) { int64_t t = I; I = J; J = t; }

    // A = sum of the slot's partial segments in segment order (as k_inner)
    {
        const double *P0 = a.Apart + (int64_t)slot * a.maxseg * (B2 * B2);
        const int nseg = (int)a.part.NSEG;
        constexpr int PER = B2 * B2 / kThreads;
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
                    const int e = tid + k * kThreads;
                    x[u][k] = (s0 + u < nseg && e / B2 <= e % B2)
                                  ? P0[(int64_t)(s0 + u) * B2 * B2 + e] : 0.0;
                }
#pragma unroll
            for (int u = 0; u < BATCH; ++u)
#pragma unroll
                for (int k = 0; k < PER; ++k)
                    if (s0 + u < nseg) v[k] += x[u][k];
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid + k * kThreads, i = e / B2, j = e % B2;
            if (i <= j) {
                S.A[i][j] = v[k];
                S.A[j][i] = v[k];
            }
        }
    }
    if (tid < B2) S.js[tid] = (int)a.jsign[slot_pos(tid, b, I, J)];
    if (tid == 0) {
        S.rot = S.skip = S.big = 0;
        S.maxt_bits = 0;
        S.fail = kNoError;
        S.touched = 0;
    }
    __syncthreads();

    // registers in the layout of round 0
    double X[4][2][2], Wv[8][2];
    {
        const int c0 = circle_col(q, 0, 0), c1 = circle_col(q, 1, 0);
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int r0 = circle_col(4 * w + k, s, 0);
                X[k][s][0] = S.A[r0][c0];
                X[k][s][1] = S.A[r0][c1];
            }
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            Wv[m][0] = (8 * w + m == c0) ? 1.0 : 0.0;
            Wv[m][1] = (8 * w + m == c1) ? 1.0 : 0.0;
        }
        if (w == 0) {
            S.D[0][q][0] = S.A[c0][c0];
            S.D[0][q][1] = S.A[c0][c1];
            S.D[0][q][2] = S.A[c1][c0];
            S.D[0][q][3] = S.A[c1][c1];
        }
    }
    __syncthreads();

    unsigned int my_rot = 0, my_skip = 0, my_big = 0;
    unsigned long long my_touch = 0;
    double my_max = 0.0;
    bool failed = false;
    const int rounds = (B2 - 1) * a.passes;
    long long *tr = (a.trace && blockIdx.x == 0 && tid == 0) ? a.trace : nullptr;
    int rd = 0;
    for (int it = 0; it < rounds; ++it) {
        const int buf = it & 1;
        if (tr && it < 64) tr[8 * it] = clock64();
        const int ca = circle_col(q, 0, rd), cb = circle_col(q, 1, rd);
        const double4 dg = *reinterpret_cast<const double4 *>(&S.D[buf][q][0]);
        const double a_ii = dg.x, a_jj = dg.w, a_ij = ca < cb ? dg.y : dg.z;
        double t = 0.0, c = 1.0, st = 0.0;
        int act = 0, bad = 0;
        if (!(a_ij == 0.0 ||
              (a.use_skip && a_ij * a_ij < (a.eps * a.eps) * (a_ii * a_jj)))) {
            const int hyp = S.js[ca] == S.js[cb] ? -1 : 1;
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
        if (w == 0) {
            const int lo = ca < cb ? ca : cb, hi = ca < cb ? cb : ca;
            if (bad) atomicMin(&S.fail, pack_err(a.slot_base + slot, slot_pos(lo, b, I, J),
                                                 slot_pos(hi, b, I, J)));
            else if (act) {
                ++my_rot;
                my_touch |= (1ull << ca) | (1ull << cb);
                const double at = fabs(t);
                my_big |= at > a.teps;
                my_max = fmax(my_max, at);
            } else {
                ++my_skip;
            }
        }
        if (__any_sync(0xffffffffu, bad)) { failed = true; break; }  // identical in every warp
        if (tr && it < 64) tr[8 * it + 1] = clock64();
        if (__any_sync(0xffffffffu, act)) {
            // the rotations of this warp's row-pairs
            if ((q >> 2) == w) *reinterpret_cast<double4 *>(&S.R[w][q & 3][0]) = make_double4(t, c, st, 0.0);
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double4 rp = *reinterpret_cast<const double4 *>(&S.R[w][k][0]);
                const double tp = rp.x, cp = rp.y, sp = rp.z;
                if (t == 0.0 && tp == 0.0) continue;
                const double x00 = X[k][0][0], x01 = X[k][0][1], x10 = X[k][1][0], x11 = X[k][1][1];
                // Y = X R_q (columns), X' = R_p^T Y (rows)
                const double y00 = fma(st, x01, x00) * c;
                const double y01 = fma(t, x00, x01) * c;
                const double y10 = fma(st, x11, x10) * c;
                const double y11 = fma(t, x10, x11) * c;
                X[k][0][0] = fma(sp, y10, y00) * cp;
                X[k][1][1] = fma(tp, y01, y11) * cp;
                if (4 * w + k == q) {  // the pair itself: annihilated
                    X[k][0][1] = 0.0;
                    X[k][1][0] = 0.0;
                } else {
                    X[k][0][1] = fma(sp, y11, y01) * cp;
                    X[k][1][0] = fma(tp, y00, y10) * cp;
                }
            }
            if (t != 0.0) {  // W <- W R_q on this warp's rows
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const double wx = Wv[m][0], wy = Wv[m][1];
                    Wv[m][0] = fma(st, wy, wx) * c;
                    Wv[m][1] = fma(t, wx, wy) * c;
                }
            }
        }
        if (tr && it < 64) tr[8 * it + 2] = clock64();
        // ---- move to the layout of the next round
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int s = 0; s < 2; ++s) circle_shift(X[k][s][0], X[k][s][1], q);
#pragma unroll
        for (int m = 0; m < 8; ++m) circle_shift(Wv[m][0], Wv[m][1], q);
        const int nb = buf ^ 1;
        // rows: (p, a) -> (p - 1, a) for p >= 2, (1, a) -> (0, b), (0, a) stays;
        // (p, b) -> (p + 1, b) for p <= 30, (31, b) -> (31, a)
        if (w > 0) *reinterpret_cast<double2 *>(&S.up[nb][w - 1][q][0]) = make_double2(X[0][0][0], X[0][0][1]);
        if (w < 7) *reinterpret_cast<double2 *>(&S.dn[nb][w + 1][q][0]) = make_double2(X[3][1][0], X[3][1][1]);
        // the next round's diagonal blocks, published by the lanes holding them
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int p = 4 * w + k;
                int dp, ds;
                if (s == 0) {
                    dp = p <= 1 ? 0 : p - 1;
                    ds = p == 1 ? 1 : 0;
                } else {
                    dp = p == 31 ? 31 : p + 1;
                    ds = p == 31 ? 0 : 1;
                }
                if (dp == q)
                    *reinterpret_cast<double2 *>(&S.D[nb][q][2 * ds]) = make_double2(X[k][s][0], X[k][s][1]);
            }
        double n00[2], n01[2], n30[2], n31[2];
        if (w == 0) {
            n00[0] = X[0][0][0]; n00[1] = X[0][0][1];
            n01[0] = X[1][0][0]; n01[1] = X[1][0][1];
        } else {
            n00[0] = X[1][0][0]; n00[1] = X[1][0][1];
        }
        if (w == 7) { n30[0] = X[3][1][0]; n30[1] = X[3][1][1]; }
        n31[0] = X[2][1][0]; n31[1] = X[2][1][1];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const double a1 = X[2][0][u], a2 = X[3][0][u], b0 = X[0][1][u], b1 = X[1][1][u];
            X[1][0][u] = a1;  // (2, a) -> (1, a)
            X[2][0][u] = a2;  // (3, a) -> (2, a)
            X[1][1][u] = b0;  // (0, b) -> (1, b)
            X[2][1][u] = b1;  // (1, b) -> (2, b)
            X[0][0][u] = n00[u];
            X[3][1][u] = n31[u];
            if (w == 0) X[0][1][u] = n01[u];
            if (w == 7) X[3][0][u] = n30[u];
        }
        if (tr && it < 64) tr[8 * it + 3] = clock64();
        __syncthreads();
        if (w < 7) {
            const double2 v = *reinterpret_cast<const double2 *>(&S.up[nb][w][q][0]);
            X[3][0][0] = v.x;
            X[3][0][1] = v.y;
        }
        if (w > 0) {
            const double2 v = *reinterpret_cast<const double2 *>(&S.dn[nb][w][q][0]);
            X[0][1][0] = v.x;
            X[0][1][1] = v.y;
        }
        rd = rd == 62 ? 0 : rd + 1;
        if (tr && it < 64) tr[8 * it + 4] = clock64();
    }
    if (w == 0) {
        atomicAdd(&S.rot, my_rot);
        atomicAdd(&S.skip, my_skip);
        atomicOr(&S.big, my_big);
        atomicMax(&S.maxt_bits, (unsigned long long)__double_as_longlong(my_max));
        atomicOr(&S.touched, my_touch);
    }
    // W into the staging area (the rows of A are no longer read)
    if (!failed) {
        const int c0 = circle_col(q, 0, rd), c1 = circle_col(q, 1, rd);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            S.A[8 * w + m][c0] = Wv[m][0];
            S.A[8 * w + m][c1] = Wv[m][1];
        }
    }
    __syncthreads();
    if (S.fail != kNoError) {
        if (tid == 0) atomicMin(a.err, S.fail);
        return;
    }
    if (tid < B2) a.colidx[(int64_t)slot * B2 + tid] = a.colmap[slot_pos(tid, b, I, J)];
    double *Wout = a.Wg + (int64_t)slot * B2 * B2;
    for (int e = tid; e < B2 * B2; e += kThreads) Wout[e] = S.A[e % B2][e / B2];
    if (tid == 0) {
        uint8_t *ts = a.tset + (int64_t)slot * kTsetStride;
        unsigned long long m = S.touched;
        int cnt = 0;
        while (m) {
            const int cc = __ffsll((long long)m) - 1;
            m &= m - 1;
            ts[1 + cnt++] = (uint8_t)cc;
        }
        ts[0] = (uint8_t)cnt;
        if (S.big) a.C[slot] = 3;
        else if (S.rot) a.C[slot] |= 1;
        a.rotk[slot] += S.rot;
        a.skipk[slot] += S.skip;
        const double mt = __longlong_as_double((long long)S.maxt_bits);
        if (mt > a.maxt[slot]) a.maxt[slot] = mt;
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
}

