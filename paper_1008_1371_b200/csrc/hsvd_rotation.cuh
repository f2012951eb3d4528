// hsvd_rotation.cuh -- the double-double rotation of the reference
// (_kernels.py:84-173), shared by the pointwise (bit-exact) and block kernels.
// Every operation is an explicit round-to-nearest intrinsic, so the result
// does not depend on the translation unit's -fmad setting.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace hsvd {

// ---- double-double helpers: _kernels.py:84-125 ------------------------
__device__ __forceinline__ void dd_two_sum(double a, double b, double &s,
                                           double &e)
{
    s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void dd_quick(double a, double b, double &s,
                                         double &e)
{
    s = __dadd_rn(a, b);
    e = __dsub_rn(b, __dsub_rn(s, a));
}
__device__ __forceinline__ void dd_add(double xh, double xl, double yh,
                                       double yl, double &rh, double &rl)
{
    double s, e;
    dd_two_sum(xh, yh, s, e);
    dd_quick(s, __dadd_rn(e, __dadd_rn(xl, yl)), rh, rl);
}
__device__ __forceinline__ void dd_mul(double xh, double xl, double yh,
                                       double yl, double &rh, double &rl)
{
    double p = __dmul_rn(xh, yh);
    double e = __fma_rn(xh, yh, -p);
    double cross = __dadd_rn(__dmul_rn(xh, yl), __dmul_rn(xl, yh));
    dd_quick(p, __dadd_rn(e, cross), rh, rl);
}
__device__ __forceinline__ void dd_div(double xh, double xl, double yh,
                                       double yl, double &rh, double &rl)
{
    double q1 = __ddiv_rn(xh, yh);
    double ph = __dmul_rn(yh, q1);
    double pe = __dadd_rn(__fma_rn(yh, q1, -ph), __dmul_rn(yl, q1));
    double h, l;
    dd_add(xh, xl, -ph, -pe, h, l);
    dd_quick(q1, __ddiv_rn(__dadd_rn(h, l), yh), rh, rl);
}
__device__ __forceinline__ void dd_sqrt(double xh, double xl, double &rh,
                                        double &rl)
{
    double r = __dsqrt_rn(xh);
    double ph = __dmul_rn(r, r);
    double pe = __fma_rn(r, r, -ph);
    double dh, dl;
    dd_add(xh, xl, -ph, -pe, dh, dl);
    dd_quick(r, __ddiv_rn(__dadd_rn(dh, dl), __dmul_rn(2.0, r)), rh, rl);
}

// ---- rotation_tc: _kernels.py:128-173 ---------------------------------
__device__ __forceinline__ int rotation_tc(double a_ii, double a_jj, double a_ij, int64_t hyp,
                           double &t_out, double &c_out)
{
    t_out = 0.0;
    c_out = 1.0;
    if (a_ij == 0.0) return 0;
    double t, c;
    if (hyp < 0) {
        double zeta_est = __ddiv_rn(__dsub_rn(a_jj, a_ii), __dmul_rn(2.0, a_ij));
        if (fabs(zeta_est) > 6.7e7) {
            t_out = __ddiv_rn(0.5, zeta_est);
            return 0;
        }
        double nh, nl, zh, zl, sh, sl, oh, ol, wh, wl, bh, bl, th, tl;
        dd_two_sum(a_jj, -a_ii, nh, nl);
        dd_div(nh, nl, __dmul_rn(2.0, a_ij), 0.0, zh, zl);
        double sgn = zh >= 0.0 ? 1.0 : -1.0;
        zh = __dmul_rn(zh, sgn);
        zl = __dmul_rn(zl, sgn);
        dd_mul(zh, zl, zh, zl, sh, sl);
        dd_add(1.0, 0.0, sh, sl, oh, ol);
        dd_sqrt(oh, ol, wh, wl);
        dd_add(zh, zl, wh, wl, bh, bl);
        dd_div(sgn, 0.0, bh, bl, th, tl);
        t = __dadd_rn(th, tl);
        c = __ddiv_rn(1.0, __dsqrt_rn(__fma_rn(t, t, 1.0)));
    } else {
        double sh, sl, th0, tl0, qh, ql, dh, dl, wh, wl, bh, bl, th, tl;
        dd_two_sum(a_ii, a_jj, sh, sl);
        dd_div(__dmul_rn(-2.0, a_ij), 0.0, sh, sl, th0, tl0);
        dd_mul(th0, tl0, th0, tl0, qh, ql);
        dd_add(1.0, 0.0, -qh, -ql, dh, dl);
        if (dh <= 0.0) return 1;
        dd_sqrt(dh, dl, wh, wl);
        dd_add(1.0, 0.0, wh, wl, bh, bl);
        dd_div(th0, tl0, bh, bl, th, tl);
        t = __dadd_rn(th, tl);
        double u = __fma_rn(-t, t, 1.0);
        if (u <= 0.0) return 1;
        c = __ddiv_rn(1.0, __dsqrt_rn(u));
    }
    t_out = t;
    c_out = c;
    return 0;
}

}  // namespace hsvd
