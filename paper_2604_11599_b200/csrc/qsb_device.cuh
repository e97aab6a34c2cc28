// Device helpers: complex arithmetic on interleaved amplitudes, the gate-matrix
// builder for ParamRef angles, and the 2x2 update rules per gate class.
#pragma once
#ifndef QSB_JIT
#include <cuda_runtime.h>
#include <math_constants.h>

#include "qsb_internal.h"
#else
#define CUDART_PI 3.1415926535897931e+0
#endif

namespace qsb {

template <typename R> struct Amp;
template <> struct Amp<double> { using T = double2; };
template <> struct Amp<float> { using T = float2; };

template <typename R> __device__ __forceinline__ typename Amp<R>::T mk(R x, R y) {
  typename Amp<R>::T a;
  a.x = x;
  a.y = y;
  return a;
}

// m * a  (m given as double re/im, converted to R)
template <typename R>
__device__ __forceinline__ typename Amp<R>::T cmul(R mr, R mi, typename Amp<R>::T a) {
  return mk<R>(fma(mr, a.x, -mi * a.y), fma(mr, a.y, mi * a.x));
}

// m0 * a + m1 * b
template <typename R>
__device__ __forceinline__ typename Amp<R>::T cmac2(R m0r, R m0i, typename Amp<R>::T a, R m1r, R m1i,
                                                    typename Amp<R>::T b) {
  R re = fma(m0r, a.x, fma(-m0i, a.y, fma(m1r, b.x, -m1i * b.y)));
  R im = fma(m0r, a.y, fma(m0i, a.x, fma(m1r, b.y, m1i * b.x)));
  return mk<R>(re, im);
}

template <typename R> __device__ __forceinline__ double norm2(typename Amp<R>::T a) {
  double x = (double)a.x, y = (double)a.y;
  // numpy: re**2 + im**2, each square rounded, then added (sim.py:240); no FMA contraction
  return __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
}

// Apply a 2x2 of class `gc` to the pair (a0 = bit 0, a1 = bit 1).  m = 8 doubles.
template <typename R>
__device__ __forceinline__ void apply_pair(int gc, const double* m, typename Amp<R>::T& a0,
                                           typename Amp<R>::T& a1) {
  typename Amp<R>::T b0, b1;
  switch (gc) {
    case GC_XPERM:
      b0 = a1;
      b1 = a0;
      break;
    case GC_ANTI:
      b0 = cmul<R>((R)m[2], (R)m[3], a1);
      b1 = cmul<R>((R)m[4], (R)m[5], a0);
      break;
    case GC_DIAG:
      b0 = cmul<R>((R)m[0], (R)m[1], a0);
      b1 = cmul<R>((R)m[6], (R)m[7], a1);
      break;
    default:
      b0 = cmac2<R>((R)m[0], (R)m[1], a0, (R)m[2], (R)m[3], a1);
      b1 = cmac2<R>((R)m[4], (R)m[5], a0, (R)m[6], (R)m[7], a1);
      break;
  }
  a0 = b0;
  a1 = b1;
}

// gate_matrix (sim.py:190-200) for one op with angles resolved from `params`.
__device__ __forceinline__ void build_matrix(const MatSrc& s, const double* params, double* m) {
  if (s.has_matrix) {
    for (int i = 0; i < 8; ++i) m[i] = s.mat[i];
    return;
  }
  double a[3];
  for (int i = 0; i < 3; ++i) a[i] = s.slot[i] >= 0 ? params[s.slot[i]] : s.angle[i];
  for (int i = 0; i < 8; ++i) m[i] = 0.0;
  const double r2 = 1.0 / sqrt(2.0);
  switch (s.base) {
    case QSB_G_X: m[2] = 1; m[4] = 1; break;
    case QSB_G_Y: m[3] = -1; m[5] = 1; break;
    case QSB_G_Z: m[0] = 1; m[6] = -1; break;
    case QSB_G_H: m[0] = r2; m[2] = r2; m[4] = r2; m[6] = -r2; break;
    case QSB_G_S: m[0] = 1; m[7] = 1; break;
    case QSB_G_T: m[0] = 1; sincos(CUDART_PI / 4, &m[7], &m[6]); break;
    case QSB_G_SX: m[0] = 0.5; m[1] = 0.5; m[2] = 0.5; m[3] = -0.5; m[4] = 0.5; m[5] = -0.5; m[6] = 0.5; m[7] = 0.5; break;
    case QSB_G_RX: {
      double sn, c;
      sincos(a[0] / 2, &sn, &c);
      m[0] = c; m[3] = -sn; m[5] = -sn; m[6] = c;
    } break;
    case QSB_G_RY: {
      double sn, c;
      sincos(a[0] / 2, &sn, &c);
      m[0] = c; m[2] = -sn; m[4] = sn; m[6] = c;
    } break;
    case QSB_G_RZ: {
      double sn, c;
      sincos(0.5 * a[0], &sn, &c);
      m[0] = c; m[1] = -sn; m[6] = c; m[7] = sn;
    } break;
    case QSB_G_P: {
      double sn, c;
      sincos(a[0], &sn, &c);
      m[0] = 1; m[6] = c; m[7] = sn;
    } break;
    case QSB_G_U: {
      double th = a[0], ph = a[1], la = a[2];
      double sn, c, sl, cl, sp, cp, spl, cpl;
      sincos(th / 2, &sn, &c);
      sincos(la, &sl, &cl);
      sincos(ph, &sp, &cp);
      sincos(ph + la, &spl, &cpl);
      m[0] = c;
      m[2] = -cl * sn; m[3] = -sl * sn;
      m[4] = cp * sn; m[5] = sp * sn;
      m[6] = cpl * c; m[7] = spl * c;
    } break;
    default: break;
  }
  if (s.adjoint) {  // conjugate transpose
    double t0 = m[2], t1 = m[3];
    m[2] = m[4]; m[3] = -m[5];
    m[4] = t0; m[5] = -t1;
    m[1] = -m[1];
    m[7] = -m[7];
  }
}

}  // namespace qsb
