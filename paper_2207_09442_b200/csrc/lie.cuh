// Device Lie-group math for the Between / Prior costs (PAPER.md:157 closed forms, :479
// relative-pose error).  fp64, register-resident, one thread per cost.  Written from the
// formulas in DESIGN.md "Readings" A1-A7 (right perturbation, SE3 xi = (rho, omega)).
//
// Small-angle handling (reading A7): every coefficient function is evaluated from a form
// without cancellation or by a factorial-coefficient Taylor polynomial below the pinned switch
// points theta < 0.5 (A, C, D) and theta < 1.0 (c2, c3):
//   A  = sin t / t                      B = (1 - cos t)/t^2 = 0.5 (sin(t/2)/(t/2))^2
//   C  = (t - sin t)/t^3                D = 1/t^2 - (1 + cos t)/(2 t sin t) = G / (2B),
//        G = (2B - A)/t^2 = sum_{k>=1} (-1)^(k+1) 2k t^(2k-2)/(2k+2)!
//   f  = t/(2 sin t) = 1/(2A)           c2 = (t^2 + 2cos t - 2)/(2t^4), c3 = (2t - 3 sin t + t cos t)/(2t^5)
#pragma once
#include <cuda_runtime.h>

namespace dnls {
namespace dev {

// ----------------------------------------------------------------------------- coefficients
__device__ __forceinline__ double horner(const double* c, int n, double x) {
  double r = c[n - 1];
  for (int i = n - 2; i >= 0; --i) r = fma(r, x, c[i]);
  return r;
}

struct Coef {
  double A, B, C, D, f;
};

// 1/(2k+1)!, (-1)^k
__device__ __forceinline__ double coefA_series(double t2) {
  const double c[9] = {1.0, -1.0 / 6.0, 1.0 / 120.0, -1.0 / 5040.0, 1.0 / 362880.0,
                       -1.0 / 39916800.0, 1.0 / 6227020800.0, -1.0 / 1307674368000.0,
                       1.0 / 355687428096000.0};
  return horner(c, 9, t2);
}
// 1/(2k+3)!
__device__ __forceinline__ double coefC_series(double t2) {
  const double c[9] = {1.0 / 6.0, -1.0 / 120.0, 1.0 / 5040.0, -1.0 / 362880.0, 1.0 / 39916800.0,
                       -1.0 / 6227020800.0, 1.0 / 1307674368000.0, -1.0 / 355687428096000.0,
                       1.0 / 121645100408832000.0};
  return horner(c, 9, t2);
}
// G = sum_{k>=1} (-1)^(k+1) 2k t^(2k-2) / (2k+2)!
__device__ __forceinline__ double coefG_series(double t2) {
  const double c[9] = {2.0 / 24.0, -4.0 / 720.0, 6.0 / 40320.0, -8.0 / 3628800.0,
                       10.0 / 479001600.0, -12.0 / 87178291200.0, 14.0 / 20922789888000.0,
                       -16.0 / 6402373705728000.0, 18.0 / 2432902008176640000.0};
  return horner(c, 9, t2);
}
// c2 = sum (-1)^k t^2k / (2k+4)!
__device__ __forceinline__ double coefc2_series(double t2) {
  const double c[11] = {1.0 / 24.0, -1.0 / 720.0, 1.0 / 40320.0, -1.0 / 3628800.0,
                        1.0 / 479001600.0, -1.0 / 87178291200.0, 1.0 / 20922789888000.0,
                        -1.0 / 6402373705728000.0, 1.0 / 2432902008176640000.0,
                        -1.0 / 1.1240007277776077e21, 1.0 / 6.204484017332394e23};
  return horner(c, 11, t2);
}
// c3 = sum (-1)^k (k+1) t^2k / (2k+5)!
__device__ __forceinline__ double coefc3_series(double t2) {
  const double c[11] = {1.0 / 120.0, -2.0 / 5040.0, 3.0 / 362880.0, -4.0 / 39916800.0,
                        5.0 / 6227020800.0, -6.0 / 1307674368000.0, 7.0 / 355687428096000.0,
                        -8.0 / 121645100408832000.0, 9.0 / 51090942171709440000.0,
                        -10.0 / 2.585201673888498e22, 11.0 / 1.5511210043330986e25};
  return horner(c, 11, t2);
}

__device__ __forceinline__ Coef coefs(double t) {
  Coef k;
  const double t2 = t * t;
  double s, c;
  sincos(t, &s, &c);
  if (t < 0.5) {
    k.A = coefA_series(t2);
    double h = coefA_series(0.25 * t2);  // sin(t/2)/(t/2)
    k.B = 0.5 * h * h;
    k.C = coefC_series(t2);
    k.D = coefG_series(t2) / (2.0 * k.B);
  } else {
    k.A = s / t;
    double h = sin(0.5 * t) / (0.5 * t);
    k.B = 0.5 * h * h;
    k.C = (t - s) / (t2 * t);
    k.D = 1.0 / t2 - (1.0 + c) / (2.0 * t * s);
  }
  k.f = 0.5 / k.A;
  return k;
}

__device__ __forceinline__ void coefs_c23(double t, double& c2, double& c3) {
  const double t2 = t * t;
  if (t < 1.0) {
    c2 = coefc2_series(t2);
    c3 = coefc3_series(t2);
  } else {
    double s, c;
    sincos(t, &s, &c);
    double t4 = t2 * t2;
    c2 = (t2 + 2.0 * c - 2.0) / (2.0 * t4);
    c3 = (2.0 * t - 3.0 * s + t * c) / (2.0 * t4 * t);
  }
}

// ----------------------------------------------------------------------------- 3x3 helpers
struct M3 {
  double m[3][3];
};

__device__ __forceinline__ M3 mul(const M3& a, const M3& b) {
  M3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j] + a.m[i][2] * b.m[2][j];
  return r;
}
__device__ __forceinline__ M3 hat(const double* v) {
  M3 r;
  r.m[0][0] = 0.0;   r.m[0][1] = -v[2]; r.m[0][2] = v[1];
  r.m[1][0] = v[2];  r.m[1][1] = 0.0;   r.m[1][2] = -v[0];
  r.m[2][0] = -v[1]; r.m[2][1] = v[0];  r.m[2][2] = 0.0;
  return r;
}
// a*I + b*W + c*W^2 with W = hat(w), W^2 = w w^T - |w|^2 I
__device__ __forceinline__ M3 poly_hat(double a, double b, double c, const double* w) {
  M3 r;
  double n2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.m[i][j] = c * w[i] * w[j];
#pragma unroll
  for (int i = 0; i < 3; ++i) r.m[i][i] += a - c * n2;
  r.m[0][1] += -b * w[2]; r.m[0][2] += b * w[1];
  r.m[1][0] += b * w[2];  r.m[1][2] += -b * w[0];
  r.m[2][0] += -b * w[1]; r.m[2][1] += b * w[0];
  return r;
}

// ----------------------------------------------------------------------------- SE(3)
// pose: row-major [3][4] = [R | t]
struct SE3 {
  double R[3][3];
  double t[3];
};

// Poses and measurements live in global memory, one pose per thread: a warp's accesses are 96 B
// apart, so each row [R_i0 R_i1 R_i2 t_i] (32 B) is moved with one 256-bit access when aligned.
__device__ __forceinline__ SE3 se3_load(const double* p) {
  SE3 T;
  if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
      asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(T.R[i][0]), "=d"(T.R[i][1]), "=d"(T.R[i][2]), "=d"(T.t[i])
                   : "l"(p + 4 * i)
                   : "memory");
    return T;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    T.R[i][0] = p[4 * i + 0];
    T.R[i][1] = p[4 * i + 1];
    T.R[i][2] = p[4 * i + 2];
    T.t[i] = p[4 * i + 3];
  }
  return T;
}
__device__ __forceinline__ void se3_store(const SE3& T, double* p) {
  if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p + 4 * i), "d"(T.R[i][0]), "d"(T.R[i][1]),
                   "d"(T.R[i][2]), "d"(T.t[i])
                   : "memory");
    return;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    p[4 * i + 0] = T.R[i][0];
    p[4 * i + 1] = T.R[i][1];
    p[4 * i + 2] = T.R[i][2];
    p[4 * i + 3] = T.t[i];
  }
}
// a^-1 b
__device__ __forceinline__ SE3 se3_between(const SE3& a, const SE3& b) {
  SE3 r;
  double dt[3] = {b.t[0] - a.t[0], b.t[1] - a.t[1], b.t[2] - a.t[2]};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) r.R[i][j] = a.R[0][i] * b.R[0][j] + a.R[1][i] * b.R[1][j] + a.R[2][i] * b.R[2][j];
    r.t[i] = a.R[0][i] * dt[0] + a.R[1][i] * dt[1] + a.R[2][i] * dt[2];
  }
  return r;
}
__device__ __forceinline__ SE3 se3_mul(const SE3& a, const SE3& b) {
  SE3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) r.R[i][j] = a.R[i][0] * b.R[0][j] + a.R[i][1] * b.R[1][j] + a.R[i][2] * b.R[2][j];
    r.t[i] = a.R[i][0] * b.t[0] + a.R[i][1] * b.t[1] + a.R[i][2] * b.t[2] + a.t[i];
  }
  return r;
}

// Log: theta = atan2(|v|/2, (tr R - 1)/2), v = vee(R - R^T), omega = f v;  rho = Jl^-1(omega) t
__device__ __forceinline__ void se3_log(const SE3& T, double* xi) {
  double v[3] = {T.R[2][1] - T.R[1][2], T.R[0][2] - T.R[2][0], T.R[1][0] - T.R[0][1]};
  double s = 0.5 * sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  double c = 0.5 * (T.R[0][0] + T.R[1][1] + T.R[2][2] - 1.0);
  double th = atan2(s, c);
  Coef k = coefs(th);
  double w[3] = {k.f * v[0], k.f * v[1], k.f * v[2]};
  M3 Jli = poly_hat(1.0, -0.5, k.D, w);   // Jl^-1 = I - W/2 + D W^2
#pragma unroll
  for (int i = 0; i < 3; ++i) xi[i] = Jli.m[i][0] * T.t[0] + Jli.m[i][1] * T.t[1] + Jli.m[i][2] * T.t[2];
  xi[3] = w[0];
  xi[4] = w[1];
  xi[5] = w[2];
}

// Exp(rho, omega) = [R(omega) | Jl(omega) rho],  R = I + A W + B W^2, Jl = I + B W + C W^2
__device__ __forceinline__ SE3 se3_exp(const double* xi) {
  const double* w = xi + 3;
  double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  Coef k = coefs(th);
  M3 R = poly_hat(1.0, k.A, k.B, w);
  M3 Jl = poly_hat(1.0, k.B, k.C, w);
  SE3 T;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) T.R[i][j] = R.m[i][j];
    T.t[i] = Jl.m[i][0] * xi[0] + Jl.m[i][1] * xi[1] + Jl.m[i][2] * xi[2];
  }
  return T;
}

// Jr^-1(xi) = [[Ji, -Ji Q(-rho,-omega) Ji], [0, Ji]],  Ji = Jr^-1(omega) = I + W/2 + D W^2.
// Returns the two distinct 3x3 blocks: Ji (diagonal) and U (upper right).
__device__ __forceinline__ void se3_jr_inv(const double* xi, M3& Ji, M3& U) {
  const double* w = xi + 3;
  double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  Coef k = coefs(th);
  double c2, c3;
  coefs_c23(th, c2, c3);
  Ji = poly_hat(1.0, 0.5, k.D, w);
  // Q(rho', phi) at rho' = -rho, phi = -omega (Barfoot)
  double nr[3] = {-xi[0], -xi[1], -xi[2]};
  double nw[3] = {-w[0], -w[1], -w[2]};
  M3 P = hat(nw), Rh = hat(nr);
  M3 PR = mul(P, Rh), RP = mul(Rh, P);
  M3 PRP = mul(PR, P);
  M3 PPR = mul(P, PR), RPP = mul(RP, P);
  M3 PRPP = mul(PRP, P), PPRP = mul(P, PRP);
  M3 Q;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      Q.m[i][j] = 0.5 * Rh.m[i][j] + k.C * (PR.m[i][j] + RP.m[i][j] + PRP.m[i][j]) +
                  c2 * (PPR.m[i][j] + RPP.m[i][j] - 3.0 * PRP.m[i][j]) + c3 * (PRPP.m[i][j] + PPRP.m[i][j]);
  M3 T1 = mul(Ji, Q);
  M3 T2 = mul(T1, Ji);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) U.m[i][j] = -T2.m[i][j];
}

// ----------------------------------------------------------------------------- SE(2)
struct SE2 {
  double c, s;   // R = [[c, -s], [s, c]] (stored as read, not re-normalised)
  double R[2][2];
  double t[2];
};

__device__ __forceinline__ SE2 se2_load(const double* p) {
  SE2 T;
  T.R[0][0] = p[0]; T.R[0][1] = p[1]; T.t[0] = p[2];
  T.R[1][0] = p[3]; T.R[1][1] = p[4]; T.t[1] = p[5];
  T.c = p[0];
  T.s = p[3];
  return T;
}
__device__ __forceinline__ void se2_store(const SE2& T, double* p) {
  p[0] = T.R[0][0]; p[1] = T.R[0][1]; p[2] = T.t[0];
  p[3] = T.R[1][0]; p[4] = T.R[1][1]; p[5] = T.t[1];
}
__device__ __forceinline__ SE2 se2_between(const SE2& a, const SE2& b) {
  SE2 r;
  double dt0 = b.t[0] - a.t[0], dt1 = b.t[1] - a.t[1];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) r.R[i][j] = a.R[0][i] * b.R[0][j] + a.R[1][i] * b.R[1][j];
  r.t[0] = a.R[0][0] * dt0 + a.R[1][0] * dt1;
  r.t[1] = a.R[0][1] * dt0 + a.R[1][1] * dt1;
  r.c = r.R[0][0];
  r.s = r.R[1][0];
  return r;
}
__device__ __forceinline__ SE2 se2_mul(const SE2& a, const SE2& b) {
  SE2 r;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j) r.R[i][j] = a.R[i][0] * b.R[0][j] + a.R[i][1] * b.R[1][j];
    r.t[i] = a.R[i][0] * b.t[0] + a.R[i][1] * b.t[1] + a.t[i];
  }
  r.c = r.R[0][0];
  r.s = r.R[1][0];
  return r;
}
// V(w) = [[A, -wB], [wB, A]];  Exp = [R(w) | V rho];  Log: w = atan2(R10, R00), rho = V^-1 t
__device__ __forceinline__ void se2_log(const SE2& T, double* xi) {
  double w = atan2(T.R[1][0], T.R[0][0]);
  Coef k = coefs(fabs(w));
  double a = k.A, bb = w * k.B;
  double det = a * a + bb * bb;
  xi[0] = (a * T.t[0] + bb * T.t[1]) / det;
  xi[1] = (-bb * T.t[0] + a * T.t[1]) / det;
  xi[2] = w;
}
__device__ __forceinline__ SE2 se2_exp(const double* xi) {
  double w = xi[2];
  Coef k = coefs(fabs(w));
  double s, c;
  sincos(w, &s, &c);
  SE2 T;
  T.R[0][0] = c; T.R[0][1] = -s;
  T.R[1][0] = s; T.R[1][1] = c;
  double a = k.A, bb = w * k.B;
  T.t[0] = a * xi[0] - bb * xi[1];
  T.t[1] = bb * xi[0] + a * xi[1];
  T.c = c;
  T.s = s;
  return T;
}
// Jr(xi) = [[A, wB, wC r1 - B r2], [-wB, A, B r1 + wC r2], [0, 0, 1]];  Jr^-1 = [[M^-1, -M^-1 v], [0, 1]]
__device__ __forceinline__ void se2_jr_inv(const double* xi, double J[3][3]) {
  double r1 = xi[0], r2 = xi[1], w = xi[2];
  Coef k = coefs(fabs(w));
  double a = k.A, bb = w * k.B;
  double v0 = w * k.C * r1 - k.B * r2;
  double v1 = k.B * r1 + w * k.C * r2;
  double det = a * a + bb * bb;            // M = [[a, bb], [-bb, a]]
  double m00 = a / det, m01 = -bb / det, m10 = bb / det, m11 = a / det;
  J[0][0] = m00; J[0][1] = m01; J[0][2] = -(m00 * v0 + m01 * v1);
  J[1][0] = m10; J[1][1] = m11; J[1][2] = -(m10 * v0 + m11 * v1);
  J[2][0] = 0.0; J[2][1] = 0.0; J[2][2] = 1.0;
}

}  // namespace dev
}  // namespace dnls
