// fk_device.cuh — batched standard-DH forward kinematics (Eq. 1-2)
// as a per-thread register chain, shared by the FK kernel (K1) and the fused edge
// prologue (K4).
//
// One configuration per thread. The chain wA_i = wA_0 0A_1 ... (i-1)A_i
// is carried as three rotation columns + the origin in fp64 registers; each joint
// applies Eq. 1 in structured form:
//   c0' = c(th) c0 + s(th) c1              (x axis of frame i)
//   v   = -s(th) c0 + c(th) c1
//   c1' = c(al) v + s(al) c2,   c2' = -s(al) v + c(al) c2
//   p'  = p + a c0' + d c2                 (the last column of Eq. 1, rotated)
// which is Eq. 1's 3x3 block and translation multiplied out. Control point m on
// frame j_m is pos(wA_{j_m} T_m) = p_{j_m} + R_{j_m} t_m (Eq. 2). fp64 keeps the
// position error at the final fp32 rounding (DESIGN.md §5 error budget).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fastron {

struct FkParams {
  int32_t dof;
  int32_t n_cp;
  double theta_off[16];
  double d[16];
  double a[16];
  double ca[16];  // cos(alpha_i), computed on the host in double from the fp32 alpha
  double sa[16];  // sin(alpha_i)
  double base_c[3][3];  // columns of the base rotation
  double base_p[3];
  int32_t frame_begin[18];  // control points of frame j (0..16): frame_list[frame_begin[j] .. frame_begin[j+1])
  int32_t frame_list[32];
  double cp_off[32][3];  // t_m, indexed by m
};

// Runs the chain for one configuration; q(j) returns joint value j (double);
// emit(m, x, y, z) receives every control point once (in frame order).
template <class QFun, class Emit>
__device__ __forceinline__ void fk_chain(const FkParams& P, QFun q, Emit emit) {
  double c0x = P.base_c[0][0], c0y = P.base_c[0][1], c0z = P.base_c[0][2];
  double c1x = P.base_c[1][0], c1y = P.base_c[1][1], c1z = P.base_c[1][2];
  double c2x = P.base_c[2][0], c2y = P.base_c[2][1], c2z = P.base_c[2][2];
  double px = P.base_p[0], py = P.base_p[1], pz = P.base_p[2];
  auto emit_frame = [&](int j) {
    for (int idx = P.frame_begin[j]; idx < P.frame_begin[j + 1]; ++idx) {
      const int m = P.frame_list[idx];
      const double tx = P.cp_off[m][0], ty = P.cp_off[m][1], tz = P.cp_off[m][2];
      emit(m, px + c0x * tx + c1x * ty + c2x * tz, py + c0y * tx + c1y * ty + c2y * tz,
           pz + c0z * tx + c1z * ty + c2z * tz);
    }
  };
  emit_frame(0);
#pragma unroll 1
  for (int j = 0; j < P.dof; ++j) {
    double s, c;
    sincos(q(j) + P.theta_off[j], &s, &c);
    const double ca = P.ca[j], sa = P.sa[j], a = P.a[j], d = P.d[j];
    const double n0x = c * c0x + s * c1x, n0y = c * c0y + s * c1y, n0z = c * c0z + s * c1z;
    const double vx = c * c1x - s * c0x, vy = c * c1y - s * c0y, vz = c * c1z - s * c0z;
    px += a * n0x + d * c2x;
    py += a * n0y + d * c2y;
    pz += a * n0z + d * c2z;
    const double n1x = ca * vx + sa * c2x, n1y = ca * vy + sa * c2y, n1z = ca * vz + sa * c2z;
    const double n2x = ca * c2x - sa * vx, n2y = ca * c2y - sa * vy, n2z = ca * c2z - sa * vz;
    c0x = n0x; c0y = n0y; c0z = n0z;
    c1x = n1x; c1y = n1y; c1z = n1z;
    c2x = n2x; c2y = n2y; c2z = n2z;
    emit_frame(j + 1);
  }
}

// The same chain for NC configurations per thread: the per-joint parameters and the
// frame table are read once for all NC, and the NC chains give the scheduler independent
// fp64 work. Each configuration's arithmetic is fk_chain's, expression for expression,
// so its positions are the same bits. q(c, j): joint j of configuration c;
// emit(c, m, x, y, z).
template <int NC, class QFun, class Emit>
__device__ __forceinline__ void fk_chain_multi(const FkParams& P, QFun q, Emit emit) {
  double c0x[NC], c0y[NC], c0z[NC], c1x[NC], c1y[NC], c1z[NC], c2x[NC], c2y[NC], c2z[NC], px[NC], py[NC], pz[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    c0x[c] = P.base_c[0][0]; c0y[c] = P.base_c[0][1]; c0z[c] = P.base_c[0][2];
    c1x[c] = P.base_c[1][0]; c1y[c] = P.base_c[1][1]; c1z[c] = P.base_c[1][2];
    c2x[c] = P.base_c[2][0]; c2y[c] = P.base_c[2][1]; c2z[c] = P.base_c[2][2];
    px[c] = P.base_p[0]; py[c] = P.base_p[1]; pz[c] = P.base_p[2];
  }
  auto emit_frame = [&](int j) {
    for (int idx = P.frame_begin[j]; idx < P.frame_begin[j + 1]; ++idx) {
      const int m = P.frame_list[idx];
      const double tx = P.cp_off[m][0], ty = P.cp_off[m][1], tz = P.cp_off[m][2];
#pragma unroll
      for (int c = 0; c < NC; ++c)
        emit(c, m, px[c] + c0x[c] * tx + c1x[c] * ty + c2x[c] * tz, py[c] + c0y[c] * tx + c1y[c] * ty + c2y[c] * tz,
             pz[c] + c0z[c] * tx + c1z[c] * ty + c2z[c] * tz);
    }
  };
  emit_frame(0);
#pragma unroll 1
  for (int j = 0; j < P.dof; ++j) {
    const double ca = P.ca[j], sa = P.sa[j], a = P.a[j], d = P.d[j], off = P.theta_off[j];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      double s, c;
      sincos(q(k, j) + off, &s, &c);
      const double n0x = c * c0x[k] + s * c1x[k], n0y = c * c0y[k] + s * c1y[k], n0z = c * c0z[k] + s * c1z[k];
      const double vx = c * c1x[k] - s * c0x[k], vy = c * c1y[k] - s * c0y[k], vz = c * c1z[k] - s * c0z[k];
      px[k] += a * n0x + d * c2x[k];
      py[k] += a * n0y + d * c2y[k];
      pz[k] += a * n0z + d * c2z[k];
      const double n1x = ca * vx + sa * c2x[k], n1y = ca * vy + sa * c2y[k], n1z = ca * vz + sa * c2z[k];
      const double n2x = ca * c2x[k] - sa * vx, n2y = ca * c2y[k] - sa * vy, n2z = ca * c2z[k] - sa * vz;
      c0x[k] = n0x; c0y[k] = n0y; c0z[k] = n0z;
      c1x[k] = n1x; c1y[k] = n1y; c1z[k] = n1z;
      c2x[k] = n2x; c2y[k] = n2y; c2z[k] = n2z;
    }
    emit_frame(j + 1);
  }
}

}  // namespace fastron
