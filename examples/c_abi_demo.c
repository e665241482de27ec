/*
 * c_abi_demo.c — the library used from plain C (no Python, no torch): FK of a 2-link planar
 * arm's configurations, a packed two-support model and the proxy collision check
 * (include/fastron.h). Prints one line per query: "score label".
 *
 *   gcc -O2 -Iinclude -I/usr/local/cuda/include examples/c_abi_demo.c \
 *       -Lpaper_1910_06451_b200 -lfastron_b200 -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1910_06451_b200 -o build/c_abi_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "fastron.h"

#define CHECK(call)                                                                 \
  do {                                                                              \
    fastron_status s_ = (call);                                                     \
    if (s_ != FASTRON_OK) {                                                         \
      fprintf(stderr, "%s failed (%d): %s\n", #call, (int)s_, fastron_last_error()); \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

int main(void) {
  /* planar 2-link arm, a1 = a2 = 1: control points at both joint origins */
  fastron_robot robot;
  memset(&robot, 0, sizeof(robot));
  robot.dof = 2;
  robot.n_cp = 2;
  for (int i = 0; i < 2; ++i) robot.dh[i][2] = 1.0f; /* theta_off, d, a, alpha */
  robot.base[0][0] = robot.base[1][1] = robot.base[2][2] = 1.0f;
  robot.cp_frame[0] = 1;
  robot.cp_frame[1] = 2;

  /* supports x' = (pi, 0) with alpha = 2 and x = (0, 0) with alpha = -1; queries (0,0), (pi,0), (pi/2,pi/2) */
  const float sup[4] = {(float)M_PI, 0.f, 0.f, 0.f};
  const float alpha[2] = {2.f, -1.f};
  const float q[6] = {0.f, 0.f, (float)M_PI, 0.f, (float)(M_PI / 2), (float)(M_PI / 2)};
  const int64_t ns = 2, nq = 3;
  const fastron_kernel k = {FASTRON_RBF_GAUSSIAN, 0.6931471805599453f}; /* gamma = ln 2 */

  float *d_sup, *d_alpha, *d_q, *d_spos, *d_qpos, *d_score;
  int8_t* d_label;
  void *d_model, *d_ws;
  cudaMalloc((void**)&d_sup, sizeof(sup));
  cudaMalloc((void**)&d_alpha, sizeof(alpha));
  cudaMalloc((void**)&d_q, sizeof(q));
  cudaMalloc((void**)&d_spos, 4 * sizeof(float) * robot.n_cp * ns);
  cudaMalloc((void**)&d_qpos, 4 * sizeof(float) * robot.n_cp * nq);
  cudaMalloc((void**)&d_score, sizeof(float) * nq);
  cudaMalloc((void**)&d_label, nq);
  cudaMemcpy(d_sup, sup, sizeof(sup), cudaMemcpyHostToDevice);
  cudaMemcpy(d_alpha, alpha, sizeof(alpha), cudaMemcpyHostToDevice);
  cudaMemcpy(d_q, q, sizeof(q), cudaMemcpyHostToDevice);

  const size_t model_bytes = fastron_model_bytes(ns, robot.n_cp);
  const size_t ws_bytes = fastron_score_packed_workspace_bytes(nq, ns, robot.n_cp);
  cudaMalloc(&d_model, model_bytes);
  cudaMalloc(&d_ws, ws_bytes > 256 ? ws_bytes : 256);

  CHECK(fastron_fk(&robot, d_sup, ns, 2, d_spos, ns, NULL));                    /* Eq. 1-2 */
  CHECK(fastron_model_pack(d_spos, d_alpha, ns, ns, robot.n_cp, k, d_model, model_bytes, NULL));
  CHECK(fastron_fk(&robot, d_q, nq, 2, d_qpos, nq, NULL));
  CHECK(fastron_score_packed(d_qpos, nq, nq, d_model, ns, robot.n_cp, k, d_score, d_label, d_ws,
                             ws_bytes > 256 ? ws_bytes : 256, NULL));
  /* an invalid argument is reported, not crashed on */
  if (fastron_fk(&robot, d_q, -1, 2, d_qpos, nq, NULL) != FASTRON_ERR_INVALID_ARG) return 2;

  float score[3];
  int8_t label[3];
  cudaMemcpy(score, d_score, sizeof(score), cudaMemcpyDeviceToHost);
  cudaMemcpy(label, d_label, sizeof(label), cudaMemcpyDeviceToHost);
  for (int i = 0; i < nq; ++i) printf("%.9g %d\n", score[i], (int)label[i]);
  printf("%s\n", fastron_version());
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 3;
}
