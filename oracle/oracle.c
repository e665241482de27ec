/*
 * oracle.c — plain, slow, obviously-correct fp64 CPU reference for the Fastron FK
 * hot path (arXiv 1910.06451, "Forward Kinematics Kernel for Improved Proxy
 * Collision Checking").
 *
 * *** TEST INFRASTRUCTURE ONLY. ***
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library. The product path
 * (paper_1910_06451_b200/) never links, imports or calls it, and this file
 * shares no code, header, table or constant with the CUDA path.
 *
 * Every quantity is computed in double from the exact fp32 inputs promoted to
 * double. Each function cites the passage of /root/reference/PAPER.md it
 * restates (PAPER.md:<line> (§, Eq./Alg.)). Where the paper is silent the
 * reading is the one listed in DESIGN.md §"Readings" (R-numbers below).
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"):
 *   oracle_dh_transform  — DH-definition product Rz*Tz*Tx*Rx; SPEC.md:63-65 examples
 *   oracle_fk            — planar 2-link closed form; elbow-manipulator closed form;
 *                          link-length invariant
 *   oracle_kernel_value  — k(q,q)=1; RQ worked values SPEC.md:130-131; Gaussian
 *                          gamma=ln2,d2=1 -> 0.5; hand-computed planar values
 *   oracle_score         — brute force on tiny inputs (hand values), linearity
 *   oracle_gram          — symmetry, diag 1, PD (Claim 1), summand decomposition
 *   oracle_train         — hand-derived 2-point traces (tests/golden/), Claim 2
 *                          loss decrease, sign constraint, F = K alpha audit
 *   oracle_edge          — a=b and endpoint cases; OR of per-point scores
 *   oracle_*_joint       — RQ worked values on 7-D vectors; Fig. 2 equality; PD Gram
 * No function here is "parity unpinned".
 *
 * Build (also done by __graft_entry__.build()):
 *   gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC oracle/oracle.c -o oracle/liboracle.so -lm
 * -ffp-contract=off keeps every multiply and add separately rounded, so the
 * Algorithm-1 arithmetic (Eq. 6-8) is the textbook one the trace-exact test
 * relies on (R13).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_GAUSSIAN 0 /* exp(-gamma d^2): BASELINE.json north_star (R1) */
#define ORACLE_RQ 1       /* (1 + gamma/2 d^2)^-2: PAPER.md:115-117 (Eq. 3)           */

/* ------------------------------------------------------------------------ */
/* 4x4 homogeneous matrices, row-major, generic product.                    */
/* ------------------------------------------------------------------------ */

static void mat4_mul(const double A[16], const double B[16], double C[16]) {
  double tmp[16];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      double s = 0.0;
      for (int k = 0; k < 4; ++k) s += A[4 * r + k] * B[4 * k + c];
      tmp[4 * r + c] = s;
    }
  memcpy(C, tmp, sizeof(tmp));
}

static void mat4_identity(double A[16]) {
  memset(A, 0, 16 * sizeof(double));
  A[0] = A[5] = A[10] = A[15] = 1.0;
}

/*
 * Eq. 1, PAPER.md:88-96 (§II-A): the standard D-H link transform
 *   [ c(th)  -c(al)s(th)   s(al)s(th)  a c(th) ]
 *   [ s(th)   c(al)c(th)  -s(al)c(th)  a s(th) ]
 *   [   0       s(al)        c(al)        d    ]
 *   [   0         0            0          1    ]
 * The matrix is authoritative over the prose of PAPER.md:97, which swaps the
 * axes of d and a (R5).
 */
void oracle_dh_transform(double theta, double d, double a, double alpha, double out[16]) {
  double ct = cos(theta), st = sin(theta), ca = cos(alpha), sa = sin(alpha);
  out[0] = ct;   out[1] = -ca * st; out[2] = sa * st;  out[3] = a * ct;
  out[4] = st;   out[5] = ca * ct;  out[6] = -sa * ct; out[7] = a * st;
  out[8] = 0.0;  out[9] = sa;       out[10] = ca;      out[11] = d;
  out[12] = 0.0; out[13] = 0.0;     out[14] = 0.0;     out[15] = 1.0;
}

/*
 * Joint poses wA_0 .. wA_D for one configuration, PAPER.md:99:
 *   wA_i = wA_0 0A_1 ... (i-1)A_i,  theta_i = q_i + theta_offset_i (R6).
 * dh: dof rows of (theta_offset, d, a, alpha). base: 3x4 row-major affine of wA_0.
 * poses: (dof+1) x 16.
 */
static void joint_poses_d(int dof, const double* dh, const double* base, const double* q, double* poses) {
  double T[16];
  mat4_identity(T);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 4; ++c) T[4 * r + c] = base[4 * r + c];
  memcpy(poses, T, sizeof(T));
  for (int i = 0; i < dof; ++i) {
    double A[16];
    double theta = q[i] + dh[4 * i + 0];
    oracle_dh_transform(theta, dh[4 * i + 1], dh[4 * i + 2], dh[4 * i + 3], A);
    mat4_mul(T, A, T);
    memcpy(poses + 16 * (i + 1), T, sizeof(T));
  }
}

void oracle_joint_poses(int dof, const double* dh, const double* base, const float* q, double* poses) {
  double qd[16];
  for (int i = 0; i < dof; ++i) qd[i] = (double)q[i];
  joint_poses_d(dof, dh, base, qd, poses);
}

/* pos(wA_{j_m} T_m) for every control point, from precomputed joint poses. */
static void control_points(int n_cp, const int* cp_frame, const double* cp_offset, const double* poses, double* u) {
  for (int m = 0; m < n_cp; ++m) {
    double Tm[16], P[16];
    mat4_identity(Tm);
    Tm[3] = cp_offset[3 * m + 0];
    Tm[7] = cp_offset[3 * m + 1];
    Tm[11] = cp_offset[3 * m + 2];
    mat4_mul(poses + 16 * cp_frame[m], Tm, P);
    /* pos(.) = first three elements of the last column */
    u[3 * m + 0] = P[3];
    u[3 * m + 1] = P[7];
    u[3 * m + 2] = P[11];
  }
}

/*
 * Eq. 2: FK_m(x) = pos(wA_{j_m} T_m), T_m a static transform
 * (here a pure translation cp_offset[m]; T_m = I when the offset is 0).
 * cp_frame[m] in [0, dof] (0 = base frame wA_0).
 * q: n x ldq fp32 configurations; pos: n x M x 3 doubles.
 */
void oracle_fk(int dof, const double* dh, const double* base, int n_cp, const int* cp_frame,
               const double* cp_offset, const float* q, int64_t n, int64_t ldq, double* pos) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < n; ++k) {
    double poses[17 * 16];
    oracle_joint_poses(dof, dh, base, q + k * ldq, poses);
    control_points(n_cp, cp_frame, cp_offset, poses, pos + k * n_cp * 3);
  }
}

/* ------------------------------------------------------------------------ */
/* Kernels                                                                  */
/* ------------------------------------------------------------------------ */

/* One RBF term of squared distance d2.
 * RQ, Eq. 3: (1 + gamma/2 * d2)^-2.
 * Gaussian (north_star, R1/R2): exp(-gamma * d2). */
double oracle_rbf_term(int kind, double gamma, double d2) {
  if (kind == ORACLE_RQ) return pow(1.0 + 0.5 * gamma * d2, -2.0);
  return exp(-gamma * d2);
}

/* Eq. 4: K_FK(x,x') = (1/M) sum_m K_RBF(FK_m(x), FK_m(x')).
 * u, v: M x 3 control-point positions of the two configurations. */
double oracle_kernel_value(int kind, double gamma, int n_cp, const double* u, const double* v) {
  double s = 0.0;
  for (int m = 0; m < n_cp; ++m) {
    double dx = u[3 * m + 0] - v[3 * m + 0];
    double dy = u[3 * m + 1] - v[3 * m + 1];
    double dz = u[3 * m + 2] - v[3 * m + 2];
    s += oracle_rbf_term(kind, gamma, dx * dx + dy * dy + dz * dz);
  }
  return s / (double)n_cp;
}

/* Fastron model: f(x) = sum_i K(X_i, x) alpha_i, summed in double.
 * qpos: nq x M x 3, spos: ns x M x 3, alpha: ns. f: nq. label: nq (+1 iff f > 0, R8). */
void oracle_score(int kind, double gamma, int n_cp, const double* qpos, int64_t nq, const double* spos,
                  const double* alpha, int64_t ns, double* f, int8_t* label) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < nq; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < ns; ++i)
      acc += oracle_kernel_value(kind, gamma, n_cp, spos + i * n_cp * 3, qpos + j * n_cp * 3) * alpha[i];
    f[j] = acc;
    if (label) label[j] = acc > 0.0 ? 1 : -1;
  }
}

/* Kernel matrix: K_ij = K(X_i, X_j), dense double loop. K: n x n. */
void oracle_gram(int kind, double gamma, int n_cp, const double* pos, int64_t n, double* K) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j)
      K[i * n + j] = oracle_kernel_value(kind, gamma, n_cp, pos + i * n_cp * 3, pos + j * n_cp * 3);
}

/* Joint-space RBF kernel of the "Fastron RBF" baseline (Table I):
 * K(x, x') = term(||x - x'||^2) on the raw D-dimensional joint vectors (fp32 inputs). */
double oracle_joint_kernel(int kind, double gamma, int dof, const float* x, const float* xp) {
  double d2 = 0.0;
  for (int i = 0; i < dof; ++i) {
    double d = (double)x[i] - (double)xp[i];
    d2 += d * d;
  }
  return oracle_rbf_term(kind, gamma, d2);
}

/* f(x) = sum_i K(S_i, x) alpha_i with the joint-space kernel. */
void oracle_score_joint(int kind, double gamma, int dof, const float* q, int64_t nq, int64_t ldq, const float* s,
                        int64_t ns, int64_t lds, const double* alpha, double* f, int8_t* label) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < nq; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < ns; ++i) acc += oracle_joint_kernel(kind, gamma, dof, s + i * lds, q + j * ldq) * alpha[i];
    f[j] = acc;
    if (label) label[j] = acc > 0.0 ? 1 : -1;
  }
}

void oracle_gram_joint(int kind, double gamma, int dof, const float* x, int64_t n, int64_t ldx, double* K) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) K[i * n + j] = oracle_joint_kernel(kind, gamma, dof, x + i * ldx, x + j * ldx);
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1, literally.                               */
/* ------------------------------------------------------------------------ */

/* Loss, Eq. 5: L = 1/2 a^T K a - y^T B a, b_i = beta^(0.5 (y_i + 1)). */
double oracle_loss(const double* K, int64_t n, const int8_t* y, double beta, const double* alpha) {
  double quad = 0.0, lin = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double row = 0.0;
    for (int64_t j = 0; j < n; ++j) row += K[i * n + j] * alpha[j];
    quad += alpha[i] * row;
    double b = pow(beta, 0.5 * ((double)y[i] + 1.0));
    lin += (double)y[i] * b * alpha[i];
  }
  return 0.5 * quad - lin;
}

/*
 * Algorithm 1, "Fastron Model Update Algorithm", with Eq. 6-9
 * (PAPER.md:191-201). Readings: R9 lowest index wins ties; R10 one
 * add/adjust/remove = one iteration, the break does not count; misclassification
 * test `min yF <= 0`; removal test strict `> 0`.
 *
 * K: n x n (row i = column i, K symmetric). alpha, F: in/out (loadPreviousModel,
 * zeros = cold start). trace (nullable, iter_max entries): i for an
 * add/adjust of index i, -(i+1) for a removal. loss_trace (nullable, iter_max+1):
 * L(alpha) before the first step and after every step (O(n^2) each; small n only).
 * support_idx (nullable, n): ascending indices with alpha != 0
 * (removeNonsupportPoints). out[5] = {iterations, n_add, n_remove,
 * converged (min yF > 0 at exit), n_support}.
 */
void oracle_train(const double* K, int64_t n, const int8_t* y, double beta, int64_t iter_max, int64_t s_max,
                  double* alpha, double* F, int32_t* trace, double* loss_trace, int32_t* support_idx,
                  int64_t out[5]) {
  int64_t iters = 0, n_add = 0, n_remove = 0;
  if (loss_trace) loss_trace[0] = oracle_loss(K, n, y, beta, alpha);
  for (int64_t iter = 1; iter <= iter_max; ++iter) {
    /* Check for misclassifications: i = argmin_j y_j F_j (Eq. 9), lowest index on ties. */
    int64_t imin = -1;
    double mmin = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double m = (double)y[j] * F[j];
      if (imin < 0 || m < mmin) { imin = j; mmin = m; }
    }
    if (n > 0 && mmin <= 0.0) {
      int64_t i = imin;
      /* computeKernelMatrixColumn(i): K is given in full here. */
      int64_t nnz = 0;
      for (int64_t j = 0; j < n; ++j) nnz += (alpha[j] != 0.0);
      if (nnz < s_max || alpha[i] != 0.0) {
        double b = pow(beta, 0.5 * ((double)y[i] + 1.0));
        double delta = b * (double)y[i] - F[i];                       /* Eq. 6 */
        alpha[i] = alpha[i] + delta;                                  /* Eq. 7 */
        for (int64_t j = 0; j < n; ++j) F[j] = F[j] + delta * K[i * n + j]; /* Eq. 8 */
        if (trace) trace[iters] = (int32_t)i;
        ++iters; ++n_add;
        if (loss_trace) loss_trace[iters] = oracle_loss(K, n, y, beta, alpha);
        continue;
      }
    }
    /* Remove redundant support points: argmax y(F - alpha) s.t. alpha != 0. */
    int64_t imax = -1;
    double rmax = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      if (alpha[j] == 0.0) continue;
      double r = (double)y[j] * (F[j] - alpha[j]);
      if (imax < 0 || r > rmax) { imax = j; rmax = r; }
    }
    if (imax >= 0 && rmax > 0.0) {
      int64_t i = imax;
      double a = alpha[i];
      for (int64_t j = 0; j < n; ++j) F[j] = F[j] - a * K[i * n + j];
      alpha[i] = 0.0;
      if (trace) trace[iters] = (int32_t)(-(i + 1));
      ++iters; ++n_remove;
      if (loss_trace) loss_trace[iters] = oracle_loss(K, n, y, beta, alpha);
      continue;
    }
    break;
  }
  double mmin = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    double m = (double)y[j] * F[j];
    if (j == 0 || m < mmin) mmin = m;
  }
  int64_t ns = 0;
  for (int64_t j = 0; j < n; ++j)
    if (alpha[j] != 0.0) {
      if (support_idx) support_idx[ns] = (int32_t)j;
      ++ns;
    }
  out[0] = iters;
  out[1] = n_add;
  out[2] = n_remove;
  out[3] = (n > 0 && mmin > 0.0) ? 1 : 0;
  out[4] = ns;
}

/* ------------------------------------------------------------------------ */
/* Discrete edge check (BASELINE.json cfg4; R11). */
/* ------------------------------------------------------------------------ */

/*
 * For each edge e and k = 0..n_interp-1: q_k = qa + (k/(n_interp-1)) (qb - qa) in
 * double (t = 0 when n_interp == 1), FK (Eq. 1-2), score f(q_k).
 * in_collision[e] = OR_k (f(q_k) > 0); fmax[e] = max_k f(q_k); f_all (nullable)
 * = all n_edges x n_interp scores. No early exit. spos: ns x M x 3 (double).
 */
void oracle_edge(int dof, const double* dh, const double* base, int n_cp, const int* cp_frame,
                 const double* cp_offset, const float* qa, const float* qb, int64_t n_edges, int n_interp,
                 int kind, double gamma, const double* spos, const double* alpha, int64_t ns,
                 uint8_t* in_collision, double* fmax, double* f_all) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t e = 0; e < n_edges; ++e) {
    double best = -INFINITY;
    int hit = 0;
    double poses[17 * 16];
    double* u = (double*)malloc(sizeof(double) * 3 * (size_t)n_cp);
    for (int k = 0; k < n_interp; ++k) {
      double t = n_interp > 1 ? (double)k / (double)(n_interp - 1) : 0.0;
      /* joint-space linear interpolation in double, then Eq. 1-2 as in oracle_fk */
      double qd[16];
      for (int i = 0; i < dof; ++i) {
        double a = (double)qa[e * dof + i], b = (double)qb[e * dof + i];
        qd[i] = a + t * (b - a);
      }
      joint_poses_d(dof, dh, base, qd, poses);
      control_points(n_cp, cp_frame, cp_offset, poses, u);
      double f = 0.0;
      for (int64_t i = 0; i < ns; ++i) f += oracle_kernel_value(kind, gamma, n_cp, spos + i * n_cp * 3, u) * alpha[i];
      if (f_all) f_all[e * n_interp + k] = f;
      if (f > best) best = f;
      if (f > 0.0) hit = 1;
    }
    free(u);
    in_collision[e] = (uint8_t)hit;
    if (fmax) fmax[e] = best;
  }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of the OpenMP loops (timing only: the per-element arithmetic and its order
 * do not depend on it). */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  omp_set_num_threads(n > 0 ? n : 1);
#else
  (void)n;
#endif
}
