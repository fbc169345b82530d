/*
 * utv_oracle.c -- plain, slow, obviously-correct CPU oracle for randUTV + the
 * least-squares solve of arXiv 2408.05238 (Chillaron, Quintana-Orti, Vidal,
 * Martinsson).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (libutv.so) shares no source with this file and never calls it.
 *
 * Conventions: FP64, column-major, 0-based, leading dimensions as in LAPACK.
 * Citations: "P:n" = line n of the paper's LaTeX; "S8c" = the
 * reading of the paper fixed in SURVEY.md section 8(c) and listed in DESIGN.md
 * ("R1".."R18").  Every function follows the paper's algorithm step by step,
 * with plain loops; there is no blocking, fusion or reordering beyond what the
 * cited formula states.
 *
 * Parity status:
 *   philox4x32_10 .......... pinned (Random123 known-answer tests)
 *   gauss .................. pinned (moments; Box-Muller closed form per entry)
 *   hqr .................... pinned (dlarfg closed form [3;4] -> -5; QR = P;
 *                             Q orthogonal; T-factor vs explicit H0..Hb-1)
 *   svd_small .............. pinned (numpy.linalg.svd singular values;
 *                             closed forms diag(3,1), [[0,1],[1,0]])
 *   randutv ................ pinned (A = U T V^T, orthogonality, structure,
 *                             RSVD identity P:848-858)
 *   rank / solve / lstsq ... pinned (pinv brute force on exact-rank inputs,
 *                             numpy.linalg.solve for full rank, known solution)
 *   nullify ................ pinned (T12 == 0, V orthogonal, A = U T V^T kept, and
 *                             x = pinv(U_1 [T11 T12] V^T) b by brute force)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_ARG -1
#define ORACLE_ERR_SHAPE -2
#define ORACLE_ERR_ALLOC -3
#define ORACLE_ERR_NUMERICAL -6

#define IDX(i, j, ld) ((size_t)(i) + (size_t)(j) * (size_t)(ld))

/* ------------------------------------------------------------------------- */
/* Threads: every output element is always reduced by one thread in the same  */
/* order, so results are bit-identical for any thread count.                   */
/* ------------------------------------------------------------------------- */
void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
int oracle_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------- */
/* a1. Random numbers ("generate_iid_stdnorm_matrix";     */
/* the generator itself is unspecified -> reading R6: Philox4x32-10).          */
/* ------------------------------------------------------------------------- */

/* Philox4x32-10 (Salmon et al., SC'11): 10 rounds of
 *   (hi0,lo0) = M0*c0 ; (hi1,lo1) = M1*c2 ;
 *   c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0) ; k += (W0, W1).          */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* (hi, lo) -> u in (0, 1]: u = ((((hi << 32) | lo) >> 11) + 1) * 2^-53.  R6 */
static double u01_from_pair(uint32_t hi, uint32_t lo) {
  uint64_t x = ((uint64_t)hi << 32) | (uint64_t)lo;
  return (double)((x >> 11) + 1) * 0x1.0p-53;
}

/* G (mrows x b), entry (i, c) is the standard normal for global row row0 + i,
 * column c of sketch step `step` (R6):
 *   key = (lo32(seed), hi32(seed)); ctr = (lo32(g), hi32(g), c/2, step)
 *   u1 from (x0, x1), u2 from (x2, x3);
 *   z_even = sqrt(-2 ln u1) cos(2 pi u2), z_odd = sqrt(-2 ln u1) sin(2 pi u2). */
void oracle_gauss(uint64_t seed, int64_t step, int64_t row0, int64_t mrows, int64_t b,
                  double* G, int64_t ldg) {
  const double two_pi = 6.283185307179586476925286766559;
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int64_t i = 0; i < mrows; ++i) {
    uint64_t g = (uint64_t)(row0 + i);
    for (int64_t c = 0; c < b; c += 2) {
      uint32_t ctr[4] = {(uint32_t)g, (uint32_t)(g >> 32), (uint32_t)(c / 2), (uint32_t)step};
      uint32_t x[4];
      oracle_philox4x32_10(ctr, key, x);
      double u1 = u01_from_pair(x[0], x[1]);
      double u2 = u01_from_pair(x[2], x[3]);
      double rad = sqrt(-2.0 * log(u1));
      double ang = two_pi * u2;
      G[IDX(i, c, ldg)] = rad * cos(ang);
      if (c + 1 < b) G[IDX(i, c + 1, ldg)] = rad * sin(ang);
    }
  }
}

/* ------------------------------------------------------------------------- */
/* Plain matrix products (library-primitive role; one thread per output column */
/* and a fixed summation order l = 0..K-1).                                    */
/* ------------------------------------------------------------------------- */

/* C(M x N) = op(A) * op(B), op = transpose if t != 0.  C is overwritten.     */
static void matmul(int ta, int tb, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* C, int64_t ldc) {
  if (ta) {
    /* C[i, j] = sum_{l=0}^{K-1} A[l, i] * op(B)[l, j]: a dot product of two columns */
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < N; ++j)
      for (int64_t i = 0; i < M; ++i) {
        const double* a = A + (size_t)i * lda;
        double acc = 0.0;
        for (int64_t l = 0; l < K; ++l) acc += a[l] * (tb ? B[IDX(j, l, ldb)] : B[IDX(l, j, ldb)]);
        C[IDX(i, j, ldc)] = acc;
      }
    return;
  }
  /* C[:, j] = sum_{l=0}^{K-1} A[:, l] * op(B)[l, j], accumulated in order l = 0..K-1 */
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < N; ++j) {
    double* c = C + (size_t)j * ldc;
    for (int64_t i = 0; i < M; ++i) c[i] = 0.0;
    for (int64_t l = 0; l < K; ++l) {
      double blj = tb ? B[IDX(j, l, ldb)] : B[IDX(l, j, ldb)];
      const double* a = A + (size_t)l * lda;
      for (int64_t i = 0; i < M; ++i) c[i] += a[i] * blj;
    }
  }
}

static double* dalloc(int64_t n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

/* ------------------------------------------------------------------------- */
/* a3 / a5. Householder QR ("unpivoted_QR"; compact WY   */
/* "W unit lower trapezoidal" P:663-666).  Reading R8: LAPACK dlarfg/dlarft.  */
/* In place: R in the upper triangle of P, the Householder vectors (implicit  */
/* unit diagonal) strictly below it.  tau[0:n], T (n x n upper triangular).    */
/* Q = H_0 ... H_{n-1} = I - W T W^T.                                          */
/* ------------------------------------------------------------------------- */
void oracle_hqr(int64_t m, int64_t n, double* P, int64_t ldp, double* tau, double* T, int64_t ldt) {
  int64_t kmax = n < m ? n : m;
  for (int64_t j = 0; j < kmax; ++j) {
    /* dlarfg on x = P[j:m, j] */
    double alpha = P[IDX(j, j, ldp)];
    double xi2 = 0.0;
    for (int64_t i = j + 1; i < m; ++i) xi2 += P[IDX(i, j, ldp)] * P[IDX(i, j, ldp)];
    double xi = sqrt(xi2);
    double tj;
    if (xi == 0.0) {
      tj = 0.0;                         /* H = I, v = e0, R_jj = alpha */
    } else {
      double beta = -copysign(hypot(alpha, xi), alpha);
      tj = (beta - alpha) / beta;
      double scal = 1.0 / (alpha - beta);
      for (int64_t i = j + 1; i < m; ++i) P[IDX(i, j, ldp)] *= scal;
      P[IDX(j, j, ldp)] = beta;
    }
    tau[j] = tj;
    /* apply H_j = I - tau v v^T to P[j:m, j+1:n] from the left */
    if (tj != 0.0) {
#pragma omp parallel for schedule(static)
      for (int64_t l = j + 1; l < n; ++l) {
        double w = P[IDX(j, l, ldp)];   /* v_0 = 1 */
        for (int64_t i = j + 1; i < m; ++i) w += P[IDX(i, j, ldp)] * P[IDX(i, l, ldp)];
        w *= tj;
        P[IDX(j, l, ldp)] -= w;
        for (int64_t i = j + 1; i < m; ++i) P[IDX(i, l, ldp)] -= P[IDX(i, j, ldp)] * w;
      }
    }
  }
  /* dlarft (forward, columnwise): T_jj = tau_j;
     T[0:j, j] = -tau_j * T[0:j, 0:j] * (W[:, 0:j]^T w_j) */
  if (T) {
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) T[IDX(i, j, ldt)] = 0.0;
    double* s = dalloc(n);
    for (int64_t j = 0; j < kmax; ++j) {
      for (int64_t p = 0; p < j; ++p) {
        /* (w_p)^T w_j with w_p[p] = 1, w_p[i<p] = 0, w_j[j] = 1, w_j[i<j] = 0 */
        double acc = P[IDX(j, p, ldp)];      /* row j: w_p[j] * 1 */
        for (int64_t i = j + 1; i < m; ++i) acc += P[IDX(i, p, ldp)] * P[IDX(i, j, ldp)];
        s[p] = acc;
      }
      for (int64_t p = 0; p < j; ++p) {
        double acc = 0.0;
        for (int64_t l = p; l < j; ++l) acc += T[IDX(p, l, ldt)] * s[l];
        T[IDX(p, j, ldt)] = -tau[j] * acc;
      }
      T[IDX(j, j, ldt)] = tau[j];
    }
    free(s);
  }
}

/* Dense W (m x n, unit lower trapezoidal) from the in-place hqr output. */
static void extract_w(int64_t m, int64_t n, const double* P, int64_t ldp, double* W, int64_t ldw) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i)
      W[IDX(i, j, ldw)] = i < j ? 0.0 : (i == j ? 1.0 : P[IDX(i, j, ldp)]);
}

/* ------------------------------------------------------------------------- */
/* a7. Small SVD of the b x b block R ("SVD(A11)"; the method is     */
/* unspecified -> reading R9): one-sided Hestenes Jacobi on W := R^T,          */
/* cyclic-by-rows pair order, skip when |w_i^T w_j| <= sqrt(b) eps ||w_i||     */
/* ||w_j||, w_i^T w_j == 0, or either column is numerically zero (R9b: squared */
/* norm <= eps^2 ||R||_F^2); rotations accumulated into U_s; stop after a      */
/* sweep without rotations (> 30 sweeps = error).  Columns stably sorted by    */
/* norm (descending); (V_s, R') = Householder QR of the sorted W with explicit */
/* Q; signs flipped so R'_jj >= 0; sigma_j = R'_jj.  R ~= U_s diag(s) V_s^T.   */
/* ------------------------------------------------------------------------- */
int oracle_svd_small(int64_t b, const double* R, int64_t ldr, double* Us, int64_t ldu, double* sigma,
                     double* Vs, int64_t ldv, int* sweeps_out) {
  const double eps = 0x1.0p-52; /* DBL_EPSILON */
  const double tol = sqrt((double)b) * eps;
  double* W = dalloc(b * b);
  double* J = dalloc(b * b);
  for (int64_t j = 0; j < b; ++j)
    for (int64_t i = 0; i < b; ++i) {
      W[IDX(i, j, b)] = R[IDX(j, i, ldr)]; /* W = R^T */
      J[IDX(i, j, b)] = i == j ? 1.0 : 0.0;
    }
  /* Reading R9b: a column whose squared norm is <= (eps ||R||_F)^2 is numerically zero and is
     not rotated (an exactly rank-deficient R otherwise regenerates a rounding-noise column
     parallel to a large one on every sweep and never converges). */
  double fro2 = 0.0;
  for (int64_t j = 0; j < b; ++j)
    for (int64_t i = 0; i < b; ++i) fro2 += W[IDX(i, j, b)] * W[IDX(i, j, b)];
  const double small2 = eps * eps * fro2;
  int sweeps = 0, converged = 0;
  while (!converged) {
    if (sweeps >= 30) { free(W); free(J); if (sweeps_out) *sweeps_out = sweeps; return ORACLE_ERR_NUMERICAL; }
    ++sweeps;
    long rotations = 0;
    for (int64_t i = 0; i < b - 1; ++i) {
      for (int64_t j = i + 1; j < b; ++j) {
        double* wi = W + (size_t)i * b;
        double* wj = W + (size_t)j * b;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int64_t r = 0; r < b; ++r) { al += wi[r] * wi[r]; be += wj[r] * wj[r]; ga += wi[r] * wj[r]; }
        if (ga == 0.0 || al <= small2 || be <= small2 || fabs(ga) <= tol * sqrt(al) * sqrt(be)) continue;
        double zeta = (be - al) / (2.0 * ga);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = c * t;
        for (int64_t r = 0; r < b; ++r) {
          double x = wi[r], y = wj[r];
          wi[r] = c * x - s * y;
          wj[r] = s * x + c * y;
        }
        double* ji = J + (size_t)i * b;
        double* jj = J + (size_t)j * b;
        for (int64_t r = 0; r < b; ++r) {
          double x = ji[r], y = jj[r];
          ji[r] = c * x - s * y;
          jj[r] = s * x + c * y;
        }
        ++rotations;
      }
    }
    if (rotations == 0) converged = 1;
  }
  if (sweeps_out) *sweeps_out = sweeps;
  /* stable sort of the columns by ||w|| descending (insertion sort on an index) */
  double* nrm = dalloc(b);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(b > 0 ? b : 1));
  for (int64_t j = 0; j < b; ++j) {
    double s = 0.0;
    for (int64_t r = 0; r < b; ++r) s += W[IDX(r, j, b)] * W[IDX(r, j, b)];
    nrm[j] = sqrt(s);
    perm[j] = j;
  }
  for (int64_t a = 1; a < b; ++a) {
    int64_t p = perm[a];
    int64_t c = a - 1;
    while (c >= 0 && nrm[perm[c]] < nrm[p]) { perm[c + 1] = perm[c]; --c; }
    perm[c + 1] = p;
  }
  double* Ws = dalloc(b * b);
  for (int64_t j = 0; j < b; ++j)
    for (int64_t r = 0; r < b; ++r) {
      Ws[IDX(r, j, b)] = W[IDX(r, perm[j], b)];
      Us[IDX(r, j, ldu)] = J[IDX(r, perm[j], b)];
    }
  /* (V_s, R') := QR(Ws) with explicit Q = (I - Wh T Wh^T) I[:, 0:b] */
  double* tau = dalloc(b);
  double* T = dalloc(b * b);
  oracle_hqr(b, b, Ws, b, tau, T, b);
  double* Wh = dalloc(b * b);
  extract_w(b, b, Ws, b, Wh, b);
  double* TWt = dalloc(b * b);  /* T * Wh^T */
  matmul(0, 1, b, b, b, T, b, Wh, b, TWt, b);
  double* Q = dalloc(b * b);    /* Wh * (T Wh^T) */
  matmul(0, 0, b, b, b, Wh, b, TWt, b, Q, b);
  for (int64_t j = 0; j < b; ++j)
    for (int64_t r = 0; r < b; ++r) Vs[IDX(r, j, ldv)] = (r == j ? 1.0 : 0.0) - Q[IDX(r, j, b)];
  for (int64_t j = 0; j < b; ++j) {
    double d = Ws[IDX(j, j, b)];
    if (d < 0.0) {
      d = -d;
      for (int64_t r = 0; r < b; ++r) Vs[IDX(r, j, ldv)] = -Vs[IDX(r, j, ldv)];
    }
    sigma[j] = d;
  }
  free(W); free(J); free(nrm); free(perm); free(Ws); free(tau); free(T); free(Wh); free(TWt); free(Q);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------- */
/* a1..a7. randUTV (P:467-473 eq:UTVdef; fig:alg_utv), with the     */
/* readings R1 (right update on all rows), R3 (left update Q_U^T), R5 (no      */
/* sketch when n' <= b), R13 (strictly-lower part of T exactly zero) and the   */
/* on-the-fly C := U^T B of v23t.                                */
/* A (m x n, m >= n) is overwritten by T; V (n x n) must be provided; U        */
/* (m x m) and B (m x k) are optional (NULL).                                  */
/* ------------------------------------------------------------------------- */
int oracle_randutv(int64_t m, int64_t n, int64_t k, double* A, int64_t lda, double* V, int64_t ldv,
                   double* U, int64_t ldu, double* B, int64_t ldb, int64_t nb, int32_t q, uint64_t seed,
                   int* max_sweeps_out) {
  if (m < n) return ORACLE_ERR_SHAPE;
  if (nb < 1 || q < 0 || lda < m || ldv < n || (U && ldu < m) || (B && k > 0 && ldb < m)) return ORACLE_ERR_ARG;
  int max_sweeps = 0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) V[IDX(i, j, ldv)] = i == j ? 1.0 : 0.0;
  if (U)
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < m; ++i) U[IDX(i, j, ldu)] = i == j ? 1.0 : 0.0;
  /* scratch, sized for step 0 */
  double* G = dalloc(m * nb);
  double* Y = dalloc(n * nb);
  double* Z = dalloc(m * nb);
  double* Wv = dalloc(n * nb);
  double* Tv = dalloc(nb * nb);
  double* tau = dalloc(nb);
  double* X = dalloc((m > n ? m : n) * nb);
  double* X2 = dalloc((m > n ? m : n) * nb);
  double* Wu = dalloc(m * nb);
  double* Tu = dalloc(nb * nb);
  double* Pm = dalloc(nb * (n > k ? n : k));
  double* P2 = dalloc(nb * (n > k ? n : k));
  double* R = dalloc(nb * nb);
  double* Us = dalloc(nb * nb);
  double* Vs = dalloc(nb * nb);
  double* sig = dalloc(nb);
  double* tmp = dalloc(m * (n > k ? n : k) + nb * nb);
  if (!G || !Y || !Z || !Wv || !Tv || !tau || !X || !X2 || !Wu || !Tu || !Pm || !P2 || !R || !Us || !Vs || !sig || !tmp)
    return ORACLE_ERR_ALLOC;
  int status = ORACLE_OK;

  for (int64_t j0 = 0, step = 0; j0 < n; j0 += nb, ++step) {
    int64_t bw = nb < n - j0 ? nb : n - j0;
    int64_t mp = m - j0, np = n - j0;
    double* Ap = A + IDX(j0, j0, lda);          /* A' = A[j0:m, j0:n] */
    /* ---- apply transformations from the right ---- */
    if (np > nb) {                              /* R5: not the last block */
      oracle_gauss(seed, step, j0, mp, nb, G, mp);                  /* a1 */
      matmul(1, 0, np, nb, mp, Ap, lda, G, mp, Y, np);              /* Y = A'^T G */
      for (int32_t it = 0; it < q; ++it) {                          /* a2, R7 */
        matmul(0, 0, mp, nb, np, Ap, lda, Y, np, Z, mp);            /* Z = A' Y */
        matmul(1, 0, np, nb, mp, Ap, lda, Z, mp, Y, np);            /* Y = A'^T Z */
      }
      oracle_hqr(np, nb, Y, np, tau, Tv, nb);                       /* a3 */
      extract_w(np, nb, Y, np, Wv, np);
      /* a4, R1: A[0:m, j0:n] -= (A[0:m, j0:n] W_V) T_V W_V^T */
      double* Ac = A + IDX(0, j0, lda);
      matmul(0, 0, m, nb, np, Ac, lda, Wv, np, X, m);
      matmul(0, 0, m, nb, nb, X, m, Tv, nb, X2, m);
      matmul(0, 1, m, np, nb, X2, m, Wv, np, tmp, m);
      for (int64_t j = 0; j < np; ++j)
        for (int64_t i = 0; i < m; ++i) Ac[IDX(i, j, lda)] -= tmp[IDX(i, j, m)];
      /* V[0:n, j0:n] -= (V[0:n, j0:n] W_V) T_V W_V^T */
      double* Vc = V + IDX(0, j0, ldv);
      matmul(0, 0, n, nb, np, Vc, ldv, Wv, np, X, n);
      matmul(0, 0, n, nb, nb, X, n, Tv, nb, X2, n);
      matmul(0, 1, n, np, nb, X2, n, Wv, np, tmp, n);
      for (int64_t j = 0; j < np; ++j)
        for (int64_t i = 0; i < n; ++i) Vc[IDX(i, j, ldv)] -= tmp[IDX(i, j, n)];
    }
    /* ---- apply transformations from the left ---- */
    oracle_hqr(mp, bw, Ap, lda, tau, Tu, nb);                       /* a5 */
    extract_w(mp, bw, Ap, lda, Wu, mp);
    for (int64_t j = 0; j < bw; ++j)                                /* R = upper triangle */
      for (int64_t i = 0; i < bw; ++i) R[IDX(i, j, nb)] = i <= j ? Ap[IDX(i, j, lda)] : 0.0;
    /* a6, R3: A[j0:m, j0+bw:n] -= W_U T_U^T (W_U^T A[j0:m, j0+bw:n]) */
    int64_t nr = np - bw;
    if (nr > 0) {
      double* Ar = A + IDX(j0, j0 + bw, lda);
      matmul(1, 0, bw, nr, mp, Wu, mp, Ar, lda, Pm, bw);            /* W_U^T A_r */
      matmul(1, 0, bw, nr, bw, Tu, nb, Pm, bw, P2, bw);             /* T_U^T (...) */
      matmul(0, 0, mp, nr, bw, Wu, mp, P2, bw, tmp, mp);
      for (int64_t j = 0; j < nr; ++j)
        for (int64_t i = 0; i < mp; ++i) Ar[IDX(i, j, lda)] -= tmp[IDX(i, j, mp)];
    }
    if (B && k > 0) {                                               /* C := Q_U^T C (v23t) */
      double* Cr = B + IDX(j0, 0, ldb);
      matmul(1, 0, bw, k, mp, Wu, mp, Cr, ldb, Pm, bw);
      matmul(1, 0, bw, k, bw, Tu, nb, Pm, bw, P2, bw);
      matmul(0, 0, mp, k, bw, Wu, mp, P2, bw, tmp, mp);
      for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < mp; ++i) Cr[IDX(i, j, ldb)] -= tmp[IDX(i, j, mp)];
    }
    if (U) {                                                        /* U[0:m, j0:m] -= (U W_U) T_U W_U^T */
      double* Uc = U + IDX(0, j0, ldu);
      matmul(0, 0, m, bw, mp, Uc, ldu, Wu, mp, X, m);
      matmul(0, 0, m, bw, bw, X, m, Tu, nb, X2, m);
      double* big = dalloc(m * mp);
      if (!big) { status = ORACLE_ERR_ALLOC; break; }
      matmul(0, 1, m, mp, bw, X2, m, Wu, mp, big, m);
      for (int64_t j = 0; j < mp; ++j)
        for (int64_t i = 0; i < m; ++i) Uc[IDX(i, j, ldu)] -= big[IDX(i, j, m)];
      free(big);
    }
    /* R13: zero below the diagonal of the panel, R into A11 */
    for (int64_t j = 0; j < bw; ++j)
      for (int64_t i = j + 1; i < mp; ++i) Ap[IDX(i, j, lda)] = 0.0;
    /* ---- small SVD and the four updates ---- */
    int sw = 0;
    int st = oracle_svd_small(bw, R, nb, Us, nb, sig, Vs, nb, &sw);   /* a7 */
    if (sw > max_sweeps) max_sweeps = sw;
    if (st != ORACLE_OK) { status = st; break; }
    for (int64_t j = 0; j < bw; ++j)
      for (int64_t i = 0; i < bw; ++i) Ap[IDX(i, j, lda)] = i == j ? sig[j] : 0.0;
    if (j0 > 0) {                                                   /* A01 := A01 V_s */
      double* A01 = A + IDX(0, j0, lda);
      matmul(0, 0, j0, bw, bw, A01, lda, Vs, nb, tmp, j0);
      for (int64_t j = 0; j < bw; ++j)
        for (int64_t i = 0; i < j0; ++i) A01[IDX(i, j, lda)] = tmp[IDX(i, j, j0)];
    }
    if (nr > 0) {                                                   /* A12 := U_s^T A12 */
      double* A12 = A + IDX(j0, j0 + bw, lda);
      matmul(1, 0, bw, nr, bw, Us, nb, A12, lda, tmp, bw);
      for (int64_t j = 0; j < nr; ++j)
        for (int64_t i = 0; i < bw; ++i) A12[IDX(i, j, lda)] = tmp[IDX(i, j, bw)];
    }
    {                                                               /* V1 := V1 V_s */
      double* V1 = V + IDX(0, j0, ldv);
      matmul(0, 0, n, bw, bw, V1, ldv, Vs, nb, tmp, n);
      for (int64_t j = 0; j < bw; ++j)
        for (int64_t i = 0; i < n; ++i) V1[IDX(i, j, ldv)] = tmp[IDX(i, j, n)];
    }
    if (B && k > 0) {                                               /* C1 := U_s^T C1 */
      double* C1 = B + IDX(j0, 0, ldb);
      matmul(1, 0, bw, k, bw, Us, nb, C1, ldb, tmp, bw);
      for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < bw; ++i) C1[IDX(i, j, ldb)] = tmp[IDX(i, j, bw)];
    }
    if (U) {                                                        /* U1 := U1 U_s */
      double* U1 = U + IDX(0, j0, ldu);
      matmul(0, 0, m, bw, bw, U1, ldu, Us, nb, tmp, m);
      for (int64_t j = 0; j < bw; ++j)
        for (int64_t i = 0; i < m; ++i) U1[IDX(i, j, ldu)] = tmp[IDX(i, j, m)];
    }
  }
  if (max_sweeps_out) *max_sweeps_out = max_sweeps;
  free(G); free(Y); free(Z); free(Wv); free(Tv); free(tau); free(X); free(X2); free(Wu); free(Tu);
  free(Pm); free(P2); free(R); free(Us); free(Vs); free(sig); free(tmp);
  return status;
}

/* ------------------------------------------------------------------------- */
/* a8. Compute_rank.  Reading R10: relative to the largest */
/* diagonal entry, prefix rule: r = first j with T_jj <= tau * max_l T_ll      */
/* (n if none), r = 0 when max_l T_ll == 0.                                   */
/* ------------------------------------------------------------------------- */
int64_t oracle_rank(int64_t n, const double* T, int64_t ldt, double tau) {
  double dmax = 0.0;
  for (int64_t j = 0; j < n; ++j)
    if (T[IDX(j, j, ldt)] > dmax) dmax = T[IDX(j, j, ldt)];
  if (dmax == 0.0) return 0;
  for (int64_t j = 0; j < n; ++j)
    if (T[IDX(j, j, ldt)] <= tau * dmax) return j;
  return n;
}

/* ------------------------------------------------------------------------- */
/* a9. x_simple = V(:, 1:r) T11^{-1} U_1^T b (eq:simplesoln P:894-901, with   */
/* C = U^T B from the factorization).  z by back substitution, X = V(:,0:r) z. */
/* r == 0 -> X = 0 (R17).                                                      */
/* ------------------------------------------------------------------------- */
void oracle_solve(int64_t n, int64_t r, const double* T, int64_t ldt, const double* V, int64_t ldv,
                  const double* C, int64_t ldc, int64_t k, double* X, int64_t ldx) {
  double* z = dalloc(r > 0 ? r : 1);
  for (int64_t c = 0; c < k; ++c) {
    for (int64_t i = r - 1; i >= 0; --i) {
      double s = C[IDX(i, c, ldc)];
      for (int64_t l = i + 1; l < r; ++l) s -= T[IDX(i, l, ldt)] * z[l];
      z[i] = s / T[IDX(i, i, ldt)];
    }
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t l = 0; l < r; ++l) s += V[IDX(i, l, ldv)] * z[l];
      X[IDX(i, c, ldx)] = s;
    }
  }
  free(z);
}

/* ------------------------------------------------------------------------- */
/* Nullify_top_right_part_of_T (fig:alg_nullify_t12; "conforming to */
/* the xGELSY functions" P:902-907): an RZ sweep from the right that zeroes    */
/* T12 = T(0:r, r:n) and updates V.  Row by row from the bottom (the blocked    */
/* Nullify / Update of the figure, one row per block): for i = r-1 .. 0,       */
/* dlarfg on x = [T(i,i), T(i, r:n)] gives beta, tau, v = [1; z]; the           */
/* reflector H = I - tau v v^T acts on columns (i, r:n) of the rows above       */
/* (Update(C11, D1, C01, D0)) and of V (Update(C11, D1, E1, F)); then           */
/* T(i,i) = beta and T(i, r:n) = 0.  Rows below i already have zeros in T12    */
/* and in column i, so they are unaffected.                                    */
/* ------------------------------------------------------------------------- */
void oracle_nullify(int64_t n, int64_t r, double* T, int64_t ldt, double* V, int64_t ldv) {
  const int64_t nz = n - r;
  if (nz <= 0 || r <= 0) return;
  double* z = dalloc(nz);
  for (int64_t i = r - 1; i >= 0; --i) {
    const double alpha = T[IDX(i, i, ldt)];
    double xi2 = 0.0;
    for (int64_t l = 0; l < nz; ++l) xi2 += T[IDX(i, r + l, ldt)] * T[IDX(i, r + l, ldt)];
    const double xi = sqrt(xi2);
    if (xi == 0.0) continue;                       /* tau = 0: H = I */
    const double beta = -copysign(hypot(alpha, xi), alpha);
    const double tau = (beta - alpha) / beta;
    const double scal = 1.0 / (alpha - beta);
    for (int64_t l = 0; l < nz; ++l) z[l] = T[IDX(i, r + l, ldt)] * scal;
    for (int64_t k = 0; k < i; ++k) {              /* rows above: x_k <- x_k H */
      double w = T[IDX(k, i, ldt)];
      for (int64_t l = 0; l < nz; ++l) w += T[IDX(k, r + l, ldt)] * z[l];
      w *= tau;
      T[IDX(k, i, ldt)] -= w;
      for (int64_t l = 0; l < nz; ++l) T[IDX(k, r + l, ldt)] -= w * z[l];
    }
    if (V) {
      for (int64_t k = 0; k < n; ++k) {            /* V <- V H */
        double w = V[IDX(k, i, ldv)];
        for (int64_t l = 0; l < nz; ++l) w += V[IDX(k, r + l, ldv)] * z[l];
        w *= tau;
        V[IDX(k, i, ldv)] -= w;
        for (int64_t l = 0; l < nz; ++l) V[IDX(k, r + l, ldv)] -= w * z[l];
      }
    }
    T[IDX(i, i, ldt)] = beta;
    for (int64_t l = 0; l < nz; ++l) T[IDX(i, r + l, ldt)] = 0.0;
  }
  free(z);
}

/* ------------------------------------------------------------------------- */
/* Solve_linear_system, fast option (fig:alg_axb P:1075-1108 without the       */
/* Nullify line, "Fast option" P:1114-1121; v24s/v34s).  A and B consumed.    */
/* ------------------------------------------------------------------------- */
int oracle_lstsq_ex(int64_t m, int64_t n, int64_t k, double* A, int64_t lda, double* B, int64_t ldb,
                    double* X, int64_t ldx, int64_t nb, int32_t q, double tau, uint64_t seed, int nullify,
                    int64_t* rank) {
  if (m < n) return ORACLE_ERR_SHAPE;
  if (!(tau >= 0.0 && tau < 1.0) || ldx < n) return ORACLE_ERR_ARG;
  double* V = dalloc(n * n);
  if (!V) return ORACLE_ERR_ALLOC;
  int st = oracle_randutv(m, n, k, A, lda, V, n, NULL, 0, B, ldb, nb, q, seed, NULL);
  if (st != ORACLE_OK) { free(V); return st; }
  int64_t r = oracle_rank(n, A, lda, tau);
  if (nullify) oracle_nullify(n, r, A, lda, V, n);     /* fig:alg_axb line 3 */
  oracle_solve(n, r, A, lda, V, n, B, ldb, k, X, ldx);
  if (rank) *rank = r;
  free(V);
  return ORACLE_OK;
}

int oracle_lstsq(int64_t m, int64_t n, int64_t k, double* A, int64_t lda, double* B, int64_t ldb,
                 double* X, int64_t ldx, int64_t nb, int32_t q, double tau, uint64_t seed, int64_t* rank) {
  return oracle_lstsq_ex(m, n, k, A, lda, B, ldb, X, ldx, nb, q, tau, seed, 0, rank);
}
