/* osc_oracle.c — plain-C restatement of the reference MLMC sample path.
 * TEST INFRASTRUCTURE ONLY: see osc_oracle.h for the contract and citations.
 * Reference paths are relative to /root/reference/proj. */
#include "osc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- RNG: Philox4x32-10 + Box-Muller (src/rng.cpp:10-67) ------------------ */
void oo_philox_block(const uint32_t key[2], const uint32_t ctr_in[4], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) { /* rng.cpp:29-40 */
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static double uniform53(uint32_t hi, uint32_t lo) { /* rng.cpp:22-25 */
  const uint64_t bits = ((uint64_t)hi << 32) | lo;
  return ((double)(bits >> 11) + 0.5) * 0x1p-53;
}

void oo_normals(uint64_t seed, uint32_t level, uint64_t index, double* out, int64_t n) {
  /* key = seed words, counter = (block, level, idx lo, idx hi) (rng.cpp:42-46);
   * one block per two normals: cos first, sin second (rng.cpp:48-63). */
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int64_t j = 0; 2 * j < n; ++j) {
    const uint32_t ctr[4] = {(uint32_t)j, level, (uint32_t)index, (uint32_t)(index >> 32)};
    uint32_t r[4];
    oo_philox_block(key, ctr, r);
    const double u1 = uniform53(r[0], r[1]), u2 = uniform53(r[2], r[3]);
    const double mag = sqrt(-2.0 * log(u1));
    const double ang = 2.0 * 3.14159265358979323846 * u2;
    out[2 * j] = mag * cos(ang);
    if (2 * j + 1 < n) out[2 * j + 1] = mag * sin(ang);
  }
}

/* ---- DFT (src/fft.cpp:20-56): unitary, + sign, real input ------------------ */
typedef struct { int n; double* tw; } dft_plan; /* tw[2t..] = exp(+2 pi i t / n) */

static void dft_plan_init(dft_plan* p, int n) {
  p->n = n;
  p->tw = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  for (int t = 0; t < n; ++t) {
    const long double a = 6.283185307179586476925286766559005768L * (long double)t / n;
    p->tw[2 * t] = (double)cosl(a);
    p->tw[2 * t + 1] = (double)sinl(a);
  }
}

/* In-place unnormalised 1-D DFT with + sign of a contiguous complex line. */
static void dft_line(const dft_plan* p, double* x, double* scratch) {
  const int n = p->n;
  if ((n & (n - 1)) == 0) { /* radix-2 DIT, bit-reversed input */
    for (int i = 1, j = 0; i < n; ++i) {
      int bit = n >> 1;
      for (; j & bit; bit >>= 1) j ^= bit;
      j ^= bit;
      if (i < j) {
        double t0 = x[2 * i], t1 = x[2 * i + 1];
        x[2 * i] = x[2 * j]; x[2 * i + 1] = x[2 * j + 1];
        x[2 * j] = t0; x[2 * j + 1] = t1;
      }
    }
    for (int len = 2; len <= n; len <<= 1) {
      const int half = len >> 1, step = n / len;
      for (int s = 0; s < n; s += len)
        for (int k = 0; k < half; ++k) {
          const double wr = p->tw[2 * k * step], wi = p->tw[2 * k * step + 1];
          double* a = x + 2 * (s + k);
          double* b = x + 2 * (s + k + half);
          const double tr = b[0] * wr - b[1] * wi, ti = b[0] * wi + b[1] * wr;
          b[0] = a[0] - tr; b[1] = a[1] - ti;
          a[0] += tr; a[1] += ti;
        }
    }
    return;
  }
  for (int k = 0; k < n; ++k) { /* direct DFT for other lengths */
    double sr = 0.0, si = 0.0;
    for (int j = 0; j < n; ++j) {
      const int e = (int)(((int64_t)j * k) % n);
      const double wr = p->tw[2 * e], wi = p->tw[2 * e + 1];
      sr += x[2 * j] * wr - x[2 * j + 1] * wi;
      si += x[2 * j] * wi + x[2 * j + 1] * wr;
    }
    scratch[2 * k] = sr; scratch[2 * k + 1] = si;
  }
  memcpy(x, scratch, sizeof(double) * 2 * (size_t)n);
}

/* sample_into (src/embedding.cpp:165-174): w = sqrt(lam) xi; v = F w; u = Re v + Im v */
int oo_sample(int n, const double* sqrt_lam, const double* xi, double* u) {
  const int64_t s = (int64_t)n * n;
  double* buf = (double*)malloc(sizeof(double) * 2 * (size_t)s);
  double* line = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  double* scratch = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  if (!buf || !line || !scratch) { free(buf); free(line); free(scratch); return -1; }
  dft_plan p;
  dft_plan_init(&p, n);
  for (int64_t i = 0; i < s; ++i) { buf[2 * i] = sqrt_lam[i] * xi[i]; buf[2 * i + 1] = 0.0; }
  for (int q1 = 0; q1 < n; ++q1) dft_line(&p, buf + 2 * (int64_t)q1 * n, scratch); /* along x */
  for (int q0 = 0; q0 < n; ++q0) {                                                  /* along y */
    for (int q1 = 0; q1 < n; ++q1) {
      line[2 * q1] = buf[2 * ((int64_t)q1 * n + q0)];
      line[2 * q1 + 1] = buf[2 * ((int64_t)q1 * n + q0) + 1];
    }
    dft_line(&p, line, scratch);
    for (int q1 = 0; q1 < n; ++q1) {
      buf[2 * ((int64_t)q1 * n + q0)] = line[2 * q1];
      buf[2 * ((int64_t)q1 * n + q0) + 1] = line[2 * q1 + 1];
    }
  }
  const double scale = 1.0 / sqrt((double)s); /* fft.cpp:54-55 */
  for (int64_t i = 0; i < s; ++i) u[i] = buf[2 * i] * scale + buf[2 * i + 1] * scale;
  free(p.tw); free(buf); free(line); free(scratch);
  return 0;
}

/* restrict_to (src/embedding.cpp:183-203) */
void oo_restrict(int n, int m, const double* u, int m_t, double* out) {
  const int r = m / m_t;
  for (int p1 = 0; p1 <= m_t; ++p1)
    for (int p0 = 0; p0 <= m_t; ++p0)
      out[(int64_t)p1 * (m_t + 1) + p0] = u[(int64_t)p1 * r * n + (int64_t)p0 * r];
}

/* ---- FEM (src/fem.cpp) ------------------------------------------------------ */
typedef struct { int64_t n; int64_t* row_ptr; int64_t* col; double* val; } csr_t;

static void csr_free(csr_t* A) { free(A->row_ptr); free(A->col); free(A->val); memset(A, 0, sizeof(*A)); }

static void spmv(const csr_t* A, const double* x, double* y) { /* fem.cpp:19-25 */
  for (int64_t i = 0; i < A->n; ++i) {
    double acc = 0.0;
    for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) acc += A->val[k] * x[A->col[k]];
    y[i] = acc;
  }
}

/* fem.cpp:28-30, widened by the DIRICHLET_ALL extension. */
static int is_dir(int bc, int m, int p0, int p1) {
  if (p0 == 0 || p0 == m) return 1;
  return bc == OSC_BC_DIRICHLET_ALL && (p1 == 0 || p1 == m);
}
static double dir_val(int bc, int p0) { return (bc == OSC_BC_FLOWCELL && p0 == 0) ? 1.0 : 0.0; }

static const int OFF0[7] = {-1, 0, -1, 0, 1, 0, 1}; /* fem.cpp:48-49 */
static const int OFF1[7] = {-1, -1, 0, 0, 0, 1, 1};
static int slot_of(int d0, int d1) {
  for (int s = 0; s < 7; ++s) if (OFF0[s] == d0 && OFF1[s] == d1) return s;
  return -1;
}

/* Raw 7-slot stencil + load (fem.cpp:56-97), no Dirichlet handling. */
static void assemble_raw(int m, const double* k, int forcing, double fval, int homogeneous,
                         double* stencil, double* b) {
  const int n0 = m + 1;
  const int64_t n = (int64_t)n0 * n0;
  const double hx = 1.0 / m, hy = 1.0 / m, area = 0.5 * hx * hy;
  memset(stencil, 0, sizeof(double) * 7 * (size_t)n);
  memset(b, 0, sizeof(double) * (size_t)n);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i)
      for (int t = 0; t < 2; ++t) {
        const int lo0[3] = {i, i + 1, i + 1}, lo1[3] = {j, j, j + 1};
        const int up0[3] = {i, i + 1, i}, up1[3] = {j, j + 1, j + 1};
        const int* p0 = t == 0 ? lo0 : up0;
        const int* p1 = t == 0 ? lo1 : up1;
        double xs[3], ys[3], bb[3], cc[3], ke = 0.0;
        int64_t idx[3];
        for (int a = 0; a < 3; ++a) { xs[a] = p0[a] * hx; ys[a] = p1[a] * hy; }
        for (int a = 0; a < 3; ++a) { idx[a] = (int64_t)p1[a] * n0 + p0[a]; ke += k[idx[a]]; }
        ke /= 3.0;
        for (int a = 0; a < 3; ++a) {
          const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
          bb[a] = ys[a1] - ys[a2];
          cc[a] = xs[a2] - xs[a1];
        }
        for (int a = 0; a < 3; ++a) {
          for (int c = 0; c < 3; ++c) {
            const int s = slot_of(p0[c] - p0[a], p1[c] - p1[a]);
            stencil[idx[a] * 7 + s] += ke * (bb[a] * bb[c] + cc[a] * cc[c]) / (4.0 * area);
          }
          if (forcing && !homogeneous) b[idx[a]] += fval * area / 3.0;
        }
      }
}

/* assemble (fem.cpp:38-138): raw stencil, symmetric Dirichlet elimination, CSR. */
static void assemble(int m, const double* k, int bc, int forcing, double fval, int homogeneous,
                     csr_t* A, double* b) {
  const int n0 = m + 1;
  const int64_t n = (int64_t)n0 * n0;
  double* st = (double*)malloc(sizeof(double) * 7 * (size_t)n);
  assemble_raw(m, k, forcing, fval, homogeneous, st, b);
  for (int p1 = 0; p1 <= m; ++p1)
    for (int p0 = 0; p0 <= m; ++p0) {
      const int64_t i = (int64_t)p1 * n0 + p0;
      if (is_dir(bc, m, p0, p1)) {
        for (int s = 0; s < 7; ++s) st[i * 7 + s] = 0.0;
        st[i * 7 + 3] = 1.0;
        b[i] = homogeneous ? 0.0 : dir_val(bc, p0);
        continue;
      }
      for (int s = 0; s < 7; ++s) {
        const int q0 = p0 + OFF0[s], q1 = p1 + OFF1[s];
        if (q0 < 0 || q0 > m || q1 < 0 || q1 > m || !is_dir(bc, m, q0, q1)) continue;
        if (!homogeneous) b[i] -= st[i * 7 + s] * dir_val(bc, q0);
        st[i * 7 + s] = 0.0;
      }
    }
  A->n = n;
  A->row_ptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  A->col = (int64_t*)malloc(sizeof(int64_t) * 7 * (size_t)n);
  A->val = (double*)malloc(sizeof(double) * 7 * (size_t)n);
  int64_t nnz = 0;
  for (int p1 = 0; p1 <= m; ++p1)
    for (int p0 = 0; p0 <= m; ++p0) {
      const int64_t i = (int64_t)p1 * n0 + p0;
      for (int s = 0; s < 7; ++s) {
        const int q0 = p0 + OFF0[s], q1 = p1 + OFF1[s];
        if (q0 < 0 || q0 > m || q1 < 0 || q1 > m) continue;
        const double v = st[i * 7 + s];
        if (v == 0.0 && s != 3) continue;
        A->col[nnz] = i + OFF1[s] * n0 + OFF0[s];
        A->val[nnz] = v;
        ++nnz;
      }
      A->row_ptr[i + 1] = nnz;
    }
  free(st);
}

/* prolong_add (fem.cpp:144-165) */
static void prolong_add(int mf, const double* ec, double* zf) {
  const int nf = mf + 1, nc = mf / 2 + 1;
  for (int J = 0; J <= mf; ++J)
    for (int I = 0; I <= mf; ++I) {
      const int64_t i = (int64_t)J * nf + I;
      const int ex = (I % 2) == 0, ey = (J % 2) == 0;
      if (ex && ey) zf[i] += ec[(J / 2) * nc + I / 2];
      else if (!ex && ey) zf[i] += 0.5 * (ec[(J / 2) * nc + (I - 1) / 2] + ec[(J / 2) * nc + (I + 1) / 2]);
      else if (ex && !ey) zf[i] += 0.5 * (ec[((J - 1) / 2) * nc + I / 2] + ec[((J + 1) / 2) * nc + I / 2]);
      else zf[i] += 0.5 * (ec[((J - 1) / 2) * nc + (I - 1) / 2] + ec[((J + 1) / 2) * nc + (I + 1) / 2]);
    }
}

/* restrict_residual (fem.cpp:168-195); coarse Dirichlet zeroing widened per bc. */
static void restrict_residual(int mf, int bc, const double* rf, double* rc) {
  const int nf = mf + 1, mc = mf / 2, nc = mc + 1;
  memset(rc, 0, sizeof(double) * (size_t)nc * nc);
  for (int J = 0; J <= mf; ++J)
    for (int I = 0; I <= mf; ++I) {
      const double v = rf[(int64_t)J * nf + I];
      if (v == 0.0) continue;
      const int ex = (I % 2) == 0, ey = (J % 2) == 0;
      if (ex && ey) rc[(J / 2) * nc + I / 2] += v;
      else if (!ex && ey) {
        rc[(J / 2) * nc + (I - 1) / 2] += 0.5 * v;
        rc[(J / 2) * nc + (I + 1) / 2] += 0.5 * v;
      } else if (ex && !ey) {
        rc[((J - 1) / 2) * nc + I / 2] += 0.5 * v;
        rc[((J + 1) / 2) * nc + I / 2] += 0.5 * v;
      } else {
        rc[((J - 1) / 2) * nc + (I - 1) / 2] += 0.5 * v;
        rc[((J + 1) / 2) * nc + (I + 1) / 2] += 0.5 * v;
      }
    }
  for (int J = 0; J <= mc; ++J)
    for (int I = 0; I <= mc; ++I)
      if (is_dir(bc, mc, I, J)) rc[J * nc + I] = 0.0;
}

/* gauss_seidel (fem.cpp:197-212) */
static void gauss_seidel(const csr_t* A, const double* r, double* z, int backward) {
  for (int64_t ii = 0; ii < A->n; ++ii) {
    const int64_t i = backward ? A->n - 1 - ii : ii;
    double acc = r[i], diag = 1.0;
    for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) {
      if (A->col[k] == i) diag = A->val[k];
      else acc -= A->val[k] * z[A->col[k]];
    }
    z[i] = acc / diag;
  }
}

#define MG_MAX 32
typedef struct {
  int nlev;
  int m[MG_MAX];
  csr_t A[MG_MAX];
  double *r[MG_MAX], *z[MG_MAX], *t[MG_MAX];
  double* chol;
  int bc;
} mg_t;

/* Multigrid ctor (fem.cpp:227-249) + factor_coarsest (fem.cpp:255-272) */
static void mg_init(mg_t* mg, int m, const double* k_nodal, int bc) {
  memset(mg, 0, sizeof(*mg));
  mg->bc = bc;
  int g = m;
  double* k = (double*)malloc(sizeof(double) * (size_t)(m + 1) * (m + 1));
  memcpy(k, k_nodal, sizeof(double) * (size_t)(m + 1) * (m + 1));
  for (;;) {
    const int l = mg->nlev++;
    const int64_t nn = (int64_t)(g + 1) * (g + 1);
    double* dummy = (double*)malloc(sizeof(double) * (size_t)nn);
    mg->m[l] = g;
    assemble(g, k, bc, 0, 0.0, 1, &mg->A[l], dummy);
    free(dummy);
    mg->r[l] = (double*)calloc((size_t)nn, sizeof(double));
    mg->z[l] = (double*)calloc((size_t)nn, sizeof(double));
    mg->t[l] = (double*)calloc((size_t)nn, sizeof(double));
    if (g <= 4 || g % 2 != 0 || mg->nlev == MG_MAX) break;
    const int gc = g / 2;
    double* kc = (double*)malloc(sizeof(double) * (size_t)(gc + 1) * (gc + 1));
    for (int J = 0; J <= gc; ++J)
      for (int I = 0; I <= gc; ++I) kc[J * (gc + 1) + I] = k[(int64_t)(2 * J) * (g + 1) + 2 * I];
    free(k);
    k = kc;
    g = gc;
  }
  free(k);
  const csr_t* A = &mg->A[mg->nlev - 1];
  const int64_t n = A->n;
  mg->chol = (double*)calloc((size_t)(n * n), sizeof(double));
  double* L = mg->chol;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t q = A->row_ptr[i]; q < A->row_ptr[i + 1]; ++q) L[i * n + A->col[q]] = A->val[q];
  for (int64_t j = 0; j < n; ++j) {
    double d = L[j * n + j];
    for (int64_t q = 0; q < j; ++q) d -= L[j * n + q] * L[j * n + q];
    L[j * n + j] = sqrt(d);
    for (int64_t i = j + 1; i < n; ++i) {
      double v = L[i * n + j];
      for (int64_t q = 0; q < j; ++q) v -= L[i * n + q] * L[j * n + q];
      L[i * n + j] = v / L[j * n + j];
    }
  }
}

static void mg_free(mg_t* mg) {
  for (int l = 0; l < mg->nlev; ++l) { csr_free(&mg->A[l]); free(mg->r[l]); free(mg->z[l]); free(mg->t[l]); }
  free(mg->chol);
}

static void solve_coarsest(const mg_t* mg, const double* r, double* z) { /* fem.cpp:274-286 */
  const int64_t n = mg->A[mg->nlev - 1].n;
  const double* L = mg->chol;
  for (int64_t i = 0; i < n; ++i) {
    double v = r[i];
    for (int64_t q = 0; q < i; ++q) v -= L[i * n + q] * z[q];
    z[i] = v / L[i * n + i];
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double v = z[i];
    for (int64_t q = i + 1; q < n; ++q) v -= L[q * n + i] * z[q];
    z[i] = v / L[i * n + i];
  }
}

static void mg_cycle(mg_t* mg, int d, const double* r, double* z) { /* fem.cpp:288-303 */
  if (d + 1 == mg->nlev) { solve_coarsest(mg, r, z); return; }
  const csr_t* A = &mg->A[d];
  memset(z, 0, sizeof(double) * (size_t)A->n);
  gauss_seidel(A, r, z, 0);
  spmv(A, z, mg->t[d]);
  for (int64_t i = 0; i < A->n; ++i) mg->t[d][i] = r[i] - mg->t[d][i];
  restrict_residual(mg->m[d], mg->bc, mg->t[d], mg->r[d + 1]);
  mg_cycle(mg, d + 1, mg->r[d + 1], mg->z[d + 1]);
  prolong_add(mg->m[d], mg->z[d + 1], z);
  gauss_seidel(A, r, z, 1);
}

static double norm2(const double* v, int64_t n) { /* fem.cpp:309-313 */
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

/* assemble_and_solve (fem.cpp:317-400) */
int oo_solve(int m, const double* Z, int bc, int forcing, double fval, double tol,
             int max_iter_factor, int precond, double* u, int* iters, double* hist, int hist_cap,
             int* hist_len) {
  const int n0 = m + 1;
  const int64_t n = (int64_t)n0 * n0;
  int status = 0, hl = 0;
  double* k = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    if (!isfinite(Z[i])) { free(k); return -3; }
    k[i] = exp(Z[i]);
  }
  csr_t A;
  double* b = (double*)malloc(sizeof(double) * (size_t)n);
  assemble(m, k, bc, forcing, fval, 0, &A, b);
  memset(u, 0, sizeof(double) * (size_t)n);
  for (int p1 = 0; p1 <= m; ++p1) { /* Dirichlet lift, fem.cpp:335-339 */
    for (int p0 = 0; p0 <= m; ++p0)
      if (is_dir(bc, m, p0, p1)) u[(int64_t)p1 * n0 + p0] = dir_val(bc, p0);
  }
  mg_t mg;
  double* inv_diag = NULL;
  if (precond) mg_init(&mg, m, k, bc);
  else {
    inv_diag = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t q = A.row_ptr[i]; q < A.row_ptr[i + 1]; ++q)
        if (A.col[q] == i) inv_diag[i] = 1.0 / A.val[q];
  }
  double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n),
         *p = malloc(sizeof(double) * n), *Ap = malloc(sizeof(double) * n);
  spmv(&A, u, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  const double bnorm = norm2(b, n);
  const int64_t max_iter = (int64_t)max_iter_factor * n;
  double last = norm2(r, n) / bnorm;
  if (hist && hl < hist_cap) hist[hl] = last;
  ++hl;
  int64_t iter = 0;
  if (last > tol) {
#define PRECOND(rr, zz) do { if (precond) mg_cycle(&mg, 0, rr, zz); \
      else for (int64_t i_ = 0; i_ < n; ++i_) zz[i_] = inv_diag[i_] * rr[i_]; } while (0)
    PRECOND(r, z);
    memcpy(p, z, sizeof(double) * (size_t)n);
    double rz = 0.0;
    for (int64_t i = 0; i < n; ++i) rz += r[i] * z[i];
    for (;;) {
      if (iter++ >= max_iter) { status = -4; break; }
      spmv(&A, p, Ap);
      double pAp = 0.0;
      for (int64_t i = 0; i < n; ++i) pAp += p[i] * Ap[i];
      const double alpha = rz / pAp;
      for (int64_t i = 0; i < n; ++i) { u[i] += alpha * p[i]; r[i] -= alpha * Ap[i]; }
      last = norm2(r, n) / bnorm;
      if (hist && hl < hist_cap) hist[hl] = last;
      ++hl;
      if (last <= tol) break;
      PRECOND(r, z);
      double rz_new = 0.0;
      for (int64_t i = 0; i < n; ++i) rz_new += r[i] * z[i];
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
#undef PRECOND
  }
  if (iters) *iters = (int)(status == -4 ? iter - 1 : iter);
  if (hist_len) *hist_len = hl;
  if (precond) mg_free(&mg);
  free(inv_diag); free(r); free(z); free(p); free(Ap); free(b); free(k); csr_free(&A);
  return status;
}

/* ---- QoIs (fem.cpp:402-436 + extensions) ------------------------------------ */
static double qoi_point(int m, const double* u, double x, double y) { /* fem.cpp:402-418 */
  const int n0 = m + 1;
  int i = (int)(x * m), j = (int)(y * m);
  if (i > m - 1) i = m - 1;
  if (j > m - 1) j = m - 1;
  const double xi = x * m - i, eta = y * m - j;
  const double ull = u[j * n0 + i], ulr = u[j * n0 + i + 1], uur = u[(j + 1) * n0 + i + 1],
               uul = u[(j + 1) * n0 + i];
  if (eta <= xi) return (1.0 - xi) * ull + (xi - eta) * ulr + eta * uur;
  return (1.0 - eta) * ull + xi * uur + (eta - xi) * uul;
}

static double qoi_tri_sum(int m, const double* u, int l2) { /* fem.cpp:420-436 (+ integral) */
  const int n0 = m + 1;
  const double h = 1.0 / m, area = 0.5 * h * h;
  double acc = 0.0;
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) {
      const int64_t a = (int64_t)j * n0 + i;
      const int64_t tri[2][3] = {{a, a + 1, a + n0 + 1}, {a, a + n0 + 1, a + n0}};
      for (int t = 0; t < 2; ++t) {
        const double ua = u[tri[t][0]], ub = u[tri[t][1]], uc = u[tri[t][2]];
        const double sum = ua + ub + uc;
        if (l2) acc += area / 12.0 * (ua * ua + ub * ub + uc * uc + sum * sum);
        else acc += area * sum / 3.0;
      }
    }
  return l2 ? sqrt(acc) : acc;
}

/* Outflow flux through x = 1 (extension): -sum_{p1} (K_raw u - F)_{(m,p1)} with K_raw the
 * assembled stiffness BEFORE Dirichlet elimination (consistent reaction flux). */
static double qoi_flux(int m, const double* u, const double* Z, int forcing, double fval) {
  const int n0 = m + 1;
  const int64_t n = (int64_t)n0 * n0;
  double* k = (double*)malloc(sizeof(double) * (size_t)n);
  double* st = (double*)malloc(sizeof(double) * 7 * (size_t)n);
  double* F = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) k[i] = exp(Z[i]);
  assemble_raw(m, k, forcing, fval, 0, st, F);
  double flux = 0.0;
  for (int p1 = 0; p1 <= m; ++p1) {
    const int64_t i = (int64_t)p1 * n0 + m;
    double Ku = 0.0;
    for (int s = 0; s < 7; ++s) {
      const int q0 = m + OFF0[s], q1 = p1 + OFF1[s];
      if (q0 < 0 || q0 > m || q1 < 0 || q1 > m) continue;
      Ku += st[i * 7 + s] * u[(int64_t)q1 * n0 + q0];
    }
    flux -= Ku - F[i];
  }
  free(k); free(st); free(F);
  return flux;
}

double oo_qoi(int m, const double* u, int bc, int qoi, double qx, double qy, const double* Z,
              int forcing, double fval) {
  (void)bc;
  switch (qoi) {
    case OSC_QOI_POINT: return qoi_point(m, u, qx, qy);
    case OSC_QOI_L2: return qoi_tri_sum(m, u, 1);
    case OSC_QOI_INTEGRAL: return qoi_tri_sum(m, u, 0);
    default: return qoi_flux(m, u, Z, forcing, fval);
  }
}

/* ---- coupled samples (estimators.cpp:200-237) over pthreads (:32-63) --------- */
typedef struct {
  const oo_level* L;
  int64_t from, lo, hi;
  const double* xi_host;
  double *qf, *qc;
  int *itf, *itc;
  int status;
} job_t;

static void* run_job(void* arg) {
  job_t* jb = (job_t*)arg;
  const oo_level* L = jb->L;
  const int n = L->n, m = L->m;
  const int64_t s = (int64_t)n * n;
  double* xi = (double*)malloc(sizeof(double) * (size_t)s);
  double* u = (double*)malloc(sizeof(double) * (size_t)s);
  double* u2 = (double*)malloc(sizeof(double) * (size_t)s);
  double* Z = (double*)malloc(sizeof(double) * (size_t)(m + 1) * (m + 1));
  double* sol = (double*)malloc(sizeof(double) * (size_t)(m + 1) * (m + 1));
  for (int64_t i = jb->lo; i < jb->hi && jb->status == 0; ++i) {
    const int64_t slot = i - jb->from;
    if (jb->xi_host) memcpy(xi, jb->xi_host + slot * s, sizeof(double) * (size_t)s);
    else oo_normals(L->seed, L->ell, (uint64_t)i, xi, s);
    oo_sample(n, L->sqrt_fine, xi, u);
    oo_restrict(n, m, u, m, Z);
    int it = 0;
    int st = oo_solve(m, Z, L->bc, L->forcing, L->forcing_value, L->tol, L->max_iter_factor,
                      L->precond, sol, &it, NULL, 0, NULL);
    if (st) { jb->status = st; break; }
    jb->qf[slot] = oo_qoi(m, sol, L->bc, L->qoi, L->qx, L->qy, Z, L->forcing, L->forcing_value);
    if (jb->itf) jb->itf[slot] = it;
    if (L->has_coarse) {
      const double* uc = u;
      if (L->sqrt_coarse != L->sqrt_fine) { oo_sample(n, L->sqrt_coarse, xi, u2); uc = u2; }
      const int mc = m / 2;
      oo_restrict(n, m, uc, mc, Z);
      st = oo_solve(mc, Z, L->bc, L->forcing, L->forcing_value, L->tol, L->max_iter_factor,
                    L->precond, sol, &it, NULL, 0, NULL);
      if (st) { jb->status = st; break; }
      jb->qc[slot] = oo_qoi(mc, sol, L->bc, L->qoi, L->qx, L->qy, Z, L->forcing, L->forcing_value);
      if (jb->itc) jb->itc[slot] = it;
    } else if (jb->qc) {
      jb->qc[slot] = 0.0;
    }
  }
  free(xi); free(u); free(u2); free(Z); free(sol);
  return NULL;
}

int oo_coupled(const oo_level* L, int64_t from, int64_t to, const double* xi_host, double* q_fine,
               double* q_coarse, int* it_fine, int* it_coarse) {
  const int64_t count = to - from;
  if (count <= 0) return 0;
  int workers = L->threads > 0 ? L->threads : 1;
  if (workers > count) workers = (int)count;
  job_t* jobs = (job_t*)calloc((size_t)workers, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
  const int64_t chunk = (count + workers - 1) / workers;
  int started = 0;
  for (int w = 0; w < workers; ++w) {
    const int64_t lo = from + w * chunk, hi = lo + chunk < to ? lo + chunk : to;
    if (lo >= hi) break;
    jobs[w] = (job_t){L, from, lo, hi, xi_host, q_fine, q_coarse, it_fine, it_coarse, 0};
    pthread_create(&th[w], NULL, run_job, &jobs[w]);
    ++started;
  }
  int status = 0;
  for (int w = 0; w < started; ++w) {
    pthread_join(th[w], NULL);
    if (!status && jobs[w].status) status = jobs[w].status;
  }
  free(jobs); free(th);
  return status;
}

void oo_moments(const double* qf, const double* qc, int64_t n, int has_coarse, double out[5]) {
  double mean_y = 0.0, mean_q = 0.0, m2y = 0.0, m2q = 0.0; /* estimators.cpp:82-101 */
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double y = has_coarse ? qf[i] - qc[i] : qf[i];
    ++cnt;
    double d = y - mean_y;
    mean_y += d / cnt;
    m2y += d * (y - mean_y);
    d = qf[i] - mean_q;
    mean_q += d / cnt;
    m2q += d * (qf[i] - mean_q);
  }
  out[0] = (double)cnt;
  out[1] = mean_y;
  out[2] = cnt >= 2 ? m2y / (cnt - 1) : 0.0;
  out[3] = mean_q;
  out[4] = cnt >= 2 ? m2q / (cnt - 1) : 0.0;
}
