/* osc_oracle — plain-C CPU restatement of the reference's MLMC sample path.
 *
 * TEST INFRASTRUCTURE ONLY. Imported/called only by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs, as the CHECKER. The product
 * (paper_2306_13493_b200/) never links, loads or calls it.
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Parity pin: tests/test_oracle_pin.py checks this
 * restatement against the pristine reference compiled into oracle/_ref/ and
 * against the committed golden fixtures in tests/golden/.
 *
 * Extensions NOT present in the reference (BASELINE configs 1/3/4/5 ask for them):
 *   bc = OSC_BC_DIRICHLET_ALL (u = 0 on all four sides), qoi = OSC_QOI_INTEGRAL (∫u dx)
 *   and OSC_QOI_FLUX (outflow flux through x = 1). Their parity is UNPINNED by the
 *   reference; they follow the same assembly (fem.cpp:38-138) with the Dirichlet test
 *   (fem.cpp:28-30) widened, and are cross-checked by analytic cases in tests/.
 */
#ifndef OSC_ORACLE_H
#define OSC_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { OSC_BC_FLOWCELL = 0, OSC_BC_DIRICHLET_ALL = 1 };
enum { OSC_QOI_POINT = 0, OSC_QOI_L2 = 1, OSC_QOI_INTEGRAL = 2, OSC_QOI_FLUX = 3 };

void oo_philox_block(const uint32_t key[2], const uint32_t ctr[4], uint32_t out[4]);
void oo_normals(uint64_t seed, uint32_t level, uint64_t index, double* out, int64_t n);

/* u = Re(F w) + Im(F w), w = sqrt_lam .* xi, F unitary 2-D DFT with + sign; n x n. */
int oo_sample(int n, const double* sqrt_lam, const double* xi, double* u);
/* R-block of u (row stride n) subsampled by r = m/m_t onto (m_t+1)^2 nodes. */
void oo_restrict(int n, int m, const double* u, int m_t, double* out);

/* assemble_and_solve: Z nodal log field on (m+1)^2 nodes; precond 0 Jacobi, 1 MG.
 * Returns 0, -3 non-finite Z, -4 not converged. iters/history optional. */
int oo_solve(int m, const double* Z, int bc, int forcing, double forcing_value, double tol,
             int max_iter_factor, int precond, double* u, int* iters, double* hist, int hist_cap,
             int* hist_len);
double oo_qoi(int m, const double* u, int bc, int qoi, double qx, double qy, const double* Z,
              int forcing, double forcing_value);

typedef struct {
  int m;                      /* fine cells per side */
  int n;                      /* embedding size per dim, 2(m+J) */
  const double* sqrt_fine;    /* sqrt eigenvalues used for the fine field (n*n) */
  const double* sqrt_coarse;  /* used for the coarse field; == sqrt_fine when shared */
  int has_coarse;
  uint64_t seed;
  uint32_t ell;
  int bc, forcing, qoi, precond, max_iter_factor;
  double forcing_value, qx, qy, tol;
  int threads;
} oo_level;

/* coupled_sample (estimators.cpp:200-237) for indices [from, to); xi_host optional
 * (row i-from of length n*n) replaces NormalStream. Outputs by slot. */
int oo_coupled(const oo_level* L, int64_t from, int64_t to, const double* xi_host, double* q_fine,
               double* q_coarse, int* it_fine, int* it_coarse);

/* Welford moments over slot-ordered draws (estimators.cpp:82-101). */
void oo_moments(const double* q_fine, const double* q_coarse, int64_t n, int has_coarse,
                double out[5] /* n, mean_y, var_y, mean_q, var_q */);

#ifdef __cplusplus
}
#endif
#endif
