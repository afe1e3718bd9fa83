/* TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * si_oracle: a plain-C, single-threaded CPU restatement of the reference's
 * multilevel ORAS inpainting path (schwarz-inpaint, /root/reference/proj).
 * It is the parity checker for the CUDA path: only tests/, the smoke() entry
 * and bench.py's cpu_baseline leg may load it.
 *
 * Parity pin: tests/test_oracle.py checks this restatement against the
 * reference itself (headers compiled by oracle/Makefile into oracle/_ref/)
 * and against the committed fixtures in tests/golden/ produced by
 * tests/golden/make_golden.py from that compiled reference.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj/include/schwarz_inpaint/.
 */
#ifndef SI_ORACLE_H
#define SI_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_MAX_LEVELS 32

/* Mirrors RunOptions (methods.hpp:40-55) plus the solver choice. */
typedef struct {
  double tolerance;            /* finest-level relative residual target */
  int levels;                  /* pyramid depth requested */
  int block_size;
  int overlap;
  double alpha;                /* Robin weight, schwarz.hpp:34 */
  double coarse_tolerance;
  int averaging;               /* 0 KnownOnly, 1 AllPixels (multilevel.hpp:25) */
  double local_tolerance;      /* SolverConfig local{1e-2,30,30} */
  int local_max_iterations;
  int local_check_interval;
  int max_outer_iterations;
  int normalizer;              /* 0 InitialGuess, 1 RhsNorm (schwarz.hpp:36) */
  int flavour;                 /* 0 RAS, 1 ORAS (schwarz.hpp:29), 2 CG level solver */
  int cg_max_iterations;       /* RunOptions::cg_max_iterations (methods.hpp:51) */
  int cg_check_interval;       /* RunOptions::cg_check_interval (methods.hpp:54) */
} or_options;

typedef struct {
  int iterations;              /* finest-level outer sweeps */
  double final_rel;
  int converged;
  int depth;                   /* levels actually built */
  int level_iterations[OR_MAX_LEVELS];   /* index 0 = finest */
  double level_final_rel[OR_MAX_LEVELS];
  int level_converged[OR_MAX_LEVELS];
  long long local_solves;
  long long local_failures;
  long long local_cg_iterations;
  int trace_rows;              /* finest-level rows written (<= cap) */
  int error;                   /* 0 ok, 1 invalid argument */
} or_report;

void or_default_options(or_options* o);

/* multilevel_solve (multilevel.hpp:239-310) for ORAS/RAS level solvers.
 * f, out: planar [c][y][x] doubles; mask: [y][x] uint8.  trace_rel receives
 * the finest-level relative residual per outer iteration (row 0 included). */
int or_multilevel_solve(const double* f, const uint8_t* mask, int w, int h, int c,
                        const or_options* opt, double* out, or_report* rep,
                        double* trace_rel, int trace_cap);

/* Building blocks, exported for the fine-grained parity tests. */
void or_partition_axis(int extent, int block, int overlap, int* anchors, int* count,
                       int* owned_end);
double or_residual_sumsq(const uint8_t* mask, int w, int h, const double* u, const double* b);
int or_restrict_level(const uint8_t* mask, const double* values, int fw, int fh, int c,
                      int averaging, uint8_t* cmask, double* cvalues);
void or_prolongate(const double* coarse, int cw, int ch, int fw, int fh, double* fine);
/* One outer sweep of run_schwarz_level on a fixed partition (block, overlap
 * already clamped): u_new = u + sum_i R_i^T D_i v_i. */
void or_schwarz_sweep(const uint8_t* mask, int w, int h, int c, const double* b, const double* u,
                      int block, int overlap, const or_options* opt, double* u_new,
                      long long* failures, long long* cg_iterations);
/* Local operator of one block applied to a cell-ordered vector
 * (LocalOperator::apply, schwarz.hpp:50-76). */
void or_local_operator_apply(const uint8_t* mask, int w, int h, int x0, int y0, int bw, int bh,
                             int flavour, double alpha, const double* v, double* out);

/* assign_nearest_site (masks.hpp:54-139): sites = known pixel indices
 * ascending (capacity w*h), site_of[p] = index into sites.  Returns 1 when the
 * mask has no known pixel. */
int or_assign_nearest_site(const uint8_t* mask, int w, int h, int32_t* sites, int32_t* site_of,
                           int* num_sites);
/* voronoi_densify (masks.hpp:155-212) from the seed mask random_mask drew. */
int or_voronoi_densify(const double* f, int w, int h, int c, const uint8_t* seed_mask,
                       long long target_k, double cell_fraction, double inner_tolerance,
                       int max_sweeps, const or_options* solve, uint8_t* mask, int* sweeps);

#ifdef __cplusplus
}
#endif
#endif
