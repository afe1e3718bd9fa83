/* schwarz_b200 — C ABI of the B200-native multilevel ORAS inpainting solver.
 *
 * Drop-in replacement for the solver entry points of the reference
 * schwarz-inpaint library (header-only C++20, /root/reference/proj).  Every
 * entry point cites the reference interface it replaces; paths are relative
 * to proj/include/schwarz_inpaint/.  Plain pointers and sizes only: no C++
 * or CUDA types cross this boundary, and no exception escapes it.
 *
 * Data layout (identical to the reference's ImageBuffer / InpaintingMask,
 * image.hpp:24-94): images are planar double, channel c occupying
 * [c*w*h, (c+1)*w*h), row-major; masks are uint8 per pixel, nonzero = known.
 *
 * Errors: every call returns an si_status.  SI_ERR_INVALID_ARGUMENT is
 * returned exactly where the reference throws std::invalid_argument (the
 * message, retrievable with si_last_error(), names the same check).
 * Non-convergence is not an error: it is reported in si_report.converged
 * and si_report.diagnostic, as the reference's SolveReport does.
 *
 * Threading: one si_ctx per host thread (or per GPU); contexts are
 * independent.  si_last_error() is thread-local.
 */
#ifndef SCHWARZ_B200_H
#define SCHWARZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SI_ABI_VERSION 2
#define SI_MAX_LEVELS 32

typedef enum {
  SI_OK = 0,
  SI_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument (image.hpp:18-20) */
  SI_ERR_CUDA = 2,
  SI_ERR_OOM = 3,
  SI_ERR_UNSUPPORTED = 4,      /* e.g. block_size > 32 */
  SI_ERR_NO_DEVICE = 5,
  SI_ERR_RUNTIME = 6           /* reference: std::runtime_error (reduction.hpp:109-110) */
} si_status;

/* Method (methods.hpp:13). */
typedef enum {
  SI_METHOD_CG = 0,
  SI_METHOD_MLCG = 1,
  SI_METHOD_RAS = 2,
  SI_METHOD_ORAS = 3,
  SI_METHOD_MLORAS = 4
} si_method;

typedef enum { SI_AVERAGING_KNOWN_ONLY = 0, SI_AVERAGING_ALL_PIXELS = 1 } si_averaging;    /* multilevel.hpp:25 */
typedef enum { SI_NORMALIZER_INITIAL_GUESS = 0, SI_NORMALIZER_RHS_NORM = 1 } si_normalizer; /* schwarz.hpp:36 */
typedef enum { SI_FLAVOUR_RAS = 0, SI_FLAVOUR_ORAS = 1 } si_flavour;                      /* schwarz.hpp:29 */
/* FP64: the reference's arithmetic everywhere.  FP32: everything in float.
 * MIXED: the image, residual norms and outer iteration in double, the local
 * CG solves (tolerance 1e-2 by default) in float. */
typedef enum {
  SI_PRECISION_FP64 = 0,
  SI_PRECISION_FP32 = 1,
  SI_PRECISION_MIXED = 2
} si_precision;

/* RunOptions (methods.hpp:40-55), field for field, plus the device
 * arithmetic type.  si_default_options() fills the reference defaults. */
typedef struct si_options {
  double tolerance;             /* 1e-3 */
  int levels;                   /* 3 (mlcg / mloras only) */
  int block_size;               /* 32 */
  int overlap;                  /* 6 */
  double alpha;                 /* 0.25 = kDefaultOrasAlpha (schwarz.hpp:34) */
  double coarse_tolerance;      /* 1e-2 */
  int averaging;                /* si_averaging, KnownOnly */
  double local_tolerance;       /* SolverConfig local{1e-2, 30, 30} */
  int local_max_iterations;
  int local_check_interval;
  int max_outer_iterations;     /* 1000 */
  int cg_max_iterations;        /* 100000 (cg / mlcg level solver) */
  int cg_check_interval;        /* 4 */
  int normalizer;               /* si_normalizer, InitialGuess */
  int precision;                /* si_precision, FP64 (the reference's type) */
} si_options;

/* SolveReport (cg.hpp:29-34) + LevelRunStats (schwarz.hpp:254-260) per level. */
typedef struct si_report {
  int iterations;               /* finest-level outer sweeps */
  double final_relative_residual;
  int converged;
  char diagnostic[128];
  int depth;                    /* pyramid levels actually built */
  int level_iterations[SI_MAX_LEVELS];     /* index 0 = finest */
  double level_final_rel[SI_MAX_LEVELS];
  int level_converged[SI_MAX_LEVELS];
  long long local_solves;       /* blocks x channels x sweeps, all levels */
  long long local_failures;     /* local CG cap reached or breakdown */
  long long local_cg_iterations;/* sum of local CG iterations (device-counted) */
  double elapsed_ms;            /* host wall clock around the solve */
  long long h2d_bytes;          /* host->device bytes this frame moved (host entries) */
  long long d2h_bytes;          /* device->host bytes this frame moved (host entries) */
} si_report;

/* Trace sink: one call per finest-level outer iteration, row 0 included
 * (ConvergenceTrace::append, metrics.hpp:74-77).  psnr is NaN unless a
 * reference image was passed. */
typedef void (*si_trace_fn)(int iteration, double time_ms, double rel_residual, double psnr,
                            void* user);

typedef struct si_ctx si_ctx;

/* ---- library / context ------------------------------------------------ */
int si_abi_version(void);
const char* si_last_error(void);
const char* si_status_string(si_status s);
void si_default_options(si_options* opt);
/* Validates options as run_method/multilevel_solve would (multilevel.hpp:243-244,
 * partition.hpp:68-73, schwarz.hpp:275-276, cg.hpp:75-80).  No device needed. */
si_status si_validate_options(int method, const si_options* opt);

si_status si_create(int device, si_ctx** out);
void si_destroy(si_ctx* ctx);
/* Releases cached per-level device buffers. */
si_status si_trim(si_ctx* ctx);

/* ---- solver entry points ----------------------------------------------- */

/* run_method(method, f, mask, options, reference) (methods.hpp:57-88) with
 * HOST buffers: f and reference are w*h*c planar doubles, mask w*h bytes,
 * out receives the w*h*c reconstruction.  reference may be NULL. */
si_status si_run_method(si_ctx* ctx, int method, const double* f, const uint8_t* mask, int w,
                        int h, int c, const si_options* opt, const double* reference, double* out,
                        si_report* report, si_trace_fn trace, void* user);

/* Same, DEVICE-resident: d_f, d_mask, d_reference, d_out live in device
 * memory of ctx's device; work is issued on `stream` (a cudaStream_t, NULL =
 * the context's own stream).  The call returns when the solve is complete. */
si_status si_run_method_device(si_ctx* ctx, int method, const double* d_f, const uint8_t* d_mask,
                               int w, int h, int c, const si_options* opt,
                               const double* d_reference, double* d_out, si_report* report,
                               si_trace_fn trace, void* user, void* stream);

/* A batch of independent frames (BASELINE configs[3]): run_method on each of
 * the n frames f[k]/mask[k] -> out[k] (host buffers, each w*h*c / w*h).  The
 * host->device copy of frame k+1 and the device->host copy of frame k-1 run on
 * their own streams while frame k is solved (pinned host buffers make them
 * truly asynchronous).  reports: NULL or n entries. */
si_status si_run_method_batch(si_ctx* ctx, int method, int n, const double* const* f,
                              const uint8_t* const* mask, int w, int h, int c,
                              const si_options* opt, double* const* out, si_report* reports);

/* The CLI's wire format (pnm.hpp): pixels[k] is a P5/P6 payload (w*h*c bytes,
 * interleaved, value = byte/255, c = 1 or 3), mask_pbm[k] a P4 payload
 * ((w+7)/8 bytes per row, MSB first, bit 1 = known), out_pixels[k] receives the
 * P5/P6 payload of the result (clamp to [0,1], lround(255 v): write_pnm,
 * pnm.hpp:130-147).  Decoding and quantisation run on the device, so a 4K RGB
 * frame moves 25 MB + 1 MB in and 25 MB out instead of 207 MB + 199 MB. */
si_status si_run_pnm_batch(si_ctx* ctx, int method, int n, const uint8_t* const* pixels,
                           const uint8_t* const* mask_pbm, int w, int h, int c,
                           const si_options* opt, uint8_t* const* out_pixels, si_report* reports);

/* solve_schwarz(f, mask, partition_domain(w,h,block,overlap), options, reference)
 * (schwarz.hpp:349-389): single level on an explicit, unclamped partition.
 * flavour: si_flavour; host buffers. */
si_status si_solve_schwarz(si_ctx* ctx, const double* f, const uint8_t* mask, int w, int h, int c,
                           int block_size, int overlap, int flavour, const si_options* opt,
                           const double* reference, double* out, si_report* report,
                           si_trace_fn trace, void* user);

/* run_schwarz_level(op, part, b, u, r0, tol, opt, row) (schwarz.hpp:266-323):
 * the finest seam, u in/out, host buffers.  b and u are w*h*c planar. */
si_status si_run_schwarz_level(si_ctx* ctx, const uint8_t* mask, int w, int h, int c,
                               const double* b, double* u, int block_size, int overlap,
                               double r0_norm, double tolerance, int flavour,
                               const si_options* opt, si_report* report, si_trace_fn trace,
                               void* user);

/* canonical_r0(op, b, normalizer) (schwarz.hpp:333-345), host buffers. */
si_status si_canonical_r0(si_ctx* ctx, const uint8_t* mask, int w, int h, int c, const double* b,
                          int normalizer, double* r0_norm);

/* ---- building blocks (device-executed; host buffers) --------------------- */

/* One outer sweep: u_new = u + sum_i R_i^T D_i v_i on partition_domain(w,h,
 * block,overlap) (schwarz.hpp:305-318).  Counters may be NULL. */
si_status si_schwarz_sweep(si_ctx* ctx, const uint8_t* mask, int w, int h, int c, const double* b,
                           const double* u, int block_size, int overlap, int flavour,
                           const si_options* opt, double* u_new, long long* failures,
                           long long* cg_iterations);
/* sum_i (b - A u)_i^2 per channel (residual_into + vec::dot, operators.hpp:91-97). */
si_status si_residual_sumsq(si_ctx* ctx, const uint8_t* mask, int w, int h, int c,
                            const double* u, const double* b, double* sumsq);
/* restrict_level (multilevel.hpp:33-70): coarse grid is ceil(w/2) x ceil(h/2). */
si_status si_restrict_level(si_ctx* ctx, const uint8_t* mask, const double* values, int w, int h,
                            int c, int averaging, uint8_t* coarse_mask, double* coarse_values);
/* prolongate (multilevel.hpp:101-128) of one channel. */
si_status si_prolongate(si_ctx* ctx, const double* coarse, int cw, int ch, int fw, int fh,
                        double* fine);
/* LocalOperator::apply for block `index` of partition_domain(w,h,block,overlap)
 * (build_local_operator schwarz.hpp:115-130, apply :57-75); v, out: block cells. */
si_status si_local_operator_apply(si_ctx* ctx, const uint8_t* mask, int w, int h, int block_size,
                                  int overlap, int index, int flavour, double alpha,
                                  const double* v, double* out);

/* ---- one image over G ranks: horizontal stripes (BASELINE configs[4]) ----
 * multilevel_solve (multilevel.hpp:239-310) with every pyramid level split
 * into G stripes of whole block rows of that level's own partition
 * (partition_domain, partition.hpp:46-106).  Each rank allocates, ingests,
 * restricts, sweeps and prolongs only its rows (plus halos); per outer
 * iteration the G x C partial residual sums are all-gathered (every rank
 * takes run_schwarz_level's stop decision, schwarz.hpp:288-300, in the same
 * fixed rank order) and halo rows move between neighbours.  The image equals
 * the single-GPU solve's bit for bit whenever the stop decisions agree.
 * Schwarz methods only (ras, oras, mloras); CG methods -> SI_ERR_UNSUPPORTED.
 *
 * A communicator joins the ranks: NCCL (one process per GPU; rank 0 makes
 * the id with si_nccl_unique_id and the caller broadcasts its 128 bytes) or
 * local (G ranks as host threads of one process, possibly on one device). */
typedef struct si_stripe_comm si_stripe_comm;
#define SI_NCCL_ID_BYTES 128
si_status si_nccl_unique_id(unsigned char* id /* SI_NCCL_ID_BYTES */);
si_status si_stripe_comm_init_nccl(si_ctx* ctx, int world, int rank, const unsigned char* id,
                                   si_stripe_comm** out);
/* comms_out[r] for r < world, rank r driven on ctxs[r] (one host thread each). */
si_status si_stripe_comm_init_local(si_ctx* const* ctxs, int world, si_stripe_comm** comms_out);
void si_stripe_comm_destroy(si_stripe_comm* comm);
/* Outer iterations are decided on the device.  With speculation on (the
 * default) a solve issues, per level, as many iterations as the last solve
 * with the same shape and options took, without a host round trip; a level
 * that needed more is resumed and the finer levels after it are redone
 * (results identical).  Off: one host round trip per decision.  Every rank
 * of a group must use the same setting. */
si_status si_stripe_comm_set_speculation(si_stripe_comm* comm, int enabled);
/* The finest own rows of the last striped solve on ctx that ran without an
 * output buffer: channel k's rows start at *rows + k * *plane_stride
 * (doubles), *n_rows rows of w; device memory owned by ctx, valid until its
 * next call.  *rows is NULL when the rank owns no rows. */
si_status si_stripe_result_rows(si_ctx* ctx, const double** rows, size_t* plane_stride,
                                int* n_rows);
/* out[0] solves, out[1] solves that speculated, out[2] resumed levels. */
si_status si_stripe_comm_counters(const si_stripe_comm* comm, long long* out /* 3 */);

/* Rows of every level for `rank` (host only, no device): out receives
 * SI_STRIPE_PLAN_INTS ints per level (index 0 = finest): k0, k1 (block rows),
 * own_lo, own_hi (rows it owns), win_lo, win_hi (rows its sweeps read),
 * need_lo, need_hi (coarse rows its prolongation reads), store_lo, store_hi
 * (rows it holds), block, overlap (clamped partition).  *depth = levels. */
#define SI_STRIPE_PLAN_INTS 12
si_status si_stripe_level_plan(int method, int w, int h, int c, const si_options* opt, int world,
                               int rank, int* depth, int* out /* SI_MAX_LEVELS*12 */);

/* run_method over the ranks of `comm` (collective: every rank calls it).
 * f / mask: the full HOST image (only this rank's level-0 store rows are
 * uploaded); out: full-size host buffer, this rank writes its own finest
 * rows.  Every rank's report carries the global counts. */
si_status si_run_method_striped(si_ctx* ctx, si_stripe_comm* comm, int method, const double* f,
                                const uint8_t* mask, int w, int h, int c, const si_options* opt,
                                double* out, si_report* report, si_trace_fn trace, void* user);
/* Device-resident: d_f_rows / d_mask_rows hold level-0 rows [store_lo,
 * store_hi) (compact planar), d_out_rows receives rows [own_lo, own_hi).
 * d_out_rows may be NULL (FP64 / MIXED): the rows are then left where the
 * solve put them, see si_stripe_result_rows (no device output pass). */
si_status si_run_method_striped_device(si_ctx* ctx, si_stripe_comm* comm, int method,
                                       const double* d_f_rows, const uint8_t* d_mask_rows, int w,
                                       int h, int c, const si_options* opt, double* d_out_rows,
                                       si_report* report, void* stream);
/* Every rank of a local group (si_stripe_comm_init_local) in one call, on
 * device rows as si_run_method_striped_device: rank r on ctxs[r] and
 * comms[r] with d_f_rows[r] / d_mask_rows[r] -> d_out_rows[r] (d_out_rows or
 * an entry may be NULL: rows in place) on streams[r] (NULL: the context's).
 * Ranks 1..world-1 run on the group's persistent host threads, rank 0 on the
 * caller's.  One group call at a time per group. */
si_status si_run_method_striped_local_device(si_stripe_comm* const* comms, si_ctx* const* ctxs,
                                             int world, int method,
                                             const double* const* d_f_rows,
                                             const uint8_t* const* d_mask_rows, int w, int h,
                                             int c, const si_options* opt,
                                             double* const* d_out_rows, si_report* reports,
                                             void* const* streams);
/* Convenience: `world` ranks as threads of this process on ctxs[] over a
 * local communicator; out receives the whole image; reports: NULL or world. */
si_status si_run_method_striped_group(si_ctx* const* ctxs, int world, int method, const double* f,
                                      const uint8_t* mask, int w, int h, int c,
                                      const si_options* opt, double* out, si_report* reports);

/* ---- host-only helpers (no device needed) -------------------------------- */

/* partition_domain (partition.hpp:67-106).  rects receives 8 ints per block:
 * x0, y0, width, height, own_x0, own_y0, own_x1, own_y1 (row-major blocks). */
si_status si_partition_domain(int w, int h, int block_size, int overlap, int* blocks_x,
                              int* blocks_y, int* rects, int rects_capacity);
/* Known-sample packing of the host entries' upload (si_run_method,
 * si_run_method_batch ship a sparse frame as its mask plus these): the solver
 * reads f only at known pixels (build_pyramid, multilevel.hpp:84-88).
 * tile_off[t] = known pixels before tile t (ceil(w*h / SI_KNOWN_TILE) tiles),
 * *K = known total, vals [c][K] (NULL: count only) = f at the known pixels in
 * pixel order. */
#define SI_KNOWN_TILE 4096
si_status si_pack_known_samples(const double* f, const uint8_t* mask, int w, int h, int c,
                                uint32_t* tile_off, double* vals, long long* K);
/* synthetic_test_image (synthetic.hpp:14-59) and random_mask (masks.hpp:25-43):
 * the reference's seeded input generators (libstdc++ <random>). */
si_status si_synthetic_test_image(int w, int h, int c, uint64_t seed, double* out);
si_status si_random_mask(int w, int h, double density, uint64_t seed, uint8_t* out);
/* sqrt(sum_c sqrt(sumsq[c])^2): the joint residual norm of run_schwarz_level
 * (schwarz.hpp:290-295, accumulate contracted to an fma as in the gcc build). */
double si_joint_norm(const double* sumsq, int c);
/* mse_per_channel / psnr (metrics.hpp:30-56) on host buffers. */
si_status si_psnr(const double* u, const double* f, int w, int h, int c, double* psnr_db);

/* ---- Voronoi densification (masks.hpp:45-215) -------------------------- */

/* DensifyOptions (masks.hpp:145-151). */
typedef struct si_densify_options {
  double initial_density;  /* <= 0: start at a quarter of the target */
  double cell_fraction;    /* share of cells refined per sweep (0.20) */
  double inner_tolerance;  /* tolerance of the guiding inpainting runs (1e-3) */
  int max_sweeps;          /* 100 */
  si_options solve;        /* MultilevelSolveOptions of the guide solver (multilevel
                              ORAS); its tolerance is replaced by inner_tolerance */
} si_densify_options;
void si_default_densify_options(si_densify_options* o);
/* voronoi_densify(f, target_density, seed, options) (masks.hpp:155-212):
 * grows random_mask(w, h, initial, seed) towards round(target * w * h) known
 * pixels; every sweep inpaints with the multilevel ORAS path, assigns Voronoi
 * cells, ranks them by (squared error desc, area desc, site index asc) and
 * plants a known pixel at the worst pixel of the first
 * max(1, cell_fraction * sites) cells.  The whole loop runs on the device.
 * mask_out: w*h bytes.  Invalid targets -> SI_ERR_INVALID_ARGUMENT with the
 * reference's messages (masks.hpp:157-160). */
si_status si_voronoi_densify(si_ctx* ctx, const double* f, int w, int h, int c,
                             double target_density, uint64_t seed, const si_densify_options* opt,
                             uint8_t* mask_out, int* sweeps, int* reached_target);
/* assign_nearest_site (masks.hpp:54-139): sites = known pixel indices in
 * ascending order (capacity w*h), site_of[p] = index of p's nearest site
 * (squared Euclidean distance, ties to the lower site index). */
si_status si_assign_nearest_site(si_ctx* ctx, const uint8_t* mask, int w, int h, int32_t* sites,
                                 int32_t* site_of, int* num_sites);

/* ---- instrumentation ---------------------------------------------------- */

/* Per-kernel device time (CUDA events on the launching stream) accumulated
 * while profiling is enabled; kind: 0 residual (K1), 1 sweep (K2), 2 restrict
 * (K3), 3 prolong (K4), 4 ingest/export (K5), 5 metrics (K6), 6 Voronoi
 * densification (D1-D6).
 * total_launches counts every kernel launched by the context, always. */
typedef struct si_kernel_stats {
  long long launches[8];
  double device_ms[8];
  double algorithmic_bytes[8];
  long long total_launches;
} si_kernel_stats;
si_status si_set_profiling(si_ctx* ctx, int enabled);
/* Device self-tests of arithmetic shortcuts used by the kernels.  which = 0:
 * division through a precomputed correctly rounded reciprocal equals IEEE
 * division on n random operand pairs; *failures = mismatches. */
si_status si_selftest(si_ctx* ctx, int which, long long n, long long* failures);
si_status si_get_kernel_stats(si_ctx* ctx, si_kernel_stats* out, int reset);
/* Pinned host memory for zero-staging host<->device copies. */
si_status si_host_alloc(size_t bytes, void** ptr);
si_status si_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif
