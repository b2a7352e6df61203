/*
 * tccd -- B200-native batched Tight-Inclusion CCD (arXiv 2009.13349).
 *
 * C-ABI of libtccd.so: plain pointers, sizes and a struct; no torch types.
 * The library never allocates device memory on the batched path: the caller
 * passes a workspace sized by tccd_workspace_bytes().  All device work is
 * enqueued on the caller's stream (a cudaStream_t passed as void*).
 *
 * Reference interface each entry point replaces (paths under the reference
 * repo):
 *   tccd_solve_kernel  <- ccdkit._kernel.solve_kernel
 *                         (pkg/src/ccdkit/_kernel.py:136-146, same argument
 *                         list and the same 13-field result)
 *   tccd_solve_batch   <- a loop of ccdkit.solver.solve(q, config)
 *                         (pkg/src/ccdkit/solver.py:50-107) over a batch,
 *                         including its filter resolution
 *                         (_resolve_filters, solver.py:30-47 ->
 *                         inclusion.compute_gamma / compute_filters,
 *                         pkg/src/ccdkit/inclusion.py:85-122) and the
 *                         SolverConfig validation (core.py:176-184)
 *   tccd_workspace_bytes, tccd_error_string, tccd_abi_version: new (no
 *                         reference counterpart; numba allocates internally)
 */
#ifndef TCCD_H
#define TCCD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCCD_ABI_VERSION 3

/* Per-query status values written to tccd_batch.status. */
#define TCCD_STATUS_FREE 0           /* certified collision free, toi = +inf   */
#define TCCD_STATUS_HIT 1            /* collision, toi = witness t_lo          */
#define TCCD_STATUS_ERR_SEPARATION 2 /* d >= gamma on an axis: the reference's
                                        compute_filters ValueError
                                        (inclusion.py:110-113)                 */
#define TCCD_STATUS_ERR_NONFINITE 3  /* NaN/inf coordinate: Vec3 ValueError
                                        (core.py:49-51)                        */
#define TCCD_STATUS_ERR_PARAM 4      /* per-query delta/m_I/d/t_max/kind
                                        outside SolverConfig's domain
                                        (core.py:176-184)                      */

/* Return codes. */
#define TCCD_OK 0
#define TCCD_E_NULL 1       /* a required pointer is NULL                     */
#define TCCD_E_N 2          /* n < 0                                          */
#define TCCD_E_DELTA 3      /* broadcast delta not > 0 and finite             */
#define TCCD_E_MAXCHECKS 4  /* broadcast max_checks < 1                       */
#define TCCD_E_TMAX 5       /* broadcast t_max not in (0, 1]                  */
#define TCCD_E_SEPARATION 6 /* broadcast separation < 0 or non-finite         */
#define TCCD_E_KIND 7       /* broadcast kind not 0/1                         */
#define TCCD_E_WORKSPACE 8  /* workspace NULL or smaller than required        */
#define TCCD_E_CUDA 9       /* a CUDA runtime call failed                     */
#define TCCD_E_STRUCT 10    /* struct_size mismatch (ABI skew)                */
#define TCCD_E_CAPACITY 11  /* max_checks_max exceeds what the layout indexes */

/* flags */
#define TCCD_FLAG_HEAVY_ONLY 1u /* route every query through the block-per-query
                                   engine (testing / diagnostics)             */
#define TCCD_FLAG_NO_LANE 2u    /* skip the lane tier: every survivor of the
                                   root check goes through the group tiers
                                   (testing / diagnostics)                    */

/* Solver stages, in launch order per chunk (tccd_batch.events). */
#define TCCD_STAGE_PROLOGUE 0 /* validation, filters, kappas, root check     */
#define TCCD_STAGE_LANE 1     /* thread-per-query tier (dyadic t_max)        */
#define TCCD_STAGE_LIGHT 2    /* group tiers: light, medium, giant           */
#define TCCD_STAGE_MEDIUM 3
#define TCCD_STAGE_GIANT 4
#define TCCD_NUM_STAGES 5

/* Diagnostic counters (tccd_batch.stats, TCCD_NUM_STATS int64, summed over
 * chunks). */
#define TCCD_NUM_STATS 32
#define TCCD_STAT_GIANT_QUERIES 0   /* queries that reached the giant tier      */
#define TCCD_STAT_ROUNDS 1          /* group-engine rounds                      */
#define TCCD_STAT_DEFERRALS 2       /* group-engine level deferrals             */
#define TCCD_STAT_MEDIUM_QUERIES 3  /* queries that reached the medium tier     */
#define TCCD_STAT_BOXES 4           /* [4..6] boxes visited per group tier      */
#define TCCD_STAT_LANE_QUERIES 7    /* queries that entered the lane tier       */
#define TCCD_STAT_CLS 8             /* [8..13] box classifications per group
                                       tier and kind (light VF, light EE, medium
                                       VF, medium EE, giant VF, giant EE)       */
#define TCCD_STAT_LANE_CLS 14       /* [14..15] lane classifications VF, EE     */
#define TCCD_STAT_LANE_CHECKS 16    /* [16..17] checks the lane tier did on the
                                       reference's path (queries it finished or
                                       handed over with their level; root check
                                       excluded: the prologue's): algorithmic
                                       work                                     */
#define TCCD_STAT_LANE_DONE 18      /* [18..19] queries the lane tier finished  */
#define TCCD_STAT_LANE_EVICTED 20   /* queries the lane tier sent to the light
                                       tier (handed over or restarting)         */
#define TCCD_STAT_LANE_WASTED 21    /* lane checks of those that restart (the
                                       light tier repeats them)                 */
#define TCCD_STAT_POOL_DEMAND 22    /* [22..23] handover boxes requested light->
                                       medium, medium->giant                    */
#define TCCD_STAT_RESTARTS 24       /* [24..25] evictions light->medium,
                                       medium->giant that found the handover
                                       pool full (restart from the root)        */
#define TCCD_STAT_TIER_CHECKS 26    /* [26..28] checks of the reference's path
                                       done in the light, medium, giant tiers
                                       (classifications past a query's return
                                       point, deferral re-runs and restarted
                                       work excluded)                           */
#define TCCD_STAT_PROLOGUE_DONE 29  /* queries decided at the root (or invalid) */
#define TCCD_STAT_LANE_HANDED 30    /* lane evictions handed over with their
                                       current level (the rest restart)         */
#define TCCD_STAT_CHUNKS 31         /* library chunks                           */

/*
 * One batched solve.  All array pointers are DEVICE pointers.  For every
 * per-query parameter, a NULL array means "use the broadcast *_all value".
 *
 * points: [n][8][3] f64, row-major: the 4 points at t0 in query order
 *         (VF: p, v1, v2, v3; EE: p1, p2, p3, p4 -- core.py:86-89), then the
 *         same 4 points at t1 (Query.all_coordinates(), core.py:114-116).
 * kind:   [n] u8, 0 vertex-face, 1 edge-edge (QueryKind, core.py:75-79).
 * eps:    NULL -> per-query gamma/eps computed on device exactly as
 *         compute_gamma + compute_filters; else [n][3] caller filters
 *         (a reused FilterEps, solver.py:30-47; not re-validated, like the
 *         reference).
 * Outputs: status and toi are required; the others may be NULL.
 *         toi = +inf for status != HIT.  witness = [n][6]
 *         (t_lo, t_hi, u_lo, u_hi, v_lo, v_hi).  tol = witness t width,
 *         codom = witness hull width, checks = box classifications,
 *         early = budget ended the search, level = witness BFS level.
 */
typedef struct tccd_batch {
  uint32_t struct_size; /* = sizeof(tccd_batch)                       */
  uint32_t flags;       /* TCCD_FLAG_*                                */
  int64_t n;

  const double *points;
  const uint8_t *kind;
  int32_t kind_all;
  int32_t reserved0;
  const double *delta;
  double delta_all;
  const int64_t *max_checks;
  int64_t max_checks_all;
  int64_t max_checks_max; /* upper bound over the batch; sizes the workspace */
  const double *separation;
  double separation_all;
  const double *t_max;
  double t_max_all;
  const double *eps;

  uint8_t *status;
  double *toi;
  double *tol;
  double *codom;
  int64_t *checks;
  uint8_t *early;
  double *witness;
  int32_t *level;

  void *workspace;
  size_t workspace_bytes;
  int32_t heavy_blocks; /* concurrent block-per-query solvers; 0 = default   */
  int32_t device_sms;   /* SM count of the target device; 0 = query it      */
  int64_t *stats;       /* optional device [TCCD_NUM_STATS] diagnostics
                           (TCCD_STAT_*)                                  */
  /* Per-kernel timing on the launching stream (ABI 3): events is an
   * optional host array of n_events cudaEvent_t; the call records one after
   * each stage it launches, in launch order, writes that stage
   * (TCCD_STAGE_*) to event_stage[i] (host array, same length) and sets
   * events_used (out).  A stage's time is the gap to the previous recorded
   * event (the first: to an event the caller records before the call). */
  void *const *events;
  int32_t *event_stage;
  int32_t n_events;
  int32_t events_used;
  /* Host-input overlap (ABI 3): if input_events is non-NULL, the prologue
   * of queries [c * input_chunk, (c + 1) * input_chunk) waits for
   * input_events[c] (cudaEvent_t recorded by the caller once those
   * queries' inputs are on the device, e.g. after a copy on another
   * stream); n_input_events = ceil(n / input_chunk). */
  void *const *input_events;
  int64_t input_chunk;
  int32_t n_input_events;
  int32_t reserved1;
  /* Optional compacted hit list (ABI 3): every query with status HIT
   * appends (index, toi) -- in no particular order -- at position
   * *hit_count (device u64, NOT reset by the call: zero it once and several
   * calls append to one list), which ends as the number of entries written
   * so far; it may exceed hit_capacity (entries past the capacity are
   * dropped). */
  int64_t *hit_index;
  double *hit_toi;
  uint64_t *hit_count;
  int64_t hit_capacity;
  int64_t hit_index_base; /* added to every index written to hit_index (a
                             caller solving a slice of a larger batch)   */
  int64_t pool_boxes;   /* handover pool boxes per tier transition and
                           sub-chunk; 0 = default (tccd_workspace_bytes_ex
                           must be asked with the same value)            */
  int64_t launches;     /* out: kernels this call launched               */
} tccd_batch;

/* Bytes of device workspace tccd_solve_batch needs for a batch of n queries
 * whose largest check budget is max_checks_max, with heavy_blocks concurrent
 * block-per-query solvers (0 = default for the current device). */
size_t tccd_workspace_bytes(int64_t n, int64_t max_checks_max, int32_t heavy_blocks);
/* The same for a non-default handover pool size (tccd_batch.pool_boxes). */
size_t tccd_workspace_bytes_ex(int64_t n, int64_t max_checks_max, int32_t heavy_blocks,
                               int64_t pool_boxes);

/* Enqueue a batched solve on `stream` (cudaStream_t, NULL = legacy default).
 * Returns TCCD_OK or a TCCD_E_* code; per-query failures go to status[]. */
int tccd_solve_batch(const tccd_batch *batch, void *stream);

/* Drop-in for _kernel.solve_kernel(s, e, kind, t_max, delta, max_checks,
 * sep, ex, ey, ez) (_kernel.py:136): HOST pointers s[4][3], e[4][3];
 * out13 receives (status, toi, tol, codom, checks, early, w_t0, w_t1, w_u0,
 * w_u1, w_v0, w_v1, w_level) as doubles.  Synchronous, on the current
 * device; its device scratch is cached per device and grows with the
 * largest max_checks seen (no allocation per call once warm).  Calls are
 * serialized by a library lock.  tccd_release_cached() frees the caches. */
int tccd_solve_kernel(const double *s, const double *e, int kind, double t_max,
                      double delta, int64_t max_checks, double sep, double ex,
                      double ey, double ez, double *out13);

/*
 * GPU broad phase <- ccdkit.scene.broad_phase
 * (pkg/src/ccdkit/scene.py:225-300): the primitive pairs whose inflated
 * swept boxes overlap, minus pairs sharing a mesh vertex; vertex-face pairs
 * (vertex, triangle) sorted, then edge-edge pairs (edge_a < edge_b) sorted,
 * with their queries in the solver's [m][8][3] layout.
 *
 * Mesh arrays are DEVICE pointers; positions must be finite and indices in
 * [0, n_vertices) (the Python layer validates, like TriMeshPair).  Edges
 * are rows (i, j), i < j, unique (edges_from_triangles).
 */
typedef struct tccd_mesh {
  uint32_t struct_size; /* = sizeof(tccd_mesh) */
  uint32_t reserved;
  int64_t n_vertices, n_triangles, n_edges;
  const double *x0;          /* [n_vertices][3] positions at the step start */
  const double *x1;          /* [n_vertices][3] positions at the step end   */
  const int64_t *triangles;  /* [n_triangles][3]                            */
  const int64_t *edges;      /* [n_edges][2]                                */
} tccd_mesh;

typedef struct tccd_broad tccd_broad; /* opaque broad-phase state */

/* Boxes, grid and pair counts (stream-ordered device allocations owned by
 * the handle).  Synchronizes `stream` and returns the candidate counts. */
int tccd_broad_create(const tccd_mesh *mesh, double inflation, tccd_broad **out,
                      int64_t *n_vf, int64_t *n_ee, void *stream);
/* Writes the n_vf + n_ee candidates (VF block first) on the handle's
 * stream: kind [m] u8, pairs [m][2] i64 (vertex, triangle) / (edge_a,
 * edge_b), points [m][8][3] f64 (device buffers of the caller). */
int tccd_broad_emit(tccd_broad *h, uint8_t *kind, int64_t *pairs, double *points);
void tccd_broad_destroy(tccd_broad *h);

/*
 * IRF baseline <- ccdkit.baselines.irf_solve
 * (pkg/src/ccdkit/baselines.py:123-206): outward-rounded interval
 * bisection, best-first by (t_lo, level, push order), bit-identical to the
 * reference for every query.  Uses the tccd_batch fields points, kind,
 * delta, max_checks (any value; <= 0 returns the root box as an early
 * hit), max_checks_max, t_max (finite, >= 0), the outputs, workspace /
 * workspace_bytes, heavy_blocks (= second-pass slots, 0 = one per SM) and
 * device_sms; separation, eps, stats and events are ignored.  Per-query
 * invalid delta / t_max / kind -> status TCCD_STATUS_ERR_PARAM (the
 * reference's ValueError), non-finite coordinates -> ERR_NONFINITE.
 */
size_t tccd_irf_workspace_bytes(int64_t n, int64_t max_checks_max, int32_t big_slots);
int tccd_irf_batch(const tccd_batch *batch, void *stream);

/*
 * Copy `bytes` from device memory to pinned (page-locked) host memory with a
 * kernel on `stream` instead of a copy-engine transfer (new; no reference
 * counterpart).  A streaming caller's result copies then do not queue in
 * front of its next batch's host-to-device copy, which the copy engines
 * would otherwise serve in submission order.  host_dst must be pinned host
 * memory (device-accessible through unified addressing); returns
 * TCCD_E_CUDA if it is not, so the caller can fall back to cudaMemcpyAsync.
 */
int tccd_copy_to_host(const void *src, void *host_dst, int64_t bytes, void *stream);

void tccd_release_cached(void);

/*
 * The reference's spec-level inclusion functions, batched, on the device
 * (the solver's own arithmetic; the solver does not call them).  DEVICE
 * pointers; kind NULL -> kind_all; asynchronous on `stream`.
 *   tccd_box_hulls <- ccdkit.inclusion.box_inclusion (inclusion.py:131-156):
 *       for each i, lo[i][ax] / hi[i][ax] = min / max over the 8 corners of
 *       boxes[i] = (t0, t1, u0, u1, v0, v1) of axis ax of F (NaN if a corner
 *       value is NaN, as numpy's min / max).
 *   tccd_kappas <- ccdkit.inclusion.kappas (inclusion.py:195-217) =
 *       ccdkit._kernel._kappas (_kernel.py:98-132): out[i] = (k_t, k_u, k_v)
 *       on [0, t_max] x [0,1]^2 (t_max NULL -> t_max_all).
 */
int tccd_box_hulls(const double *points, const uint8_t *kind, int kind_all, const double *boxes,
                   int64_t n, double *lo, double *hi, void *stream);
int tccd_kappas(const double *points, const uint8_t *kind, int kind_all, const double *t_max,
                double t_max_all, int64_t n, double *out, void *stream);

/* Copy the first min(*count, max_elems) elements of elem_bytes each from
 * device array src to pinned host memory, where *count (device) was written
 * by an earlier kernel on `stream` (a compacted hit list, tccd_batch.
 * hit_count): only the live entries cross the bus, with no host
 * synchronization.  *count itself goes to host_count (pinned, may be NULL).
 * A kernel on `stream` (see tccd_copy_to_host). */
int tccd_copy_counted_to_host(const void *src, void *host_dst, int64_t elem_bytes,
                              const uint64_t *count, int64_t max_elems, void *host_count,
                              void *stream);

const char *tccd_error_string(int code);
int tccd_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TCCD_H */
