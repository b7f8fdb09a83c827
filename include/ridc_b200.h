/*
 * ridc_b200.h -- C-ABI of the B200-native RIDC-FBE marching engine.
 *
 * This is the drop-in boundary for the reference's hot path (paths relative
 * to /root/reference, package pkg/src/ridc):
 *
 *   ridc_create / ridc_run   replace  engine.run_serial / engine.run_pipelined
 *                                     (engine.py:476-522) including _prepare
 *                                     (engine.py:465-473: dt, weight tables,
 *                                     pre-factorisation, restart partition).
 *   ridc_run_device          same run with device-resident state (no H2D/D2H).
 *   ridc_op_apply            replaces ImplicitSolver.stiff_value (steppers.py:66-70)
 *                                     and SplitIVP.eval_nonstiff (problems.py:133,164)
 *   ridc_op_solve            replaces ImplicitSolver.solve_shifted -> qr_solve
 *                                     (steppers.py:72-78, linalg.py:59-63)
 *   ridc_op_step             replaces predict_step / correct_step (engine.py:193-231)
 *                                     driven by states instead of f^S/f^N rows
 *   ridc_pipe_*              the one-level-per-GPU lagged pipeline
 *                                     (engine.py:349-459, LevelBuffer :284-331)
 *   ridc_ark_*               replace  steppers.ark_step / integrate_ark
 *                                     (steppers.py:122-155) with
 *                                     kernels.stage_accumulate (kernels.py:149-158)
 *                                     for the tableaus.py imex3 / imex4 pairs
 *   ridc_shards_*            2-D row shards under the levels (no reference
 *                                     analogue)
 *
 * Conventions.  All pointers are plain; no torch types.  "_host" buffers are
 * caller-owned host memory; "_dev" buffers are caller-owned device memory on
 * the context's device.  The library owns every other device allocation.
 * Return value: 0 on success or a RIDC_E_* status; ridc_last_error() gives
 * the message.  Status codes map onto the reference's exception classes
 * (errors.py:4-47).  One host thread per context; a context is not
 * reentrant; distinct contexts may run concurrently on distinct devices.
 */
#ifndef RIDC_B200_H
#define RIDC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mapped by paper_1209_4297_b200/errors.py) */
#define RIDC_OK 0
#define RIDC_E_CONFIG 1        /* ConfigError */
#define RIDC_E_DIMENSION 2     /* DimensionMismatch */
#define RIDC_E_NONFINITE 3     /* NonFiniteStateError */
#define RIDC_E_PROTOCOL 4      /* PipelineProtocolError (watchdog / protocol) */
#define RIDC_E_DETERMINISM 5   /* DeterminismError */
#define RIDC_E_CUDA 6          /* CUDA runtime failure */

/* problem kinds */
#define RIDC_ADV_DIFF_1D 1            /* problems.py:109-138 (periodic) */
#define RIDC_BURGERS_1D 2             /* problems.py:141-168 (Dirichlet) */
#define RIDC_REACTION_DIFFUSION_1D 3  /* periodic, f^N = rho u (1-u) */
#define RIDC_ADV_DIFF_2D 4            /* periodic, x-line implicit */
#define RIDC_REACTION_DIFFUSION_2D 5  /* periodic, x-line implicit */

/* Structured problem: replaces SplitIVP's callables + dense operator
 * (ivp.py:31-66).  State layout: ny rows of nx points, row-major. */
typedef struct ridc_problem {
    int32_t kind;
    int32_t nx;        /* points per x-line (1-D: the dimension) */
    int32_t ny;        /* lines (1 for 1-D kinds) */
    int32_t reserved;
    double c_x, c_y;   /* advection speeds (adv-diff) */
    double d_x, d_y;   /* diffusivity: x (stiff, implicit), y (explicit) */
    double rho;        /* logistic reaction rate */
    double h_x, h_y;   /* grid spacings */
} ridc_problem;

typedef struct ridc_ctx ridc_ctx;

/* run flags */
#define RIDC_RECORD_TRAJECTORY 1u  /* RidcConfig.record_trajectory */
#define RIDC_TICK_ONLY 2u          /* never use the resident marches -- single-level FEBE or
                                      the multi-level one (testing: they must agree bitwise
                                      with the tick kernel) */
#define RIDC_RESIDENT_SEGMENTS 4u  /* accepted for compatibility: segmented lines march
                                      resident by default */

/* Engine geometry / accounting, for reports and tests. */
typedef struct ridc_info {
    int32_t levels;
    int32_t restarts;
    int64_t steps;
    int64_t ticks_per_interval;   /* steps/restarts + levels(levels-1)/2 */
    int64_t kernel_launches;      /* launches per ridc_run (graph nodes) */
    int32_t tile;                 /* output points per work item */
    int32_t halo;                 /* truncation halo per side (0: exact line solve) */
    int32_t items_per_level;      /* work items per level-step */
    int32_t threads;              /* CUDA threads per item */
    int64_t ring_vectors;         /* device vectors held by all level rings */
    double lambda;                /* decay factor of the shifted operator's factors */
    double r;                     /* stiffness dt*d_x/h_x^2 */
    int32_t path;                 /* marching path in effect (after the last run):
                                     RIDC_PATH_TICK / _RESIDENT_FEBE / _RESIDENT_LEVELS /
                                     _CARRY_FEBE / _SWEEP_FEBE / _SWEEP2D_FEBE /
                                     _SWEEP2D_LEVELS / _SWEEP_LEVELS / _SWEEP_WARP_FEBE /
                                     _CARRY_LEVELS / _RESIDENT_CARRY_LEVELS /
                                     _WARP_CARRY_FEBE */
    int32_t fell_back;            /* 1: a resident march could not get its co-resident
                                     SMs at run time and the tick graph replaced it */
} ridc_info;

#define RIDC_PATH_TICK 0             /* one fused tick kernel per pipeline tick (CUDA graph) */
#define RIDC_PATH_RESIDENT_FEBE 1    /* one cooperative launch marches every FEBE step */
#define RIDC_PATH_RESIDENT_LEVELS 2  /* one cooperative launch per interval, all levels */
#define RIDC_PATH_CARRY_FEBE 3       /* one cooperative launch marches every FEBE step, tiles
                                        exchange two carries per step (periodic RD lines) */
#define RIDC_PATH_SWEEP_FEBE 4       /* one launch per FEBE step, every SM sweeps a contiguous
                                        range once (long periodic RD lines, CUDA graph) */
#define RIDC_PATH_SWEEP2D_FEBE 5     /* one launch per FEBE step on a 2-D grid, every CTA sweeps a
                                        row block reading each row once (CUDA graph) */
#define RIDC_PATH_SWEEP2D_LEVELS 6   /* one launch per pipeline tick on a 2-D grid, every CTA sweeps
                                        a row block for each active level (CUDA graph) */
#define RIDC_PATH_SWEEP_LEVELS 7     /* one launch per pipeline tick on a long 1-D line, every SM
                                        sweeps its range for each active level (CUDA graph) */
#define RIDC_PATH_SWEEP_WARP_FEBE 8  /* one launch per FEBE step, every warp sweeps a contiguous
                                        range once (lines of >= 512 x 12 x SMs points, CUDA graph) */
#define RIDC_PATH_CARRY_LEVELS 9     /* one launch per pipeline tick on a 1-D line of 512-point
                                        chunks, one chunk per warp, carries exchanged between
                                        neighbouring chunks (CUDA graph) */
#define RIDC_PATH_RESIDENT_CARRY_LEVELS 10  /* RIDC-2 on a periodic RD line: one cooperative launch per
                                        interval, both levels' tiles held on the SMs, carries
                                        exchanged between tiles */
#define RIDC_PATH_WARP_CARRY_FEBE 11 /* one cooperative launch marches every FEBE step, one
                                        512-point chunk per warp, chunks exchange two carries per
                                        step (shared memory within a CTA, L2 between CTAs) */

/*
 * Create a run context (RidcConfig validation engine.py:71-87, _prepare
 * engine.py:465-473).  weights: packed quadrature tables (steady j=1..L-1,
 * then startup (j, n) for j=2..L-1, n=0..j-2; j+1 doubles each) as produced
 * by quadrature.pack_weight_tables; nweights its length.  device: CUDA
 * ordinal.  All device memory, the factor tables and the CUDA graph of the
 * whole run are set up here, outside any timed region.
 */
int ridc_create(const ridc_problem *problem, double t_start, double t_end,
                int32_t levels, int64_t steps, int32_t restarts,
                const double *weights, int64_t nweights,
                int32_t device, uint32_t flags, ridc_ctx **out);

/* One full run from host buffers (H2D of y0, marching, D2H of results).
 * final_host (n); level_finals_host (levels*n) or NULL; traj_host
 * ((steps+1)*n) or NULL (requires RIDC_RECORD_TRAJECTORY); wall_seconds:
 * device time of the marching only (engine.py:482-488), may be NULL. */
int ridc_run(ridc_ctx *ctx, const double *y0_host, double *final_host,
             double *level_finals_host, double *traj_host, double *wall_seconds);

/* Same with device-resident input/output (state already in HBM). */
int ridc_run_device(ridc_ctx *ctx, const double *y0_dev, double *final_dev,
                    double *wall_seconds);

int ridc_info_get(const ridc_ctx *ctx, ridc_info *info);
/* Watchdog of the resident marches' in-kernel neighbour waits
 * (RidcConfig.watchdog_seconds, engine.py:432-439): a wait exceeding it
 * aborts the march with RIDC_E_PROTOCOL.  Default 30 s. */
int ridc_set_watchdog(ridc_ctx *ctx, double seconds);
int ridc_destroy(ridc_ctx *ctx);
const char *ridc_last_error(const ridc_ctx *ctx);   /* ctx may be NULL: thread's last error */

/* ---- single operators (device buffers, synchronous on the device's default stream) ---- */

#define RIDC_OP_STIFF 0     /* f^S(u) */
#define RIDC_OP_NONSTIFF 1  /* f^N(u) */
int ridc_op_apply(const ridc_problem *problem, int32_t op, const double *in_dev,
                  double *out_dev, int32_t device);

/* x_dev = (I - coeff * L_S)^{-1} rhs_dev */
int ridc_op_solve(const ridc_problem *problem, double coeff, const double *rhs_dev,
                  double *x_dev, int32_t device);

/* One level step: rhs = eta + dt f^N(eta) + sum_k (cs[k] f^S(win[k]) + cn[k] f^N(win[k]))
 * then out = (I - dt L_S)^{-1} rhs.  nwin = 0 for the predictor.  win_dev is a
 * HOST array of nwin device pointers.  Returns RIDC_E_NONFINITE if out has
 * non-finite entries. */
int ridc_op_step(const ridc_problem *problem, double dt, const double *eta_dev,
                 int32_t nwin, const double *const *win_dev, const double *cs,
                 const double *cn, double *out_dev, int32_t device);

/* Reference-form level step (LevelWindow with f^S / f^N rows, engine.py:200-231):
 * rhs = eta + dt f^N(eta) + sum_k ca[k] rows[k]; out = (I - dt L_S)^{-1} rhs.
 * rows_dev: HOST array of nrows (<= 24) device pointers. */
int ridc_op_step_rows(const ridc_problem *problem, double dt, const double *eta_dev,
                      int32_t nrows, const double *const *rows_dev, const double *ca,
                      double *out_dev, int32_t device);

/* Diagnostic: clock64 phase trace of the last tick launch (CTA 0, 8 items x 16
 * stamps); only when the context was created with RIDC_PHASE_TIMING=1. */
int ridc_debug_phase_trace(const ridc_ctx *ctx, long long *out, int32_t n);

/* ---- lagged level pipeline, one level per GPU (one process per GPU) ----
 *
 * Replaces _pipelined_interval / LevelBuffer (engine.py:284-459) with levels
 * on different devices.  Rank j owns level j.  Its tick kernel writes each
 * new state tile both to its own ring and -- peer stores over NVLink -- to
 * level j+1's inbox ring; after the kernel, a device-side stream write
 * publishes the watermark into the consumer's memory (LevelBuffer.watermark,
 * :299).  Level j waits on its own inbox watermark and on the release counter
 * its consumer writes back (LevelBuffer.released, :300) with device-side
 * stream waits (cuStreamWaitValue64), so no host round trip sits between
 * ticks.  Slots are indexed by the global step number across restarts. */

typedef struct ridc_pipe ridc_pipe;

/* Size of the opaque blob a rank exports for its neighbours (IPC handle of
 * its mailbox = inbox ring + watermark + release counter). */
int64_t ridc_pipe_handle_bytes(void);

/* Create the rank owning `level` (0..levels-1) on `device`.  inbox_capacity:
 * inbox ring slots (0: default 2*level+13; at least level+3 -- the window of
 * level+1 steps plus the deferred publication of the resident march -- else
 * RIDC_E_CONFIG; >= steps/restarts+1 makes every rank runnable to completion
 * without its consumer, e.g. ranks driven one after another on one device).
 * watchdog_seconds bounds every wait (PipelineProtocolError on expiry,
 * engine.py:432-439).  Watermark waits on a producer on ANOTHER device use
 * CU_STREAM_WAIT_VALUE_FLUSH where the device supports flushing remote
 * writes, else an in-kernel acquire poll at system scope. */
int ridc_pipe_create(const ridc_problem *problem, double t_start, double t_end,
                     int32_t levels, int64_t steps, int32_t restarts,
                     const double *weights, int64_t nweights, int32_t level,
                     int32_t device, int32_t inbox_capacity, double watchdog_seconds,
                     ridc_pipe **out);
/* Export this rank's handles into blob (ridc_pipe_handle_bytes() bytes). */
int ridc_pipe_export(ridc_pipe *p, void *blob);
/* Connect to the previous level (prev_blob; NULL for level 0) and the next
 * level (next_blob; NULL for the top level).  Blobs from the same process
 * are used as direct device pointers, others through cudaIpcOpenMemHandle. */
int ridc_pipe_connect(ridc_pipe *p, const void *prev_blob, const void *next_blob);
/* Run restart interval `interval` (0..restarts-1) of this rank's level from
 * state0_dev (the interval's initial state, on this device); final_dev
 * receives this level's state at the interval end (the top rank's is the
 * solution and the next interval's state0).  Blocks until the level is done
 * (bounded by the watchdog).  wall_seconds: device time of this rank. */
int ridc_pipe_run_interval(ridc_pipe *p, int32_t interval, const double *state0_dev,
                           double *final_dev, double *wall_seconds);
/* Zero this rank's mailbox counters (watermarks, release and progress
 * counters).  The stream-memop protocol counts global step numbers, so
 * before a SECOND run of the same ranks every rank resets -- after all ranks
 * finished the previous run and before any starts the next (barrier, reset,
 * barrier; distributed.PipelineRank.run_device / ConcurrentPipeline /
 * GridPipeline do this).  The resident mode's flags carry a run epoch and
 * need no reset. */
int ridc_pipe_reset(ridc_pipe *p);
int ridc_pipe_info(const ridc_pipe *p, ridc_info *info);
/* Resident level march (default where the line qualifies: 1-D, one
 * co-resident CTA per segment): the rank's whole interval is ONE cooperative
 * launch whose CTAs poll per-segment publish / release flags in peer memory
 * (the LevelBuffer watermark / released protocol, engine.py:299-331) instead
 * of per-step stream memory operations.  enable = 0 selects the per-step
 * tick kernel + stream memops.  Call before ridc_pipe_export on EVERY rank
 * (the mode travels in the blob; neighbours must agree).  Never run ranks
 * of the resident mode concurrently on one device (their kernels wait on
 * each other).  ridc_pipe_resident reports the mode in effect. */
int ridc_pipe_set_resident(ridc_pipe *p, int32_t enable);
int ridc_pipe_resident(const ridc_pipe *p);
/* Levels x row shards (the layer that uses every GPU
 * when p < #GPUs): the rank owning level `level` of row shard `shard`
 * (global rows [ny*shard/nshards, ny*(shard+1)/nshards)), 2-D kinds, stream
 * memops only.  Besides the pipeline's watermark / release protocol with
 * (level-1, shard) and (level+1, shard), every step it delivers its first and
 * last row into the ghost rows of (level, shard-+1)'s own ring and of
 * (level+1, shard-+1)'s inbox, each with its own watermark, and releases
 * inbox slots to all three producers; ny periodic (shard 0's upper
 * neighbour is shard nshards-1).  run_interval takes the GLOBAL state0 and
 * returns this shard's rows (nrows x nx) of the level's final. */
int ridc_pipe_create_shard(const ridc_problem *problem, double t_start, double t_end,
                           int32_t levels, int64_t steps, int32_t restarts,
                           const double *weights, int64_t nweights, int32_t level,
                           int32_t shard, int32_t nshards, int32_t device,
                           int32_t inbox_capacity, double watchdog_seconds, ridc_pipe **out);
/* blobs[8]: (level-1, shard), (level-1, shard-1), (level-1, shard+1),
 * (level+1, shard), (level+1, shard-1), (level+1, shard+1), (level, shard-1),
 * (level, shard+1); NULL exactly where the level does not exist. */
int ridc_pipe_connect_shard(ridc_pipe *p, const void *const *blobs);
int ridc_pipe_destroy(ridc_pipe *p);
const char *ridc_pipe_last_error(const ridc_pipe *p);

/* ---------------------------------------------------------------------------
 * ARK (IMEX) comparators on the device: the coupled DIRK / explicit pair step
 * of steppers.ark_step (steppers.py:122-142) marched by integrate_ark
 * (steppers.py:145-155), stage sums as kernels.stage_accumulate
 * (kernels.py:149-158).  Tableaus are s x s row-major (tableaus.py:82-127 for
 * imex3 / imex4): a_implicit lower triangular, a_explicit strictly lower.
 * Non-finite results raise RIDC_E_NONFINITE with the reference's message
 * "ARK march produced non-finite entries at step k".
 */
typedef struct ridc_ark_ctx ridc_ark_ctx;

int ridc_ark_create(const ridc_problem *problem, double t_start, double t_end,
                    int64_t steps, int32_t stages, const double *a_implicit,
                    const double *a_explicit, const double *b_implicit,
                    const double *b_explicit, int32_t device, ridc_ark_ctx **out);
int ridc_ark_run(ridc_ark_ctx *ctx, const double *y0_host, double *final_host,
                 double *wall_seconds);
int ridc_ark_run_device(ridc_ark_ctx *ctx, const double *y0_dev, double *final_dev,
                        double *wall_seconds);
int ridc_ark_info(const ridc_ark_ctx *ctx, int64_t *kernel_launches, int32_t *items_per_step);
/* The path the stages run on: RIDC_PATH_CARRY_LEVELS (periodic RD lines of
 * 512-point chunks: every stage one carry-exchange launch) or RIDC_PATH_TICK;
 * -1 for a NULL context. */
int ridc_ark_path(const ridc_ark_ctx *ctx);
int ridc_ark_destroy(ridc_ark_ctx *ctx);
const char *ridc_ark_last_error(const ridc_ark_ctx *ctx);

/* ---------------------------------------------------------------------------
 * 2-D row shards under the levels: the grid's rows
 * split into nshards contiguous shards, each running every level on its rows
 * plus one ghost row per side, the boundary rows of every newly written slot
 * exchanged after each tick.  This group runs all shards on one device in
 * lockstep and reproduces ridc_run bitwise; 2-D kinds only.
 */
typedef struct ridc_shards ridc_shards;

int ridc_shards_create(const ridc_problem *problem, double t_start, double t_end,
                       int32_t levels, int64_t steps, int32_t restarts,
                       const double *weights, int64_t nweights, int32_t nshards,
                       int32_t device, ridc_shards **out);
/* The same shards, one stream per shard on devices[s] (neighbours may share a
 * device): per tick each shard waits until both neighbours copied their
 * boundary rows of the previous tick into its ghost rows (device-side
 * mailbox, cuStreamWaitValue64), runs its tick, copies its own boundary rows
 * into the neighbours' ghost rows (peer copies across devices) and raises
 * their mailboxes.  No host synchronisation per tick; a stalled neighbour
 * becomes RIDC_E_PROTOCOL after watchdog_seconds. */
int ridc_shards_create_multi(const ridc_problem *problem, double t_start, double t_end,
                             int32_t levels, int64_t steps, int32_t restarts,
                             const double *weights, int64_t nweights, int32_t nshards,
                             const int32_t *devices, double watchdog_seconds,
                             ridc_shards **out);
int ridc_shards_run(ridc_shards *g, const double *y0_host, double *final_host,
                    double *wall_seconds);
int ridc_shards_info(const ridc_shards *g, int64_t *kernel_launches);
int ridc_shards_destroy(ridc_shards *g);
const char *ridc_shards_last_error(const ridc_shards *g);

#ifdef __cplusplus
}
#endif

#endif /* RIDC_B200_H */
