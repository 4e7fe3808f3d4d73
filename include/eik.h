/*
 * eik.h -- C ABI of the B200-native cell-sweep Eikonal solver (pHCM hot path, arXiv 1306.4743).
 *
 * Problem exported (Eq. (1)-(2)):
 *   |grad u| F = 1 on the (n+1)^3 uniform grid of [0, n h]^3, u = q on the exit set Q'
 *   (exits may be anywhere; reading R8), values outside the cube are +inf,
 *   discretised by the first-order upwind scheme of Eq. (2) and solved to the
 *   discrete fixed point (kappa = 0; reading R13) by cell-level Gauss-Seidel
 *   processing (HCM, Alg. 1-2) scheduled on the GPU (pHCM Alg. 3 analogue).
 *
 * Layout of every array argument: contiguous, lexicographic with i fastest,
 *   idx = i + (n+1)*(j + (n+1)*k),  M = (n+1)^3
 * dtype: float (EIK_F32) or double (EIK_F64) for F, exit_vals and U_out; uint8 for exit_mask.
 *
 * Ownership: the caller owns F, exit_mask, exit_vals, U_out (valid until the call returns).
 * The ctx owns its scratch (padded cell tiles, keys, flags, worklists), grown lazily, reused
 * across solves, freed by eik_destroy.  One ctx per host thread; no internal locking.
 *
 * Errors: every call returns an eik_status; text via eik_last_error.  Nothing throws or aborts
 * across the ABI.  On EIK_EINVAL U_out is untouched.
 */
#ifndef EIK_H_
#define EIK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EIK_ABI_VERSION 4   /* 3: eik_stats gained h2d_bytes, d2h_bytes; 4: eik_get_trace, EIK_OPT_TRACE */

typedef struct eik_ctx eik_ctx;

typedef enum {
    EIK_OK = 0,
    EIK_EINVAL = 1,     /* bad argument or input data (see eik_solve); U_out untouched      */
    EIK_ENOMEM = 2,     /* device scratch allocation failed                                  */
    EIK_ECUDA = 3,      /* a CUDA runtime error (message carries cudaGetErrorString)          */
    EIK_ENOTSUP = 4,    /* device is not compute capability 10.x (sm_100a build)              */
    EIK_EINTERNAL = 5   /* internal limit hit (e.g. max rounds) -- a bug or a debug knob      */
} eik_status;

typedef enum { EIK_F32 = 0, EIK_F64 = 1 } eik_precision;
typedef enum { EIK_DFSM = 0, EIK_DLSM = 1 } eik_sweep_method;   /* eik_solve_sweep */

/* Options for eik_set_option (all optional; defaults in brackets). */
typedef enum {
    EIK_OPT_BIN_WIDTH = 0,   /* Delta of the priority bins, in units of time (same units as U).
                                Cells whose key lies in [kmin, kmin + Delta] are processed in a
                                round ("cells in the lowest range of values").  <= 0 or
                                +inf = every queued cell each round.  [+inf]                    */
    EIK_OPT_MAX_ROUNDS = 1,  /* safety cap on scheduler rounds; exceeding it = EIK_EINTERNAL
                                [1e9]                                                           */
    EIK_OPT_LOOP_MODE = 2,   /* 0 = asynchronous persistent kernel (CTAs pull cells from a
                                device ring with ticket pops; no rounds, no host round-trip)
                                [default];
                                1 = bulk-synchronous rounds driven by the host (debug);
                                2 = bulk-synchronous rounds in a CUDA graph WHILE node, no host
                                round-trip per round.  The bin width applies to modes 1-2.       */
    EIK_OPT_COLLECT_STATS = 3, /* 1 = count point updates/writes/sweeps on device [1]           */
    EIK_OPT_TIME_CELL_EVENTS = 4, /* 1 = (host loop and async modes) bracket every cell-sweep
                                    kernel launch with CUDA events; sum in
                                    eik_stats.ms_cell_events [0]                                 */
    EIK_OPT_ASYNC_DEFER = 5, /* async mode readiness test on a popped cell (it is re-queued if
                                an adjacent cell blocks it): 0 none; 1 a neighbour is running;
                                2 ... or is queued with a smaller (key, index); 3 ... with a key
                                smaller by > bin width; 4 as 2 across inflow faces only; 5 ...
                                or is queued from an older activation generation; 6 ... or is
                                queued with a smaller (generation, key, index); 7 ... with a
                                smaller (key, generation, index); 8 automatic: 6 until the solve
                                has run more than 6 processings per processed cell, then 2 [8];
                                9 as 6 with the activation LEVEL (1 + the smallest level of a
                                cell's taggers) in place of the generation (1 + the largest):
                                30-60 % fewer processings but a narrower front -- faster on
                                maze-like inputs (shell maze at 320^3: 29.8 -> 20.4 ms), slower
                                on open ones (C3 5.5 -> 7.0 ms).
                                2, 6, 7 and 9 are strict total orders: the smallest queued cell
                                is never deferred                                               */
    EIK_OPT_MAX_SWEEPS = 6,  /* sweeps per cell processing before the cell saves its active
                                points and re-queues itself (bounds the round length, which is
                                the slowest cell's); 0 = until convergence; -1 = automatic: 4
                                in the round modes, 0 in async mode [-1]                         */
    EIK_OPT_TIMEOUT_S = 7,   /* device-side watchdog: the scheduler loop stops and the solve
                                returns EIK_EINTERNAL after this many seconds [120]              */
    EIK_OPT_KAPPA = 8,       /* early termination threshold kappa >= 0 [0 = exact].
                                eik_solve: a point change <= kappa activates no neighbour point
                                and a border change <= kappa tags no neighbour cell (P:1192-
                                1193).  eik_solve_sweep: stop after the first sweep whose
                                largest change is <= kappa.  kappa > 0 returns an
                                approximation of the discrete solution (values >= it; P:1187
                                gives no error bound)                                            */
    EIK_OPT_CELL_KEY = 9,    /* cell value of a tag (Alg. 1 line 9): 0 = Eq. (3), the smallest
                                newly updated inflow value, reset to +inf on removal [0];
                                1 = the legacy Eq. (4): V_max + D / F(y), never
                                reset.  Orders work only (bin width < inf, async readiness);
                                the fixed point is the same                          */
    EIK_OPT_TRACE = 10,      /* diagnostics, async mode: record up to this many cell processings
                                (cell, tagger, pop / swept / end times, sweeps, flags, generation)
                                for eik_get_trace; 0 = off [0]                                  */
    EIK_OPT_CELL_KERNEL = 11 /* cell-sweep kernel of the async scheduler for r = 16 (kappa = 0,
                                no sweep cap): 0 = one thread per point, the point wavefront
                                used for every configuration [0]; 1 = 2x2x2 micro-blocks, one
                                thread per block and block activity flags (an experiment that
                                measured slower; kept for comparison).  Same fixed point
                                                                                      */
} eik_option;

/* Work and time counters of the last successful solve. */
typedef struct {
    int64_t  M;                 /* (n+1)^3 real gridpoints                                   */
    int64_t  padded_points;     /* (cps*r)^3 stored points                                   */
    int64_t  J;                 /* cells, cps^3                                              */
    int32_t  cells_per_side;    /* cps = ceil((n+1)/r)                                       */
    int32_t  cell_size;         /* r                                                         */
    int32_t  precision;         /* eik_precision                                             */
    int32_t  pad_;
    uint64_t point_updates;     /* local solves executed (Alg. 2 line 5)                     */
    uint64_t point_writes;      /* strict decreases (Alg. 2 line 7)                          */
    uint64_t cell_processings;  /* heap-removal analogue (Alg. 1 line 4)                     */
    uint64_t cell_sweeps;       /* sweeps over all processings (AvS numerator)       */
    uint64_t real_points_processed; /* sum over processings of real points in the cell      */
    uint32_t rounds;            /* scheduler rounds (select -> process -> re-activate)       */
    uint32_t max_worklist;      /* largest number of cells processed in one round            */
    uint64_t bytes_min;         /* north-star minimum bytes: P_eq * M * (sF + sU), D.4       */
    uint64_t bytes_cell_alg;    /* algorithmic cell-sweep bytes: per processing
                                   (2 r^3 + 6 r^2) s read + (changed points) s written          */
    double   ms_ingest, ms_loop, ms_egress, ms_total;   /* CUDA events on the ctx stream      */
    double   ms_cell_device;    /* sum over rounds of the cell-sweep kernel's span (first CTA
                                   start to last CTA end, %globaltimer), any loop mode          */
    double   ms_cell_events;    /* sum of CUDA-event durations of the cell-sweep launches
                                   (EIK_OPT_TIME_CELL_EVENTS in host loop mode), else 0         */
    uint64_t cell_launches;     /* cell-sweep kernel launches that processed >= 1 cell
                                   (eik_solve_sweep: diagonal launches)                         */
    uint64_t grid_sweeps;       /* eik_solve_sweep: whole-grid sweeps, the last of which changed
                                   nothing (the FSM count of P:803, Table 4); else 0            */
    uint64_t h2d_bytes;         /* eik_solve_host: host->device bytes of the call (F and the mask
                                   copied; exit_vals copied, or -- page-locked -- only its exit
                                   values read in place); else 0                                */
    uint64_t d2h_bytes;         /* eik_solve_host: device->host bytes (U); else 0               */
} eik_stats;

/* Create a context on `device`.  cuda_stream: a cudaStream_t to enqueue on (e.g. torch's
 * current stream), or NULL to let the ctx create and own a non-blocking stream.
 * Returns EIK_ENOTSUP if the device is not sm_100. */
int eik_create(eik_ctx** out, int device, void* cuda_stream);

/* Change the stream subsequent solves enqueue on (NULL = the ctx's own stream). */
int eik_set_stream(eik_ctx* ctx, void* cuda_stream);

/* Set an eik_option.  EIK_EINVAL for an unknown option or a bad value. */
int eik_set_option(eik_ctx* ctx, int option, double value);

/* Solve with DEVICE pointers (CUDA device memory, e.g. torch CUDA tensors).
 *   n          >= 1 intervals per side (n+1 points per side)
 *   h          > 0, finite grid spacing (the problem's 1/n for [0,1]^3)
 *   F          M x dtype speeds; finite, >= 0; 0 = impassable (reading R11)
 *   exit_mask  M x uint8; nonzero = exit gridpoint; at least one exit (R10)
 *   exit_vals  M x dtype; q, read where exit_mask != 0; finite, >= 0 (R9; -0 -> +0)
 *   U_out      M x dtype; written only on EIK_OK: q at exits, the discrete solution at
 *              reachable points, +inf at unreachable ones (F = 0 walls, enclosed pockets)
 *   precision  EIK_F32 (storage and arithmetic in fp32, R14) or EIK_F64
 *   cell_size  r in {4, 8, 16} gridpoints per cell side; (n+1) need not be a
 *              multiple of r: cells are padded with never-updated "outside" points (R12)
 * Blocking: returns after the work on the ctx stream completes, so the status (including
 * device-detected input errors) is final.
 * EIK_EINVAL: null ctx/pointer, n < 1, h <= 0 or non-finite, bad precision or cell_size,
 * any F < 0 / NaN / inf, any exit q < 0 / NaN / inf, or no exit point. */
int eik_solve(eik_ctx* ctx, int64_t n, double h, const void* F, const uint8_t* exit_mask,
              const void* exit_vals, void* U_out, int precision, int cell_size);

/* Same contract with HOST pointers (pageable or pinned).  The host->device copies of the
 * inputs and the device->host copy of U happen inside the call (the e2e path). */
int eik_solve_host(eik_ctx* ctx, int64_t n, double h, const void* F, const uint8_t* exit_mask,
                   const void* exit_vals, void* U_out, int precision, int cell_size);

/* Whole-grid sweeping: the paper's comparison methods (P:140-149 FSM / LSM, P:175-186
 * Detrixhe's DFSM, P:795-801 DLSM) on the same device tiles, same contract
 * and arguments as eik_solve plus
 *   method     EIK_DFSM: Gauss-Seidel sweeps of Eq. (2) in the 2^3 directions, sweep s in
 *              direction s mod 8 (bit 0/1/2 = x/y/z descending), until a sweep changes
 *              nothing (counted).  The ordering is a cell-diagonal wavefront with a
 *              point-plane wavefront inside each cell: the same values after every sweep as
 *              the lexicographic FSM, hence the same sweep count.
 *              EIK_DLSM: DFSM that skips a cell whose inputs did not change since it last
 *              ran (locking at cell granularity): same values and sweep count as DFSM.
 * The sweep count is eik_stats.grid_sweeps; EIK_OPT_MAX_ROUNDS caps it (EIK_EINTERNAL).
 * EIK_EINVAL additionally for an unknown method. */
int eik_solve_sweep(eik_ctx* ctx, int64_t n, double h, const void* F, const uint8_t* exit_mask,
                    const void* exit_vals, void* U_out, int precision, int cell_size, int method);

/* Stats of the last successful solve.  EIK_EINVAL if ctx/out is NULL. */
int eik_get_stats(const eik_ctx* ctx, eik_stats* out);

/* Diagnostics of the last solve (for profiling; layout may change between ABI versions):
 * out[0] sum of per-processing SM cycles, out[1] max, out[2] wavefront plane steps executed,
 * out[3] processings, out[4 + s] number of processings that ran s sweeps (s = 31: >= 31),
 * out[36..39] cycles in staging / plane-mask / plane steps / write-back, out[40] active-list
 * iterations, out[41] async-mode deferrals, out[42 + 2r], out[43 + 2r] = cells and span (ns) of
 * round r (round modes, r < 1024), out[2090], out[2091] cycles in tile loads / halo loads.
 * Copies min(n, 2092) values.  EIK_EINVAL if ctx/out is NULL or n < 0. */
int eik_get_debug(const eik_ctx* ctx, uint64_t* out, int n);

/* Processing trace of the last solve (EIK_OPT_TRACE > 0, async mode): copies up to
 * max_entries entries of 8 uint32 each into out (host memory, 32 bytes per entry):
 *   {cell, id of the processing that last tagged it (0xFFFFFFFF: seeded), t_pop, t_swept,
 *    t_end, sweeps, state flags taken at the pop, point writes}
 * with times in ns since the solve's start (t_swept: sweeps and write-back done, before the
 * neighbour tags; t_end: tags done).  The entry index is the processing id.
 * Returns the number of entries copied (0 if tracing is off), or -EIK_EINVAL / -EIK_ECUDA. */
int64_t eik_get_trace(const eik_ctx* ctx, uint32_t* out, int64_t max_entries);

/* Message of the last failing call on ctx (owned by ctx; valid until its next call).
 * eik_last_error(NULL) returns the message of the last failed eik_create. */
const char* eik_last_error(const eik_ctx* ctx);

/* Free scratch (and the ctx's own stream). NULL-safe. */
void eik_destroy(eik_ctx* ctx);

/* EIK_ABI_VERSION of the loaded library. */
int eik_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EIK_H_ */
