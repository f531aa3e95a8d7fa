/*
 * orca.h -- C ABI of liborca, the B200-native (sm_100a) ORCA crowd step.
 *
 * What it computes (arXiv 1908.10107, PAPER.md; "P:NN" = PAPER.md line NN):
 *   one synchronous time step of the ORCA agent update (§3):
 *     1. spatial binning of agents into a uniform grid of cell size r_obs (FLAME messages
 *        organised into spatial bins, Fig. 2 caption P:94);
 *     2. each agent reads its own and the 8 surrounding bins and keeps the k nearest
 *        agents strictly within r_obs, in (distance, id) order;
 *     3. one ORCA half-plane per observed neighbour (Fig. 1(b)-(c));
 *     4. the closest permitted velocity to the preferred one by an incremental 2-D LP
 *        (P:82-86), or the least-penetrating velocity when infeasible;
 *     5. explicit integration p' = p + dt v'.
 *   The cited ORCA geometry and every reading of a silent/garbled passage are listed in
 *   DESIGN.md §3.  No buffer or argument here carries a torch type.
 *
 * Conventions (all entry points):
 *   - Every function returns orca_status (0 = OK) except orca_destroy / orca_status_string
 *     / orca_last_error.  No C++ exception crosses the ABI.
 *   - Vectors are float32 x,y interleaved: "float[2n]" means n agents, element 2i = x of
 *     agent i, 2i+1 = y.  Agent id = index in the orca_set_agents arrays.
 *   - Pointer arguments may be HOST (pageable or pinned) or DEVICE (CUDA, same device as
 *     the context) memory; the library dispatches through unified addressing.  The library
 *     copies inputs (the caller keeps ownership of its buffers) and writes outputs into
 *     caller-allocated buffers.
 *   - A context is used by one host thread at a time.  orca_step is asynchronous on the
 *     context's stream (a call of more than two 64-step chunks waits for chunk q-2 before
 *     queuing chunk q, to re-derive the grid while it runs); every getter synchronises that
 *     stream.  orca_set_state_async / orca_get_state_async do not synchronise: their buffers
 *     are in use until orca_io_wait returns.
 *   - On error, orca_last_error() returns a thread-local human-readable message.
 */
#ifndef ORCA_H
#define ORCA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------------ */
typedef int32_t orca_status;
#define ORCA_OK 0
#define ORCA_ERR_INVALID_ARGUMENT 1 /* bad parameter, NaN/Inf input, null pointer */
#define ORCA_ERR_NOT_READY 2        /* step/get before set_agents */
#define ORCA_ERR_OUT_OF_MEMORY 3    /* cudaMalloc failed */
#define ORCA_ERR_CUDA 4             /* any other CUDA runtime error */
#define ORCA_ERR_NCCL 5             /* NCCL error (multi-GPU contexts) */
#define ORCA_ERR_CAPACITY 6         /* grid / halo / migration buffer too small */
#define ORCA_ERR_INTERNAL 7

/* Largest supported maxNeighbors (compile-time bound of the per-agent LP). */
#define ORCA_MAX_K 32

/* ---- parameters (BASELINE.json north_star order) ------------------------------------ *
 * timeStep      dt > 0, seconds: integration step ("simulation iteration").
 * neighborDist  r_obs > 0, metres: observation radius (Fig. 2 caption); it is also
 *               the grid cell size, so the 3x3 bins cover the r_obs disc.
 * maxNeighbors  k in [0, ORCA_MAX_K]: at most k nearest neighbours give half-planes.
 * timeHorizon   tau > 0, seconds: lookahead of the velocity obstacle (Fig. 1(b)).
 * radius        r > 0, metres: agent radius, global (Fig. 1(a)); R = 2r per pair.
 * maxSpeed      >= 0, m/s: speed cap |v| <= maxSpeed ("capped maximum speed").
 * All finite. */
typedef struct {
    float timeStep;
    float neighborDist;
    int32_t maxNeighbors;
    float timeHorizon;
    float radius;
    float maxSpeed;
} orca_params;

typedef struct orca_ctx orca_ctx; /* opaque, library-owned */

/* Per-context counters accumulated over all steps since creation / the last reset. */
typedef struct {
    int64_t steps;          /* orca_step iterations executed */
    int64_t agent_updates;  /* sum over steps of the agent count */
    int64_t infeasible;     /* agent-steps whose LP2 failed -> LP3 */
    int64_t degenerate;     /* agent-steps with a g1 or g2 event (DESIGN.md §3 Q15/Q9) */
    int64_t coincident;     /* g1: collision branch with w == 0 (Q15) */
    int64_t eps_parallel;   /* g2: an LP pair with |det| <= 1e-5 (Q9) */
    int64_t marginal;       /* g3: infeasible with max penetration < 1e-6 (reported only) */
    int64_t collision_pairs;/* neighbour pairs that took the collision branch (Q4) */
    int64_t removed;        /* agents removed at their goal (orca_set_goal_removal) */
    int64_t rebalances;     /* strip re-partitions since creation (orca_rebalance; automatic) */
    int64_t regrids;        /* grid re-derivations since creation (an agent reached the outer
                               cell ring; automatic, reading Q12) */
} orca_stats;

/* ---- lifecycle -------------------------------------------------------------------- */

/* Create a single-GPU context on CUDA device `device` (its own non-blocking stream).
 * Errors: INVALID_ARGUMENT (params out of range, out == NULL), CUDA. */
orca_status orca_create(const orca_params *params, int32_t device, orca_ctx **out);

/* Release all device memory, graphs and the stream.  NULL is a no-op. */
void orca_destroy(orca_ctx *ctx);

/* ---- state ------------------------------------------------------------------------ */

/* Load n >= 0 agents (copied).  pos, vel, prefVel: float[2n] (x,y interleaved); prefVel
 * is the preferred velocity held constant over steps (reading Q16) unless orca_set_goals
 * is called afterwards.  Freezes the grid: origin = fl32(min - r_obs) per axis, dims =
 * floor((max - origin)/r_obs) + 2 (reading Q12); later positions outside are clamped to
 * edge cells.  Bins the agents.  Clears any goals.  With the same n as the loaded state,
 * each agent keeps its last k-th-neighbour distance as its first search radius (by id; a
 * performance hint only -- the neighbour selection is exact for any radius).
 * Errors: INVALID_ARGUMENT (n < 0, NULL with n > 0, NaN/Inf), CAPACITY (grid larger than
 * 2^28 cells), OUT_OF_MEMORY, CUDA. */
orca_status orca_set_agents(orca_ctx *ctx, int64_t n, const float *pos, const float *vel,
                            const float *prefVel);

/* Replace the positions and velocities (float[2n] by id, host or device) of the loaded
 * agents and keep everything else: preferred velocities or goals, per-agent properties,
 * removals (entries of removed agents are ignored), counters, the LP-order step index and
 * each agent's search-radius hint.  The grid stays unless the new positions leave its
 * interior (then it is re-derived, reading Q12).  The per-frame upload of an application
 * that moves agents itself, or reloads a checkpoint of the same crowd.  Multi-rank
 * contexts: every rank calls it with the same arrays.  Synchronises.  Errors: NOT_READY,
 * INVALID_ARGUMENT (NULL, NaN/Inf for an agent present), CAPACITY, CUDA, NCCL. */
orca_status orca_set_state(orca_ctx *ctx, const float *pos, const float *vel);

/* Goal seeking ("The agent's velocity is in the direction of the goal location,
 * scaled to the walking speed"): goal float[2n] by id; from the next step on, the
 * preferred velocity is recomputed every step as g*min(1, prefSpeed/|g|), g = goal - pos.
 * Errors: NOT_READY, INVALID_ARGUMENT (NULL, NaN/Inf, prefSpeed < 0). */
orca_status orca_set_goals(orca_ctx *ctx, const float *goal, float prefSpeed);

/* Removal at the goal ("Once a person reaches the goal location they are removed from
 * the simulation. Once all people have reached their goal the simulation is ended."): with
 * goals set and radius > 0, an agent whose new position lies strictly within `radius` of its
 * goal leaves the simulation after that step -- it is no longer stepped or observed;
 * orca_get_state then reports NaN for it, orca_get_count counts the remaining agents (0 =
 * ended).  radius 0 disables.  Persists across orca_set_agents.  Errors: INVALID_ARGUMENT. */
orca_status orca_set_goal_removal(orca_ctx *ctx, float radius);

/* Constraint order of the per-agent LP ("based on the randomized incremental linear
 * program solver of Seidel"; reading Q8).  The feasible optimum does not depend on
 * the order; only the work does, and infeasible agents with a non-unique least-penetration
 * velocity can.
 *   mode 0 (default): greedy -- at each step the most violated half-plane not yet processed
 *          goes next, re-solved against the processed ones only; the LP ends as soon as no
 *          remaining half-plane is violated.
 *   mode 1: randomized -- the half-planes of agent `id` at step `t` are processed in the
 *          Fisher-Yates order of the counter-based hash of (seed, t, id) -- splitmix64
 *          finaliser, spelled out in DESIGN.md §3 -- where t = first_step for the next
 *          orca_step and grows by one per step (orca_set_agents does not reset it: to resume
 *          a checkpoint taken at step t, pass first_step = t).
 *   mode 2: neighbour order (nearest first), the sequential incremental LP as the oracle
 *          runs it; the work-unit kernel variant (orca_set_variant 3) runs in modes 1 and 2.
 * Persists across orca_set_agents.  Synchronises.  Errors: INVALID_ARGUMENT (mode not
 * 0/1/2, first_step outside [0, 2^31 - 2^24)). */
orca_status orca_set_lp_order(orca_ctx *ctx, int32_t mode, uint64_t seed, int64_t first_step);

/* Heterogeneous crowds ("an equal chance of being of radius 0.5 m, 0.75 m or 1 m ...
 * desired speed of 1 m/s, 1.33 m/s or 2 m/s. The maximum speed is adjusted to be 125% of
 * the desired speed"): per-agent radius, maxSpeed and prefSpeed, float[n] by id, each
 * nullable (NULL -> the global radius / maxSpeed / the orca_set_goals speed).  A pair uses
 * R = r_i + r_j; agent i's LP uses its own maxSpeed; with goals its preferred speed is its
 * own.  All three NULL returns to the global parameters.  Call after orca_set_agents (which
 * clears them).  The cell size stays neighborDist.  Errors: NOT_READY, INVALID_ARGUMENT
 * (radius <= 0, negative speed, NaN/Inf; on strips maxSpeed * timeStep >= neighborDist). */
orca_status orca_set_agent_props(orca_ctx *ctx, const float *radius, const float *maxSpeed,
                                 const float *prefSpeed);

/* active uint8[n] by id: 1 while the agent is in the simulation, 0 once removed.
 * Synchronises.  Errors: NOT_READY. */
orca_status orca_get_active(orca_ctx *ctx, uint8_t *active);

/* Enqueue n_steps >= 0 synchronous steps on the context stream: CUDA graphs of up to 64
 * step bodies, replayed, and re-captured only when a captured argument changed.  Before each
 * chunk of up to 64 steps, two maintenance checks run:
 *   - the grid is re-derived (reading Q12) once an agent reached its outer cell ring (a
 *     host-mapped flag: no synchronisation unless it is set);
 *   - strip contexts read one small fill report (a synchronisation) and re-partition when a
 *     strip could outgrow its buffers within the chunk (orca_rebalance).
 * Multi-rank contexts: every rank calls it with the same n_steps.  Errors: NOT_READY,
 * INVALID_ARGUMENT, CUDA, NCCL, CAPACITY, INTERNAL (an exchange timed out: a neighbour
 * rank did not step). */
orca_status orca_step(orca_ctx *ctx, int32_t n_steps);

/* Trace dump ("saving the agent data for each simulation step to a binary file",
 * P:177): run n_steps steps and write every step's positions (and velocities if vframes
 * != NULL) in id order into frames[s][n][2] (float, caller-owned; pinned host memory
 * lets the copy engine overlap frame s with step s+1 on a separate stream, double
 * buffered).  Removed agents read NaN.  Synchronises at the end.
 * Errors: INVALID_ARGUMENT (NULL frames, multi-rank context), NOT_READY, CUDA. */
orca_status orca_step_trace(orca_ctx *ctx, int32_t n_steps, float *frames, float *vframes);

/* Current positions / velocities in id order into caller buffers float[2n] (either may
 * be NULL).  Synchronises.  Errors: NOT_READY, CUDA. */
orca_status orca_get_state(orca_ctx *ctx, float *pos, float *vel);

/* ---- asynchronous per-step I/O ---------------------------------------------------------
 * The same operations as orca_set_state / orca_get_state (each iteration observes the
 * agents' positions and velocities; the per-step state leaves the GPU), enqueued
 * without any host synchronisation, so that an application streaming state in and out
 * every frame overlaps step s with the upload of frame s+1 and the read-back of frame s-1
 * (host->device and device->host run on two copy streams; two slots each, so at most two
 * uploads and two read-backs are in flight).  Pass pinned host memory (or device memory)
 * for the overlap; pageable memory works but is staged synchronously by CUDA.
 *
 * orca_set_state_async: pos, vel float[2n] by id, as orca_set_state.  The caller must not
 * modify them until orca_io_wait returns.  The grid stays; positions outside its interior
 * are clamped for the steps already enqueued (exact, reading Q12) and the grid is re-derived
 * before a later step.  A NaN/Inf is reported by orca_io_wait, or earlier by an orca_step
 * that re-derives the grid first (INVALID_ARGUMENT; the context then needs orca_set_agents).  Strip contexts (more than one strip) take the synchronous
 * orca_set_state.  Errors: NOT_READY, INVALID_ARGUMENT (NULL), OUT_OF_MEMORY, CUDA.
 *
 * orca_get_state_async: the state after all previously enqueued steps into caller buffers
 * float[2n] (either may be NULL), valid once orca_io_wait returns.  Loopback strip contexts
 * take the synchronous orca_get_state.  Errors: NOT_READY, INVALID_ARGUMENT (multi-rank),
 * OUT_OF_MEMORY, CUDA.
 *
 * orca_io_wait: blocks until every enqueued upload, step and read-back is complete.
 * Errors: INVALID_ARGUMENT (a non-finite upload, see above), CUDA. */
orca_status orca_set_state_async(orca_ctx *ctx, const float *pos, const float *vel);
orca_status orca_get_state_async(orca_ctx *ctx, float *pos, float *vel);
orca_status orca_io_wait(orca_ctx *ctx);

/* One frame of the per-frame loop in one call: upload pos_in / vel_in (float[2n] by id, like
 * orca_set_state_async), step once, and read the stepped positions / velocities back into
 * pos_out / vel_out (float[2n] by id, either may be NULL; like orca_get_state_async) -- no host
 * synchronisation; complete after orca_io_wait.  Results equal orca_set_state_async ->
 * orca_step(1) -> orca_get_state_async bit for bit.  On one strip it skips work those three
 * calls repeat: the step's own next-step binning is left undone, the next frame bins its upload
 * in place in the work arrays, the read-back un-permutes the work arrays, and any other call
 * first completes the pending binning.  Strips, n = 0 or a pending grid re-derivation take the
 * three calls.  The buffers must stay untouched until orca_io_wait (pinned host memory for the
 * overlap).  Errors: as the three calls. */
orca_status orca_step_io_async(orca_ctx *ctx, const float *pos_in, const float *vel_in, float *pos_out,
                               float *vel_out);

/* Number of agents currently held (multi-GPU: held by this rank). */
orca_status orca_get_count(orca_ctx *ctx, int64_t *n);

/* ---- introspection (tests / bench; not needed for simulation) ----------------------- */

/* Frozen grid: origin[2] (fp32 values widened to double), cell size, dims {nx, ny}. */
orca_status orca_get_grid(orca_ctx *ctx, double origin[2], float *cs, int32_t dims[2]);

/* Cell (cx, cy) of every agent for the current state, id order, int32[n] each. */
orca_status orca_debug_cells(orca_ctx *ctx, int32_t *cx, int32_t *cy);

/* Compute (but do NOT apply) the next step for the current state, id order:
 * vnew float[2n] (nullable), flags uint8[n] (nullable; bit0 infeasible, bit1 g1
 * coincident, bit2 g2 eps-parallel, bit3 g3 marginal), nbr int32[n*k] neighbour ids in
 * (distance, id) order padded with -1 (nullable), cnt int32[n] (nullable).
 * Runs the same device code as orca_step.  Synchronises. */
orca_status orca_debug_step(orca_ctx *ctx, float *vnew, uint8_t *flags, int32_t *nbr,
                            int32_t *cnt);

/* Work of one step on the current state, counted by an instrumented dry run of the same
 * kernel (not applied): out[0] candidates the kernel read (its fine-column runs within the
 * search radius), out[1] half-planes built, out[2] LP constraint checks, out[3] LP1 inner
 * iterations, out[4] LP3 projected lines, out[5] agents in the 3x3 bins around every agent
 * (the paper's candidate set, P:94 / P:98: SURVEY §8(d)'s c_cand).  Used for the ALU
 * roofline.  Synchronises. */
orca_status orca_debug_work(orca_ctx *ctx, int64_t out[6]);

/* Counters (synchronises).  orca_reset_stats zeroes them. */
orca_status orca_get_stats(orca_ctx *ctx, orca_stats *out);
orca_status orca_reset_stats(orca_ctx *ctx);

/* Kernel variant of the fused step (all compute the same result bit for bit; chosen by
 * measurement): -1 = automatic (default: 1 for strips of fewer than ~17k
 * agents, where the step is latency bound, else 0), 0 = one thread per agent with a
 * shared-memory top-k list, 1 = an 8-lane group per agent, 2 = one thread per agent with a
 * register top-k list (k <= 16; else shared memory), 3 = variant 0 with the paper's
 * work-unit LP2 (lanes that need no re-solve evaluate the constraints of lanes
 * that do) in the sequential LP orders (orca_set_lp_order modes 1 and 2; in the greedy order
 * it runs variant 0's LP), 4 = two lanes per agent (each scans every other candidate into its
 * own top-k list, the lists are merged exactly, the lanes build every other half-plane and
 * share the greedy LP2; k <= 14 and the greedy order, else it runs as 0).  Same results bit
 * for bit.  Errors: INVALID_ARGUMENT. */
orca_status orca_set_variant(orca_ctx *ctx, int32_t variant);

/* Lanes per queued infeasible agent in the least-penetration kernel: 1 = one thread
 * per agent, 4 / 8 / 16 = a lane group per agent (projected lines one per lane, LP1 bounds
 * by an exact group scan), -1 = automatic (default; one thread per agent at every size since
 * the greedy LP3, chosen by measurement).  Same results bit for bit.  Only
 * strips whose LP3 is queued use it: where LP3 runs inside the step kernel (see
 * orca_set_lp3_inline) this setting has no effect.  Errors: INVALID_ARGUMENT. */
orca_status orca_set_lp3_lanes(orca_ctx *ctx, int32_t lanes);

/* Where the least-penetration LP of infeasible agents runs: -1 = automatic (default:
 * inside the thread-per-agent step kernel on the block's queue (mode 2) for strips that fit
 * one wave of its blocks at the occupancy its shared memory allows -- computed at
 * orca_create from the CUDA occupancy API for the context's k -- else queued for the k_lp3
 * kernel; measured), 0 = always queued
 * (k_lp3, honouring orca_set_lp3_lanes), 1 = always inside the step kernel, each thread on
 * its own agent, 2 = inside the step kernel on the block's compacted queue (after a block
 * barrier, the block's infeasible agents are solved by its first threads, their projected
 * half-planes in the shared-memory columns of finished agents).  The 8-lane group variant
 * always queues.  Same results bit for bit.  Synchronises.  Errors: INVALID_ARGUMENT. */
orca_status orca_set_lp3_inline(orca_ctx *ctx, int32_t mode);

/* The context's cudaStream_t (as void*), e.g. for CUDA-event timing by the caller. */
orca_status orca_get_stream(orca_ctx *ctx, void **stream);

/* Per-stage device time of the last orca_step_timed call, milliseconds:
 * ms[0] = step kernel (query+ORCA+LP+integrate+hash), ms[1] = scan, ms[2] = scatter,
 * ms[3] = exchange (multi-GPU).  orca_step_timed runs n_steps un-graphed with CUDA events
 * around every launch on the context stream and synchronises. */
orca_status orca_step_timed(orca_ctx *ctx, int32_t n_steps, double ms[4]);

/* ---- errors ----------------------------------------------------------------------- */
const char *orca_status_string(orca_status s);
const char *orca_last_error(void);

/* ---- multi-GPU: spatial strips over NCCL ------------------------------ */

/* NCCL unique id (128 bytes) for rank 0 to broadcast through any process group.
 * Errors: NCCL (libnccl.so.2 not loadable). */
orca_status orca_nccl_unique_id(void *id128);

/* Create the rank-th of `world` strip contexts on `device`; every rank must call it with
 * the same params and id.  world == 1 behaves like orca_create.  Each rank must then call
 * orca_set_agents with the SAME global arrays (every rank keeps only its strip; ids are
 * global).  Errors: INVALID_ARGUMENT, NCCL, CUDA. */
orca_status orca_create_dist(const orca_params *params, int32_t device, int32_t rank,
                             int32_t world, const void *nccl_id128, orca_ctx **out);

/* Local agents of this rank: ids int32[n_local] (nullable), pos/vel float[2 n_local]
 * (nullable), in the context's sorted order; n_local from orca_get_count.  Synchronises.
 * Errors: NOT_READY, CAPACITY (a strip buffer overflowed; re-partition with set_agents). */
orca_status orca_get_local_state(orca_ctx *ctx, int32_t *ids, float *pos, float *vel);

/* In-process strip decomposition for testing on ONE GPU: `nstrips` strips held by one
 * context, exchanging halos and migrants by device copies instead of NCCL (the same
 * kernels and exchange buffers as orca_create_dist).  Results are bit-identical to
 * orca_create (same ordered neighbour lists, global-id ties).  Errors: INVALID_ARGUMENT
 * (nstrips outside [1, 64], maxSpeed * timeStep >= neighborDist), CUDA. */
orca_status orca_create_strips(const orca_params *params, int32_t device, int32_t nstrips,
                               orca_ctx **out);

/* Strip partition (host only, no GPU): split columns [0, nx) into `world` contiguous
 * strips of >= 1 column with near-equal agent counts.  colCount int64[nx] (agents per
 * column), bounds int32[world + 1] out (strip s = [bounds[s], bounds[s+1])).
 * Errors: INVALID_ARGUMENT (world < 1, world > nx, NULL, negative count). */
orca_status orca_partition_columns(const int64_t *colCount, int32_t nx, int32_t world,
                                   int32_t *bounds);

/* Re-partition the strips from the current state (agent-count quantiles of the columns
 * on the frozen grid) and re-size their buffers.  Done automatically before every chunk of
 * up to 64 steps when a strip could outgrow its capacities within the chunk (a crowd
 * converging into one strip); every rank of a multi-GPU context must call it together
 * (it all-gathers the state over NCCL).  Results are unchanged (bit-identical to one
 * strip); goals, per-agent properties, removals and counters carry over.  Single-strip
 * contexts: no-op.  Synchronises.  Errors: NOT_READY, CUDA, NCCL, CAPACITY. */
orca_status orca_rebalance(orca_ctx *ctx);

/* Transport of the per-step strip exchange: 0 = peer memory (default of
 * in-process loopback strips) -- a
 * k_push kernel stores exactly the used halo/migration records into the neighbour's receive
 * buffer (cudaIpc mapping over NVLink between ranks; the neighbour strip's buffer in
 * loopback) and raises an arrival flag the neighbour's k_receive waits on (bounded: a
 * missing neighbour step is an error, never a hang); 1 = NCCL send/recv of the whole
 * buffers (loopback: device copies; the default of orca_create_dist until an NVLink
 * measurement shows the peer-memory path faster).  Multi-rank contexts: every rank must
 * call it together.  Synchronises.  Errors: INVALID_ARGUMENT, CUDA, NCCL. */
orca_status orca_set_transport(orca_ctx *ctx, int32_t mode);

/* Halo overlap of the strips (SURVEY §8(e) "interior columns compute during the
 * exchange"): the agents of the two boundary columns on each side of a strip -- every agent
 * that can end the step in an edge column or leave the strip, since maxSpeed * timeStep < one
 * column -- step first; the exchange and k_receive then run on a second stream while the
 * interior columns step, joined before the next binning.  -1 = automatic (default: on for
 * strips of >= 4 columns on the thread-per-agent kernels), 0 = off, 1 = on where possible.
 * Overlapping strips run LP3 on the block queue (orca_set_lp3_inline mode 2).  Results are
 * bit-identical either way.  Synchronises.  Errors: INVALID_ARGUMENT. */
orca_status orca_set_overlap(orca_ctx *ctx, int32_t mode);

/* The transport in use (0 / 1 as above).  A multi-rank context falls back from 0 to 1 on
 * every rank when some pair of neighbouring GPUs cannot map each other's memory. */
orca_status orca_get_transport(orca_ctx *ctx, int32_t *mode);

/* The kernels one step launches, as chosen for the loaded agents:
 * info[0] = step kernel variant of the first strip (0, 1, 2 or 3), info[1] = lanes per
 * agent of the first strip's least-penetration kernel (0 = LP3 runs inside the step kernel,
 * no k_lp3 launch), info[2] = this library's CUDA kernels launched per step, summed over
 * the strips this context holds (per strip: step kernel, k_lp3 unless inline, k_scan and
 * k_scatter -- one fused cooperative k_bin for a one-strip context -- plus k_receive and
 * one k_push per neighbour with the peer-memory exchange;
 * NCCL's own kernels under transport 1 are not counted), info[3] = the transport.
 * Errors: INVALID_ARGUMENT, NOT_READY. */
orca_status orca_get_launch_info(orca_ctx *ctx, int32_t info[4]);

/* The step-kernel instantiation the first strip runs (DESIGN.md §10, §12 r02ai-au): cfg[0] =
 * kernel variant (0 thread per agent with the shared-memory top-k list, 1 8-lane group, 2
 * register list, 3 work-unit LP2, 4 lane pair), cfg[1] = LP3 placement (0 k_lp3 kernel, 1 per
 * thread inside the step kernel, 2 the step kernel's block queue), cfg[2] = -1 for the general
 * instantiation, else the LP3 placement it is compiled for (0 or 2; greedy LP order), cfg[3] = 1
 * if compiled for one strip of homogeneous agents, cfg[4] = threads per block, cfg[5] = the
 * blocks per SM its register budget is sized for (0: 1024 threads per SM, 64 registers).
 * Informational: every configuration gives the same results bit for bit.
 * Errors: INVALID_ARGUMENT, NOT_READY. */
orca_status orca_get_kernel_config(orca_ctx *ctx, int32_t cfg[6]);

/* Owned column ranges of the strips held by this context: bounds int32[2 * strips held]
 * = (c0, c1) pairs.  Errors: INVALID_ARGUMENT, NOT_READY. */
orca_status orca_get_strips(orca_ctx *ctx, int32_t *bounds);

/* The context's ranks: info[0] = world, info[1] = rank, info[2] = the rank count of
 * liborca's own NCCL communicator as NCCL reports it (ncclCommCount; -1 if the library
 * lacks the call; 1 for single-rank contexts).  Errors: INVALID_ARGUMENT. */
orca_status orca_get_comm_info(orca_ctx *ctx, int32_t info[3]);

/* Measured ALU denominators of the roofline (SURVEY §8(d) "confirm with an
 * FFMA microbenchmark at the run's clock"): on `device`, 8 independent FMA chains per
 * thread, 2048 threads per SM; out[0] = FP32 FFMA lane-ops/s, out[1] = FP64 DFMA lane-ops/s,
 * out[2] = the SM clock (MHz) the FP32 probe ran at (clock64 over its duration), out[3] =
 * FP32 FMA lanes per SM per clock implied by out[0] and out[2] (128 on B200).  Best of two
 * ~1 ms launches each; synchronises the device.  Not part of the step.
 * Errors: INVALID_ARGUMENT, CUDA. */
orca_status orca_probe_alu(int32_t device, double out[4]);

#ifdef __cplusplus
}
#endif
#endif /* ORCA_H */
