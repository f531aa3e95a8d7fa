/*
 * orca_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded fp64 CPU oracle of one ORCA time step as described
 * in arXiv 1908.10107 "Fast Simulation of Crowd Collision Avoidance".
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  The product path (paper_1908_10107_b200/) never links,
 * imports or executes anything under oracle/, and shares no code, header, constant or
 * table with it.
 *
 * Citations use "P:NN" = PAPER.md line NN, "S:NN" = SPEC.md line NN.  The ORCA geometry
 * itself is deferred by the paper to van den Berg et al. (§3); DESIGN.md §3 and
 * SURVEY.md Appendix A restate those semantics, and every reading of a silent/garbled
 * passage is listed in DESIGN.md §3 ("readings").
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off is part of the definition: every product and sum is separately
 * rounded, which is what the bit-exact cell / neighbour / branch decisions rely on.
 *
 * Pins: see tests/test_oracle_pins.py (each function below names its pin).
 */
#ifndef ORCA_ORACLE_H
#define ORCA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One ORCA line in the point/direction form of the cited ORCA library:
 * permitted side is det(d, p - v) <= 0 (v lies on the left of d). */
typedef struct {
    double px, py;  /* a point on the line */
    double dx, dy;  /* unit direction */
} or_line;

/* Global simulation parameters, same meaning as orca_params of the product ABI but an
 * independent declaration (the oracle shares no header with the product). */
typedef struct {
    float timeStep;       /* dt, s        ("simulation iteration") */
    float neighborDist;   /* r_obs, m     (Fig. 2 "observation radius") */
    int32_t maxNeighbors; /* k            (S:257 cap) */
    float timeHorizon;    /* tau, s       (Fig. 1(b) "look-ahead period") */
    float radius;         /* r, m         (Fig. 1(a) "radius r_a, r_b") */
    float maxSpeed;       /* m/s          ("capped maximum speed") */
} or_params;

/* Optional per-agent properties (P:128 heterogeneous crowds: "radius 0.5 m, 0.75 m or 1 m
 * ... desired speed of 1 m/s, 1.33 m/s or 2 m/s ... maximum speed ... 125% of the desired
 * speed").  Each array is float[n] by id, or NULL for the global value of or_params
 * (radius, maxSpeed) / the prefSpeed argument. */
typedef struct {
    const float *radius;
    const float *maxSpeed;
    const float *prefSpeed;
} or_agents;

/* Optional constraint order of the LP (reading Q8): randomized = 0 -> nearest first (the
 * neighbour order); 1 -> a Fisher-Yates shuffle per agent and step keyed by the
 * counter-based hash of (seed, step, agent id) ("randomized incremental").  `step`
 * counts steps since the state was loaded. */
typedef struct {
    int32_t randomized;
    uint64_t seed;
    int64_t step;
} or_lp_order;

/* The shuffle: idx[slot] = neighbour-order index of the line processed at `slot`. */
void or_lp_permutation(uint64_t seed, int64_t step, int64_t id, int32_t c, int32_t *idx);

/* Per-agent diagnostic flags written by or_step. */
#define OR_FLAG_INFEASIBLE 0x01u /* LP2 failed, LP3 (least penetration) used */
#define OR_FLAG_G1_COINCIDENT 0x02u /* collision branch with w == 0 (reading Q15) */
#define OR_FLAG_G2_PARALLEL 0x04u   /* an evaluated line pair with |det| <= OR_G2_DET */
#define OR_FLAG_G3_MARGINAL 0x08u   /* infeasible with 0 < delta* < 1e-6 (marginal feasibility) */
#define OR_FLAG_G4_NONUNIQUE 0x10u  /* reversed-order re-solve: same delta, different v */
/* Degenerate = excluded from the 1e-4 velocity parity (g1 | g2 | g4).  g3 is reported
 * but not excluded: the solution is continuous across the feasibility boundary (reading
 * Q21 in DESIGN.md), e.g. head-on flows pinch the feasible set to v = 0 exactly. */
#define OR_FLAG_DEGENERATE 0x16u
/* Diagnostic only (NOT degenerate): a successful main-LP LP1 interval shorter than 1e-6,
 * i.e. the optimum is a vertex where the feasible set pinches to a point.  Common and
 * well-conditioned in head-on flows (leg lines of exactly opposed pairs all pass through
 * the origin); reading Q21. */
#define OR_FLAG_NARROW 0x20u

/* ---- grid (Fig. 2) ---------------------------------------------------- */

/* Derive the frozen grid from the initial positions (reading Q12):
 * origin = fl32(min - cs) per axis, dims = floor((max - origin)/cs) + 2.
 * n == 0 -> origin (0,0), dims (1,1).  Returns 0, or -1 on bad arguments. */
int or_grid_derive(int64_t n, const float *pos, float cs, float origin[2], int32_t dims[2]);

/* Cell of every agent: cx = clamp(floor((fl64(x) - fl64(x0)) / fl64(cs)), 0, nx-1),
 * likewise cy (reading Q11).  Pin: exact rational floor (Python fractions). */
void or_cells(int64_t n, const float *pos, const float origin[2], float cs,
              const int32_t dims[2], int32_t *cx, int32_t *cy);

/* Neighbour lists through the paper's bins: read own + 8 surrounding bins, keep those
 * strictly within r_obs (P:94 caption), order by (kappa, id), keep first k.
 * kappa = fl64(dx)*fl64(dx) + fl64(dy)*fl64(dy) with dx = fl64(x_j) - fl64(x_i).
 * nbr is n*k (padded with -1), cnt is n.  Pin: brute-force O(N^2) numpy. */
void or_neighbors(int64_t n, const float *pos, const float origin[2], float cs,
                  const int32_t dims[2], float nd, int32_t k, int32_t *nbr, int32_t *cnt);

/* ---- ORCA half-plane (Fig. 1(b)-(c)) ------------------------------------ */

/* Line ORCA_{i|j} for agent i against neighbour j with combined radius R = ri + rj.
 * Returns a bitmask: 1 = collision branch, 2 = cutoff branch, 4 = left leg, 8 = right
 * leg, 16 = degenerate (coincident with w == 0).  Pin: closed forms (head-on, crossing,
 * cutoff, collision), reciprocity, VO-boundary tightness, pairwise no-collision. */
int or_orca_line(const float pi[2], const float vi[2], const float pj[2], const float vj[2],
                 int64_t idi, int64_t idj, float ri, float rj, float tau, float dt, or_line *out);

/* ---- LP (Seidel incremental) ------------------------------------ */

/* LP2 (2-D incremental): returns the number of lines processed without failure (== n on
 * success).  v is the result (the last feasible point on failure).  diag (nullable)
 * receives OR_FLAG_G2/G3 bits raised during the solve.
 * Pin: vertex enumeration (numpy) within 1e-9; SPEC examples S:103-115. */
int or_lp2(const or_line *lines, int n, double r, const double opt[2], int dirOpt,
           double v[2], uint32_t *diag);

/* LP3 (least penetration): starting from the LP2 failure index `begin` and the
 * LP2 point v, minimise max_j penetration_j(v) over the speed disc.
 * Pin: dense grid search over the disc (numpy), empty triangle. */
void or_lp3(const or_line *lines, int n, int begin, double r, double v[2], uint32_t *diag);

/* Maximum penetration max(0, max_j det(d_j, p_j - v)) of v into the lines. */
double or_penetration(const or_line *lines, int n, const double v[2]);

/* One agent's velocity solve as or_step does it: LP2 over the lines in the given
 * order, LP3 from the failure index, then the classification: returns the flags
 * (INFEASIBLE, G2, G3, G4; n <= 32), writes v and delta = or_penetration(lines, v).
 * Pins: g4 fires on a non-unique least-penetration argmin (S:123 pair) and not on a
 * unique one (empty triangle); g2 fires on near-parallel pairs crossing inside the disc. */
uint32_t or_solve(const or_line *lines, int n, double maxSpeed, const double pref[2], double v[2],
                  double *delta);

/* ---- one synchronous time step (reading Q13) ---------------------------- */

/* Computes, for every agent i in `agents` (or all agents when agents == NULL, m ignored),
 * the new velocity / position from the pre-step state.  The grid (origin, dims) is the
 * frozen grid of or_grid_derive.  goals != NULL -> pref = g*min(1, prefSpeed/|g|),
 * g = goal - pos (reading Q16); otherwise pref is used as given.
 * Outputs are indexed like `agents` (or by agent id when agents == NULL):
 *   vnew[2m], pnew[2m] (fp64), flags[m], delta[m] (max penetration at vnew),
 *   nbr[m*k] / cnt[m] (nullable).  vtest[2m] (nullable): velocities to judge -- dtest[q]
 *   receives their maximum penetration into agent q's own half-planes (the parity tests'
 *   infeasible-agent check).  Returns 0 or -1 on bad arguments. */
int or_step(const or_params *p, int64_t n, const float *pos, const float *vel,
            const float *pref, const float *goals, float prefSpeed, const or_agents *ag,
            const or_lp_order *order, const float origin[2],
            const int32_t dims[2], int64_t m, const int64_t *agents, double *vnew,
            double *pnew, uint8_t *flags, double *delta, int32_t *nbr, int32_t *cnt,
            const double *vtest, double *dtest);

/* Runs nsteps full steps in place on fp32 state (state is fp32 between steps, as in the
 * product ABI): vel <- fl32(v'), pos <- fl32(p + dt*v').  The grid is derived once from
 * the initial positions (frozen, reading Q12).  Returns the number of infeasible
 * agent-steps, or -1 on bad arguments. */
int64_t or_run(const or_params *p, int64_t n, float *pos, float *vel, const float *pref,
               const float *goals, float prefSpeed, const or_agents *ag, const or_lp_order *order,
               int32_t nsteps);

#ifdef __cplusplus
}
#endif
#endif
