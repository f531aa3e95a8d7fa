/*
 * orca_oracle.c -- TEST INFRASTRUCTURE ONLY (see orca_oracle.h header comment).
 *
 * A plain, slow, obviously-correct fp64 single-threaded ORCA step, written from
 * arXiv 1908.10107 and, where the paper defers to it ("For more
 * in-depth description of the ORCA algorithm, see the work of van den Berg et al."),
 * the cited ORCA semantics restated in DESIGN.md §3 / SURVEY.md Appendix A.
 *
 * Compiled with -ffp-contract=off: every "a*b + c*d" below is two separately rounded
 * products and one rounded sum.  No blocking, fusion or reordering beyond the
 * algorithm's own order.
 *
 * Pins (tests/test_oracle_pins.py): cells vs exact rationals; neighbours vs brute force;
 * lines vs closed forms; LP2 vs vertex enumeration; LP3 vs grid search; step invariants.
 */
#include "orca_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Parallel-line tolerance of the oracle's own LP (reading Q9: the oracle takes the
 * near-exact reading; the product's fp32 tolerance 1e-5 is covered by flag g2). */
#define OR_EPS 1e-12
/* g2 flag threshold: pairs whose |det| is this small may be decided differently by an
 * fp32 solver that uses a 1e-5 tolerance (reading Q9 + fp32 rounding slack). */
#define OR_G2_DET 2e-5
#define OR_G2_SLACK 1e-6 /* fp32 rounding slack on line offsets */
/* g3 thresholds (SURVEY §8(c) degenerate class g3). */
#define OR_G3_EPS 1e-6

static double det2(double ax, double ay, double bx, double by) { return ax * by - ay * bx; }

/* ---------------------------------------------------------------------------------- */
/* Grid: FLAME spatial bins, P:91-98 (Fig. 2).                                           */
/* ---------------------------------------------------------------------------------- */

int or_grid_derive(int64_t n, const float *pos, float cs, float origin[2], int32_t dims[2]) {
    if (n < 0 || !(cs > 0.0f) || !origin || !dims) return -1;
    if (n == 0) {
        origin[0] = origin[1] = 0.0f;
        dims[0] = dims[1] = 1;
        return 0;
    }
    for (int a = 0; a < 2; ++a) {
        float mn = pos[a], mx = pos[a];
        for (int64_t i = 1; i < n; ++i) {
            float x = pos[2 * i + a];
            if (x < mn) mn = x;
            if (x > mx) mx = x;
        }
        /* origin in fp32: one margin cell below the minimum (reading Q12) */
        volatile float o = mn - cs;
        origin[a] = o;
        double t = floor(((double)mx - (double)origin[a]) / (double)cs);
        dims[a] = (int32_t)t + 2; /* + one margin cell above the maximum */
    }
    return 0;
}

/* floor((x - x0)/cs) clamped to [0, nc-1] -- reading Q11 (exact for fp32 inputs). */
static int32_t cell_of(float x, float x0, float cs, int32_t nc) {
    double t = ((double)x - (double)x0) / (double)cs;
    double f = floor(t);
    if (f < 0.0) f = 0.0;
    if (f > (double)(nc - 1)) f = (double)(nc - 1);
    return (int32_t)f;
}

void or_cells(int64_t n, const float *pos, const float origin[2], float cs,
              const int32_t dims[2], int32_t *cx, int32_t *cy) {
    for (int64_t i = 0; i < n; ++i) {
        cx[i] = cell_of(pos[2 * i], origin[0], cs, dims[0]);
        cy[i] = cell_of(pos[2 * i + 1], origin[1], cs, dims[1]);
    }
}

/* kappa_ij: squared distance in fp64 from fp32 inputs, separately rounded (Q11). */
static double kappa(const float *pos, int64_t i, int64_t j) {
    double dx = (double)pos[2 * j] - (double)pos[2 * i];
    double dy = (double)pos[2 * j + 1] - (double)pos[2 * i + 1];
    return dx * dx + dy * dy;
}

typedef struct {
    double key;
    int64_t id;
} cand_t;

static int cand_cmp(const void *a, const void *b) {
    const cand_t *x = (const cand_t *)a, *y = (const cand_t *)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    return (x->id < y->id) ? -1 : (x->id > y->id);
}

/* Bins: agents listed per cell in ascending id order ("bin contents are ordered
 * by agent_id").  binStart has C+1 entries; binList holds agent ids. */
typedef struct {
    int32_t nx, ny;
    int64_t *binStart;
    int64_t *binList;
    int32_t *cx, *cy;
} bins_t;

static int bins_build(bins_t *b, int64_t n, const float *pos, const float origin[2], float cs,
                      const int32_t dims[2]) {
    int64_t C = (int64_t)dims[0] * dims[1];
    b->nx = dims[0];
    b->ny = dims[1];
    b->binStart = (int64_t *)calloc((size_t)C + 1, sizeof(int64_t));
    b->binList = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    b->cx = (int32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    b->cy = (int32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    if (!b->binStart || !b->binList || !b->cx || !b->cy) return -1;
    or_cells(n, pos, origin, cs, dims, b->cx, b->cy);
    for (int64_t i = 0; i < n; ++i) b->binStart[(int64_t)b->cx[i] * b->ny + b->cy[i] + 1]++;
    for (int64_t c = 0; c < C; ++c) b->binStart[c + 1] += b->binStart[c];
    int64_t *fill = (int64_t *)malloc((size_t)C * sizeof(int64_t));
    if (!fill) return -1;
    memcpy(fill, b->binStart, (size_t)C * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) b->binList[fill[(int64_t)b->cx[i] * b->ny + b->cy[i]]++] = i;
    free(fill);
    return 0;
}

static void bins_free(bins_t *b) {
    free(b->binStart);
    free(b->binList);
    free(b->cx);
    free(b->cy);
}

/* Neighbours of agent i: read own and neighbouring bins, keep strictly
 * within r_obs (reading Q10), order by (kappa, id), truncate to k.
 * cand is scratch of size n.  Returns the count. */
static int32_t neighbors_of(const bins_t *b, int64_t n, const float *pos, int64_t i, double nd2,
                            int32_t k, cand_t *cand, int32_t *out) {
    (void)n;
    int64_t m = 0;
    for (int32_t cx = b->cx[i] - 1; cx <= b->cx[i] + 1; ++cx) {
        if (cx < 0 || cx >= b->nx) continue;
        for (int32_t cy = b->cy[i] - 1; cy <= b->cy[i] + 1; ++cy) {
            if (cy < 0 || cy >= b->ny) continue;
            int64_t c = (int64_t)cx * b->ny + cy;
            for (int64_t q = b->binStart[c]; q < b->binStart[c + 1]; ++q) {
                int64_t j = b->binList[q];
                if (j == i) continue;
                double key = kappa(pos, i, j);
                if (key < nd2) {
                    cand[m].key = key;
                    cand[m].id = j;
                    ++m;
                }
            }
        }
    }
    qsort(cand, (size_t)m, sizeof(cand_t), cand_cmp);
    int32_t cnt = (int32_t)(m < k ? m : k);
    for (int32_t q = 0; q < cnt; ++q) out[q] = (int32_t)cand[q].id;
    return cnt;
}

void or_neighbors(int64_t n, const float *pos, const float origin[2], float cs,
                  const int32_t dims[2], float nd, int32_t k, int32_t *nbr, int32_t *cnt) {
    bins_t b;
    if (bins_build(&b, n, pos, origin, cs, dims) != 0) return;
    cand_t *cand = (cand_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(cand_t));
    double nd2 = (double)nd * (double)nd;
    for (int64_t i = 0; i < n; ++i) {
        for (int32_t q = 0; q < k; ++q) nbr[i * k + q] = -1;
        cnt[i] = neighbors_of(&b, n, pos, i, nd2, k, cand, nbr + i * k);
    }
    free(cand);
    bins_free(&b);
}

/* ---------------------------------------------------------------------------------- */
/* ORCA half-plane, Fig. 1(b)-(c) with the cited geometry.         */
/* ---------------------------------------------------------------------------------- */

int or_orca_line(const float pi[2], const float vi[2], const float pj[2], const float vj[2],
                 int64_t idi, int64_t idj, float ri, float rj, float tau, float dt, or_line *out) {
    const double rpx = (double)pj[0] - (double)pi[0]; /* relative position p_b - p_a */
    const double rpy = (double)pj[1] - (double)pi[1];
    const double rvx = (double)vi[0] - (double)vj[0]; /* relative velocity v_a - v_b (Q3) */
    const double rvy = (double)vi[1] - (double)vj[1];
    const double d2 = rpx * rpx + rpy * rpy;
    const double R = (double)ri + (double)rj; /* r_a + r_b (Fig. 1(a)) */
    const double R2 = R * R;
    double dirx, diry, ux, uy;
    int branch;

    if (d2 > R2) {
        /* No collision: VO truncated at lookahead tau (Fig. 1(b)). */
        const double invTau = 1.0 / (double)tau;
        const double wx = rvx - invTau * rpx; /* w = v_rel - p_rel / tau */
        const double wy = rvy - invTau * rpy;
        const double wl2 = wx * wx + wy * wy;
        const double dot1 = wx * rpx + wy * rpy;
        if (dot1 < 0.0 && dot1 * dot1 > R2 * wl2) {
            /* project on the cut-off circle */
            const double wl = sqrt(wl2);
            const double nx = wx / wl, ny = wy / wl;
            dirx = ny;
            diry = -nx;
            ux = (R * invTau - wl) * nx;
            uy = (R * invTau - wl) * ny;
            branch = 2;
        } else {
            /* project on a leg; det > 0 -> left leg, else (incl. 0) right leg (Q5) */
            const double leg = sqrt(d2 - R2);
            if (rpx * wy - rpy * wx > 0.0) {
                dirx = (rpx * leg - rpy * R) / d2;
                diry = (rpx * R + rpy * leg) / d2;
                branch = 4;
            } else {
                dirx = -(rpx * leg + rpy * R) / d2;
                diry = -(-rpx * R + rpy * leg) / d2;
                branch = 8;
            }
            const double dp = rvx * dirx + rvy * diry;
            ux = dp * dirx - rvx;
            uy = dp * diry - rvy;
        }
    } else {
        /* Collision (reading Q4): horizon = one time step. */
        const double invDt = 1.0 / (double)dt;
        const double wx = rvx - invDt * rpx;
        const double wy = rvy - invDt * rpy;
        const double wl2 = wx * wx + wy * wy;
        double nx, ny, wl;
        branch = 1;
        if (wl2 == 0.0) {
            /* coincident with equal velocity (reading Q15): lower id is pushed to -x */
            nx = (idi < idj) ? -1.0 : 1.0;
            ny = 0.0;
            wl = 0.0;
            branch |= 16;
        } else {
            wl = sqrt(wl2);
            nx = wx / wl;
            ny = wy / wl;
        }
        dirx = ny;
        diry = -nx;
        ux = (R * invDt - wl) * nx;
        uy = (R * invDt - wl) * ny;
    }
    /* ORCA_{a|b} passes through v_a + u/2 (reciprocity, reading Q2) */
    out->px = (double)vi[0] + 0.5 * ux;
    out->py = (double)vi[1] + 0.5 * uy;
    out->dx = dirx;
    out->dy = diry;
    return branch;
}

/* ---------------------------------------------------------------------------------- */
/* LP: Seidel incremental 2-D LP with a disc, and the 3-D fallback.            */
/* ---------------------------------------------------------------------------------- */

/* LP1: optimum on line `no`, clipped to the disc and to lines 0..no-1.  Returns 1 on
 * success (v written), 0 if the admissible segment is empty. */
static int lp1(const or_line *L, int no, double r, const double opt[2], int dirOpt, double v[2],
               uint32_t *diag) {
    const double dotProduct = L[no].px * L[no].dx + L[no].py * L[no].dy;
    const double disc = dotProduct * dotProduct + r * r - (L[no].px * L[no].px + L[no].py * L[no].py);
    if (disc < 0.0) return 0; /* line misses the speed disc */
    const double sq = sqrt(disc);
    double tL = -dotProduct - sq, tR = -dotProduct + sq;
    for (int i = 0; i < no; ++i) {
        const double den = det2(L[no].dx, L[no].dy, L[i].dx, L[i].dy);
        const double num = det2(L[i].dx, L[i].dy, L[no].px - L[i].px, L[no].py - L[i].py);
        /* g2: nearly parallel AND the crossing t = num/den lies inside the chord's reach,
         * i.e. an fp32 solver's "parallel -> fail if pointing away, else skip" rule could
         * decide differently from the exact crossing (reading Q9) */
        if (fabs(den) <= OR_G2_DET && fabs(num) <= OR_G2_DET * r + OR_G2_SLACK && diag)
            *diag |= OR_FLAG_G2_PARALLEL;
        if (fabs(den) <= OR_EPS) {
            if (num < 0.0) return 0; /* parallel and pointing away */
            continue;
        }
        const double t = num / den;
        if (den >= 0.0) {
            if (t < tR) tR = t;
        } else {
            if (t > tL) tL = t;
        }
        if (tL > tR) return 0;
    }
    if (!dirOpt && diag && (tR - tL) < OR_G3_EPS) *diag |= OR_FLAG_NARROW;
    double t;
    if (dirOpt) {
        t = (opt[0] * L[no].dx + opt[1] * L[no].dy > 0.0) ? tR : tL;
    } else {
        t = L[no].dx * (opt[0] - L[no].px) + L[no].dy * (opt[1] - L[no].py);
        if (t < tL) t = tL;
        if (t > tR) t = tR;
    }
    v[0] = L[no].px + t * L[no].dx;
    v[1] = L[no].py + t * L[no].dy;
    return 1;
}

int or_lp2(const or_line *L, int n, double r, const double opt[2], int dirOpt, double v[2],
           uint32_t *diag) {
    if (dirOpt) {
        /* opt is a unit direction: start at the far end of the disc */
        v[0] = opt[0] * r;
        v[1] = opt[1] * r;
    } else if (opt[0] * opt[0] + opt[1] * opt[1] > r * r) {
        const double l = sqrt(opt[0] * opt[0] + opt[1] * opt[1]);
        v[0] = opt[0] / l * r;
        v[1] = opt[1] / l * r;
    } else {
        v[0] = opt[0];
        v[1] = opt[1];
    }
    for (int i = 0; i < n; ++i) {
        if (det2(L[i].dx, L[i].dy, L[i].px - v[0], L[i].py - v[1]) > 0.0) {
            double keep[2] = {v[0], v[1]};
            if (!lp1(L, i, r, opt, dirOpt, v, diag)) {
                v[0] = keep[0];
                v[1] = keep[1];
                return i;
            }
        }
    }
    return n;
}

void or_lp3(const or_line *L, int n, int begin, double r, double v[2], uint32_t *diag) {
    double distance = 0.0;
    or_line *proj = (or_line *)malloc((size_t)(n > 0 ? n : 1) * sizeof(or_line));
    for (int i = begin; i < n; ++i) {
        if (det2(L[i].dx, L[i].dy, L[i].px - v[0], L[i].py - v[1]) > distance) {
            int m = 0;
            for (int j = 0; j < i; ++j) {
                or_line q;
                const double determinant = det2(L[i].dx, L[i].dy, L[j].dx, L[j].dy);
                /* g2: nearly parallel, same direction (an fp32 solver skips the pair) and the
                 * lines so close that their bisector still crosses the speed disc (reading Q9) */
                if (fabs(determinant) <= OR_G2_DET && L[i].dx * L[j].dx + L[i].dy * L[j].dy > 0.0 &&
                    fabs(det2(L[i].dx, L[i].dy, L[j].px - L[i].px, L[j].py - L[i].py)) <= OR_G2_DET * r + OR_G2_SLACK &&
                    diag)
                    *diag |= OR_FLAG_G2_PARALLEL;
                if (fabs(determinant) <= OR_EPS) {
                    if (L[i].dx * L[j].dx + L[i].dy * L[j].dy > 0.0) continue; /* same direction */
                    q.px = 0.5 * (L[i].px + L[j].px);                            /* opposite */
                    q.py = 0.5 * (L[i].py + L[j].py);
                } else {
                    const double t = det2(L[j].dx, L[j].dy, L[i].px - L[j].px, L[i].py - L[j].py) / determinant;
                    q.px = L[i].px + t * L[i].dx;
                    q.py = L[i].py + t * L[i].dy;
                }
                const double ddx = L[j].dx - L[i].dx, ddy = L[j].dy - L[i].dy;
                const double l = sqrt(ddx * ddx + ddy * ddy);
                q.dx = ddx / l;
                q.dy = ddy / l;
                proj[m++] = q;
            }
            const double keep[2] = {v[0], v[1]};
            const double dirOpt[2] = {-L[i].dy, L[i].dx};
            if (or_lp2(proj, m, r, dirOpt, 1, v, diag) < m) {
                /* in principle impossible (v is feasible for the projected LP); only
                 * floating-point error gets here: keep the current result */
                v[0] = keep[0];
                v[1] = keep[1];
            }
            distance = det2(L[i].dx, L[i].dy, L[i].px - v[0], L[i].py - v[1]);
        }
    }
    free(proj);
}

double or_penetration(const or_line *L, int n, const double v[2]) {
    double d = 0.0;
    for (int i = 0; i < n; ++i) {
        const double pen = det2(L[i].dx, L[i].dy, L[i].px - v[0], L[i].py - v[1]);
        if (pen > d) d = pen;
    }
    return d;
}

/* Full velocity solve of one agent: LP2 over the lines in neighbour
 * order (reading Q8), LP3 from the failure index if infeasible. */
static int solve_agent(const or_line *L, int n, double maxSpeed, const double pref[2], double v[2],
                       uint32_t *diag) {
    int f = or_lp2(L, n, maxSpeed, pref, 0, v, diag);
    if (f < n) {
        or_lp3(L, n, f, maxSpeed, v, diag);
        return 1;
    }
    return 0;
}

/* The solve and its classification (SURVEY 8(c) degenerate classes; DESIGN reading Q21):
 * infeasible, g2 (raised inside LP1/LP3), g3 (0 < delta < 1e-6 after LP3) and g4 (a
 * reversed-order re-solve reaches the same delta, within 1e-9, at a v more than 1e-6
 * away: the least-penetration argmin is not unique). */
uint32_t or_solve(const or_line *L, int n, double maxSpeed, const double pref[2], double v[2], double *delta) {
    uint32_t diag = 0;
    or_line Lrev[32];
    int infeasible = solve_agent(L, n, maxSpeed, pref, v, &diag);
    double dl = or_penetration(L, n, v);
    if (infeasible) {
        diag |= OR_FLAG_INFEASIBLE;
        if (dl > 0.0 && dl < OR_G3_EPS) diag |= OR_FLAG_G3_MARGINAL;
        for (int a = 0; a < n; ++a) Lrev[a] = L[n - 1 - a];
        double v2[2];
        uint32_t d2 = 0;
        solve_agent(Lrev, n, maxSpeed, pref, v2, &d2);
        double dl2 = or_penetration(L, n, v2);
        if (fabs(dl2 - dl) <= 1e-9 && hypot(v2[0] - v[0], v2[1] - v[1]) > 1e-6)
            diag |= OR_FLAG_G4_NONUNIQUE;
    }
    if (delta) *delta = dl;
    return diag;
}

/* ---------------------------------------------------------------------------------- */
/* One synchronous step (reading Q13: all reads are of the pre-step state). */
/* ---------------------------------------------------------------------------------- */

static int params_ok(const or_params *p) {
    return p && p->timeStep > 0.0f && p->neighborDist > 0.0f && p->timeHorizon > 0.0f &&
           p->radius > 0.0f && p->maxSpeed >= 0.0f && p->maxNeighbors >= 0 && p->maxNeighbors <= 32 &&
           isfinite(p->timeStep) && isfinite(p->neighborDist) && isfinite(p->timeHorizon) &&
           isfinite(p->radius) && isfinite(p->maxSpeed);
}

/* preferred velocity toward the goal at walking speed ("The agent's velocity is in
 * the direction of the goal location, scaled to the walking speed"; reading Q16). */
static void pref_of(const float *pos, const float *pref, const float *goals, float prefSpeed,
                    const or_agents *ag, int64_t i, double out[2]) {
    if (ag && ag->prefSpeed) prefSpeed = ag->prefSpeed[i]; /* P:128 per-person desired speed */
    if (!goals) {
        out[0] = (double)pref[2 * i];
        out[1] = (double)pref[2 * i + 1];
        return;
    }
    const double gx = (double)goals[2 * i] - (double)pos[2 * i];
    const double gy = (double)goals[2 * i + 1] - (double)pos[2 * i + 1];
    const double gl = sqrt(gx * gx + gy * gy);
    const double s = (gl > (double)prefSpeed) ? (double)prefSpeed / gl : 1.0;
    out[0] = gx * s;
    out[1] = gy * s;
}

/* splitmix64 finaliser: the counter-based generator of the randomized LP order; integer
 * only, so the CUDA path reproduces it bit for bit from the same inputs (no shared code) */
static uint64_t or_mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

void or_lp_permutation(uint64_t seed, int64_t step, int64_t id, int32_t c, int32_t *idx) {
    const uint64_t key = or_mix64(seed ^ or_mix64(((uint64_t)step << 32) ^ (uint64_t)id));
    for (int32_t a = 0; a < c; ++a) idx[a] = a;
    for (int32_t a = c - 1; a >= 1; --a) {
        const uint64_t h = or_mix64(key ^ ((uint64_t)a * 0x9e3779b97f4a7c15ULL));
        const int32_t b = (int32_t)(h % (uint64_t)(a + 1));
        const int32_t t = idx[a];
        idx[a] = idx[b];
        idx[b] = t;
    }
}

int or_step(const or_params *p, int64_t n, const float *pos, const float *vel, const float *pref,
            const float *goals, float prefSpeed, const or_agents *ag, const or_lp_order *order,
            const float origin[2], const int32_t dims[2],
            int64_t m, const int64_t *agents, double *vnew, double *pnew, uint8_t *flags,
            double *delta, int32_t *nbr, int32_t *cnt, const double *vtest, double *dtest) {
    if (!params_ok(p) || n < 0 || (n > 0 && (!pos || !vel || (!pref && !goals)))) return -1;
    if (!agents) m = n;
    if (m < 0) return -1;
    const int32_t k = p->maxNeighbors;
    const double nd2 = (double)p->neighborDist * (double)p->neighborDist;
    bins_t b;
    if (bins_build(&b, n, pos, origin, p->neighborDist, dims) != 0) return -1;
    cand_t *cand = (cand_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(cand_t));
    or_line L[32];
    int32_t nb[32];
    for (int64_t q = 0; q < m; ++q) {
        const int64_t i = agents ? agents[q] : q;
        if (i < 0 || i >= n) {
            free(cand);
            bins_free(&b);
            return -1;
        }
        /* 1. observe: neighbours through the bins */
        const int32_t c = neighbors_of(&b, n, pos, i, nd2, k, cand, nb);
        uint32_t diag = 0;
        /* per-person radius and maximum speed, else the global ones */
        const float ri = (ag && ag->radius) ? ag->radius[i] : p->radius;
        const double maxSpeed = (double)((ag && ag->maxSpeed) ? ag->maxSpeed[i] : p->maxSpeed);
        /* 2. one ORCA half-plane per neighbour, nearest first (Fig. 1) */
        for (int32_t a = 0; a < c; ++a) {
            const int64_t j = nb[a];
            const float rj = (ag && ag->radius) ? ag->radius[j] : p->radius;
            int br = or_orca_line(pos + 2 * i, vel + 2 * i, pos + 2 * j, vel + 2 * j, i, j, ri, rj,
                                  p->timeHorizon, p->timeStep, &L[a]);
            if (br & 16) diag |= OR_FLAG_G1_COINCIDENT;
        }
        /* optional randomized constraint order ("based on the randomized incremental
         * linear program solver of Seidel"; reading Q8): Fisher-Yates keyed by the
         * counter-based hash of (seed, step, id) */
        if (order && order->randomized && c > 1) {
            or_line tmp[32];
            int32_t idx[32];
            or_lp_permutation(order->seed, order->step, i, c, idx);
            for (int32_t a = 0; a < c; ++a) tmp[a] = L[idx[a]];
            for (int32_t a = 0; a < c; ++a) L[a] = tmp[a];
        }
        /* 3. LP: closest permitted velocity to the preferred one, else least
         *    penetration */
        double pv[2], v[2];
        pref_of(pos, pref, goals, prefSpeed, ag, i, pv);
        double dl;
        diag |= or_solve(L, c, maxSpeed, pv, v, &dl);
        /* 4. integrate ("take the chosen velocity"; explicit Euler) */
        vnew[2 * q] = v[0];
        vnew[2 * q + 1] = v[1];
        if (pnew) {
            pnew[2 * q] = (double)pos[2 * i] + (double)p->timeStep * v[0];
            pnew[2 * q + 1] = (double)pos[2 * i + 1] + (double)p->timeStep * v[1];
        }
        if (flags) flags[q] = (uint8_t)diag;
        if (delta) delta[q] = dl;
        /* a candidate velocity (e.g. the product's) judged on this agent's own lines */
        if (vtest && dtest) dtest[q] = or_penetration(L, c, vtest + 2 * q);
        if (nbr) {
            for (int32_t a = 0; a < k; ++a) nbr[q * k + a] = (a < c) ? nb[a] : -1;
        }
        if (cnt) cnt[q] = c;
    }
    free(cand);
    bins_free(&b);
    return 0;
}

int64_t or_run(const or_params *p, int64_t n, float *pos, float *vel, const float *pref,
               const float *goals, float prefSpeed, const or_agents *ag, const or_lp_order *order,
               int32_t nsteps) {
    if (!params_ok(p) || n < 0 || nsteps < 0) return -1;
    float origin[2];
    int32_t dims[2];
    if (or_grid_derive(n, pos, p->neighborDist, origin, dims) != 0) return -1;
    double *vn = (double *)malloc((size_t)(n > 0 ? 2 * n : 1) * sizeof(double));
    double *pn = (double *)malloc((size_t)(n > 0 ? 2 * n : 1) * sizeof(double));
    uint8_t *fl = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
    int64_t infeasible = 0;
    for (int32_t s = 0; s < nsteps; ++s) {
        or_lp_order ord;
        if (order) {
            ord = *order;
            ord.step = order->step + s;
        }
        if (or_step(p, n, pos, vel, pref, goals, prefSpeed, ag, order ? &ord : NULL, origin, dims, 0, NULL, vn, pn,
                    fl, NULL, NULL, NULL, NULL, NULL) != 0) {
            infeasible = -1;
            break;
        }
        for (int64_t i = 0; i < n; ++i) {
            vel[2 * i] = (float)vn[2 * i];
            vel[2 * i + 1] = (float)vn[2 * i + 1];
            pos[2 * i] = (float)pn[2 * i];
            pos[2 * i + 1] = (float)pn[2 * i + 1];
            infeasible += (fl[i] & OR_FLAG_INFEASIBLE) ? 1 : 0;
        }
    }
    free(vn);
    free(pn);
    free(fl);
    return infeasible;
}
