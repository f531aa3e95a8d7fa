// orca_step_group.cuh -- the fused step with an 8-lane group per agent (sm_100a).
//
// Same computation as k_step (orca_kernels.cuh), bit for bit: stages 2-5 of the ORCA
// step for one agent, but spread over 8 lanes so that the data-dependent loops
// of one agent do not serialise a whole warp (SURVEY §8(a) kernel option (ii)):
//   * scan: the group strides a column run 8 candidates at a time (coalesced loads);
//     candidates under the running bound are appended with ballot + popc;
//   * selection: every buffered candidate's rank among all candidates is counted with the
//     exact (kappa, id) order, branch-free; ranks < k form the sorted list;
//   * half-planes: one lane per neighbour;
//   * LP2: a ballot finds the first violated line, LP1's bounds over the earlier lines are
//     a group min/max reduction (exact operations, so the result is the sequential one).
// LP3 agents are queued for k_lp3 exactly as in k_step.
#pragma once
#include "orca_kernels.cuh"

namespace orca {

constexpr int kG = 8;                    // lanes per agent
constexpr int kGroupThreads = 128;       // 16 agents per block
constexpr int kGroupAgents = kGroupThreads / kG;
constexpr int kBufE = 48;                // candidate buffer entries per agent

// per-agent shared words: buffer (f, j) x kBufE, two lists (f, j) x k, lines 3 x k
__host__ __device__ constexpr int group_words(int k) { return 2 * kBufE + 4 * k + 3 * k + 1; }

struct GroupCtx {
    unsigned gmask;  // the group's lanes in the warp
    int gbase;       // first lane of the group
    int gl;          // lane in group
};

__device__ __forceinline__ unsigned gballot(const GroupCtx& G, bool p) {
    return (__ballot_sync(G.gmask, p) >> G.gbase) & 0xffu;
}

__device__ __forceinline__ float gmax(const GroupCtx& G, float v) {
    v = fmaxf(v, __shfl_xor_sync(G.gmask, v, 4));
    v = fmaxf(v, __shfl_xor_sync(G.gmask, v, 2));
    return fmaxf(v, __shfl_xor_sync(G.gmask, v, 1));
}

__device__ __forceinline__ float gmin(const GroupCtx& G, float v) {
    v = fminf(v, __shfl_xor_sync(G.gmask, v, 4));
    v = fminf(v, __shfl_xor_sync(G.gmask, v, 2));
    return fminf(v, __shfl_xor_sync(G.gmask, v, 1));
}

// Merge buffer entries (bf, bj)[0, nb) with the current list (lf, lj)[0, cnt) into the
// other list (of, oj): rank every candidate by the exact (kappa, id) order among all
// valid candidates, keep ranks < k.  Buffer entries outside r_obs are invalid.
__device__ __forceinline__ int group_merge(const GroupCtx& G, float* bf, uint32_t* bj, int nb, const float* lf,
                                           const uint32_t* lj, int cnt, float* of, uint32_t* oj, int k, float2 pi,
                                           const Model& m, const float2* __restrict__ posS,
                                           const uint32_t* __restrict__ idS) {
    // validity of the new candidates (exact only near the r_obs boundary)
    for (int e = G.gl; e < nb; e += kG)
        if (!in_radius(bf[e], bj[e], pi, m.nd2Lo, m.nd2Fup, m.nd2D, posS)) bf[e] = INFINITY;
    __syncwarp(G.gmask);
    const int M = cnt + nb;
    int valid = 0;
    for (int e = G.gl; e < M; e += kG) {
        const float fe = (e < cnt) ? lf[e] : bf[e - cnt];
        const uint32_t je = (e < cnt) ? lj[e] : bj[e - cnt];
        if (fe == INFINITY) continue;
        ++valid;
        int rank = 0;
        for (int q = 0; q < M; ++q) {
            const float fq = (q < cnt) ? lf[q] : bf[q - cnt];
            if (fq == INFINITY || q == e) continue;
            const uint32_t jq = (q < cnt) ? lj[q] : bj[q - cnt];
            rank += cand_less(fq, jq, fe, je, pi, posS, idS) ? 1 : 0;
        }
        if (rank < k) {
            of[rank] = fe;
            oj[rank] = je;
        }
    }
    // valid count over the group
    valid += __shfl_xor_sync(G.gmask, valid, 4);
    valid += __shfl_xor_sync(G.gmask, valid, 2);
    valid += __shfl_xor_sync(G.gmask, valid, 1);
    __syncwarp(G.gmask);
    return min(valid, k);
}

// LP1 on line `no` against lines [0, no), lanes split the earlier lines; tL/tR are
// exact group max/min and any parallel-fail is a ballot, so the outcome is the sequential
// lp1's.
__device__ __forceinline__ bool lp1_group(const GroupCtx& G, const float* nx, const float* ny, const float* sv, int no,
                                          float r, float optx, float opty, bool dirOpt, float& vx, float& vy,
                                          uint32_t& fl) {
    const float nix = nx[no], niy = ny[no], si = sv[no];
    const float disc = (r - si) * (r + si);
    if (disc < 0.0f) return false;
    const float sq = sqrtf(disc);
    float tL = -sq, tR = sq;
    const float Dx = niy, Dy = -nix;
    bool failp = false;
    for (int j = G.gl; j < no; j += kG) {
        const float njx = nx[j], njy = ny[j], sj = sv[j];
        const float den = fmaf(njx, Dx, njy * Dy);
        const float num = sj - si * fmaf(njx, nix, njy * niy);
        if (fabsf(den) <= kEps) {
            if (fabsf(num) <= 2e-5f * r + 1e-6f) fl |= FL_G2;
            if (num > 0.0f) failp = true;
            continue;
        }
        const float t = num / den;
        if (den > 0.0f)
            tL = fmaxf(tL, t);
        else
            tR = fminf(tR, t);
    }
    tL = gmax(G, tL);
    tR = gmin(G, tR);
    if (gballot(G, failp) || tL > tR) return false;
    const float od = fmaf(optx, Dx, opty * Dy);
    float t;
    if (dirOpt)
        t = (od > 0.0f) ? tR : tL;
    else
        t = fminf(fmaxf(od, tL), tR);
    vx = fmaf(t, Dx, si * nix);
    vy = fmaf(t, Dy, si * niy);
    return true;
}

__device__ __forceinline__ int lp2_group(const GroupCtx& G, const float* nx, const float* ny, const float* sv, int n,
                                         float r, float optx, float opty, float& vx, float& vy, uint32_t& fl,
                                         uint32_t& checks, uint32_t& lp1it) {
    const float l2 = fmaf(optx, optx, opty * opty);
    if (l2 > r * r) {
        const float sc = r / sqrtf(l2);
        vx = optx * sc;
        vy = opty * sc;
    } else {
        vx = optx;
        vy = opty;
    }
    int i0 = 0;
    while (true) {
        int first = n;
        for (int q0 = i0; q0 < n; q0 += kG) {
            const int q = q0 + G.gl;
            const bool viol = q < n && (sv[q] - fmaf(nx[q], vx, ny[q] * vy) > 0.0f);
            const unsigned mk = gballot(G, viol);
            if (mk) {
                first = q0 + __ffs(mk) - 1;
                break;
            }
        }
        checks += (uint32_t)(min(first + 1, n) - i0);
        if (first >= n) return n;
        lp1it += (uint32_t)first;
        const float tx = vx, ty = vy;
        if (!lp1_group(G, nx, ny, sv, first, r, optx, opty, false, vx, vy, fl)) {
            vx = tx;
            vy = ty;
            return first;
        }
        i0 = first + 1;
    }
}

// lp2_greedy (orca_kernels.cuh) over the group: the lanes evaluate the remaining half-planes
// (slot t + lane, + 8, ...), a group reduction picks the largest violation (the lowest slot
// among equal ones, as the sequential scan does), lane 0 swaps it into slot t, and
// lp1_group re-solves against slots [0, t).  Same choices, same arithmetic, same result.
__device__ __forceinline__ int lp2_group_greedy(const GroupCtx& G, float* nx, float* ny, float* sv, int n, float r,
                                                float optx, float opty, float& vx, float& vy, uint32_t& fl,
                                                uint32_t& checks, uint32_t& lp1it) {
    const float l2 = fmaf(optx, optx, opty * opty);
    if (l2 > r * r) {
        const float sc = r / sqrtf(l2);
        vx = optx * sc;
        vy = opty * sc;
    } else {
        vx = optx;
        vy = opty;
    }
    for (int t = 0; t < n; ++t) {
        float best = 0.0f;
        int bi = -1;
        for (int q = t + G.gl; q < n; q += kG) {
            const float pen = sv[q] - fmaf(nx[q], vx, ny[q] * vy);
            if (pen > best) {
                best = pen;
                bi = q;
            }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            const float ob = __shfl_xor_sync(G.gmask, best, o);
            const int oi = __shfl_xor_sync(G.gmask, bi, o);
            if (oi >= 0 && (bi < 0 || ob > best || (ob == best && oi < bi))) {
                best = ob;
                bi = oi;
            }
        }
        checks += (uint32_t)(n - t);
        if (bi < 0) return n;
        if (bi != t) {
            __syncwarp(G.gmask);
            if (G.gl == 0) {
                const float ax = nx[t], ay = ny[t], as = sv[t];
                nx[t] = nx[bi];
                ny[t] = ny[bi];
                sv[t] = sv[bi];
                nx[bi] = ax;
                ny[bi] = ay;
                sv[bi] = as;
            }
            __syncwarp(G.gmask);
        }
        lp1it += (uint32_t)t;
        const float tx = vx, ty = vy;
        if (!lp1_group(G, nx, ny, sv, t, r, optx, opty, false, vx, vy, fl)) {
            vx = tx;
            vy = ty;
            return t;
        }
    }
    return n;
}

template <bool DRY>
__global__ void __launch_bounds__(kGroupThreads, 8) k_step_group(StepArgs a) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char smemg[];
    const int k = a.m.k;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    GroupCtx G;
    G.gbase = lane & ~(kG - 1);
    G.gmask = 0xffu << G.gbase;
    G.gl = lane & (kG - 1);
    const int ag = tid / kG;  // agent slot in the block
    float* base = reinterpret_cast<float*>(smemg) + ag * group_words(k);
    float* bf = base;
    uint32_t* bj = reinterpret_cast<uint32_t*>(base + kBufE);
    float* lfA = base + 2 * kBufE;
    uint32_t* ljA = reinterpret_cast<uint32_t*>(lfA + k);
    float* lfB = lfA + 2 * k;
    uint32_t* ljB = reinterpret_cast<uint32_t*>(lfB + k);
    float* Lnx = lfA + 4 * k;
    float* Lny = Lnx + k;
    float* Ls = Lny + k;

    const int o0 = (int)a.binStart[(a.g.c0 - a.g.e0) * a.g.colBins];
    const int o1 = (int)a.binStart[(a.g.c1 - a.g.e0) * a.g.colBins];
    const int ws = blockIdx.x * kGroupAgents + ag;
    const int i = o0 + ws;
    const bool active = i < o1;  // group-uniform
    if (!DRY && blockIdx.x == 0 && tid == 0) {
        a.ctr[CT_NOWN] = o1 - o0;
        a.ctr[CT_EXTRA] = 0;
    }
    uint32_t fl = 0;
    int nColl = 0;
    bool deferred = false;
    uint32_t wCand = 0, wChecks = 0, wLp1 = 0;
    int cnt = 0;
    if (active) {
        const float2 pi = a.posS[i];
        const float2 vi = a.velS[i];
        const float2 aux = a.auxS[i];
        const uint32_t idi = a.idS[i];
        // per-agent (radius, maxSpeed, prefSpeed) of heterogeneous crowds
        const bool het = a.propS != nullptr;
        const float4 pr = het ? a.propS[i] : make_float4(0.5f * a.m.R, a.m.maxSpeed, a.m.prefSpeed, 0.0f);
        const float ri = pr.x, vmaxi = pr.y, vprefi = (pr.z >= 0.0f) ? pr.z : a.m.prefSpeed;
        const int cx = cell_coord(pi.x, a.g.ox, a.g.csD, a.g.invCs, a.g.nx);
        const int lgS = a.g.lgS;
        const int nyS = a.g.ny << lgS;
        const int cy = subrow_coord(pi.y, a.g) >> lgS;
        float fk = INFINITY;
        bool useA = true;  // current list is A
        if (k > 0) {
            const int rlo = max(cy - 1, 0) << lgS;
            const int rhi = (min(cy + 1, a.g.ny - 1) + 1) << lgS;
            const int c0 = max(cx - 1, 0), c1 = min(cx + 1, a.g.nx - 1);
            const int lgC = a.g.lgC;
            const int fe0 = a.g.e0 << lgC;                         // first local fine column
            const int f0 = c0 << lgC, f1 = ((c1 + 1) << lgC) - 1;  // fine columns of the stencil
            float thr = a.m.nd2Fup;
            bool guessed = false;
            const float rk2p = a.rk2S[i];
            if (rk2p < a.m.nd2Fup) {
                const float marg = 2.0002f * a.m.maxSpeedAll * a.m.dt + 4e-7f * (fabsf(pi.x) + fabsf(pi.y)) + 1e-5f;
                const float r = sqrtf(rk2p) * (1.0f + 1e-5f) + marg;
                const float b = r * r * (1.0f + 1e-3f);
                if (b < thr) {
                    thr = b;
                    guessed = true;
                }
            } else {
                int ncand = 0;  // agents in the 3x3 stencil
                for (int fc = f0; fc <= f1; ++fc)
                    ncand += (int)a.binStart[(fc - fe0) * nyS + rhi] - (int)a.binStart[(fc - fe0) * nyS + rlo];
                const float g = 2.2f * (float)k * 9.0f * a.g.cs * a.g.cs / (3.14159265f * (float)ncand);
                if (ncand > 4 * k && g < thr) {
                    thr = g;
                    guessed = true;
                }
            }
            for (int pass = 0; pass < 2; ++pass) {
                const float thrPass = thr;
                int lo = rlo, hi = rhi - 1, fa = f0, fb = f1;
                if (guessed) {
                    const float rg = sqrtf(thr) * (1.0f + 1e-6f) + 1e-6f;
                    const double ty = __dmul_rn(__dsub_rn((double)pi.y, (double)a.g.oy), a.g.invCsSub);
                    const double rs = (double)rg * a.g.invCsSub + 1e-6;
                    lo = max(lo, (int)fmin(fmax(floor(ty - rs), 0.0), (double)(nyS - 1)));
                    hi = min(hi, (int)fmin(fmax(floor(ty + rs), 0.0), (double)(nyS - 1)));
                    const double tx = __dmul_rn(__dsub_rn((double)pi.x, (double)a.g.ox), a.g.invCsSubX);
                    const double rsx = (double)rg * a.g.invCsSubX + 1e-6;
                    fa = max(fa, (int)fmin(fmax(floor(tx - rsx), 0.0), (double)((a.g.nx << lgC) - 1)));
                    fb = min(fb, (int)fmin(fmax(floor(tx + rsx), 0.0), (double)((a.g.nx << lgC) - 1)));
                }
                cnt = 0;
                useA = true;
                int nb = 0;
                for (int fc = fa; fc <= fb; ++fc) {  // one run per fine column
                    const int b = (int)a.binStart[(fc - fe0) * nyS + lo];
                    const int e = (int)a.binStart[(fc - fe0) * nyS + hi + 1];
                    if (DRY) wCand += (uint32_t)max(e - b, 0);
                    for (int j0 = b; j0 < e; j0 += kG) {
                        const int j = j0 + G.gl;
                        bool pass = false;
                        float d2 = 0.0f;
                        if (j < e) {
                            const float2 pj = a.posS[j];
                            const float dx = pj.x - pi.x, dy = pj.y - pi.y;
                            d2 = fmaf(dx, dx, dy * dy);
                            pass = d2 <= thr && j != i;
                        }
                        const unsigned mk = gballot(G, pass);
                        if (pass) {
                            const int s = nb + __popc(mk & ((1u << G.gl) - 1u));
                            bf[s] = d2;
                            bj[s] = (uint32_t)j;
                        }
                        nb += __popc(mk);
                        if (nb > kBufE - kG) {  // buffer nearly full: merge, tighten the bound
                            __syncwarp(G.gmask);
                            cnt = useA ? group_merge(G, bf, bj, nb, lfA, ljA, cnt, lfB, ljB, k, pi, a.m, a.posS, a.idS)
                                       : group_merge(G, bf, bj, nb, lfB, ljB, cnt, lfA, ljA, k, pi, a.m, a.posS, a.idS);
                            useA = !useA;
                            nb = 0;
                            if (cnt == k)
                                thr = fminf(thr, __fmul_ru((useA ? lfA : lfB)[k - 1], 1.0f + 0x1p-20f));
                        }
                    }
                }
                __syncwarp(G.gmask);
                cnt = useA ? group_merge(G, bf, bj, nb, lfA, ljA, cnt, lfB, ljB, k, pi, a.m, a.posS, a.idS)
                           : group_merge(G, bf, bj, nb, lfB, ljB, cnt, lfA, ljA, k, pi, a.m, a.posS, a.idS);
                useA = !useA;
                if (!guessed) break;
                const float* lf = useA ? lfA : lfB;
                if (cnt == k && (double)lf[k - 1] < (double)thrPass * (1.0 - 0x1p-20)) break;
                thr = a.m.nd2Fup;  // rescan the full 3x3 stencil at the full radius
                guessed = false;
            }
            if (cnt == k) fk = (useA ? lfA : lfB)[k - 1];
        }
        const float* lf = useA ? lfA : lfB;
        const uint32_t* lj = useA ? ljA : ljB;
        (void)lf;
        if (!DRY && G.gl == 0) a.rk2W[ws] = fk;

        // ---- 3. half-planes, one lane per neighbour (Fig. 1) ----------------------
        if (DRY && a.dbgNbr)  // neighbours in (distance, id) order
            for (int q = G.gl; q < cnt; q += kG) a.dbgNbr[(size_t)idi * k + q] = (int32_t)a.idS[lj[q]];
        if (a.m.lpRandom && cnt > 1) {  // randomized LP order (reading Q8): one lane shuffles
            __syncwarp(G.gmask);
            if (G.gl == 0) lp_shuffle(const_cast<uint32_t*>(lj), 1, cnt, a.m.lpSeed, a.ctr[CT_STEP], idi);
            __syncwarp(G.gmask);
        }
        for (int q = G.gl; q < cnt; q += kG) {
            const uint32_t j = lj[q];
            const float2 pj = a.posS[j];
            const float2 vj = a.velS[j];
            float nx, ny, s;
            int coll;
            // combined radius R = r_i + r_j (Fig. 1(a)); per agent when heterogeneous
            float Rp = a.m.R;
            double R2p = a.m.R2D;
            if (het) {
                const double Rd = (double)ri + (double)a.propS[j].x;
                R2p = Rd * Rd;
                Rp = (float)Rd;
            }
            fl |= orca_line(pi.x, pi.y, vi.x, vi.y, pj.x, pj.y, vj.x, vj.y, idi, a.idS, j, Rp, R2p, a.m, nx, ny, s, coll);
            nColl += coll;
            Lnx[q] = nx;
            Lny[q] = ny;
            Ls[q] = s;
        }
        __syncwarp(G.gmask);

        // ---- 4. LP2; LP3 agents are queued for k_lp3 --------------------
        float px, py;
        if (a.m.goals) {
            const float gx = aux.x - pi.x, gy = aux.y - pi.y;
            const float gl = sqrtf(fmaf(gx, gx, gy * gy));
            const float sc = (gl > vprefi) ? vprefi / gl : 1.0f;
            px = gx * sc;
            py = gy * sc;
        } else {
            px = aux.x;
            py = aux.y;
        }
        float vx, vy;
        const int f = a.m.lpGreedy ? lp2_group_greedy(G, Lnx, Lny, Ls, cnt, vmaxi, px, py, vx, vy, fl, wChecks, wLp1)
                                   : lp2_group(G, Lnx, Lny, Ls, cnt, vmaxi, px, py, vx, vy, fl, wChecks, wLp1);
        // flags of all lanes of the group
        fl |= __shfl_xor_sync(G.gmask, fl, 4);
        fl |= __shfl_xor_sync(G.gmask, fl, 2);
        fl |= __shfl_xor_sync(G.gmask, fl, 1);
        if (f < cnt) {
            fl |= FL_INFEASIBLE;
            deferred = true;
            int q = 0;
            if (G.gl == 0) q = (int)atomicAdd(a.qCount, 1u);
            q = __shfl_sync(G.gmask, q, G.gbase);
            if (G.gl == 0)
                a.qEntry[q] = make_int4(i, cnt | (f << 8) | ((int)fl << 16), __float_as_int(vx), __float_as_int(vy));
            for (int m2 = G.gl; m2 < cnt; m2 += kG)
                a.qLines[(size_t)m2 * a.qcap + q] = make_float4(Lnx[m2], Lny[m2], Ls[m2], 0.0f);
        }
        if (DRY) {
            if (G.gl == 0) {
                if (!deferred && a.dbgV) a.dbgV[idi] = make_float2(vx, vy);
                if (!deferred && a.dbgFlags) a.dbgFlags[idi] = (uint8_t)fl;
                if (a.dbgCnt) a.dbgCnt[idi] = cnt;
            }
            if (a.dbgNbr)
                for (int q = cnt + G.gl; q < k; q += kG) a.dbgNbr[(size_t)idi * k + q] = -1;
        } else if (!deferred && G.gl == 0) {
            finish_agent(a, ws, o1 - o0, pi, vx, vy, aux, idi, fk, pr);
        }
    }
    // ---- counters: one lane per agent counts ---------------------------------------------
    const bool rep = active && G.gl == 0;
    if (DRY) {
        if (a.work) {
            unsigned long long c[3] = {rep ? wCand : 0u, rep ? (unsigned long long)cnt : 0ull,
                                       rep ? wChecks : 0u};
            unsigned long long c1 = rep ? wLp1 : 0u;
            for (int o = 16; o > 0; o >>= 1) {
                c[0] += __shfl_xor_sync(0xffffffffu, c[0], o);
                c[1] += __shfl_xor_sync(0xffffffffu, c[1], o);
                c[2] += __shfl_xor_sync(0xffffffffu, c[2], o);
                c1 += __shfl_xor_sync(0xffffffffu, c1, o);
            }
            if (lane == 0) {
                atomicAdd(&a.work->cand, c[0]);
                atomicAdd(&a.work->lines, c[1]);
                atomicAdd(&a.work->checks, c[2]);
                atomicAdd(&a.work->lp1, c1);
            }
        }
    } else {
        const uint32_t f2 = (rep && !deferred) ? fl : 0u;
        const int cInf = __popc(__ballot_sync(0xffffffffu, f2 & FL_INFEASIBLE));
        const int cDeg = __popc(__ballot_sync(0xffffffffu, f2 & (FL_G1 | FL_G2)));
        const int cG1 = __popc(__ballot_sync(0xffffffffu, f2 & FL_G1));
        const int cG2 = __popc(__ballot_sync(0xffffffffu, f2 & FL_G2));
        const int cG3 = __popc(__ballot_sync(0xffffffffu, f2 & FL_G3));
        int c = nColl;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) {
            if (c) atomicAdd(&a.stats[ST_COLLISION], (unsigned long long)c);
            if (cInf) atomicAdd(&a.stats[ST_INFEASIBLE], (unsigned long long)cInf);
            if (cDeg) atomicAdd(&a.stats[ST_DEGENERATE], (unsigned long long)cDeg);
            if (cG1) atomicAdd(&a.stats[ST_G1], (unsigned long long)cG1);
            if (cG2) atomicAdd(&a.stats[ST_G2], (unsigned long long)cG2);
            if (cG3) atomicAdd(&a.stats[ST_G3], (unsigned long long)cG3);
        }
    }
}

}  // namespace orca
