// orca_lp3_group.cuh -- LP3 on the queue with a GW-lane group per infeasible agent.
//
// k_lp3 (orca_kernels.cuh) gives each queued agent one thread; its projected-LP loops are
// data dependent, and ncu shows ~7.6 of 32 threads active (profiles/).  Here
// a group of GW lanes shares one agent: the projected lines are built one per lane and
// compacted with a ballot, LP2's "first violated line" is a ballot, and LP1's chord interval
// over the earlier lines is a prefix max/min scan across the group.  max/min are exact, and
// the scan reproduces the serial loop's state after every line, so the first failing line,
// the g2 flags up to it and the result equal the thread-per-agent LP3's bit for bit.
#pragma once
#include "orca_kernels.cuh"

namespace orca {


template <int GW>
struct Grp {
    unsigned mask;  // the group's lanes in the warp
    int base;       // first lane of the group
    int gl;         // lane in the group
};

template <int GW>
__device__ __forceinline__ unsigned grp_ballot(const Grp<GW>& G, bool p) {
    const unsigned b = __ballot_sync(G.mask, p) >> G.base;
    return (GW == 32) ? b : (b & ((1u << GW) - 1u));
}

template <int GW>
__device__ __forceinline__ float grp_max(const Grp<GW>& G, float v) {
#pragma unroll
    for (int o = GW / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(G.mask, v, o));
    return v;
}

// LP1 on line `no` against lines [0, no), GW lines per chunk.  runL/runR carry the
// interval across chunks; inside a chunk an inclusive scan gives lane j the serial state
// after line j.
template <int GW, bool CNT>
__device__ __forceinline__ bool lp1_grp(const Grp<GW>& G, const float* nx, const float* ny, const float* sv, int no,
                                        float r, float optx, float opty, bool dirOpt, float& vx, float& vy,
                                        uint32_t& fl, WorkT& w) {
    const float nix = nx[no], niy = ny[no], si = sv[no];
    const float disc = (r - si) * (r + si);
    if (disc < 0.0f) return false;
    const float sq = sqrtf(disc);
    float runL = -sq, runR = sq;
    const float Dx = niy, Dy = -nix;
    for (int j0 = 0; j0 < no; j0 += GW) {
        const int j = j0 + G.gl;
        float tL = runL, tR = runR;
        bool parF = false, g2 = false;
        if (j < no) {
            const float njx = nx[j], njy = ny[j], sj = sv[j];
            const float den = fmaf(njx, Dx, njy * Dy);
            const float num = sj - si * fmaf(njx, nix, njy * niy);
            if (fabsf(den) <= kEps) {
                g2 = fabsf(num) <= 2e-5f * r + 1e-6f;
                parF = num > 0.0f;
            } else {
                const float t = num / den;
                if (den > 0.0f)
                    tL = fmaxf(tL, t);
                else
                    tR = fminf(tR, t);
            }
        }
#pragma unroll
        for (int q = 1; q < GW; q <<= 1) {
            const float uL = __shfl_up_sync(G.mask, tL, q, GW);
            const float uR = __shfl_up_sync(G.mask, tR, q, GW);
            if (G.gl >= q) {
                tL = fmaxf(tL, uL);
                tR = fminf(tR, uR);
            }
        }
        const bool fail = j < no && (parF || tL > tR);
        const unsigned bf = grp_ballot(G, fail);
        const int f = bf ? __ffs(bf) - 1 : GW;  // first failing line of the chunk
        if (grp_ballot(G, g2 && G.gl <= f)) fl |= FL_G2;
        if (bf) {
            if (CNT) w.lp1 += (uint32_t)(j0 + f + 1);
            return false;
        }
        const int last = min(no - j0, GW) - 1;
        runL = __shfl_sync(G.mask, tL, G.base + last);
        runR = __shfl_sync(G.mask, tR, G.base + last);
    }
    if (CNT) w.lp1 += (uint32_t)no;
    const float od = fmaf(optx, Dx, opty * Dy);
    float t;
    if (dirOpt)
        t = (od > 0.0f) ? runR : runL;
    else
        t = fminf(fmaxf(od, runL), runR);
    vx = fmaf(t, Dx, si * nix);
    vy = fmaf(t, Dy, si * niy);
    return true;
}

// LP2: the first violated line from the current point is a ballot over chunks.
template <int GW, bool CNT>
__device__ __forceinline__ int lp2_grp(const Grp<GW>& G, const float* nx, const float* ny, const float* sv, int n,
                                       float r, float optx, float opty, bool dirOpt, float& vx, float& vy,
                                       uint32_t& fl, WorkT& w) {
    if (dirOpt) {
        vx = optx * r;
        vy = opty * r;
    } else {
        const float l2 = fmaf(optx, optx, opty * opty);
        if (l2 > r * r) {
            const float sc = r / sqrtf(l2);
            vx = optx * sc;
            vy = opty * sc;
        } else {
            vx = optx;
            vy = opty;
        }
    }
    int i0 = 0;
    while (true) {
        int first = n;
        for (int q0 = i0; q0 < n; q0 += GW) {
            const int q = q0 + G.gl;
            const bool viol = q < n && (sv[q] - fmaf(nx[q], vx, ny[q] * vy) > 0.0f);
            const unsigned mk = grp_ballot(G, viol);
            if (mk) {
                first = q0 + __ffs(mk) - 1;
                break;
            }
        }
        if (CNT) w.checks += (uint32_t)(min(first + 1, n) - i0);
        if (first >= n) return n;
        const float tx = vx, ty = vy;
        if (!lp1_grp<GW, CNT>(G, nx, ny, sv, first, r, optx, opty, dirOpt, vx, vy, fl, w)) {
            vx = tx;
            vy = ty;
            return first;
        }
        i0 = first + 1;
    }
}

// LP3 from the LP2 failure index, as lp3(): for every line i the current point
// violates by more than the running penetration, the projected lines (n_j - n_i, s_j - s_i)
// / |n_j - n_i| of the earlier lines are built one per lane (compacted in j order) and the
// direction-optimal LP2 along n_i runs on them.
template <int GW, bool CNT>
__device__ __forceinline__ void lp3_grp(const Grp<GW>& G, float* Lnx, float* Lny, float* Ls, float* Pnx, float* Pny,
                                        float* Ps, int n, int begin, float r, bool greedy, float& vx, float& vy,
                                        uint32_t& fl, WorkT& w) {
    float dist = 0.0f;
    for (int i = begin; i < n; ++i) {
        if (greedy) {
            // lp3_greedy's choice: the largest penetration beyond dist among slots [i, n)
            // (lowest slot among equals), swapped into slot i; none: the point is optimal
            float best = dist;
            int bi = -1;
            for (int q = i + G.gl; q < n; q += GW) {
                const float pen = Ls[q] - fmaf(Lnx[q], vx, Lny[q] * vy);
                if (pen > best) {
                    best = pen;
                    bi = q;
                }
            }
#pragma unroll
            for (int o = GW / 2; o > 0; o >>= 1) {
                const float ob = __shfl_xor_sync(G.mask, best, o);
                const int oi = __shfl_xor_sync(G.mask, bi, o);
                if (oi >= 0 && (bi < 0 || ob > best || (ob == best && oi < bi))) {
                    best = ob;
                    bi = oi;
                }
            }
            if (CNT) w.checks += (uint32_t)(n - i);
            if (bi < 0) break;
            if (bi != i) {
                __syncwarp(G.mask);
                if (G.gl == 0) {
                    const float ax = Lnx[i], ay = Lny[i], as = Ls[i];
                    Lnx[i] = Lnx[bi];
                    Lny[i] = Lny[bi];
                    Ls[i] = Ls[bi];
                    Lnx[bi] = ax;
                    Lny[bi] = ay;
                    Ls[bi] = as;
                }
                __syncwarp(G.mask);
            }
        }
        const float nix = Lnx[i], niy = Lny[i], si = Ls[i];
        if (!(si - fmaf(nix, vx, niy * vy) > dist)) continue;
        int m = 0;
        bool g2 = false;
        for (int j0 = 0; j0 < i; j0 += GW) {
            const int j = j0 + G.gl;
            bool keep = false;
            float px = 0.0f, py = 0.0f, ps = 0.0f;
            if (j < i) {
                const float njx = Lnx[j], njy = Lny[j], sj = Ls[j];
                const float det = fmaf(nix, njy, -niy * njx);
                if (fabsf(det) <= kEps && fmaf(nix, njx, niy * njy) > 0.0f) {
                    if (fabsf(sj - si) <= 2e-5f * r + 1e-6f) g2 = true;
                } else {
                    keep = true;
                    const float dx = njx - nix, dy = njy - niy;
                    const float il = 1.0f / sqrtf(fmaf(dx, dx, dy * dy));
                    px = dx * il;
                    py = dy * il;
                    ps = (sj - si) * il;
                }
            }
            const unsigned mk = grp_ballot(G, keep);
            if (keep) {
                const int pos = m + __popc(mk & ((1u << G.gl) - 1u));
                Pnx[pos] = px;
                Pny[pos] = py;
                Ps[pos] = ps;
            }
            m += __popc(mk);
        }
        if (grp_ballot(G, g2)) fl |= FL_G2;
        if (CNT) w.proj += (uint32_t)m;
        __syncwarp(G.mask);
        const float tx = vx, ty = vy;
        if (lp2_grp<GW, CNT>(G, Pnx, Pny, Ps, m, r, nix, niy, true, vx, vy, fl, w) < m) {
            vx = tx;  // floating-point failure: keep the current point
            vy = ty;
        }
        dist = si - fmaf(nix, vx, niy * vy);
        __syncwarp(G.mask);  // the projected lines are rebuilt for the next i
    }
}

__host__ __device__ constexpr int lp3_grp_words(int k) { return 6 * k + 1; }

template <bool DRY, int GW>
__global__ void __launch_bounds__(kStepThreads) k_lp3_grp(StepArgs a) {
    pdl_entry();
    constexpr bool CNT = DRY;
    constexpr int PPB = kStepThreads / GW;  // queued agents per block
    WorkT w{0, 0, 0, 0, 0};
    extern __shared__ __align__(16) float smem3[];
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    Grp<GW> G;
    G.base = lane & ~(GW - 1);
    G.mask = (GW == 32) ? 0xffffffffu : (((1u << GW) - 1u) << G.base);
    G.gl = lane & (GW - 1);
    const int slot = tid / GW;
    const int k = a.m.k;
    float* Lnx = smem3 + slot * lp3_grp_words(k);
    float* Lny = Lnx + k;
    float* Ls = Lny + k;
    float* Pnx = Ls + k;
    float* Pny = Pnx + k;
    float* Ps = Pny + k;
    const int nq = (int)*a.qCount;
    const int o0 = (int)a.binStart[(a.g.c0 - a.g.e0) * a.g.colBins];
    const int nOwn = (int)a.binStart[(a.g.c1 - a.g.e0) * a.g.colBins] - o0;
    int cInf = 0, cDeg = 0, cG1 = 0, cG2 = 0, cG3 = 0;
    // persistent grid (a few waves of groups), group-uniform stride over the queue
    for (int q = blockIdx.x * PPB + slot; q < nq; q += gridDim.x * PPB) {
        const int4 e = a.qEntry[q];
        const int i = e.x;
        const int cnt = e.y & 0xff, f = (e.y >> 8) & 0xff;
        uint32_t fl = (uint32_t)(e.y >> 16);
        float vx = __int_as_float(e.z), vy = __int_as_float(e.w);
        for (int m = G.gl; m < cnt; m += GW) {
            const float4 l = a.qLines[(size_t)m * a.qcap + q];
            Lnx[m] = l.x;
            Lny[m] = l.y;
            Ls[m] = l.z;
        }
        __syncwarp(G.mask);
        const float4 pr = a.propS ? a.propS[i] : make_float4(0.5f * a.m.R, a.m.maxSpeed, a.m.prefSpeed, 0.0f);
        lp3_grp<GW, CNT>(G, Lnx, Lny, Ls, Pnx, Pny, Ps, cnt, f, pr.y, a.m.lpGreedy != 0, vx, vy, fl, w);
        float dl = 0.0f;
        for (int m = G.gl; m < cnt; m += GW) dl = fmaxf(dl, Ls[m] - fmaf(Lnx[m], vx, Lny[m] * vy));
        dl = grp_max(G, dl);
        if (dl > 0.0f && dl < 1e-6f) fl |= FL_G3;
        if (G.gl == 0) {
            const float2 pi = a.posS[i];
            const uint32_t idi = a.idS[i];
            if (DRY) {
                if (a.dbgV) a.dbgV[idi] = make_float2(vx, vy);
                if (a.dbgFlags) a.dbgFlags[idi] = (uint8_t)fl;
            } else {
                finish_agent(a, i - o0, nOwn, pi, vx, vy, a.auxS[i], idi, a.rk2W[i - o0], pr);
            }
            cInf += 1;
            cDeg += (fl & (FL_G1 | FL_G2)) != 0;
            cG1 += (fl & FL_G1) != 0;
            cG2 += (fl & FL_G2) != 0;
            cG3 += (fl & FL_G3) != 0;
        }
        __syncwarp(G.mask);  // the group's smem is refilled for the next entry
    }
    const bool rep = G.gl == 0;  // one lane per agent counts
    if (DRY) {
        if (a.work) {
            unsigned long long c[3] = {rep ? w.checks : 0u, rep ? w.lp1 : 0u, rep ? w.proj : 0u};
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int r = 0; r < 3; ++r) c[r] += __shfl_xor_sync(0xffffffffu, c[r], o);
            if (lane == 0) {
                atomicAdd(&a.work->checks, c[0]);
                atomicAdd(&a.work->lp1, c[1]);
                atomicAdd(&a.work->proj, c[2]);
            }
        }
    } else {
        int c[5] = {cInf, cDeg, cG1, cG2, cG3};  // nonzero on the groups' lane 0 only
#pragma unroll
        for (int r = 0; r < 5; ++r)
            for (int o = 16; o > 0; o >>= 1) c[r] += __shfl_xor_sync(0xffffffffu, c[r], o);
        if (lane == 0) {
            if (c[0]) atomicAdd(&a.stats[ST_INFEASIBLE], (unsigned long long)c[0]);
            if (c[1]) atomicAdd(&a.stats[ST_DEGENERATE], (unsigned long long)c[1]);
            if (c[2]) atomicAdd(&a.stats[ST_G1], (unsigned long long)c[2]);
            if (c[3]) atomicAdd(&a.stats[ST_G2], (unsigned long long)c[3]);
            if (c[4]) atomicAdd(&a.stats[ST_G3], (unsigned long long)c[4]);
        }
    }
}

}  // namespace orca
