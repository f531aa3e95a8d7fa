// orca_kernels.cuh -- sm_100a device code of the ORCA step (arXiv 1908.10107).
//
// Product path.  Shares no code with oracle/.  Every stage of the step runs here:
//   k_select    pick a strip's agents (owned + ghost columns), hash + histogram
//   k_scan      exclusive scan (decoupled look-back) of the per-bin counts -> binStart
//   k_scatter   counting-sort permutation into cell-sorted SoA
//   k_step      3x3 k-nearest query -> ORCA half-planes -> LP2/LP3 -> integrate -> next hash
//               (P:77 model, Fig. 1 geometry, P:80 fallback, P:82 incremental LP)
//
// Numerics:
//   * discrete decisions that must match the fp64 oracle bit-for-bit (cell floor, the
//     neighbour key kappa, the ORCA branch predicates) are evaluated in fp64 with explicit
//     round-to-nearest intrinsics (__dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn), i.e. the
//     oracle's expression trees without contraction;
//   * the continuous geometry and the LP run in fp32 in Hessian normal form (n, s):
//     permitted set n.v >= s, |n| = 1, which keeps r^2 - s^2 and the LP3 bisectors
//     well conditioned.
#pragma once
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdint.h>
#include <climits>

namespace cg = cooperative_groups;
namespace orca {

constexpr int kMaxK = 32;
constexpr float kEps = 1e-5f;  // parallel-line tolerance (reading Q9)

// per-agent flag bits (match orca_debug_step)
constexpr uint32_t FL_INFEASIBLE = 1u;
constexpr uint32_t FL_G1 = 2u;
constexpr uint32_t FL_G2 = 4u;
constexpr uint32_t FL_G3 = 8u;

// indices into the device stats block (uint64)
enum { ST_INFEASIBLE = 0, ST_DEGENERATE, ST_G1, ST_G2, ST_G3, ST_COLLISION, ST_REMOVED, ST_COUNT };

// Work counters of an instrumented dry step (orca_debug_work): per-launch totals used by
// the bench's ALU roofline.
struct Work {
    unsigned long long cand;   // candidates read (the fine-column runs within the search radius)
    unsigned long long lines;  // ORCA half-planes built
    unsigned long long checks; // LP2 constraint checks (incl. inside LP3)
    unsigned long long lp1;    // LP1 inner iterations
    unsigned long long proj;   // LP3 projected lines
    unsigned long long stencil;  // agents in the 3x3 cell stencil of each agent (SURVEY §8(d) c_cand)
};
struct WorkT {
    uint32_t cand, lines, checks, lp1, proj;
};

// Programmatic dependent launch: the step kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so kernel N+1 is launched while kernel N
// drains.  Every such kernel first releases its own dependent (launch_dependents: the next
// kernel may be scheduled once all our blocks are running) and then waits for its
// predecessor to complete and flush (griddepcontrol.wait) before touching any data.  Both are
// no-ops for a launch without the attribute.
#ifndef ORCA_PDL
#define ORCA_PDL 0  // measured r01ay: 100k 0.0665 -> 0.0739 ms, corridor 0.050 -> 0.056 with it; off
#endif
__device__ __forceinline__ void pdl_entry() {
#if ORCA_PDL
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

struct Grid {
    float ox, oy, cs;  // origin, cell size (fp32 values; widened exactly to fp64)
    int nx, ny;        // dims (cells of size cs = r_obs)
    int lgS;           // each cell is split into 2^lgS sub-rows for the sort order ...
    int lgC;           // ... and 2^lgC sub-columns (fine columns)
    int colBins;       // sort bins per cell column: 2^lgC fine columns x (ny << lgS) sub-rows
    double csD, invCs;        // fl64(cs), fl64(1/cs)
    double csSub, invCsSub;   // cs / 2^lgS (exact), 2^lgS / cs
    double csSubX, invCsSubX; // cs / 2^lgC (exact), 2^lgC / cs
    // strip of this domain: owned columns [c0, c1); the local bins cover
    // columns [e0, e1) = owned plus one ghost column on each side that exists
    int c0, c1, e0, e1;
    int hasL, hasR;           // a neighbour strip exists on that side
};

struct Model {
    float dt, maxSpeed, R;        // R = 2 r (combined radius, Fig. 1(a))
    float invTauF, invDtF;        // fp32 copies for the continuous geometry
    float pad0;                   // explicit (no implicit padding: the host compares the bytes)
    double invTauD, invDtD;       // 1/fl64(tau), 1/fl64(dt) for the predicates
    double R2D;                   // fl64(R)^2
    double nd2D;                  // fl64(nd)^2 (exact: nd is fp32)
    float nd2Fup;                 // fp32 prefilter bound, rounded up with margin
    float nd2Lo;                  // below this fp32 d2 a candidate is surely inside r_obs
    int k;                        // maxNeighbors
    int goals;                    // 1: aux holds goals, pref = g min(1, s/|g|)
    float prefSpeed;
    float removeR2;               // > 0: remove agents within sqrt(removeR2) of their goal
    float maxSpeedAll;            // largest maxSpeed of any agent (history search bound)
    int lpRandom;                 // 1: randomized LP constraint order (reading Q8)
    unsigned long long lpSeed;
    int lpGreedy;                 // 1: LP2 takes the most violated remaining half-plane next (Q8)
    int pad1;
};

// ------------------------------------------------------------------ cell (reading Q11)
// floor(d / cs) of d = fl64(x) - fl64(o) without a division: q = floor(d * inv) is off by
// at most one, and the residual r = d - q*cs is computed exactly by one fma (q*cs has
// <= 53 bits for |q| < 2^29 and |r| < 2 cs), so the corrected q is the exact rational
// floor -- which equals the oracle's floor(fl64(d / cs)): fl64 rounding of d/cs can never
// reach an integer from below for fp32 inputs.  Clamped to [0, nc-1].
__device__ __forceinline__ int floor_div_clamped(double d, double cs, double inv, int nc) {
    const double q0 = __dmul_rn(d, inv);
    if (q0 < -2.0) return 0;
    if (q0 > (double)nc + 2.0) return nc - 1;
    double q = floor(q0);
    const double r = fma(-q, cs, d);
    if (r < 0.0) q -= 1.0;
    else if (r >= cs) q += 1.0;
    q = fmax(q, 0.0);
    q = fmin(q, (double)(nc - 1));
    return (int)q;
}

__device__ __forceinline__ int cell_coord(float x, float o, double cs, double inv, int nc) {
    return floor_div_clamped(__dsub_rn((double)x, (double)o), cs, inv, nc);
}

// Sub-row of y: floor((y - oy) / (cs / 2^lgS)), clamped; cs / 2^lgS is exact, and the
// sub-row >> lgS is exactly the clamped cell row.
__device__ __forceinline__ int subrow_coord(float y, const Grid& g) {
    return floor_div_clamped(__dsub_rn((double)y, (double)g.oy), g.csSub, g.invCsSub, g.ny << g.lgS);
}

// Fine column of x: floor((x - ox) / (cs / 2^lgC)), clamped, by the same exact rule; the
// fine column >> lgC is exactly the clamped cell column (cell_coord).
__device__ __forceinline__ int finecol_coord(float x, const Grid& g) {
    return floor_div_clamped(__dsub_rn((double)x, (double)g.ox), g.csSubX, g.invCsSubX, g.nx << g.lgC);
}

// Local bin id of the sort order: column-major over (fine column - 2^lgC e0, sub-row), so
// the owned strip (cell columns [c0, c1)) is one contiguous id range, a cell column is
// colBins consecutive bins, and each fine column's run is ordered by y at sub-row
// granularity: the agents within a distance of (x, y) lie in a few short runs.
__device__ __forceinline__ uint32_t bin_of(int fx, int sy, const Grid& g) {
    return (uint32_t)(fx - (g.e0 << g.lgC)) * (uint32_t)(g.ny << g.lgS) + (uint32_t)sy;
}

constexpr uint32_t kInvalid = 0xffffffffu;  // work entry that left the strip

// per-domain device counters
// CT_STEP: the LP-order step index; CT_XSTEP: steps since the strips were built (the
// exchange sequence number, equal on every rank)
enum { CT_NOWN = 0, CT_EXTRA, CT_OVF, CT_STEP, CT_XSTEP, CT_COUNT };
constexpr int OVF_WORK = 1, OVF_MIG = 2, OVF_HALO = 4, OVF_TIMEOUT = 8;

// One direction of the neighbour exchange (fixed capacity; one NCCL send per step):
// hdr = {emigrants, halo agents}; emigrants carry the full state, halo agents only what a
// ghost needs (position, velocity, id).
struct ExBuf {
    int* hdr;
    float2 *mpos, *mvel, *maux;
    uint32_t* mid;
    float* mrk2;
    float2 *hpos, *hvel;
    uint32_t* hid;
    float4* mprop;  // heterogeneous crowds: emigrant (radius, maxSpeed, prefSpeed, 0)
    float* hrad;    // heterogeneous crowds: halo agent radius
    int capM, capH;
};

// ------------------------------------------------------------------------- binning
// Select the agents of a strip (columns [e0, e1)) from the global input arrays into the
// work buffers: ids = input index, no search-bound history; bin + atomic rank.
__global__ void k_select(int n, const float2* __restrict__ pos, const float2* __restrict__ vel,
                         const float2* __restrict__ aux, Grid g, float2* __restrict__ posW, float2* __restrict__ velW,
                         float2* __restrict__ auxW, uint32_t* __restrict__ idW, float* __restrict__ rk2W,
                         uint32_t* __restrict__ cellW, uint32_t* __restrict__ rankW, uint32_t* __restrict__ count,
                         int* __restrict__ ctr, int capW, const float* __restrict__ hist,
                         const uint8_t* __restrict__ active) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (active && !active[i]) continue;  // removed at its goal
        const float2 p = pos[i];
        const int fx = finecol_coord(p.x, g);
        const int cx = fx >> g.lgC;  // = cell_coord(p.x, ...)
        if (cx < g.e0 || cx >= g.e1) continue;
        const int w = atomicAdd(&ctr[CT_EXTRA], 1);
        if (w >= capW) {
            atomicOr(&ctr[CT_OVF], OVF_WORK);
            continue;
        }
        const uint32_t c = bin_of(fx, subrow_coord(p.y, g), g);
        posW[w] = p;
        velW[w] = vel[i];
        auxW[w] = aux[i];
        idW[w] = (uint32_t)i;
        rk2W[w] = hist ? hist[i] : INFINITY;  // search-radius hint only (results are exact either way)
        cellW[w] = c;
        rankW[w] = atomicAdd(&count[c], 1u);
    }
}

// Previous k-th neighbour distances of the owned agents by id (out is +inf-filled): the
// first search radius of the next orca_set_agents with the same agent count.
__global__ void k_hist_by_id(const uint32_t* __restrict__ binStart, Grid g, const uint32_t* __restrict__ idS,
                             const float* __restrict__ rk2S, float* __restrict__ out) {
    const int cb = g.colBins;
    const int o0 = (int)binStart[(g.c0 - g.e0) * cb], o1 = (int)binStart[(g.c1 - g.e0) * cb];
    for (int i = o0 + blockIdx.x * blockDim.x + threadIdx.x; i < o1; i += gridDim.x * blockDim.x)
        out[idS[i]] = rk2S[i];
}

// ---- strip rebalance: the owned agents of every strip back to by-id arrays
// Owned agents -> by-id global arrays (pos, vel, aux, search-radius history) + active flag.
__global__ void k_gather_state(const uint32_t* __restrict__ binStart, Grid g, const uint32_t* __restrict__ idS,
                               const float2* __restrict__ posS, const float2* __restrict__ velS,
                               const float2* __restrict__ auxS, const float* __restrict__ rk2S,
                               float2* __restrict__ pos, float2* __restrict__ vel, float2* __restrict__ aux,
                               float* __restrict__ rk2, uint8_t* __restrict__ active) {
    const int cb = g.colBins;
    const int o0 = (int)binStart[(g.c0 - g.e0) * cb], o1 = (int)binStart[(g.c1 - g.e0) * cb];
    for (int i = o0 + blockIdx.x * blockDim.x + threadIdx.x; i < o1; i += gridDim.x * blockDim.x) {
        const uint32_t id = idS[i];
        pos[id] = posS[i];
        vel[id] = velS[i];
        aux[id] = auxS[i];
        rk2[id] = rk2S[i];
        active[id] = 1;
    }
}

// Owned agents -> fixed-size records for the all-gather between ranks: record q =
// (id bits, rk2, pos.x, pos.y), (vel.x, vel.y, aux.x, aux.y); unused records have id ~0.
__global__ void k_pack_owned(const uint32_t* __restrict__ binStart, Grid g, const uint32_t* __restrict__ idS,
                             const float2* __restrict__ posS, const float2* __restrict__ velS,
                             const float2* __restrict__ auxS, const float* __restrict__ rk2S,
                             float4* __restrict__ out, int cap) {
    const int cb = g.colBins;
    const int o0 = (int)binStart[(g.c0 - g.e0) * cb], o1 = (int)binStart[(g.c1 - g.e0) * cb];
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < cap; q += gridDim.x * blockDim.x) {
        const int i = o0 + q;
        if (i < o1) {
            const float2 p = posS[i], v = velS[i], x = auxS[i];
            out[2 * q] = make_float4(__uint_as_float(idS[i]), rk2S[i], p.x, p.y);
            out[2 * q + 1] = make_float4(v.x, v.y, x.x, x.y);
        } else {
            out[2 * q] = make_float4(__uint_as_float(0xffffffffu), 0.0f, 0.0f, 0.0f);
        }
    }
}

__global__ void k_unpack_gathered(const float4* __restrict__ in, int total, float2* __restrict__ pos,
                                  float2* __restrict__ vel, float2* __restrict__ aux, float* __restrict__ rk2,
                                  uint8_t* __restrict__ active) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
        const float4 a = in[2 * q];
        const uint32_t id = __float_as_uint(a.x);
        if (id == 0xffffffffu) continue;
        const float4 b = in[2 * q + 1];
        pos[id] = make_float2(a.z, a.w);
        vel[id] = make_float2(b.x, b.y);
        aux[id] = make_float2(b.z, b.w);
        rk2[id] = a.y;
        active[id] = 1;
    }
}

// Fill report of a strip: owned agents and the populations of its two edge columns.
__global__ void k_fill_report(const uint32_t* __restrict__ binStart, Grid g, int* __restrict__ out) {
    if (threadIdx.x != 0) return;
    const int cb = g.colBins;
    const int b0 = (int)binStart[(g.c0 - g.e0) * cb], b1 = (int)binStart[(g.c0 - g.e0 + 1) * cb];
    const int b2 = (int)binStart[(g.c1 - 1 - g.e0) * cb], b3 = (int)binStart[(g.c1 - g.e0) * cb];
    out[0] = b3 - b0;
    out[1] = b1 - b0;
    out[2] = b3 - b2;
}

// Single-pass exclusive scan (decoupled look-back) over C bin counts: tiles of 4096
// (1024 threads x 4).  status[] (64-bit: flag << 62 | value) and the tile ticket must be
// zero at launch.  Writes binStart[0..C] and re-zeroes count for the next histogram.
constexpr unsigned long long kAggFlag = 1ull << 62, kIncFlag = 2ull << 62, kValMask = (1ull << 62) - 1;
#ifndef ORCA_SCAN_ITEMS
#define ORCA_SCAN_ITEMS 4  // bins per thread (multiple of 4); tile = 1024 x this
#endif
#ifndef ORCA_SCAN_THREADS
#define ORCA_SCAN_THREADS 1024  // threads per scan tile (a multiple of 32, <= 1024)
#endif
constexpr int kScanItems = ORCA_SCAN_ITEMS;
constexpr int kScanThreads = ORCA_SCAN_THREADS;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) k_scan(uint32_t* __restrict__ count, uint32_t* __restrict__ binStart, int C,
                                               unsigned long long* __restrict__ status,
                                               unsigned int* __restrict__ ticket) {
    pdl_entry();
    __shared__ uint32_t warpSums[32];
    __shared__ uint32_t tileS, prefixS;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) tileS = atomicAdd(ticket, 1u);
    __syncthreads();
    const int tile = (int)tileS;
    const int base = tile * kScanTile;
    uint32_t v[kScanItems];
    const int i0 = base + tid * kScanItems;
    if (i0 + kScanItems - 1 < C) {
#pragma unroll
        for (int c = 0; c < kScanItems / 4; ++c) {
            const uint4 q = *reinterpret_cast<const uint4*>(count + i0 + 4 * c);
            v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < kScanItems; ++q) v[q] = (i0 + q < C) ? count[i0 + q] : 0u;
    }
    uint32_t local = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) local += v[q];
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warpSums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const uint32_t w = (lane < kScanThreads / 32) ? warpSums[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        warpSums[lane] = wi - w;  // exclusive warp offsets
        const uint32_t total = __shfl_sync(0xffffffffu, wi, 31);
        // publish the aggregate, then a warp-parallel look-back: lane l reads the status of
        // tile t - l; the nearest inclusive prefix ends the walk, else 32 aggregates are
        // summed and the window moves 32 tiles back
        volatile unsigned long long* st = status;
        if (tile == 0) {
            if (lane == 0) {
                st[0] = kIncFlag | total;
                prefixS = 0;
            }
        } else {
            if (lane == 0) st[tile] = kAggFlag | total;
            unsigned long long pre = 0;
            int t = tile - 1;
            while (true) {
                const int idx = t - lane;
                unsigned long long x = kIncFlag;  // before tile 0: an inclusive zero
                if (idx >= 0) {
                    do {
                        x = st[idx];
                    } while ((x >> 62) == 0);
                }
                const unsigned inc = __ballot_sync(0xffffffffu, (x >> 62) == 2);
                const int first = inc ? __ffs(inc) - 1 : 31;  // nearest inclusive (or the window)
                unsigned long long v = (lane <= first) ? (x & kValMask) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                pre += v;
                if (inc) break;
                t -= 32;
            }
            if (lane == 0) {
                __threadfence();
                st[tile] = kIncFlag | (pre + total);
                prefixS = (uint32_t)pre;
            }
        }
    }
    __syncthreads();
    uint32_t run = prefixS + warpSums[wid] + incl - local;
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
        if (i0 + q < C) {
            binStart[i0 + q] = run;
            count[i0 + q] = 0u;
        }
        run += v[q];
    }
    if ((C - 1) / kScanItems == tile * kScanThreads + tid) binStart[C] = run;  // owner of element C-1
}

// Counting-sort scatter of the nOwn + extra work entries (invalid = emigrated) into the
// sorted arrays (grid-stride over the device-side count).
__global__ void k_scatter(int* __restrict__ ctr, int bump, const uint32_t* __restrict__ cell,
                          const uint32_t* __restrict__ rank, const uint32_t* __restrict__ binStart,
                          const float2* __restrict__ posW, const float2* __restrict__ velW,
                          const float2* __restrict__ auxW, const uint32_t* __restrict__ idW,
                          const float* __restrict__ rk2W, float2* __restrict__ posS, float2* __restrict__ velS,
                          float2* __restrict__ auxS, uint32_t* __restrict__ idS, float* __restrict__ rk2S, int capW,
                          const float4* __restrict__ propW, float4* __restrict__ propS,
                          unsigned long long* __restrict__ scanStatus, int nStatus) {
    pdl_entry();
    // the scan is done: clear its status words, tile ticket and the LP3 queue count for the
    // next step (saves a memset node per step)
    if (blockIdx.x == 0)
        for (int q = threadIdx.x; q < nStatus; q += blockDim.x) scanStatus[q] = 0ull;
    const int n = min(ctr[CT_NOWN] + ctr[CT_EXTRA], capW);
    if (bump && blockIdx.x == 0 && threadIdx.x == 0) {  // the step is complete
        ctr[CT_STEP] += 1;
        ctr[CT_XSTEP] += 1;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t c = cell[i];
        if (c == kInvalid) continue;
        const uint32_t dst = binStart[c] + rank[i];
        posS[dst] = posW[i];
        velS[dst] = velW[i];
        auxS[dst] = auxW[i];
        idS[dst] = idW[i];
        rk2S[dst] = rk2W[i];
        if (propW) propS[dst] = propW[i];
    }
}

// Fused binning of one strip (the step graph's single-strip path): the exclusive scan of the
// bin counts and the counting-sort scatter in ONE cooperative launch of at most one resident
// wave, with two grid-wide barriers instead of a kernel boundary and a decoupled look-back:
//   (a) every block sums its contiguous chunk of bins into partial[block];
//   (b) every block adds up the partials before it (its exclusive offset) and scans its own
//       chunk (a thread per contiguous segment, one block scan), writing binStart and
//       re-zeroing the counts (binStart[C] = the total);
//   (c) the scatter of k_scatter, grid-stride over the work slots.
// The result is k_scan + k_scatter's bit for bit (integer sums).
constexpr int kBinThreads = 256;
__device__ __forceinline__ uint32_t block_sum_u32(uint32_t v, uint32_t* sm) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) sm[wid] = v;
    __syncthreads();
    uint32_t t = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += sm[q];
    return t;
}

__global__ void __launch_bounds__(kBinThreads) k_bin(int* __restrict__ ctr, int bump, uint32_t* __restrict__ count,
                                                      uint32_t* __restrict__ binStart, int C, uint32_t* __restrict__ partial,
                                                      const uint32_t* __restrict__ cell, const uint32_t* __restrict__ rank,
                                                      const float2* __restrict__ posW, const float2* __restrict__ velW,
                                                      const float2* __restrict__ auxW, const uint32_t* __restrict__ idW,
                                                      const float* __restrict__ rk2W, float2* __restrict__ posS,
                                                      float2* __restrict__ velS, float2* __restrict__ auxS,
                                                      uint32_t* __restrict__ idS, float* __restrict__ rk2S, int capW,
                                                      const float4* __restrict__ propW, float4* __restrict__ propS,
                                                      unsigned long long* __restrict__ scanStatus, int nStatus) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t sm[kBinThreads / 32];
    __shared__ uint32_t sScan[kBinThreads];
    const int G = gridDim.x, b = blockIdx.x, t = threadIdx.x;
    const int per = (C + G - 1) / G;
    const int lo = min(C, b * per), hi = min(C, lo + per);
    // (a) the block's chunk total
    uint32_t s = 0;
    for (int q = lo + t; q < hi; q += kBinThreads) s += count[q];
    s = block_sum_u32(s, sm);
    if (t == 0) partial[b] = s;
    if (b == 0)  // k_scan's status words / ticket and the LP3 queue count for the next step
        for (int q = t; q < nStatus; q += kBinThreads) scanStatus[q] = 0ull;
    grid.sync();
    // (b) offset of this chunk, then its scan
    uint32_t o = 0;
    for (int q = t; q < b; q += kBinThreads) o += partial[q];
    o = block_sum_u32(o, sm);
    const int L = (hi - lo + kBinThreads - 1) / kBinThreads;  // bins per thread (contiguous)
    const int s0 = min(hi, lo + t * L), s1 = min(hi, s0 + L);
    uint32_t mine = 0;
    for (int q = s0; q < s1; ++q) mine += count[q];
    sScan[t] = mine;
    __syncthreads();
    for (int d = 1; d < kBinThreads; d <<= 1) {  // inclusive Hillis-Steele scan of the thread sums
        const uint32_t v = (t >= d) ? sScan[t - d] : 0u;
        __syncthreads();
        sScan[t] += v;
        __syncthreads();
    }
    uint32_t run = o + sScan[t] - mine;
    for (int q = s0; q < s1; ++q) {
        const uint32_t c = count[q];
        binStart[q] = run;
        count[q] = 0u;
        run += c;
    }
    if (hi == C && lo < C && t == kBinThreads - 1) binStart[C] = o + sScan[kBinThreads - 1];
    if (C == 0 && b == 0 && t == 0) binStart[0] = 0u;
    grid.sync();
    // (c) the scatter
    const int n = min(ctr[CT_NOWN] + ctr[CT_EXTRA], capW);
    if (bump && b == 0 && t == 0) {  // the step is complete
        ctr[CT_STEP] += 1;
        ctr[CT_XSTEP] += 1;
    }
    for (int i = b * kBinThreads + t; i < n; i += G * kBinThreads) {
        const uint32_t c = cell[i];
        if (c == kInvalid) continue;
        const uint32_t dst = binStart[c] + rank[i];
        posS[dst] = posW[i];
        velS[dst] = velW[i];
        auxS[dst] = auxW[i];
        idS[dst] = idW[i];
        rk2S[dst] = rk2W[i];
        if (propW) propS[dst] = propW[i];
    }
}

__global__ void k_set_int(int* p, int v) { *p = v; }

// --------------------------------------------- randomized constraint order (Q8)
// splitmix64 finaliser; integer only, so the permutation is the oracle's bit for bit.
__device__ __forceinline__ unsigned long long lp_mix64(unsigned long long x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

// Fisher-Yates over the c entries x[0], x[T], ... keyed by (seed, step, id): applying the
// swaps of the shuffle of the identity to the list yields x'[s] = x[idx[s]].
__device__ __forceinline__ void lp_shuffle(uint32_t* x, int T, int c, unsigned long long seed, int step,
                                           uint32_t id) {
    const unsigned long long key =
        lp_mix64(seed ^ lp_mix64(((unsigned long long)(long long)step << 32) ^ (unsigned long long)id));
    for (int a = c - 1; a >= 1; --a) {
        const unsigned long long h = lp_mix64(key ^ ((unsigned long long)a * 0x9e3779b97f4a7c15ULL));
        const int b = (int)(h % (unsigned long long)(a + 1));
        const uint32_t t = x[a * T];
        x[a * T] = x[b * T];
        x[b * T] = t;
    }
}

// ------------------------------------------------------------- ORCA half-plane (Fig. 1)
// Agent i against neighbour j, R = r_i + r_j.  Branch predicates in fp64 exactly as the
// oracle's expression trees; geometry in fp32 Hessian form.  Returns flag bits
// (FL_G1) and sets *collision.
__device__ __forceinline__ uint32_t orca_line_branchy(float xi, float yi, float vxi, float vyi, float xj, float yj,
                                              float vxj, float vyj, uint32_t idi, const uint32_t* __restrict__ idS, uint32_t j, float R, double R2D,
                                              const Model& m, float& nx, float& ny, float& s, int& collision) {
    const double rpx = __dsub_rn((double)xj, (double)xi);
    const double rpy = __dsub_rn((double)yj, (double)yi);
    const double rvx = __dsub_rn((double)vxi, (double)vxj);
    const double rvy = __dsub_rn((double)vyi, (double)vyj);
    const double d2 = __dadd_rn(__dmul_rn(rpx, rpx), __dmul_rn(rpy, rpy));
    uint32_t fl = 0;
    collision = 0;
    if (d2 > R2D) {
        const double wx = __dsub_rn(rvx, __dmul_rn(m.invTauD, rpx));
        const double wy = __dsub_rn(rvy, __dmul_rn(m.invTauD, rpy));
        const double wl2 = __dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy));
        const double dot1 = __dadd_rn(__dmul_rn(wx, rpx), __dmul_rn(wy, rpy));
        if (dot1 < 0.0 && __dmul_rn(dot1, dot1) > __dmul_rn(R2D, wl2)) {
            // cut-off circle: n = w/|w|, s = n.v_i + (R/tau - |w|)/2
            const float wl = sqrtf((float)wl2);
            const float inv = 1.0f / wl;
            nx = (float)wx * inv;
            ny = (float)wy * inv;
            s = fmaf(nx, vxi, ny * vyi) + 0.5f * (R * m.invTauF - wl);
        } else {
            // legs: s = n.(v_i + v_j)/2 since n is orthogonal to the leg direction
            const float leg = sqrtf((float)__dsub_rn(d2, R2D));
            const float px = (float)rpx, py = (float)rpy;
            const float invd2 = 1.0f / (float)d2;
            const double detw = __dsub_rn(__dmul_rn(rpx, wy), __dmul_rn(rpy, wx));
            if (detw > 0.0) {  // left leg
                nx = -(px * R + py * leg) * invd2;
                ny = (px * leg - py * R) * invd2;
            } else {  // right leg (ties -> right, reading Q5)
                nx = (py * leg - px * R) * invd2;
                ny = -(px * leg + py * R) * invd2;
            }
            s = 0.5f * fmaf(nx, vxi + vxj, ny * (vyi + vyj));
        }
    } else {
        // collision (reading Q4): horizon dt
        collision = 1;
        const double wx = __dsub_rn(rvx, __dmul_rn(m.invDtD, rpx));
        const double wy = __dsub_rn(rvy, __dmul_rn(m.invDtD, rpy));
        const double wl2 = __dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy));
        float wl;
        if (wl2 == 0.0) {  // coincident, equal velocity (reading Q15)
            nx = (idi < idS[j]) ? -1.0f : 1.0f;  // (the id only here: loaded lazily)
            ny = 0.0f;
            wl = 0.0f;
            fl |= FL_G1;
        } else {
            wl = sqrtf((float)wl2);
            const float inv = 1.0f / wl;
            nx = (float)wx * inv;
            ny = (float)wy * inv;
        }
        s = fmaf(nx, vxi, ny * vyi) + 0.5f * (R * m.invDtF - wl);
    }
    return fl;
}

// The same half-plane with the three cases folded into selects (ORCA_LINE_BF, default): the
// fp64 predicates are evaluated exactly as above (same expression trees, so the same branch
// decisions bit for bit), then one sqrt and one reciprocal serve whichever case holds -- the
// lanes of a warp stay converged whatever mix of cut-off / leg / collision pairs they meet.
// Only the coincident collision (w = 0, reading Q15) keeps a branch.
#ifndef ORCA_LINE_BF
#define ORCA_LINE_BF 1
#endif
__device__ __forceinline__ uint32_t orca_line_bf(float xi, float yi, float vxi, float vyi, float xj, float yj,
                                                 float vxj, float vyj, uint32_t idi, const uint32_t* __restrict__ idS, uint32_t j, float R, double R2D,
                                                 const Model& m, float& nx, float& ny, float& s, int& collision) {
    const double rpx = __dsub_rn((double)xj, (double)xi);
    const double rpy = __dsub_rn((double)yj, (double)yi);
    const double rvx = __dsub_rn((double)vxi, (double)vxj);
    const double rvy = __dsub_rn((double)vyi, (double)vyj);
    const double d2 = __dadd_rn(__dmul_rn(rpx, rpx), __dmul_rn(rpy, rpy));
    const bool coll = !(d2 > R2D);
    const double invH = coll ? m.invDtD : m.invTauD;  // horizon dt (collision, Q4) or tau
    const double wx = __dsub_rn(rvx, __dmul_rn(invH, rpx));
    const double wy = __dsub_rn(rvy, __dmul_rn(invH, rpy));
    const double wl2 = __dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy));
    const double dot1 = __dadd_rn(__dmul_rn(wx, rpx), __dmul_rn(wy, rpy));
    const bool cut = coll || (dot1 < 0.0 && __dmul_rn(dot1, dot1) > __dmul_rn(R2D, wl2));  // w-normal cases
    const double detw = __dsub_rn(__dmul_rn(rpx, wy), __dmul_rn(rpy, wx));
    collision = coll ? 1 : 0;
    if (coll && wl2 == 0.0) {  // coincident, equal velocity (reading Q15)
        nx = (idi < idS[j]) ? -1.0f : 1.0f;  // (the id only here: loaded lazily)
        ny = 0.0f;
        s = fmaf(nx, vxi, ny * vyi) + 0.5f * (R * m.invDtF);
        return FL_G1;
    }
    // cut-off / collision: n = w/|w|, s = n.v_i + (R/h - |w|)/2;  legs: n from the leg
    // direction (left: det > 0, ties right, Q5), s = n.(v_i + v_j)/2
    const float sq = sqrtf((float)(cut ? wl2 : __dsub_rn(d2, R2D)));  // |w| or the leg length
    const float inv = 1.0f / (cut ? sq : (float)d2);
    const float px = (float)rpx, py = (float)rpy;
    const float sg = (detw > 0.0) ? 1.0f : -1.0f;
    const float lnx = -(px * R + sg * py * sq) * inv;
    const float lny = (sg * px * sq - py * R) * inv;
    nx = cut ? (float)wx * inv : lnx;
    ny = cut ? (float)wy * inv : lny;
    const float invHF = coll ? m.invDtF : m.invTauF;
    s = cut ? fmaf(nx, vxi, ny * vyi) + 0.5f * (R * invHF - sq) : 0.5f * fmaf(nx, vxi + vxj, ny * (vyi + vyj));
    return 0u;
}

__device__ __forceinline__ uint32_t orca_line(float xi, float yi, float vxi, float vyi, float xj, float yj, float vxj,
                                              float vyj, uint32_t idi, const uint32_t* __restrict__ idS, uint32_t j, float R, double R2D,
                                              const Model& m, float& nx, float& ny, float& s, int& collision) {
    if (ORCA_LINE_BF)
        return orca_line_bf(xi, yi, vxi, vyi, xj, yj, vxj, vyj, idi, idS, j, R, R2D, m, nx, ny, s, collision);
    return orca_line_branchy(xi, yi, vxi, vyi, xj, yj, vxj, vyj, idi, idS, j, R, R2D, m, nx, ny, s, collision);
}

// ------------------------------------------------------------------- LP
// Lines live in shared memory, one column per thread: half-plane m of this thread is the
// normal n[m * T] (a float2: one 64-bit access) and the offset s[m * T] (the same bank
// pattern for every m -> conflict-free under divergence apart from the 64-bit half-warp split).
struct Lines {
    float2* n;
    float* s;
};

template <bool CNT>
__device__ __forceinline__ bool lp1(const Lines& L, int T, int no, float r, float optx, float opty, bool dirOpt,
                                    float& vx, float& vy, uint32_t& fl, WorkT& w) {
    const float2 ni = L.n[no * T];
    const float nix = ni.x, niy = ni.y, si = L.s[no * T];
    const float disc = (r - si) * (r + si);  // r^2 - s^2: distance of the chord
    if (disc < 0.0f) return false;
    const float sq = sqrtf(disc);
    float tL = -sq, tR = sq;
    const float Dx = niy, Dy = -nix;  // line direction; base point s_i n_i
#ifndef ORCA_LP1_UNROLL
#define ORCA_LP1_UNROLL 1  // r01r: 4 was best with the sequential LP; with the greedy LP 1 is -1.3 % (r01ao)
#endif
#define ORCA_STR_(x) #x
#define ORCA_XSTR_(x) ORCA_STR_(x)
    _Pragma(ORCA_XSTR_(unroll ORCA_LP1_UNROLL))
    for (int j = 0; j < no; ++j) {
        if (CNT) ++w.lp1;
        const float2 nj = L.n[j * T];
        const float njx = nj.x, njy = nj.y, sj = L.s[j * T];
        const float den = fmaf(njx, Dx, njy * Dy);
        const float num = sj - si * fmaf(njx, nix, njy * niy);
        if (fabsf(den) <= kEps) {
            // parallel: fail if pointing away, else skip; an eps-hit matters only if the
            // exact crossing t = num/den could fall inside the chord (reading Q9)
            if (fabsf(num) <= 2e-5f * r + 1e-6f) fl |= FL_G2;
            if (num > 0.0f) return false;
            continue;
        }
        const float t = num / den;
        if (den > 0.0f)
            tL = fmaxf(tL, t);
        else
            tR = fminf(tR, t);
        if (tL > tR) return false;
    }
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

template <bool CNT>
__device__ __forceinline__ int lp2(const Lines& L, int T, int n, float r, float optx, float opty, bool dirOpt,
                                   float& vx, float& vy, uint32_t& fl, WorkT& w) {
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
    for (int i = 0; i < n; ++i) {
        if (CNT) ++w.checks;
        const float2 ni = L.n[i * T];
        const float pen = L.s[i * T] - fmaf(ni.x, vx, ni.y * vy);
        if (pen > 0.0f) {
            const float tx = vx, ty = vy;
            if (!lp1<CNT>(L, T, i, r, optx, opty, dirOpt, vx, vy, fl, w)) {
                vx = tx;
                vy = ty;
                return i;
            }
        }
    }
    return n;
}

// Greedy constraint order (lp order mode 0, the default; reading Q8).  Seidel's incremental
// LP reaches the same optimum for any order of the half-planes, so at every step t
// this LP2 takes, among the half-planes not yet processed (slots [t, n)), the one the current
// point violates most (the first in slot order among equal violations), swaps it into slot t
// and re-solves LP1 on it against the processed slots [0, t) only.  When no remaining
// half-plane is violated the current point is the optimum: it is optimal for the processed
// set and satisfies the rest.  An LP1 failure at step t is an infeasible LP whose first t
// slots are the processed ones -- exactly what LP3 (begin = t) expects.  Compared with the
// sequential order this re-solves only against the few binding half-planes, and the lanes of
// a warp take their steps together (one reconvergence point per step).
__device__ __forceinline__ void line_swap(const Lines& L, int T, int a, int b) {
    const float2 an = L.n[a * T];
    const float as = L.s[a * T];
    L.n[a * T] = L.n[b * T];
    L.s[a * T] = L.s[b * T];
    L.n[b * T] = an;
    L.s[b * T] = as;
}

template <bool CNT>
__device__ __forceinline__ int lp2_greedy(const Lines& L, int T, int n, int kmax, float r, float optx, float opty,
                                          float& vx, float& vy, uint32_t& fl, WorkT& w, unsigned mask) {
    const float l2 = fmaf(optx, optx, opty * opty);
    if (l2 > r * r) {
        const float sc = r / sqrtf(l2);
        vx = optx * sc;
        vy = opty * sc;
    } else {
        vx = optx;
        vy = opty;
    }
    int failed = n;
    bool done = n == 0;
    for (int t = 0; t < kmax; ++t) {
        if (!__any_sync(mask, !done)) break;  // (also the per-step reconvergence point)
        if (done) continue;
        float best = 0.0f;
        int bi = -1;
        for (int q = t; q < n; ++q) {
            if (CNT) ++w.checks;
            const float2 nq = L.n[q * T];
            const float pen = L.s[q * T] - fmaf(nq.x, vx, nq.y * vy);
            if (pen > best) {
                best = pen;
                bi = q;
            }
        }
        if (bi < 0) {
            done = true;
            continue;
        }
        if (bi != t) line_swap(L, T, t, bi);
        const float tx = vx, ty = vy;
        if (!lp1<CNT>(L, T, t, r, optx, opty, false, vx, vy, fl, w)) {
            vx = tx;
            vy = ty;
            failed = t;
            done = true;
        }
    }
    return failed;
}

// ---- LP2 on a lane pair (variant 4): the two lanes of an agent split the
// greedy violation scan and LP1's earlier lines; max/min combines are exact and the tie rule
// (lowest slot) is kept, so the result is lp2_greedy's bit for bit.  An LP1 failure (rare:
// once per infeasible agent) is redone serially by the pair's first lane, so the g2 flags and
// the work counters are exactly those of the serial LP1 (which stops at the failing line).
// Both lanes call it with identical arguments; `pm` is the pair's two lanes, h = lane & 1;
// only lane 0's fl / work counters are meaningful.
template <bool CNT>
__device__ __forceinline__ bool lp1_pair(const Lines& L, int T, int no, float r, float optx, float opty, float& vx,
                                         float& vy, uint32_t& fl, WorkT& w, unsigned pm, int h) {
    const float2 ni = L.n[no * T];
    const float nix = ni.x, niy = ni.y, si = L.s[no * T];
    const float disc = (r - si) * (r + si);
    if (disc < 0.0f) return false;  // (both lanes: the serial lp1 fails before any line)
    const float sq = sqrtf(disc);
    float tL = -sq, tR = sq;
    const float Dx = niy, Dy = -nix;
    bool failp = false;
    uint32_t g2 = 0;
    for (int j = h; j < no; j += 2) {
        const float2 nj = L.n[j * T];
        const float njx = nj.x, njy = nj.y, sj = L.s[j * T];
        const float den = fmaf(njx, Dx, njy * Dy);
        const float num = sj - si * fmaf(njx, nix, njy * niy);
        if (fabsf(den) <= kEps) {
            if (fabsf(num) <= 2e-5f * r + 1e-6f) g2 = FL_G2;
            if (num > 0.0f) failp = true;
            continue;
        }
        const float t = num / den;
        if (den > 0.0f)
            tL = fmaxf(tL, t);
        else
            tR = fminf(tR, t);
    }
    tL = fmaxf(tL, __shfl_xor_sync(pm, tL, 1));
    tR = fminf(tR, __shfl_xor_sync(pm, tR, 1));
    const int ofail = __shfl_xor_sync(pm, (int)failp, 1);  // (not inside || : both lanes must shuffle)
    failp = failp || ofail != 0;
    g2 |= __shfl_xor_sync(pm, g2, 1);
    if (failp || tL > tR) {
        if (h == 0) {  // exact flags and counters of the serial lp1 (which fails too)
            float ux = vx, uy = vy;
            lp1<CNT>(L, T, no, r, optx, opty, false, ux, uy, fl, w);
        }
        return false;
    }
    if (CNT && h == 0) w.lp1 += (uint32_t)no;
    fl |= g2;
    const float od = fmaf(optx, Dx, opty * Dy);
    const float t = fminf(fmaxf(od, tL), tR);
    vx = fmaf(t, Dx, si * nix);
    vy = fmaf(t, Dy, si * niy);
    return true;
}

template <bool CNT>
__device__ __forceinline__ int lp2_greedy_pair(const Lines& L, int T, int n, int kmax, float r, float optx,
                                               float opty, float& vx, float& vy, uint32_t& fl, WorkT& w,
                                               unsigned mask, unsigned pm, int h) {
    const float l2 = fmaf(optx, optx, opty * opty);
    if (l2 > r * r) {
        const float sc = r / sqrtf(l2);
        vx = optx * sc;
        vy = opty * sc;
    } else {
        vx = optx;
        vy = opty;
    }
    int failed = n;
    bool done = n == 0;
    for (int t = 0; t < kmax; ++t) {
        if (!__any_sync(mask, !done)) break;  // (both lanes of a pair share `done`)
        if (done) continue;
        float best = 0.0f;
        int bi = -1;
        for (int q = t + h; q < n; q += 2) {
            if (CNT) ++w.checks;
            const float2 nq = L.n[q * T];
            const float pen = L.s[q * T] - fmaf(nq.x, vx, nq.y * vy);
            if (pen > best) {
                best = pen;
                bi = q;
            }
        }
        // the larger penetration; equal ones -> the lower slot (the serial scan's first)
        const float ob = __shfl_xor_sync(pm, best, 1);
        const int oi = __shfl_xor_sync(pm, bi, 1);
        if (oi >= 0 && (ob > best || (ob == best && (bi < 0 || oi < bi)))) {
            best = ob;
            bi = oi;
        }
        if (bi < 0) {
            done = true;
            continue;
        }
        if (bi != t && h == 0) line_swap(L, T, t, bi);
        __syncwarp(pm);
        const float tx = vx, ty = vy;
        if (!lp1_pair<CNT>(L, T, t, r, optx, opty, vx, vy, fl, w, pm, h)) {
            vx = tx;
            vy = ty;
            failed = t;
            done = true;
        }
    }
    return failed;
}

// Warp-synchronised LP2 / LP3: the same arithmetic as lp2 / lp3, but every
// lane in `mask` runs the same number (kmax) of constraint iterations -- lines it does not
// have are skipped -- with a reconvergence point after each, so the lanes that re-solve on
// the same line i run that re-solve together (with equal trip counts i) instead of drifting
// apart.  Each lane in `mask` must call it exactly once with the same kmax.
#ifndef ORCA_SYNC_LP
#define ORCA_SYNC_LP 1
#endif
template <bool CNT>
__device__ __forceinline__ int lp2_sync(const Lines& L, int T, int n, int kmax, float r, float optx, float opty,
                                        float& vx, float& vy, uint32_t& fl, WorkT& w, unsigned mask) {
    const float l2 = fmaf(optx, optx, opty * opty);
    if (l2 > r * r) {
        const float sc = r / sqrtf(l2);
        vx = optx * sc;
        vy = opty * sc;
    } else {
        vx = optx;
        vy = opty;
    }
    int failed = n;
    for (int i = 0; i < kmax; ++i) {
        if (i < n && failed == n) {
            if (CNT) ++w.checks;
            const float2 ni = L.n[i * T];
            const float pen = L.s[i * T] - fmaf(ni.x, vx, ni.y * vy);
            if (pen > 0.0f) {
                const float tx = vx, ty = vy;
                if (!lp1<CNT>(L, T, i, r, optx, opty, false, vx, vy, fl, w)) {
                    vx = tx;
                    vy = ty;
                    failed = i;
                }
            }
        }
        __syncwarp(mask);
    }
    return failed;
}

// Work-unit LP2 (§8(f3)): "subdivide the calculation into work units ... If the
// thread does not need to compute a new velocity, then it can aid in another problem's
// calculation."  Same constraint loop as lp2_sync; at line i the lanes whose current point
// violates it (a warp-uniform ballot V) need the LP1 re-solve against lines 0..i-1.  One
// work unit = one (problem, line j) pair: a segment of S = 2^ceil(log2 i) lanes takes one
// problem, lane j of the segment evaluates line j of that problem (read from the owner's
// shared-memory column), and a segmented inclusive max/min scan rebuilds the chord interval
// [tL, tR] of every prefix -- the serial loop's state after line j -- so the first failing
// line, the g2 flags up to it and the final interval equal the serial lp1's bit for bit
// (max/min are exact).  32/S problems per round; with more than `maxRounds` rounds the warp
// keeps the serial per-lane re-solve for that line.  Requires the lanes of `mask` to be
// lanes 0..popc(mask)-1 (k_step's active lanes are a prefix of the warp).
#ifndef ORCA_WU_ROUNDS
#define ORCA_WU_ROUNDS 2
#endif
template <bool CNT>
__device__ __forceinline__ int lp2_wu(const Lines& L, int T, int n, int kmax, float r, float optx, float opty,
                                      float& vx, float& vy, uint32_t& fl, WorkT& w, unsigned mask) {
    const float l2 = fmaf(optx, optx, opty * opty);
    if (l2 > r * r) {
        const float sc = r / sqrtf(l2);
        vx = optx * sc;
        vy = opty * sc;
    } else {
        vx = optx;
        vy = opty;
    }
    const int lane = threadIdx.x & 31;
    const int A = __popc(mask);  // participating lanes 0..A-1
    int failed = n;
    for (int i = 0; i < kmax; ++i) {
        bool need = false;
        if (i < n && failed == n) {
            if (CNT) ++w.checks;
            const float2 ni = L.n[i * T];
            need = L.s[i * T] - fmaf(ni.x, vx, ni.y * vy) > 0.0f;
        }
        const unsigned V = __ballot_sync(mask, need);
        if (V == 0u) continue;
        const int S = (i <= 1) ? 1 : (1 << (32 - __clz(i - 1)));  // segment width >= i
        const int P = A / S;                                       // problems per round
        const int nV = __popc(V);
        if (i == 0 || P == 0 || nV > P * ORCA_WU_ROUNDS) {
            // serial per-lane re-solve (no lines to check, or too many problems)
            if (need) {
                const float tx = vx, ty = vy;
                if (!lp1<CNT>(L, T, i, r, optx, opty, false, vx, vy, fl, w)) {
                    vx = tx;
                    vy = ty;
                    failed = i;
                }
            }
            __syncwarp(mask);
            continue;
        }
        const int myRank = __popc(V & ((1u << lane) - 1u));  // owners: rank among V
        __shared__ unsigned char wuOwner[1024];                // problem rank -> owner lane
        const int wb = threadIdx.x & ~31;
        __syncwarp(mask);  // every lane's reads of the previous line's owners are done (racecheck)
        if (need) wuOwner[wb + myRank] = (unsigned char)lane;
        __syncwarp(mask);
        const int seg = lane / S, j = lane - seg * S;
        const unsigned segBits = (S == 32) ? 0xffffffffu : ((1u << S) - 1u);
        for (int base = 0; base < nV; base += P) {
            const int p = base + seg;
            const bool valid = (seg < P) && (p < nV);
            const int o = valid ? (int)wuOwner[wb + p] : lane;  // owner lane of problem p
            const int d = o - lane;                              // column offset to the owner
            const float ro = __shfl_sync(mask, r, o);
            const float2 nid = L.n[i * T + d];
            const float nix = nid.x, niy = nid.y, si = L.s[i * T + d];
            const float sq = sqrtf(fmaxf((ro - si) * (ro + si), 0.0f));
            float tL = -sq, tR = sq;
            bool parF = false, g2 = false;
            if (valid && j < i) {
                const float Dx = niy, Dy = -nix;
                const float2 njd = L.n[j * T + d];
                const float njx = njd.x, njy = njd.y, sj = L.s[j * T + d];
                const float den = fmaf(njx, Dx, njy * Dy);
                const float num = sj - si * fmaf(njx, nix, njy * niy);
                if (fabsf(den) <= kEps) {
                    g2 = fabsf(num) <= 2e-5f * ro + 1e-6f;
                    parF = num > 0.0f;
                } else {
                    const float t = num / den;
                    if (den > 0.0f)
                        tL = fmaxf(tL, t);
                    else
                        tR = fminf(tR, t);
                }
            }
            // segmented inclusive scan: (tL, tR) of lane j = the serial state after line j
            for (int q = 1; q < S; q <<= 1) {
                const float uL = __shfl_up_sync(mask, tL, q, S);
                const float uR = __shfl_up_sync(mask, tR, q, S);
                if (j >= q) {
                    tL = fmaxf(tL, uL);
                    tR = fminf(tR, uR);
                }
            }
            const bool fail = valid && j < i && (parF || tL > tR);
            const unsigned Bf = (__ballot_sync(mask, fail) >> (seg * S)) & segBits;
            const int f = Bf ? __ffs(Bf) - 1 : i;  // first failing line (i: none)
            const unsigned Bg = (__ballot_sync(mask, g2 && j <= f) >> (seg * S)) & segBits;
            const int code = (f >= i ? 1 : 0) | (Bg ? 2 : 0) | ((f < i ? f + 1 : i) << 2);
            // lane i-1 of the owner's segment holds the whole interval: deliver it
            const bool mine = need && myRank >= base && myRank < base + P;
            const int src = mine ? (myRank - base) * S + i - 1 : lane;
            const float rL = __shfl_sync(mask, tL, src), rR = __shfl_sync(mask, tR, src);
            const int rc = __shfl_sync(mask, code, src);
            if (mine) {
                const float2 oin = L.n[i * T];
                const float oix = oin.x, oiy = oin.y, osi = L.s[i * T];
                if ((r - osi) * (r + osi) < 0.0f) {
                    failed = i;  // empty chord: the serial lp1 fails before any line
                } else {
                    if (CNT) w.lp1 += (uint32_t)(rc >> 2);
                    if (rc & 2) fl |= FL_G2;
                    if (rc & 1) {
                        const float Dx = oiy, Dy = -oix;
                        const float od = fmaf(optx, Dx, opty * Dy);
                        const float t = fminf(fmaxf(od, rL), rR);
                        vx = fmaf(t, Dx, osi * oix);
                        vy = fmaf(t, Dy, osi * oiy);
                    } else {
                        failed = i;
                    }
                }
            }
        }
    }
    return failed;
}

// LP3: least penetration from the LP2 failure index.  The projected constraint
// "penetration_j <= penetration_i" is the line (n_j - n_i).v >= s_j - s_i, normalised.
template <bool CNT>
__device__ __forceinline__ void lp3(const Lines& L, const Lines& P, int T, int n, int begin, float r, float& vx,
                                    float& vy, uint32_t& fl, WorkT& w) {
    float dist = 0.0f;
    for (int i = begin; i < n; ++i) {
        const float2 ni = L.n[i * T];
        const float nix = ni.x, niy = ni.y, si = L.s[i * T];
        if (si - fmaf(nix, vx, niy * vy) > dist) {
            int m = 0;
            for (int j = 0; j < i; ++j) {
                const float2 nj = L.n[j * T];
                const float njx = nj.x, njy = nj.y, sj = L.s[j * T];
                const float det = fmaf(nix, njy, -niy * njx);
                if (fabsf(det) <= kEps && fmaf(nix, njx, niy * njy) > 0.0f) {
                    // same direction: skipped; matters only if the lines nearly coincide
                    if (fabsf(sj - si) <= 2e-5f * r + 1e-6f) fl |= FL_G2;
                    continue;
                }
                if (CNT) ++w.proj;
                const float dx = njx - nix, dy = njy - niy;
                const float il = 1.0f / sqrtf(fmaf(dx, dx, dy * dy));
                P.n[m * T] = make_float2(dx * il, dy * il);
                P.s[m * T] = (sj - si) * il;
                ++m;
            }
            const float tx = vx, ty = vy;
            if (lp2<CNT>(P, T, m, r, nix, niy, true, vx, vy, fl, w) < m) {
                vx = tx;  // floating-point failure: keep the current point
                vy = ty;
            }
            dist = si - fmaf(nix, vx, niy * vy);
        }
    }
}

// Directional LP2 of LP3's projected problem (lp2 with dirOpt), warp-synchronised like
// lp2_sync: the lanes of `mask` (all at the same LP3 line, so kmax = that line's index is
// uniform) run kmax constraint iterations with a reconvergence point after each, so the
// LP1 re-solves at the same projected line run together.
#ifndef ORCA_SYNC_LP3_INNER
#define ORCA_SYNC_LP3_INNER 0  // swept r01ae: 1 is +1.4 % (1M), +3 % (dense)
#endif
template <bool CNT>
__device__ __forceinline__ int lp2_dir_sync(const Lines& P, int T, int m, int kmax, float r, float dx, float dy,
                                            float& vx, float& vy, uint32_t& fl, WorkT& w, unsigned mask) {
    vx = dx * r;
    vy = dy * r;
    int failed = m;
    for (int i = 0; i < kmax; ++i) {
        if (i < m && failed == m) {
            if (CNT) ++w.checks;
            const float2 ni = P.n[i * T];
            const float pen = P.s[i * T] - fmaf(ni.x, vx, ni.y * vy);
            if (pen > 0.0f) {
                const float tx = vx, ty = vy;
                if (!lp1<CNT>(P, T, i, r, dx, dy, true, vx, vy, fl, w)) {
                    vx = tx;
                    vy = ty;
                    failed = i;
                }
            }
        }
        __syncwarp(mask);
    }
    return failed;
}

// LP3 in the greedy order (lp order mode 0; reading Q8): Seidel's incremental 3-D LP for the
// least-penetration velocity reaches the same penetration for any insertion order, so
// at each step the half-plane penetrated most beyond the running penetration `dist` among
// slots [t, n) (lowest slot among equals) is swapped into slot t and the projected LP over the
// processed slots [0, t) runs; when none exceeds dist the point is optimal.  One
// reconvergence point per step.
template <bool CNT>
__device__ __forceinline__ void lp3_greedy(const Lines& L, const Lines& P, int T, int TP, int n, int begin, int kmax, float r,
                                           float& vx, float& vy, uint32_t& fl, WorkT& w, unsigned mask) {
    float dist = 0.0f;
    bool done = begin >= n;
    for (int t = 0; t < kmax; ++t) {  // uniform trip count over the lanes of `mask`
        if (!__any_sync(mask, !done)) break;
        if (done || t < begin) continue;
        float best = dist;
        int bi = -1;
        for (int q = t; q < n; ++q) {
            const float2 nq = L.n[q * T];
            const float pen = L.s[q * T] - fmaf(nq.x, vx, nq.y * vy);
            if (pen > best) {
                best = pen;
                bi = q;
            }
        }
        if (CNT) w.checks += (uint32_t)(n - t);
        if (bi < 0) {
            done = true;
            continue;
        }
        if (bi != t) line_swap(L, T, t, bi);
        const float2 ni = L.n[t * T];
        const float nix = ni.x, niy = ni.y, si = L.s[t * T];
        int m = 0;
        for (int j = 0; j < t; ++j) {
            const float2 nj = L.n[j * T];
            const float njx = nj.x, njy = nj.y, sj = L.s[j * T];
            const float det = fmaf(nix, njy, -niy * njx);
            if (fabsf(det) <= kEps && fmaf(nix, njx, niy * njy) > 0.0f) {
                if (fabsf(sj - si) <= 2e-5f * r + 1e-6f) fl |= FL_G2;
                continue;
            }
            if (CNT) ++w.proj;
            const float dx = njx - nix, dy = njy - niy;
            const float il = 1.0f / sqrtf(fmaf(dx, dx, dy * dy));
            P.n[m * TP] = make_float2(dx * il, dy * il);
            P.s[m * TP] = (sj - si) * il;
            ++m;
        }
        const float tx = vx, ty = vy;
        if (lp2<CNT>(P, TP, m, r, nix, niy, true, vx, vy, fl, w) < m) {
            vx = tx;  // floating-point failure: keep the current point
            vy = ty;
        }
        dist = si - fmaf(nix, vx, niy * vy);
    }
}

// lp3 with a uniform kmax-iteration outer loop and a reconvergence point per line (see
// lp2_sync); the inner projected LP2 is lp2_dir_sync over the lanes at the same line.
template <bool CNT>
__device__ __forceinline__ void lp3_sync(const Lines& L, const Lines& P, int T, int TP, int n, int begin, int kmax, float r,
                                         float& vx, float& vy, uint32_t& fl, WorkT& w, unsigned mask) {
    float dist = 0.0f;
    for (int i = 0; i < kmax; ++i) {
        bool part = false;
        float nix = 0.0f, niy = 0.0f, si = 0.0f;
        if (i >= begin && i < n) {
            const float2 ni = L.n[i * T];
            nix = ni.x;
            niy = ni.y;
            si = L.s[i * T];
            part = si - fmaf(nix, vx, niy * vy) > dist;
        }
        const unsigned pm = ORCA_SYNC_LP3_INNER ? __ballot_sync(mask, part) : 0u;
        {
            if (part) {
                int m = 0;
                for (int j = 0; j < i; ++j) {
                    const float2 nj = L.n[j * T];
                    const float njx = nj.x, njy = nj.y, sj = L.s[j * T];
                    const float det = fmaf(nix, njy, -niy * njx);
                    if (fabsf(det) <= kEps && fmaf(nix, njx, niy * njy) > 0.0f) {
                        if (fabsf(sj - si) <= 2e-5f * r + 1e-6f) fl |= FL_G2;
                        continue;
                    }
                    if (CNT) ++w.proj;
                    const float dx = njx - nix, dy = njy - niy;
                    const float il = 1.0f / sqrtf(fmaf(dx, dx, dy * dy));
                    P.n[m * TP] = make_float2(dx * il, dy * il);
                    P.s[m * TP] = (sj - si) * il;
                    ++m;
                }
                const float tx = vx, ty = vy;
                const int fm = ORCA_SYNC_LP3_INNER ? lp2_dir_sync<CNT>(P, TP, m, i, r, nix, niy, vx, vy, fl, w, pm)
                                                   : lp2<CNT>(P, TP, m, r, nix, niy, true, vx, vy, fl, w);
                if (fm < m) {
                    vx = tx;
                    vy = ty;
                }
                dist = si - fmaf(nix, vx, niy * vy);
            }
        }
        __syncwarp(mask);
    }
}

// The least-penetration LP as an out-of-line call inside k_step (ORCA_COLD_NOINLINE): it runs
// once per infeasible agent, so a call costs little, while inlining it (twice: the per-thread
// and the block-queue placements, each in both LP orders) roughly doubles k_step's code and its
// instruction-cache footprint around the hot selection loops.
#ifndef ORCA_COLD_NOINLINE
#define ORCA_COLD_NOINLINE 0
#endif
template <bool CNT>
__device__ __noinline__ void lp3_call(Lines L, Lines P, int T, int TP, int n, int begin, int kmax, float r, float* vxy,
                                      uint32_t* fl, WorkT* w, unsigned mask, bool greedy) {
    float vx = vxy[0], vy = vxy[1];
    if (greedy)
        lp3_greedy<CNT>(L, P, T, TP, n, begin, kmax, r, vx, vy, *fl, *w, mask);
    else
        lp3_sync<CNT>(L, P, T, TP, n, begin, kmax, r, vx, vy, *fl, *w, mask);
    vxy[0] = vx;
    vxy[1] = vy;
}
template <bool CNT>
__device__ __forceinline__ void lp3_dispatch(const Lines& L, const Lines& P, int T, int TP, int n, int begin, int kmax,
                                             float r, float& vx, float& vy, uint32_t& fl, WorkT& w, unsigned mask,
                                             bool greedy) {
    if (ORCA_COLD_NOINLINE) {
        float vxy[2] = {vx, vy};
        lp3_call<CNT>(L, P, T, TP, n, begin, kmax, r, vxy, &fl, &w, mask, greedy);
        vx = vxy[0];
        vy = vxy[1];
    } else if (greedy) {
        lp3_greedy<CNT>(L, P, T, TP, n, begin, kmax, r, vx, vy, fl, w, mask);
    } else {
        lp3_sync<CNT>(L, P, T, TP, n, begin, kmax, r, vx, vy, fl, w, mask);
    }
}

// --------------------------------------------------------------------- fused step
struct StepArgs {
    Grid g;
    Model m;
    // cell-sorted (rest) state
    const float2* __restrict__ posS;
    const float2* __restrict__ velS;
    const float2* __restrict__ auxS;  // prefVel, or goal when m.goals
    const float* __restrict__ rk2S;   // previous step's fp32 d2 of the k-th neighbour (+inf: none)
    const float4* __restrict__ propS; // heterogeneous crowds: (radius, maxSpeed, prefSpeed, 0);
                                      // nullptr = the global parameters
    const uint32_t* __restrict__ idS;
    const uint32_t* __restrict__ binStart;
    // outputs of a real step (work buffers, next step's binning)
    float2* posW;
    float2* velW;
    float2* auxW;
    float* rk2W;
    float4* propW;
    uint32_t* idW;
    uint32_t* cellW;
    uint32_t* rankW;
    uint32_t* count;
    unsigned long long* stats;
    int* ctr;   // per-domain counters (CT_*)
    int capW;   // work / sorted array capacity
    int phase;  // strips' halo overlap: 0 every owned agent; 1 the agents of the
                // two boundary columns on each side (everything that can end in an edge
                // column or leave the strip); 2 the interior columns [c0 + 2, c1 - 2)
    ExBuf sendL, sendR;
    // outputs of a dry (debug) step, indexed by global id
    float2* dbgV;
    uint8_t* dbgFlags;
    int32_t* dbgNbr;
    int32_t* dbgCnt;
    Work* work;  // dry step only: instrumented work counts (nullable)
    // LP3 queue: agents whose LP2 failed are finished by k_lp3 (compacted)
    int4* qEntry;          // (i, cnt | f << 8 | flags << 16, vx bits, vy bits)
    float4* qLines;        // line m of entry q at [m * qcap + q] = (nx, ny, s, 0)
    unsigned int* qCount;  // zeroed before every step
    int qcap;
    int lp3Inline;  // 1: k_step finishes its infeasible agents itself (small strips; no k_lp3)
    int* gridFlag;  // host-mapped: set when an agent enters the grid's outer cell ring
};
static_assert(sizeof(Grid) == 104 && sizeof(Model) == 104 && sizeof(ExBuf) % 8 == 0, "padding-free layouts");

#ifndef ORCA_STEP_THREADS
#define ORCA_STEP_THREADS 128
#endif
constexpr int kStepThreads = ORCA_STEP_THREADS;

// Per-thread shared memory (32-bit words, one column per thread, stride kStepThreads):
//   [0, k)            top-k list fp32 d2   -> half-plane nx
//   [k, 2k)           top-k list j         -> half-plane ny (slot q read before written)
//   [2k, 2k + B)      candidate buffer j   -> half-plane s in its first k words
//   [2k + B, 2k + 2B) candidate buffer fp32 d2            (B = k + 8)
#ifndef ORCA_BUF_EXTRA
#define ORCA_BUF_EXTRA 14  // candidate buffer = k + this many entries
#endif
__host__ __device__ constexpr int step_buf_words(int k) { return k + ORCA_BUF_EXTRA; }
#ifndef ORCA_SHIFT2
#define ORCA_SHIFT2 0  // insertion shift loop two entries per iteration (r02 sweep)
#endif
#ifndef ORCA_SCAN_UNROLL
#define ORCA_SCAN_UNROLL 2  // candidates per scan iteration (2: r01; see DESIGN.md §12 r02)
#endif
#ifndef ORCA_SCAN_UNROLL_LM0
#define ORCA_SCAN_UNROLL_LM0 3  // r02ar: the k_lp3-placement kernel, 1M -0.7 %, dense -1 % vs 2 (4: +0.7 %)
#endif
#ifndef ORCA_BUF1
#define ORCA_BUF1 1  // 1: the buffer keeps j only; the merge recomputes the fp32 d2 (r01o: -8 %)
#endif
// projected half-plane columns of the block-queue LP3 beyond the per-thread columns (stride
// kLp3Scratch): progress when no column is free (every agent of a block infeasible)
constexpr int kLp3Scratch = 8;
__host__ __device__ constexpr int step_lp3q_scratch_bytes(int k) { return 4 * 3 * k * kLp3Scratch; }
__host__ __device__ constexpr int step_smem_per_thread(int k) {
    return 4 * (2 * k + (ORCA_BUF1 ? 1 : 2) * step_buf_words(k));
}

__device__ __forceinline__ double exact_key(float2 pj, float2 pi) {
    const double Dx = __dsub_rn((double)pj.x, (double)pi.x);
    const double Dy = __dsub_rn((double)pj.y, (double)pi.y);
    return __dadd_rn(__dmul_rn(Dx, Dx), __dmul_rn(Dy, Dy));
}

// fp32 d^2 = fma(dx, dx, dy*dy) has relative error < 2^-22 against the exact fp64 key
// kappa (reading Q11), so fa < fb (1 - 2^-20) proves kappa_a < kappa_b.  Only near-ties
// (and tiny values, where subnormals void the bound) fall back to the exact keys.
constexpr float kSep = 1.0f - 0x1p-20f;

// Exact (kappa, id) order of candidates ja (fp32 d2 fa) and jb (fb) around agent pi.
__device__ __forceinline__ bool cand_less(float fa, uint32_t ja, float fb, uint32_t jb, float2 pi,
                                          const float2* __restrict__ posS, const uint32_t* __restrict__ idS) {
    if (fa < fb * kSep && fb > 1e-30f) return true;
    if (fb < fa * kSep && fa > 1e-30f) return false;
    const double ka = exact_key(posS[ja], pi), kb = exact_key(posS[jb], pi);
    if (ka != kb) return ka < kb;
    return idS[ja] < idS[jb];
}

// Strictly within r_obs (reading Q10): exact test only near the boundary.
__device__ __forceinline__ bool in_radius(float f, uint32_t j, float2 pi, float nd2Lo, float nd2Hi, double nd2,
                                          const float2* __restrict__ posS) {
    if (f < nd2Lo) return true;
    if (f > nd2Hi) return false;
    return exact_key(posS[j], pi) < nd2;
}

// Register-resident sorted list of the KR nearest candidates (+inf padded).  Insertion
// compares in fp32 only and is branch-free (a warp stays converged however many
// candidates each thread merges); a comparison inside the 2^-20 margin (a possible
// exact-order disagreement) raises `tie`, and the caller then redoes the agent's selection
// on the exact shared-memory path.  Without a tie, every comparison agrees with the exact
// (kappa, id) order, so the list is the exact one.
template <int KR>
struct RegList {
    float f[KR];
    uint32_t j[KR];
};

template <int KR>
__device__ __forceinline__ void reg_clear(RegList<KR>& L) {
#pragma unroll
    for (int p = 0; p < KR; ++p) {
        L.f[p] = INFINITY;
        L.j[p] = 0u;
    }
}

template <int KR>
__device__ __forceinline__ void reg_insert(RegList<KR>& L, float f, uint32_t j, bool& tie) {
    int pos = 0;
    bool t = !(f > 1e-30f);  // subnormal range: the relative error bound does not hold
#pragma unroll
    for (int p = 0; p < KR; ++p) {
        const float of = L.f[p];
        const bool before = of < f * kSep;  // slot p surely nearer
        const bool after = f < of * kSep;   // slot p surely farther (also of = +inf)
        t |= !(before || after);
        pos += before ? 1 : 0;
    }
    tie |= t;
#pragma unroll
    for (int p = KR - 1; p >= 0; --p) {
        const float pf = (p > 0) ? L.f[p - 1] : f;
        const uint32_t pj = (p > 0) ? L.j[p - 1] : j;
        L.f[p] = (p > pos) ? pf : ((p == pos) ? f : L.f[p]);
        L.j[p] = (p > pos) ? pj : ((p == pos) ? j : L.j[p]);
    }
}

template <int KR>
__device__ __forceinline__ float reg_f(const RegList<KR>& L, int q) {
    float r = INFINITY;
#pragma unroll
    for (int p = 0; p < KR; ++p) r = (p == q) ? L.f[p] : r;
    return r;
}

// fp32 d2 of buffered candidate b: stored, or (ORCA_BUF1) recomputed with the scan's
// expression -- the same bits
template <int T = kStepThreads>
__device__ __forceinline__ float buf_d2(const float* Bff, int b, uint32_t j, float2 pi,
                                        const float2* __restrict__ posS) {
    if (ORCA_BUF1) {
        const float2 p = posS[j];
        const float dx = p.x - pi.x, dy = p.y - pi.y;
        return fmaf(dx, dx, dy * dy);
    }
    return Bff[b * T];
}

// buffered (j, fp32 d2) candidates into the register list (inside r_obs only)
template <int KR, int T = kStepThreads>
__device__ __forceinline__ void reg_merge(RegList<KR>& L, int& cnt, const uint32_t* Bj, const float* Bff, int nb,
                                          float2 pi, const Model& m, const float2* __restrict__ posS, bool& tie) {
    for (int b = 0; b < nb; ++b) {
        const uint32_t j = Bj[b * T];
        const float f = buf_d2<T>(Bff, b, j, pi, posS);
        if (!in_radius(f, j, pi, m.nd2Lo, m.nd2Fup, m.nd2D, posS)) continue;
        reg_insert<KR>(L, f, j, tie);
        cnt = min(cnt + 1, KR);
    }
}

// Exact (kappa, id) order of candidates ja and jb around agent pi (fp64 keys).
__device__ __forceinline__ bool exact_less(uint32_t ja, uint32_t jb, float2 pi, const float2* __restrict__ posS,
                                           const uint32_t* __restrict__ idS) {
    const double ka = exact_key(posS[ja], pi), kb = exact_key(posS[jb], pi);
    if (ka != kb) return ka < kb;
    return idS[ja] < idS[jb];
}

// Merge the nb buffered candidates (j, fp32 d2) into the sorted top-k list (Lf = fp32 d2
// bits, Lj = j).  Returns the new list length.  With f > 1e-30 (the relative error bound of
// the fp32 d2 holds) a list entry o is surely farther if f (1 + 2^-19) < o and surely nearer
// if o < f (1 - 2^-19) -- one compare per step on the insertion path; only the band between
// takes the exact fp64 keys (ORCA_FAST_MERGE; 0 = cand_less at every step).
#ifndef ORCA_FAST_MERGE
#define ORCA_FAST_MERGE 1
#endif
#ifndef ORCA_MERGE_PF
#define ORCA_MERGE_PF 1  // r02at: 1M -0.7 %. 1: the merge loads the next buffered candidate during the current insertion
#endif
// List entries are (fp32 d2 bits, j) pairs in one 64-bit shared-memory slot each: a shift
// step of the insertion is one 64-bit load and one 64-bit store.
// allIn: every buffered candidate has fp32 d2 <= a pass threshold below nd2Lo, i.e. is surely
// strictly within r_obs (in_radius would return true at its first compare).
template <int T = kStepThreads>
__device__ __forceinline__ int merge_candidates(uint2* Lst, int cnt, int k, const uint32_t* Bf,
                                                const float* Bff, int nb, float2 pi, const Model& m,
                                                const float2* __restrict__ posS, const uint32_t* __restrict__ idS,
                                                bool allIn = false) {
#if ORCA_MERGE_PF && ORCA_BUF1
    // the next buffered candidate's index and position are loaded while this one is inserted
    uint32_t jn = (nb > 0) ? Bf[0] : 0u;
    float2 pn = (nb > 0) ? posS[jn] : make_float2(0.0f, 0.0f);
#endif
    for (int b = 0; b < nb; ++b) {
#if ORCA_MERGE_PF && ORCA_BUF1
        const uint32_t j = jn;
        const float2 pj = pn;
        if (b + 1 < nb) {
            jn = Bf[(b + 1) * T];
            pn = posS[jn];
        }
        const float dxm = pj.x - pi.x, dym = pj.y - pi.y;
        const float f = fmaf(dxm, dxm, dym * dym);  // (buf_d2's expression: the scan's bits)
#else
        const uint32_t j = Bf[b * T];
        const float f = buf_d2<T>(Bff, b, j, pi, posS);
#endif
        if (!allIn && !in_radius(f, j, pi, m.nd2Lo, m.nd2Fup, m.nd2D, posS)) continue;
        if (ORCA_FAST_MERGE && f > 1e-30f) {
            const float fhi = f * (1.0f + 0x1p-19f), flo = f * (1.0f - 0x1p-19f);
            int p = cnt;
            if (cnt == k) {  // beyond the k-th: rejected
                const uint2 o = Lst[(k - 1) * T];
                const float of = __uint_as_float(o.x);
                if (!(fhi < of) && (of < flo || !exact_less(j, o.y, pi, posS, idS))) continue;
                p = k - 1;
            }
            uint2* q = Lst + p * T;
            // fast path: shift while the entry below is surely farther (one fp32 compare)
#if ORCA_SHIFT2
            // two entries per iteration: both loads in flight before the first compare
            while (p > 1) {
                const uint2 o1 = q[-T], o2 = q[-2 * T];
                if (!(fhi < __uint_as_float(o1.x))) break;
                *q = o1;
                q -= T;
                --p;
                if (!(fhi < __uint_as_float(o2.x))) break;
                *q = o2;
                q -= T;
                --p;
            }
#endif
            while (p > 0) {
                const uint2 o = q[-T];
                if (!(fhi < __uint_as_float(o.x))) break;
                *q = o;
                q -= T;
                --p;
            }
            // the entry below is not surely farther: unless surely nearer, the exact fp64 keys
            // decide (a near-tie, rare), and the shifting continues on them
            while (p > 0) {
                const uint2 o = q[-T];
                const float of = __uint_as_float(o.x);
                if (of < flo) break;
                if (!(fhi < of) && !exact_less(j, o.y, pi, posS, idS)) break;
                *q = o;
                q -= T;
                --p;
            }
            *q = make_uint2(__float_as_uint(f), j);
            if (cnt < k) ++cnt;
            continue;
        }
        if (cnt == k) {
            const uint2 o = Lst[(k - 1) * T];
            if (!cand_less(f, j, __uint_as_float(o.x), o.y, pi, posS, idS)) continue;
        }
        int p = (cnt < k) ? cnt : k - 1;
        while (p > 0) {
            const uint2 o = Lst[(p - 1) * T];
            if (!cand_less(f, j, __uint_as_float(o.x), o.y, pi, posS, idS)) break;
            Lst[p * T] = o;
            --p;
        }
        Lst[p * T] = make_uint2(__float_as_uint(f), j);
        if (cnt < k) ++cnt;
    }
    return cnt;
}

// ---------------------------------------------------------- integrate + route
__device__ __forceinline__ void push_halo(const ExBuf& x, int* ctr, float2 p, float2 v, uint32_t id, float r) {
    const int s = atomicAdd(&x.hdr[1], 1);
    if (s >= x.capH) {
        atomicOr(&ctr[CT_OVF], OVF_HALO);
        return;
    }
    x.hpos[s] = p;
    x.hvel[s] = v;
    x.hid[s] = id;
    x.hrad[s] = r;
}

// Append one entry to the work buffers at nOwn + extra (ghosts, immigrants).
__device__ __forceinline__ void append_work(const StepArgs& a, int nOwn, int fx, int sy, float2 p, float2 v, float2 aux,
                                            uint32_t id, float rk2, float4 pr) {
    const int e = nOwn + atomicAdd(&a.ctr[CT_EXTRA], 1);
    if (e >= a.capW) {
        atomicOr(&a.ctr[CT_OVF], OVF_WORK);
        return;
    }
    const uint32_t c = bin_of(fx, sy, a.g);
    a.posW[e] = p;
    a.velW[e] = v;
    a.auxW[e] = aux;
    a.idW[e] = id;
    a.rk2W[e] = rk2;
    if (a.propW) a.propW[e] = pr;
    a.cellW[e] = c;
    a.rankW[e] = atomicAdd(&a.count[c], 1u);
}

// Explicit Euler p' = p + dt v' and routing for the next step: the agent
// stays in this strip (bin + rank at its work slot w; a halo copy to the neighbour if it
// sits in an edge column), or emigrates (exchange buffer, plus a local ghost entry since
// it now sits in this strip's ghost column).  Single-GPU: always stays.  pr: the agent's
// (radius, maxSpeed, prefSpeed, 0) when heterogeneous.
// MONO: one strip (every agent stays: no halo copies, no emigration) of homogeneous agents.
template <bool MONO = false>
__device__ __forceinline__ void finish_agent(const StepArgs& a, int w, int nOwn, float2 pi, float vx, float vy,
                                             float2 aux, uint32_t id, float rk2, float4 pr) {
    const float2 pn = make_float2(fmaf(a.m.dt, vx, pi.x), fmaf(a.m.dt, vy, pi.y));
    const float2 vn = make_float2(vx, vy);
    if (a.m.removeR2 > 0.0f) {
        // P:110 "Once a person reaches the goal location they are removed from the
        // simulation": within removeR of the goal after the move -> not re-inserted
        const float gx = aux.x - pn.x, gy = aux.y - pn.y;
        if (fmaf(gx, gx, gy * gy) < a.m.removeR2) {
            a.cellW[w] = kInvalid;
            atomicAdd(&a.stats[ST_REMOVED], 1ull);
            return;
        }
    }
    const int fx = finecol_coord(pn.x, a.g);
    const int cx = fx >> a.g.lgC;  // = cell_coord(pn.x, ...)
    const int sy = subrow_coord(pn.y, a.g);
    if (a.gridFlag) {  // the outer ring: beyond it positions are clamped -> re-derive the grid
        const int cyc = sy >> a.g.lgS;
        if (cx == 0 || cx == a.g.nx - 1 || cyc == 0 || cyc == a.g.ny - 1) *a.gridFlag = 1;
    }
    if (MONO || (cx >= a.g.c0 && cx < a.g.c1)) {
        const uint32_t c = bin_of(fx, sy, a.g);
        a.posW[w] = pn;
        a.velW[w] = vn;
        a.auxW[w] = aux;
        a.idW[w] = id;
        a.rk2W[w] = rk2;
        if (!MONO && a.propW) a.propW[w] = pr;
        a.cellW[w] = c;
        a.rankW[w] = atomicAdd(&a.count[c], 1u);
        if (!MONO && cx == a.g.c0 && a.g.hasL) push_halo(a.sendL, a.ctr, pn, vn, id, pr.x);
        if (!MONO && cx == a.g.c1 - 1 && a.g.hasR) push_halo(a.sendR, a.ctr, pn, vn, id, pr.x);
    } else {
        a.cellW[w] = kInvalid;
        const ExBuf& x = (cx < a.g.c0) ? a.sendL : a.sendR;
        const int s = atomicAdd(&x.hdr[0], 1);
        if (s >= x.capM) {
            atomicOr(&a.ctr[CT_OVF], OVF_MIG);
        } else {
            x.mpos[s] = pn;
            x.mvel[s] = vn;
            x.maux[s] = aux;
            x.mid[s] = id;
            x.mrk2[s] = rk2;
            x.mprop[s] = pr;
        }
        append_work(a, nOwn, fx, sy, pn, vn, aux, id, INFINITY, pr);
    }
}

// ---- shared-memory staging of the warp's candidate runs by cp.async.bulk (ablation,
// ORCA_STAGE=1).  Per warp, the union of its 32 agents' first-pass windows --
// one contiguous run of the sorted positions per fine column -- is copied into shared memory
// by the bulk-copy engine (one elected lane issues one copy per run and arms the warp's
// mbarrier with the byte count), and the lanes scan their own windows from there.  Windows
// that do not fit kStageEntries fall back to the direct reads.
#ifndef ORCA_STAGE
#define ORCA_STAGE 0
#endif
constexpr int kStageEntries = 256;  // float2 per warp (2 KB)
constexpr int kStageCols = 6;       // fine columns per warp union
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// warp reconvergence points in k_step at the once-per-agent phase
// boundaries (PHASES); the one before the final merge is always on
#ifndef ORCA_SYNC_PHASES
#define ORCA_SYNC_PHASES 0  // swept: 1M 0.495 ms (0) vs 0.529 ms (1)
#endif
#ifndef ORCA_MARGIN
#define ORCA_MARGIN 1.0f  // 1: the rigorous displacement bound (first pass always exact)
#endif
#ifndef ORCA_COLD_LAMBDA
#define ORCA_COLD_LAMBDA 1.6f  // no history: guessed radius holds ~this x k agents on average (r01q)
#endif
#ifndef ORCA_STEP_MINBLOCKS
#define ORCA_STEP_MINBLOCKS (1024 / ORCA_STEP_THREADS)  // 32 warps/SM: 64 regs (swept r01o)
#endif
// KR > 0: the top-k selection runs in a register list (k <= KR); KR = 0: shared memory.
// WU: LP2 with the paper's work units (lp2_wu) instead of per-lane re-solves.
// PAIR (variant 4; KR = 0, k <= 14, LP3 on the block queue or k_lp3): two lanes per agent --
// each scans every other candidate of the runs into its own top-k list, the first lane merges
// the two lists (exact order) into the second lane's buffer column, the lanes build every
// other half-plane and run lp2_greedy_pair; half the per-warp dependency chain of variant 0
// for latency-bound strips.
// LM >= 0: compiled for one LP3 placement (lp3Inline == LM: 0 = k_lp3, 2 = the block queue) and
// the greedy LP order (lpGreedy, no lpRandom) -- the default configurations -- so the other
// placements and the sequential LP orders are not in this kernel's code (less than half the
// SASS of the general kernel; r02ai: 1M -2.8 %).  LM = -1: any (runtime).
// MONO (with LM >= 0): one strip of homogeneous agents (finish_agent<true>, no per-agent props).
// TB: threads per block (kStepThreads, or 256 for the block-queue kernel: DESIGN.md §12 r02al).
// MB > 0: blocks per SM the register budget is sized for (3 x 256 threads: 85 registers; the block-queue
// kernel for strips within one wave of it, r02ao), else 1024 threads per SM (64 registers).
template <bool DRY, int KR, bool WU = false, bool PAIR = false, int LM = -1, bool MONO = false, int TB = kStepThreads,
          int MB = 0>
__global__ void __launch_bounds__(TB, MB > 0 ? MB : ORCA_STEP_MINBLOCKS * kStepThreads / TB) k_step(StepArgs a) {
    pdl_entry();
    constexpr bool CNT = DRY;  // only the debug variant counts work
    WorkT w{0, 0, 0, 0, 0};
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int T = TB;
    const int tid = threadIdx.x;
    const int k = a.m.k;
    const int capB = step_buf_words(k);
    uint2* Lst = reinterpret_cast<uint2*>(smem) + tid;                    // list (d2, j) / normal n
    uint32_t* Bf = reinterpret_cast<uint32_t*>(smem) + 2 * k * T + tid;    // buffer j / s
    float* Bff = reinterpret_cast<float*>(Bf + capB * T);                  // buffer d2
    const Lines L{reinterpret_cast<float2*>(Lst), reinterpret_cast<float*>(Bf)};

    // owned agents are the contiguous sorted range of columns [c0, c1)
    const int o0 = (int)a.binStart[(a.g.c0 - a.g.e0) * a.g.colBins];
    const int o1 = (int)a.binStart[(a.g.c1 - a.g.e0) * a.g.colBins];
    constexpr int APB = PAIR ? T / 2 : T;        // agents per block
    const int h = PAIR ? (tid & 1) : 0;          // lane in the agent's pair
    const bool lead = h == 0;                    // the lane that owns the agent's results
    const unsigned pm = PAIR ? (3u << (tid & 30)) : (1u << (tid & 31));  // the pair's lanes
    if (!DRY && a.phase != 2 && blockIdx.x == 0 && tid == 0) {  // per-step counters (k_receive appends after CT_NOWN)
        a.ctr[CT_NOWN] = o1 - o0;
        a.ctr[CT_EXTRA] = 0;
    }
    // this launch's agents: [ia, ib) then [ja, jb) of the sorted order (phase 1: the two
    // boundary columns at either side; 2: the interior; 0: all owned agents)
    int ia = o0, ib = o1, ja = 0, jb = 0;
    if (a.phase != 0) {
        const int bL = (int)a.binStart[(a.g.c0 + 2 - a.g.e0) * a.g.colBins];
        const int bR = (int)a.binStart[(a.g.c1 - 2 - a.g.e0) * a.g.colBins];
        if (a.phase == 1) {
            ib = bL;
            ja = bR;
            jb = o1;
        } else {
            ia = bL;
            ib = bR;
        }
    }
    const int nPh = (ib - ia) + (jb - ja);
    if ((int)blockIdx.x * APB >= nPh) return;  // (block-uniform, before any barrier)
    const int wlin = blockIdx.x * APB + (PAIR ? (tid >> 1) : tid);
    const int i = wlin < ib - ia ? ia + wlin : ja + (wlin - (ib - ia));  // sorted index
    const int ws = i - o0;                 // work slot
    const bool active = wlin < nPh;
    // PAIR: the agent's half-planes live in the lead lane's columns; the merged neighbour
    // list (fp32 d2 at word 2q, j at 2q + 1) in the second lane's buffer column
    uint2* Lst0 = Lst - h;
    uint32_t* Bf0 = Bf - h;
    uint32_t* Bf1 = Bf0 + 1;
    const Lines L0{reinterpret_cast<float2*>(Lst0), reinterpret_cast<float*>(Bf0)};
    const unsigned activeMask = __ballot_sync(0xffffffffu, active);  // lanes that step an agent
    uint32_t fl = 0;
    int nColl = 0;
    bool deferred = false;
    // block-local LP3 queue (lp3Inline == 2): queue words of the block's
    // infeasible agents and the thread columns that are free once their agent is finished
    __shared__ uint32_t sQ[T];
    __shared__ uint8_t sFree[T];
    __shared__ int sQn;
    const int lp3Mode = LM >= 0 ? LM : a.lp3Inline;
    const bool blockQ = lp3Mode == 2;
    if (blockQ && tid == 0) sQn = 0;
    if (blockQ) __syncthreads();
    bool queued = false;
    int cInfX = 0, cDegX = 0, cG1X = 0, cG2X = 0, cG3X = 0;  // agents this thread finished from the queue
#if ORCA_STAGE
    __shared__ __align__(16) float2 sStage[T / 32][kStageEntries];
    __shared__ __align__(8) uint64_t sBar[T / 32];
    __shared__ int sStageOff[T / 32][kStageCols + 1];
    __shared__ int sStageS[T / 32][kStageCols];  // per column: staged position of index j = j - S
    if (!PAIR && (tid & 31) == 0) mbar_init(&sBar[tid >> 5]);
    __syncwarp();
    bool staged = false;
    int stF0 = 0;  // the union's first fine column
#endif
    if (active) {
        const float2 pi = a.posS[i];
        const float2 vi = a.velS[i];
        const float2 aux = a.auxS[i];
        const uint32_t idi = a.idS[i];
        // per-agent (radius, maxSpeed, prefSpeed) of heterogeneous crowds
        const bool het = !MONO && a.propS != nullptr;
        const float4 pr = het ? a.propS[i] : make_float4(0.5f * a.m.R, a.m.maxSpeed, a.m.prefSpeed, 0.0f);
        const float ri = pr.x, vmaxi = pr.y, vprefi = (pr.z >= 0.0f) ? pr.z : a.m.prefSpeed;
        (void)ri;
        const int cx = cell_coord(pi.x, a.g.ox, a.g.csD, a.g.invCs, a.g.nx);
        const int lgS = a.g.lgS;
        const int nyS = a.g.ny << lgS;
        const int cy = subrow_coord(pi.y, a.g) >> lgS;

        // ---- 2. k nearest within r_obs over the 3x3 bins -------------
        // Each column of the stencil is one contiguous run of the sorted arrays, ordered by
        // sub-row.  A search radius rg restricts every run to the sub-rows within rg of the
        // agent and skips a side column farther than rg; the result is exact by the check
        // below (else one full 3x3 rescan).  rg comes from the previous step's k-th
        // neighbour distance plus 2 maxSpeed dt (those k agents cannot have moved farther
        // apart), or, without history, from the local density.
        int cnt = 0;
        float fk = INFINITY;
        if (k > 0) {
            const int rlo = max(cy - 1, 0) << lgS;              // first sub-row of the 3 rows
            const int rhi = (min(cy + 1, a.g.ny - 1) + 1) << lgS; // one past the last
            const int c0 = max(cx - 1, 0), c1 = min(cx + 1, a.g.nx - 1);
            const int lgC = a.g.lgC;
            const int fe0 = a.g.e0 << lgC;                              // first local fine column
            const int f0 = c0 << lgC, f1 = ((c1 + 1) << lgC) - 1;       // fine columns of the stencil
            float thr = a.m.nd2Fup;
            bool guessed = false;
            const float rk2p = a.rk2S[i];
            if (rk2p < a.m.nd2Fup) {
                // this agent moved |v_i| dt since the k-th distance was measured (its stored
                // velocity is its last displacement), a neighbour at most maxSpeed dt; the guess
                // is only a hint (the exactness test below decides), ORCA_MARGIN scales it
                const float vi2 = sqrtf(fmaf(vi.x, vi.x, vi.y * vi.y));
                const float marg = ORCA_MARGIN * (1.0002f * (vi2 + a.m.maxSpeedAll) * a.m.dt) +
                                   4e-7f * (fabsf(pi.x) + fabsf(pi.y)) + 1e-5f;
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
                // r^2 = 2.2 k / (pi rho), rho = ncand / (9 cs^2): ~22 expected hits for k = 10
                const float g = ORCA_COLD_LAMBDA * (float)k * 9.0f * a.g.cs * a.g.cs / (3.14159265f * (float)ncand);
                if (ncand > 4 * k && g < thr) {
                    thr = g;
                    guessed = true;
                }
            }
            // mode 0: register list (KR > 0, fp32 compares); mode 1: exact shared-memory
            // list -- taken only if mode 0 met an fp32 near-tie (or KR == 0)
            RegList<(KR > 0 ? KR : 1)> R;
            bool tie = false;
            const float thr0 = thr;
            const bool guessed0 = guessed;
            int mode = (KR > 0) ? 0 : 1;
            bool allIn = false;  // this pass's threshold is below nd2Lo (set at each pass start)
            auto merge = [&](int nb) {
                if (KR > 0 && mode == 0)
                    reg_merge<(KR > 0 ? KR : 1), T>(R, cnt, Bf, Bff, nb, pi, a.m, a.posS, tie);
                else
                    cnt = merge_candidates<T>(Lst, cnt, k, Bf, Bff, nb, pi, a.m, a.posS, a.idS, allIn);
            };
            auto kth = [&]() -> float {  // fp32 d2 of the k-th (valid when cnt >= k)
                if (KR > 0 && mode == 0) return reg_f<(KR > 0 ? KR : 1)>(R, k - 1);
                return __uint_as_float(Lst[(k - 1) * T].x);
            };
          for (;;) {  // modes
            if (KR > 0 && mode == 0) reg_clear<(KR > 0 ? KR : 1)>(R);
            for (int pass = 0; pass < 3; ++pass) {
                const float thrPass = thr;
                allIn = thr < a.m.nd2Lo;
                // sub-row window and fine-column range for this pass
                int lo = rlo, hi = rhi - 1, fa = f0, fb = f1;
                if (guessed) {
                    const float rg = sqrtf(thr) * (1.0f + 1e-6f) + 1e-6f;
                    // sub-rows s with [oy + s h, oy + (s+1) h) within rg of y (h = cs/2^lgS):
                    // ty in fp64 is accurate to ~1e-12 sub-rows, covered by the 1e-6 margin
                    const double ty = __dmul_rn(__dsub_rn((double)pi.y, (double)a.g.oy), a.g.invCsSub);
                    const double rs = (double)rg * a.g.invCsSub + 1e-6;
                    lo = max(lo, (int)fmin(fmax(floor(ty - rs), 0.0), (double)(nyS - 1)));
                    hi = min(hi, (int)fmin(fmax(floor(ty + rs), 0.0), (double)(nyS - 1)));
                    // fine columns within rg of x, the same way.  Both windows are clamped like
                    // the agents' own bins, so an agent outside the grid searches the edge bins
                    // its neighbours are clamped into (floor and clamp are monotone)
                    const double tx = __dmul_rn(__dsub_rn((double)pi.x, (double)a.g.ox), a.g.invCsSubX);
                    const double rsx = (double)rg * a.g.invCsSubX + 1e-6;
                    fa = max(fa, (int)fmin(fmax(floor(tx - rsx), 0.0), (double)((a.g.nx << lgC) - 1)));
                    fb = min(fb, (int)fmin(fmax(floor(tx + rsx), 0.0), (double)((a.g.nx << lgC) - 1)));
                }
                int nb = 0;
#if ORCA_STAGE
                if (!PAIR && pass == 0 && mode == ((KR > 0) ? 0 : 1)) {
                    // the warp's union window, one run per fine column, into shared memory
                    __syncwarp(activeMask);
                    const int w5 = tid >> 5;
                    const int F0 = __reduce_min_sync(activeMask, fa), F1 = __reduce_max_sync(activeMask, fb);
                    int tot = 0;
                    bool oob = false;
                    const bool lw = (tid & 31) == __ffs(activeMask) - 1;  // the warp's first active lane
                    if (F1 - F0 + 1 <= kStageCols) {
                        for (int c = 0; c <= F1 - F0; ++c) {
                            const int fc = F0 + c;
                            const bool mine = fa <= fc && fc <= fb;
                            const int sb = mine ? (int)a.binStart[(fc - fe0) * nyS + lo] : INT_MAX;
                            const int se = mine ? (int)a.binStart[(fc - fe0) * nyS + hi + 1] : INT_MIN;
                            int S = __reduce_min_sync(activeMask, sb), E = __reduce_max_sync(activeMask, se);
                            if (E <= S) S = E = 0;
                            S &= ~1;               // 16-byte aligned source (even index)
                            E = (E + 1) & ~1;      // whole 16-byte units
                            oob |= E > a.capW + 2; // (the sorted arrays carry 2 spare entries)
                            if (lw) {
                                sStageOff[w5][c] = E - S;
                                sStageS[w5][c] = S - tot;
                            }
                            tot += E - S;
                        }
                    }
                    staged = tot > 0 && tot <= kStageEntries && F1 - F0 + 1 <= kStageCols && !oob;
                    if (staged) {
                        stF0 = F0;
                        if (lw) {
                            mbar_expect_tx(&sBar[w5], (uint32_t)tot * 8u);
                            int off = 0;
                            for (int c = 0; c <= F1 - F0; ++c) {
                                const int len = sStageOff[w5][c];
                                if (len > 0)
                                    bulk_g2s(&sStage[w5][off], a.posS + (off + sStageS[w5][c]), (uint32_t)len * 8u,
                                             &sBar[w5]);
                                off += len;
                            }
                        }
                        mbar_wait(&sBar[w5], 0);
                    }
                }
#endif
                for (int fc = fa; fc <= fb; ++fc) {  // one run per fine column
                    const int b = (int)a.binStart[(fc - fe0) * nyS + lo];
                    const int e = (int)a.binStart[(fc - fe0) * nyS + hi + 1];
#if ORCA_STAGE
                    // this run's positions: staged (pass 0) or the sorted array
                    const float2* __restrict__ psrc =
                        (staged && pass == 0) ? &sStage[tid >> 5][0] - sStageS[tid >> 5][fc - stF0] : a.posS;
#else
                    const float2* __restrict__ psrc = a.posS;
#endif
                    if (CNT && lead) w.cand += (uint32_t)(e - b);
                    constexpr int st = PAIR ? 2 : 1;  // PAIR: each lane every other candidate
                    // candidates per iteration (loads in flight); the k_lp3-placement kernel (large
                    // strips, throughput bound) may take another unroll than the latency-bound ones
                    constexpr int U = (LM == 0) ? ORCA_SCAN_UNROLL_LM0 : ORCA_SCAN_UNROLL;
                    int j = b + h;
                    for (; j + (U - 1) * st < e; j += U * st) {
                        float2 pu[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) pu[u] = psrc[j + u * st];
                        bool hit[U];
                        float d2u[U];
                        bool any = false;
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const float dx = pu[u].x - pi.x, dy = pu[u].y - pi.y;
                            d2u[u] = fmaf(dx, dx, dy * dy);
                            hit[u] = d2u[u] <= thr && j + u * st != i;
                            any |= hit[u];
                        }
                        if (any) {
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                if (hit[u]) {
                                    Bf[nb * T] = (uint32_t)(j + u * st);
                                    if (!ORCA_BUF1) Bff[nb * T] = d2u[u];
                                    ++nb;
                                }
                            }
                            if (nb > capB - U) {  // buffer (nearly) full: merge, tighten
                                merge(nb);
                                nb = 0;
                                if (cnt >= k)  // any key <= the k-th has fp32 d2 <= fk (1 + 2^-20)
                                    thr = fminf(thr, __fmul_ru(kth(), 1.0f + 0x1p-20f));
                            }
                        }
                    }
                    for (; j < e; j += st) {  // the remainder (< U candidates)
                        const float2 p0 = psrc[j];
                        const float dx0 = p0.x - pi.x, dy0 = p0.y - pi.y;
                        const float d20 = fmaf(dx0, dx0, dy0 * dy0);
                        if (d20 <= thr && j != i) {
                            Bf[nb * T] = (uint32_t)j;
                            if (!ORCA_BUF1) Bff[nb * T] = d20;
                            ++nb;
                        }
                        if (nb > capB - U) {
                            merge(nb);
                            nb = 0;
                            if (cnt >= k) thr = fminf(thr, __fmul_ru(kth(), 1.0f + 0x1p-20f));
                        }
                    }
                }
                // reconverge the warp after the data-dependent scan loops, so the final
                // merge runs once for all lanes instead of once per divergent subset.  Only
                // at the first pass of the first mode, which every active lane executes
                // exactly once (rescans / exact redos are per-lane and rare).
                if (pass == 0 && mode == ((KR > 0) ? 0 : 1)) __syncwarp(activeMask);
                merge(nb);
                if (PAIR) {
                    // the lead lane merges the two lanes' sorted lists (exact (kappa, id) order;
                    // disjoint candidate sets) into the second lane's buffer column
                    __syncwarp(pm);
                    const int cA = __shfl_sync(pm, cnt, tid & 30), cB = __shfl_sync(pm, cnt, (tid & 30) + 1);
                    const int cM = min(k, cA + cB);
                    if (lead) {
                        const uint2* B = Lst + 1;
                        int ia = 0, ib = 0;
                        for (int q = 0; q < cM; ++q) {
                            bool takeA;
                            if (ia >= cA) {
                                takeA = false;
                            } else if (ib >= cB) {
                                takeA = true;
                            } else {
                                const uint2 ea = Lst[ia * T], eb = B[ib * T];
                                takeA = cand_less(__uint_as_float(ea.x), ea.y, __uint_as_float(eb.x), eb.y, pi,
                                                  a.posS, a.idS);
                            }
                            const uint2 e2 = takeA ? Lst[(ia++) * T] : B[(ib++) * T];
                            Bf1[(2 * q) * T] = e2.x;
                            Bf1[(2 * q + 1) * T] = e2.y;
                        }
                    }
                    __syncwarp(pm);
                    cnt = cM;
                }
                if (!guessed) break;
                // Exact only if every candidate not kept -- rejected by the guessed radius
                // (key > thrPass (1 - 2^-22)) or pruned geometrically (distance > rg) -- is
                // strictly beyond the k-th key.
                // kappa_k <= fk (1 + 2^-22) < thrPass (1 - 2^-22) < any rejected kappa
                const float kthM = PAIR ? __uint_as_float(Bf1[(2 * (k - 1)) * T]) : (cnt >= k ? kth() : 0.0f);
                if (cnt >= k && (double)kthM < (double)thrPass * (1.0 - 0x1p-20)) break;
                // Too few within the guess (cnt < k): widen it once to ~1.5 k expected
                // agents at the observed density, else rescan the full stencil at r_obs.
                const float wid = (pass == 0 && cnt < k)
                                      ? thrPass * 1.5f * (float)k / (float)max(cnt, 1) : INFINITY;
                cnt = 0;
                if (KR > 0 && mode == 0) reg_clear<(KR > 0 ? KR : 1)>(R);
                if (wid < a.m.nd2Fup) {
                    thr = wid;
                } else {
                    thr = a.m.nd2Fup;
                    guessed = false;
                }
            }
            if (!(KR > 0 && mode == 0 && tie)) break;
            mode = 1;  // fp32 near-tie: redo this agent's selection on the exact path
            cnt = 0;
            thr = thr0;
            guessed = guessed0;
          }
            if (cnt >= k) fk = PAIR ? __uint_as_float(Bf1[(2 * (k - 1)) * T]) : kth();
            cnt = min(cnt, k);
            if (KR > 0 && mode == 0) {  // neighbour indices into the shared list slots
#pragma unroll
                for (int q = 0; q < (KR > 0 ? KR : 1); ++q)
                    if (q < cnt) Lst[q * T] = make_uint2(__float_as_uint(R.f[q]), R.j[q]);
            }
        }
        if (!DRY && lead) a.rk2W[ws] = fk;  // next step's search bound (read back by k_lp3 for queued agents)

        // Reconvergence points: each phase below runs exactly once per active lane, so the
        // warp re-forms here after the data-dependent selection (r01l).
        if (ORCA_SYNC_PHASES) __syncwarp(activeMask);
        // ---- 3. one ORCA half-plane per neighbour, nearest first (Fig. 1) -----
        // the neighbour j's: list slots (j in .y, stride 2T words) or, PAIR, the merged list
        uint32_t* nbrJ = PAIR ? Bf1 + T : reinterpret_cast<uint32_t*>(Lst) + 1;
        if (DRY && a.dbgNbr && lead)  // neighbours in (distance, id) order
            for (int q = 0; q < cnt; ++q) a.dbgNbr[(size_t)idi * k + q] = (int32_t)a.idS[nbrJ[q * 2 * T]];
        // optional randomized LP order (P:82 Seidel, reading Q8): permute the list first
        if (LM < 0 && a.m.lpRandom && cnt > 1 && lead) lp_shuffle(nbrJ, 2 * T, cnt, a.m.lpSeed, a.ctr[CT_STEP], idi);
        if (PAIR) __syncwarp(pm);
        // (half-plane q overwrites list slot q in place: j is read before the write; PAIR: the
        // lanes build every other half-plane into the lead lane's columns)
        for (int q = h; q < cnt; q += (PAIR ? 2 : 1)) {
            const uint32_t j = nbrJ[q * 2 * T];
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
            L0.n[q * T] = make_float2(nx, ny);
            L0.s[q * T] = s;
        }
        if (PAIR) {
            __syncwarp(pm);
            fl |= __shfl_xor_sync(pm, fl, 1);  // the second lane's coincidence flags (g1)
        }

        if (ORCA_SYNC_PHASES) __syncwarp(activeMask);
        // ---- 4. LP2, LP3 on failure ------------------------------------------
        float px, py;
        if (a.m.goals) {  // toward the goal at walking speed (reading Q16)
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
        if (CNT && lead) w.lines += (uint32_t)cnt;
        // LP order (reading Q8): greedy (mode 0, default) or the sequential incremental LP over
        // the neighbour / randomized order (modes 2 / 1; the work-unit variant's own loop);
        // PAIR runs the greedy order only (the host falls back to variant 0 otherwise)
#ifndef ORCA_PAIR_SERIAL_LP
#define ORCA_PAIR_SERIAL_LP 0  // debug: the lead lane alone runs lp2_greedy
#endif
        const int f = (PAIR && ORCA_PAIR_SERIAL_LP)
                          ? (lead ? lp2_greedy<CNT>(L0, T, cnt, k, vmaxi, px, py, vx, vy, fl, w, activeMask & 0x55555555u) : 0)
                      : PAIR ? lp2_greedy_pair<CNT>(L0, T, cnt, k, vmaxi, px, py, vx, vy, fl, w, activeMask, pm, h)
                      : (LM >= 0 || a.m.lpGreedy) ? lp2_greedy<CNT>(L, T, cnt, k, vmaxi, px, py, vx, vy, fl, w, activeMask)
                      : WU         ? lp2_wu<CNT>(L, T, cnt, k, vmaxi, px, py, vx, vy, fl, w, activeMask)
                      : ORCA_SYNC_LP ? lp2_sync<CNT>(L, T, cnt, k, vmaxi, px, py, vx, vy, fl, w, activeMask)
                                     : lp2<CNT>(L, T, cnt, vmaxi, px, py, false, vx, vy, fl, w);
        if (!lead) {
            fl = 0;  // PAIR: the second lane's part is done; the lead lane finishes the agent
        } else if (blockQ) {
            if (f < cnt) {
                // infeasible: into the block's queue; the least-penetration LP runs after
                // the block barrier below on a compacted set of lanes.  The LP2 point waits in
                // this thread's free buffer words (right after s)
                fl |= FL_INFEASIBLE;
                queued = true;
                Bf[k * T] = __float_as_uint(vx);
                Bf[(k + 1) * T] = __float_as_uint(vy);
                Bf[(k + 2) * T] = (uint32_t)ws;  // (the executor finds the agent from its column)
                const unsigned mask = __activemask();
                const int lane = tid & 31;
                const int leader = __ffs(mask) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(&sQn, __popc(mask));
                base = __shfl_sync(mask, base, leader);
                sQ[base + __popc(mask & ((1u << lane) - 1u))] =
                    (uint32_t)tid | ((uint32_t)cnt << 8) | ((uint32_t)f << 16) | (fl << 24);
                if (DRY && a.dbgCnt) a.dbgCnt[idi] = cnt;
                if (DRY && a.dbgNbr)
                    for (int q2 = cnt; q2 < k; ++q2) a.dbgNbr[(size_t)idi * k + q2] = -1;
            }
        } else if (lp3Mode) {
            // small strips (latency bound, spare issue slots): the least-penetration LP
            // runs here on the half-planes in shared memory -- the same lp3 as k_lp3, so the
            // same result -- and the agent is finished below like a feasible one
            const unsigned lmask = __ballot_sync(PAIR ? (activeMask & 0x55555555u) : activeMask, f < cnt);
            if (f < cnt) {
                fl |= FL_INFEASIBLE;
                // projected half-planes in the 3k words per thread the launch adds after the
                // per-thread columns (their own interleaved layout: the candidate buffers of
                // threads still selecting stay untouched)
                float* Pb = reinterpret_cast<float*>(smem) + (2 * k + capB) * T;
                const Lines P{reinterpret_cast<float2*>(Pb) + tid, Pb + 2 * k * T + tid};
                lp3_dispatch<CNT>(L, P, T, T, cnt, f, k, vmaxi, vx, vy, fl, w, lmask, a.m.lpGreedy != 0);
                float dl = 0.0f;
                for (int m = 0; m < cnt; ++m) {
                    const float2 nm = L.n[m * T];
                    dl = fmaxf(dl, L.s[m * T] - fmaf(nm.x, vx, nm.y * vy));
                }
                if (dl > 0.0f && dl < 1e-6f) fl |= FL_G3;
            }
        } else if (f < cnt) {
            // infeasible: queue the agent with its half-planes and LP2 point; k_lp3
            // runs the least-penetration LP on a compacted set of agents (full warps)
            fl |= FL_INFEASIBLE;
            deferred = true;
            const unsigned mask = __activemask();
            const int lane = tid & 31;
            const int leader = __ffs(mask) - 1;
            unsigned base = 0;
            if (lane == leader) base = atomicAdd(a.qCount, (unsigned)__popc(mask));
            base = __shfl_sync(mask, base, leader);
            const int q = (int)base + __popc(mask & ((1u << lane) - 1u));
            a.qEntry[q] = make_int4(i, cnt | (f << 8) | ((int)fl << 16), __float_as_int(vx), __float_as_int(vy));
            for (int m = 0; m < cnt; ++m)
                a.qLines[(size_t)m * a.qcap + q] = make_float4(L.n[m * T].x, L.n[m * T].y, L.s[m * T], 0.0f);
            if (DRY && a.dbgCnt) a.dbgCnt[idi] = cnt;
            if (DRY && a.dbgNbr)
                for (int q2 = cnt; q2 < k; ++q2) a.dbgNbr[(size_t)idi * k + q2] = -1;
        }

        if (ORCA_SYNC_PHASES) __syncwarp(activeMask);
        // ---- 5. integrate (explicit Euler) + next step's binning ----------------------
        if (deferred || queued || !lead) {
            // finished by k_lp3 / by the block queue below (PAIR: by the lead lane)
        } else if (DRY) {
            if (a.dbgV) a.dbgV[idi] = make_float2(vx, vy);
            if (a.dbgFlags) a.dbgFlags[idi] = (uint8_t)fl;
            if (a.dbgCnt) a.dbgCnt[idi] = cnt;
            if (a.dbgNbr)
                for (int q = cnt; q < k; ++q) a.dbgNbr[(size_t)idi * k + q] = -1;
        } else {
            finish_agent<MONO>(a, ws, o1 - o0, pi, vx, vy, aux, idi, fk, pr);
        }
    }
    if (blockQ) {
        // ---- LP3 of the block's infeasible agents on compacted lanes -----------------
        // Free columns: threads whose agent is finished (or that have none); an executor
        // thread e runs queue entry e with the owner's half-planes (owner column) and its
        // projected half-planes in free column sFree[e], then finishes the owner's agent.
        {
            const int lane = tid & 31;
            const bool fr = !queued;
            const unsigned fm = __ballot_sync(0xffffffffu, fr);
            __shared__ int sWarpFree[T / 32];
            if (lane == 0) sWarpFree[tid >> 5] = __popc(fm);
            __syncthreads();
            int off = 0;
            for (int q = 0; q < (tid >> 5); ++q) off += sWarpFree[q];
            if (fr) sFree[off + __popc(fm & ((1u << lane) - 1u))] = (uint8_t)tid;
        }
        __syncthreads();
        // Rounds (block-uniform): executors e < nfree take free column sFree[e] for their
        // projected half-planes, the next kLp3Scratch take a column of the small scratch area
        // after the per-thread columns (stride kLp3Scratch), so every round makes progress even
        // when every agent of the block is infeasible; the owners finished in a round free
        // their columns for the next.  One round whenever at most half the block is queued.
        const int nq = sQn;
        int nfree = T - nq, done = 0;
        const int o1b = o1;
        float* scratch = reinterpret_cast<float*>(smem) + (2 * k + capB) * T;
        while (done < nq) {
            const int nexec = min(nq - done, nfree + kLp3Scratch);
            const bool ex = tid < nexec;
            const unsigned xmask = __ballot_sync(0xffffffffu, ex);
            int owner = 0;
            if (ex) {
                const uint32_t e = sQ[done + tid];
                owner = (int)(e & 0xffu);
                const int cnt = (int)((e >> 8) & 0xffu), f = (int)((e >> 16) & 0xffu);
                uint32_t fl2 = e >> 24;
                float* sw = reinterpret_cast<float*>(smem);
                const Lines Lo{reinterpret_cast<float2*>(sw) + owner, sw + 2 * k * T + owner};
                const bool main = tid < nfree;
                const int TP = main ? T : kLp3Scratch;
                const int pcol = main ? (int)sFree[tid] : tid - nfree;
                const Lines P = main ? Lines{reinterpret_cast<float2*>(sw) + pcol, sw + 2 * k * T + pcol}
                                     : Lines{reinterpret_cast<float2*>(scratch) + pcol, scratch + 2 * k * TP + pcol};
                float vx = sw[3 * k * T + owner];  // the LP2 point stashed after s
                float vy = sw[(3 * k + 1) * T + owner];
                const int wso = (int)reinterpret_cast<uint32_t*>(sw)[(3 * k + 2) * T + owner];
                const int io = o0 + wso;
                const float4 pr = (!MONO && a.propS) ? a.propS[io] : make_float4(0.5f * a.m.R, a.m.maxSpeed, a.m.prefSpeed, 0.0f);
                lp3_dispatch<CNT>(Lo, P, T, TP, cnt, f, k, pr.y, vx, vy, fl2, w, xmask, LM >= 0 || a.m.lpGreedy != 0);
                float dl = 0.0f;
                for (int m = 0; m < cnt; ++m) {
                    const float2 nm = Lo.n[m * T];
                    dl = fmaxf(dl, Lo.s[m * T] - fmaf(nm.x, vx, nm.y * vy));
                }
                if (dl > 0.0f && dl < 1e-6f) fl2 |= FL_G3;
                const uint32_t ido = a.idS[io];
                if (DRY) {
                    if (a.dbgV) a.dbgV[ido] = make_float2(vx, vy);
                    if (a.dbgFlags) a.dbgFlags[ido] = (uint8_t)fl2;
                } else {
                    finish_agent<MONO>(a, wso, o1b - o0, a.posS[io], vx, vy, a.auxS[io], ido, a.rk2W[wso], pr);
                }
                cInfX += 1;
                cDegX += (fl2 & (FL_G1 | FL_G2)) != 0;
                cG1X += (fl2 & FL_G1) != 0;
                cG2X += (fl2 & FL_G2) != 0;
                cG3X += (fl2 & FL_G3) != 0;
            }
            done += nexec;
            if (done < nq) {  // (block-uniform) another round: the finished owners' columns are free
                __syncthreads();
                if (ex) sFree[nfree + tid] = (uint8_t)owner;
                nfree += nexec;
                __syncthreads();
            }
        }
    }
    if (DRY && a.work) {
        unsigned long long c[5] = {w.cand, w.lines, w.checks, w.lp1, w.proj};
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            for (int o = 16; o > 0; o >>= 1) c[q] += __shfl_xor_sync(0xffffffffu, c[q], o);
        }
        if ((tid & 31) == 0) {
            atomicAdd(&a.work->cand, c[0]);
            atomicAdd(&a.work->lines, c[1]);
            atomicAdd(&a.work->checks, c[2]);
            atomicAdd(&a.work->lp1, c[3]);
            atomicAdd(&a.work->proj, c[4]);
        }
    }
    if (!DRY) {
        // per-warp counts (ballot + popc), one relaxed atomic per warp and counter; no
        // block barrier, so fast warps never wait for a slow LP in the same block
        const int lane = tid & 31;
        if (deferred || queued) fl = 0;  // counted by k_lp3 / the queue executor with the final flags
        int cInf = __popc(__ballot_sync(0xffffffffu, fl & FL_INFEASIBLE));
        int cDeg = __popc(__ballot_sync(0xffffffffu, fl & (FL_G1 | FL_G2)));
        int cG1 = __popc(__ballot_sync(0xffffffffu, fl & FL_G1));
        int cG2 = __popc(__ballot_sync(0xffffffffu, fl & FL_G2));
        int cG3 = __popc(__ballot_sync(0xffffffffu, fl & FL_G3));
        if (blockQ) {
            int x[5] = {cInfX, cDegX, cG1X, cG2X, cG3X};
#pragma unroll
            for (int r = 0; r < 5; ++r)
                for (int o = 16; o > 0; o >>= 1) x[r] += __shfl_xor_sync(0xffffffffu, x[r], o);
            cInf += x[0];
            cDeg += x[1];
            cG1 += x[2];
            cG2 += x[3];
            cG3 += x[4];
        }
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

// ------------------------------------------------------------ LP3 on the queue
#ifndef ORCA_LP3_LOAD_UNROLL
#define ORCA_LP3_LOAD_UNROLL 4  // r01au: 1M -0.4 %, 100k -2 %, dense -1 % vs 1
#endif
#ifndef ORCA_LP3_SORT
#define ORCA_LP3_SORT 0  // r01aj: -0.8 % with the sequential LP3; with the greedy LP3 +2.2 % (r01ao)
#endif
#define ORCA_MAX_K_DEV 32  // = ORCA_MAX_K (include/orca.h); buckets 0..32 by failure index
// One thread per queued (infeasible) agent, grid-stride over the device-side queue
// count; same smem column layout as k_step (lines, then projected lines).
// MONO: one strip of homogeneous agents (finish_agent<true>, no per-agent props)
template <bool DRY, bool MONO = false>
__global__ void __launch_bounds__(kStepThreads) k_lp3(StepArgs a) {
    pdl_entry();
    constexpr bool CNT = DRY;
    WorkT w{0, 0, 0, 0, 0};
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int T = kStepThreads;
    const int tid = threadIdx.x;
    const int k = a.m.k;
    float* sw = reinterpret_cast<float*>(smem);
    const Lines L{reinterpret_cast<float2*>(sw) + tid, sw + 2 * k * T + tid};                  // words [0, 3kT)
    const Lines P{reinterpret_cast<float2*>(sw + 3 * k * T) + tid, sw + 5 * k * T + tid};      // words [3kT, 6kT)
    const int nq = (int)*a.qCount;
    if ((int)blockIdx.x * T >= nq) return;  // block-uniform: nothing queued for this block
    const int o0 = (int)a.binStart[(a.g.c0 - a.g.e0) * a.g.colBins];
    const int nOwn = (int)a.binStart[(a.g.c1 - a.g.e0) * a.g.colBins] - o0;
    int cInf = 0, cDeg = 0, cG1 = 0, cG2 = 0, cG3 = 0;
#if ORCA_LP3_SORT
    __shared__ int sHist[ORCA_MAX_K_DEV + 2];
    __shared__ int sPerm[T];
#endif
    // one queue entry per thread, grid-stride over the device-side count (block-uniform
    // trip count); lanes of a warp reconverge inside lp3_sync
    for (int qb = blockIdx.x * T; qb < nq; qb += gridDim.x * T) {
#if ORCA_LP3_SORT
    // block-local counting sort of the block's entries by LP2 failure index f, so the lanes
    // of a warp start the least-penetration loop at (nearly) the same line
    const int nv = min(T, nq - qb);
    for (int h = tid; h < ORCA_MAX_K_DEV + 2; h += T) sHist[h] = 0;
    __syncthreads();
    int key = ORCA_MAX_K_DEV + 1, rk = 0;
    if (tid < nv) {
        key = (a.qEntry[qb + tid].y >> 8) & 0xff;
        rk = atomicAdd(&sHist[key], 1);
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the <= 34 bucket counts
        int v0 = sHist[tid], v1 = (tid + 32 < ORCA_MAX_K_DEV + 2) ? sHist[tid + 32] : 0;
        int incl = v0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
        sHist[tid] = incl - v0;
        if (tid + 32 < ORCA_MAX_K_DEV + 2) sHist[tid + 32] = tot;  // (only bucket 33 = inactive)
        (void)v1;
    }
    __syncthreads();
    if (tid < nv) sPerm[sHist[key] + rk] = qb + tid;
    __syncthreads();
    const bool act = tid < nv;
    const int q = act ? sPerm[tid] : 0;
#else
    const int q = qb + tid;
    const bool act = q < nq;
#endif
    const unsigned qmask = __ballot_sync(0xffffffffu, act);
    if (act) {
        const int4 e = a.qEntry[q];
        const int i = e.x;
        const int cnt = e.y & 0xff, f = (e.y >> 8) & 0xff;
        uint32_t fl = (uint32_t)(e.y >> 16);
        float vx = __int_as_float(e.z), vy = __int_as_float(e.w);
        // the queued half-planes (L2-resident, written by k_step): unrolled so several loads
        // are in flight before the shared-memory stores wait on them
        _Pragma(ORCA_XSTR_(unroll ORCA_LP3_LOAD_UNROLL))
        for (int m = 0; m < cnt; ++m) {
            const float4 l = a.qLines[(size_t)m * a.qcap + q];
            L.n[m * T] = make_float2(l.x, l.y);
            L.s[m * T] = l.z;
        }
        const float4 pr = (!MONO && a.propS) ? a.propS[i] : make_float4(0.5f * a.m.R, a.m.maxSpeed, a.m.prefSpeed, 0.0f);
        if (a.m.lpGreedy)
            lp3_greedy<CNT>(L, P, T, T, cnt, f, k, pr.y, vx, vy, fl, w, qmask);
        else if (ORCA_SYNC_LP)
            lp3_sync<CNT>(L, P, T, T, cnt, f, k, pr.y, vx, vy, fl, w, qmask);
        else
            lp3<CNT>(L, P, T, cnt, f, pr.y, vx, vy, fl, w);
        float dl = 0.0f;
        for (int m = 0; m < cnt; ++m) {
            const float2 nm = L.n[m * T];
            dl = fmaxf(dl, L.s[m * T] - fmaf(nm.x, vx, nm.y * vy));
        }
        if (dl > 0.0f && dl < 1e-6f) fl |= FL_G3;
        const float2 pi = a.posS[i];
        const uint32_t idi = a.idS[i];
        if (DRY) {
            if (a.dbgV) a.dbgV[idi] = make_float2(vx, vy);
            if (a.dbgFlags) a.dbgFlags[idi] = (uint8_t)fl;
        } else {
            finish_agent<MONO>(a, i - o0, nOwn, pi, vx, vy, a.auxS[i], idi, a.rk2W[i - o0], pr);
        }
        cInf += 1;
        cDeg += (fl & (FL_G1 | FL_G2)) != 0;
        cG1 += (fl & FL_G1) != 0;
        cG2 += (fl & FL_G2) != 0;
        cG3 += (fl & FL_G3) != 0;
    }
    }
    const int lane = tid & 31;
    if (DRY) {
        if (a.work) {
            unsigned long long c[2] = {w.checks, w.lp1};
            unsigned long long pj = w.proj;
            for (int o = 16; o > 0; o >>= 1) {
                c[0] += __shfl_xor_sync(0xffffffffu, c[0], o);
                c[1] += __shfl_xor_sync(0xffffffffu, c[1], o);
                pj += __shfl_xor_sync(0xffffffffu, pj, o);
            }
            if (lane == 0) {
                atomicAdd(&a.work->checks, c[0]);
                atomicAdd(&a.work->lp1, c[1]);
                atomicAdd(&a.work->proj, pj);
            }
        }
    } else {
        int c[5] = {cInf, cDeg, cG1, cG2, cG3};
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

// ------------------------------------------------------------------ state utilities
// owned sorted range [o0, o1) of a domain
__device__ __forceinline__ int2 owned_range(const uint32_t* __restrict__ binStart, const Grid& g) {
    const int cb = g.colBins;
    return make_int2((int)binStart[(g.c0 - g.e0) * cb], (int)binStart[(g.c1 - g.e0) * cb]);
}

// owned agents -> id-ordered outputs (pos, vel; either nullable); optional local export
// (ids / pos / vel in sorted order starting at 0)
__global__ void k_unpermute(const uint32_t* __restrict__ binStart, Grid g, const uint32_t* __restrict__ idS,
                            const float2* __restrict__ posS, const float2* __restrict__ velS,
                            float2* __restrict__ posOut, float2* __restrict__ velOut) {
    const int2 r = owned_range(binStart, g);
    for (int i = r.x + blockIdx.x * blockDim.x + threadIdx.x; i < r.y; i += gridDim.x * blockDim.x) {
        const uint32_t id = idS[i];
        if (posOut) posOut[id] = posS[i];
        if (velOut) velOut[id] = velS[i];
    }
}

// The paper's candidate count: agents in the 3x3 bins around every owned agent ("For
// those within the same or neighboring partitioning bins, it calculates whether they are
// within the observation radius").  The per-unit figure c_cand of SURVEY §8(d)'s
// algorithmic work model; the step itself reads only the fine-column runs within its search
// radius.
__global__ void k_stencil_count(const uint32_t* __restrict__ binStart, Grid g, const float2* __restrict__ posS,
                                unsigned long long* __restrict__ out) {
    const int2 r = owned_range(binStart, g);
    const int nyS = g.ny << g.lgS, fe0 = g.e0 << g.lgC;
    unsigned long long sum = 0;
    for (int i = r.x + blockIdx.x * blockDim.x + threadIdx.x; i < r.y; i += gridDim.x * blockDim.x) {
        const float2 p = posS[i];
        const int cx = cell_coord(p.x, g.ox, g.csD, g.invCs, g.nx);
        const int cy = subrow_coord(p.y, g) >> g.lgS;
        const int rlo = max(cy - 1, 0) << g.lgS, rhi = (min(cy + 1, g.ny - 1) + 1) << g.lgS;
        const int f0 = max(cx - 1, 0) << g.lgC, f1 = (min(cx + 1, g.nx - 1) + 1) << g.lgC;
        for (int fc = f0; fc < f1; ++fc)
            sum += binStart[(fc - fe0) * nyS + rhi] - binStart[(fc - fe0) * nyS + rlo];
    }
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0 && sum) atomicAdd(out, sum);
}

// orca_set_state_async (one strip): every loaded agent, in its current sorted order, takes
// its new position / velocity by id from the upload and is binned into the work arrays
// exactly as the step epilogue bins its result (finish_agent): prefVel or goal, search-
// radius hint and per-agent properties travel along; k_scan + k_scatter then sort.  A
// non-finite input raises *bad (reported by orca_io_wait); an agent in the grid's outer
// cell ring or beyond (clamped: still exact, reading Q12) raises *gridFlag, so the grid is
// re-derived before a later step without a synchronisation here.
__global__ void k_reload(const uint32_t* __restrict__ binStart, Grid g, const uint32_t* __restrict__ idS,
                         const float2* __restrict__ auxS, const float* __restrict__ rk2S,
                         const float4* __restrict__ propS, const float2* __restrict__ pos,
                         const float2* __restrict__ vel, float2* __restrict__ posW, float2* __restrict__ velW,
                         float2* __restrict__ auxW, uint32_t* __restrict__ idW, float* __restrict__ rk2W,
                         float4* __restrict__ propW, uint32_t* __restrict__ cellW, uint32_t* __restrict__ rankW,
                         uint32_t* __restrict__ count, int* __restrict__ ctr, int* gridFlag, int* bad) {
    const int2 r = owned_range(binStart, g);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr[CT_NOWN] = r.y - r.x;
        ctr[CT_EXTRA] = 0;
    }
    bool nonfinite = false, ring = false;
    for (int i = r.x + blockIdx.x * blockDim.x + threadIdx.x; i < r.y; i += gridDim.x * blockDim.x) {
        const int w = i - r.x;
        const uint32_t id = idS[i];
        const float2 p = pos[id];
        const float2 v = vel[id];
        nonfinite |= !(isfinite(p.x) && isfinite(p.y) && isfinite(v.x) && isfinite(v.y));
        const int fx = finecol_coord(p.x, g);
        const int cx = fx >> g.lgC;
        const int sy = subrow_coord(p.y, g);
        const int cyc = sy >> g.lgS;
        ring |= cx == 0 || cx == g.nx - 1 || cyc == 0 || cyc == g.ny - 1;
        const uint32_t c = bin_of(fx, sy, g);
        posW[w] = p;
        velW[w] = v;
        auxW[w] = auxS[i];
        idW[w] = id;
        rk2W[w] = rk2S[i];
        if (propW) propW[w] = propS[i];
        cellW[w] = c;
        rankW[w] = atomicAdd(&count[c], 1u);
    }
    if (__any_sync(0xffffffffu, nonfinite) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
    if (__any_sync(0xffffffffu, ring) && (threadIdx.x & 31) == 0) *gridFlag = 1;
}

// orca_step_io_async (single strip): the upload is binned IN PLACE in the work arrays the last
// step left behind (its own next-step binning was skipped): every valid work slot takes its new
// pos / vel by id, keeps its id, preferred velocity / goal, radius hint and properties, and gets
// its bin and rank.  count[] must be zero.
__global__ void k_reload_work(const int* __restrict__ ctr, int capW, Grid g, const float2* __restrict__ pos,
                              const float2* __restrict__ vel, float2* __restrict__ posW, float2* __restrict__ velW,
                              const uint32_t* __restrict__ idW, uint32_t* __restrict__ cellW,
                              uint32_t* __restrict__ rankW, uint32_t* __restrict__ count, int* gridFlag, int* bad) {
    const int nW = min(ctr[CT_NOWN] + ctr[CT_EXTRA], capW);
    bool nonfinite = false, ring = false;
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nW; w += gridDim.x * blockDim.x) {
        if (cellW[w] == kInvalid) continue;  // removed at its goal
        const uint32_t id = idW[w];
        const float2 p = pos[id];
        const float2 v = vel[id];
        nonfinite |= !(isfinite(p.x) && isfinite(p.y) && isfinite(v.x) && isfinite(v.y));
        const int fx = finecol_coord(p.x, g);
        const int cx = fx >> g.lgC;
        const int sy = subrow_coord(p.y, g);
        const int cyc = sy >> g.lgS;
        ring |= cx == 0 || cx == g.nx - 1 || cyc == 0 || cyc == g.ny - 1;
        const uint32_t c = bin_of(fx, sy, g);
        posW[w] = p;
        velW[w] = v;
        cellW[w] = c;
        rankW[w] = atomicAdd(&count[c], 1u);
    }
    if (__any_sync(0xffffffffu, nonfinite) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
    if (__any_sync(0xffffffffu, ring) && (threadIdx.x & 31) == 0) *gridFlag = 1;
}

// The state after a step whose binning was skipped, by id, from the work arrays.
__global__ void k_unpermute_work(const int* __restrict__ ctr, int capW, const uint32_t* __restrict__ cellW,
                                 const uint32_t* __restrict__ idW, const float2* __restrict__ posW,
                                 const float2* __restrict__ velW, float2* __restrict__ posOut,
                                 float2* __restrict__ velOut) {
    const int nW = min(ctr[CT_NOWN] + ctr[CT_EXTRA], capW);
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nW; w += gridDim.x * blockDim.x) {
        if (cellW[w] == kInvalid) continue;
        const uint32_t id = idW[w];
        if (posOut) posOut[id] = posW[w];
        if (velOut) velOut[id] = velW[w];
    }
}

__global__ void k_fill1(int n, float* __restrict__ out, float v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = v;
}

// st = radius[n] | maxSpeed[n] | prefSpeed[n] (prefSpeed -1 = the set_goals speed) ->
// props[i] = (radius, maxSpeed, prefSpeed, 0); partial[b] = {max maxSpeed, -, -, -, invalid}
__global__ void k_pack_props(int n, const float* __restrict__ st, float4* __restrict__ props,
                             float* __restrict__ partial) {
    float vmax = 0.0f;
    int bad = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float r = st[i], vm = st[n + i], vp = st[2 * n + i];
        bad += !(isfinite(r) && r > 0.0f && isfinite(vm) && vm >= 0.0f && isfinite(vp) && (vp >= 0.0f || vp == -1.0f));
        vmax = fmaxf(vmax, vm);
        props[i] = make_float4(r, vm, vp, 0.0f);
    }
    for (int o = 16; o > 0; o >>= 1) {
        vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    __shared__ float s[32][2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        s[wid][0] = vmax;
        s[wid][1] = (float)bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.0f, b = 0.0f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            m = fmaxf(m, s[w][0]);
            b += s[w][1];
        }
        partial[blockIdx.x * 5 + 0] = m;
        partial[blockIdx.x * 5 + 4] = b;
    }
}

// out[i] = in[idS[i]] over all sorted entries (owned + ghosts)
__global__ void k_gather4_by_id(const uint32_t* __restrict__ binStart, int nbins, const uint32_t* __restrict__ idS,
                                const float4* __restrict__ in, float4* __restrict__ out) {
    const int n = (int)binStart[nbins];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[idS[i]];
}

__global__ void k_fill2(int n, float2* __restrict__ out, float v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = make_float2(v, v);
}

// active[id] = 1 for owned (not removed) agents
__global__ void k_mark_active(const uint32_t* __restrict__ binStart, Grid g, const uint32_t* __restrict__ idS,
                              uint8_t* __restrict__ active) {
    const int2 r = owned_range(binStart, g);
    for (int i = r.x + blockIdx.x * blockDim.x + threadIdx.x; i < r.y; i += gridDim.x * blockDim.x) active[idS[i]] = 1;
}

__global__ void k_cells(const uint32_t* __restrict__ binStart, Grid g, const uint32_t* __restrict__ idS,
                        const float2* __restrict__ posS, int32_t* __restrict__ cxOut, int32_t* __restrict__ cyOut) {
    const int2 r = owned_range(binStart, g);
    for (int i = r.x + blockIdx.x * blockDim.x + threadIdx.x; i < r.y; i += gridDim.x * blockDim.x) {
        const float2 p = posS[i];
        const uint32_t id = idS[i];
        cxOut[id] = cell_coord(p.x, g.ox, g.csD, g.invCs, g.nx);
        cyOut[id] = cell_coord(p.y, g.oy, g.csD, g.invCs, g.ny);
    }
}

// out[i] = in[idS[i]] over all sorted entries (owned + ghosts): id-ordered -> sorted
__global__ void k_gather_by_id(const uint32_t* __restrict__ binStart, int nbins, const uint32_t* __restrict__ idS,
                               const float2* __restrict__ in, float2* __restrict__ out) {
    const int n = (int)binStart[nbins];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[idS[i]];
}

// Received neighbour data -> work buffers: emigrants of the neighbour become owned agents,
// halo agents become ghosts (their columns decide which; both are just appended).
// Peer-memory exchange: copy the used records of a local send buffer into
// the neighbour's receive buffer of this step's parity -- remote stores over NVLink (a
// cudaIpc mapping between ranks; the neighbour strip's own buffer in loopback) -- and, once
// every block's stores are fenced system-wide, publish the counts and the arrival flag
// hdr[3] = step + 1.  Receive buffers alternate by step parity, so a fast sender never
// overwrites what a slow receiver is still reading (it has waited for that receiver's next
// step in between).
__global__ void k_push(ExBuf s, ExBuf d0, ExBuf d1, const int* __restrict__ ctr, unsigned int* __restrict__ done) {
    const int t = ctr[CT_XSTEP];
    const ExBuf& d = (t & 1) ? d1 : d0;
    const int nM = min(s.hdr[0], s.capM), nH = min(s.hdr[1], s.capH);
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nM + nH; q += gridDim.x * blockDim.x) {
        if (q < nM) {
            d.mpos[q] = s.mpos[q];
            d.mvel[q] = s.mvel[q];
            d.maux[q] = s.maux[q];
            d.mid[q] = s.mid[q];
            d.mrk2[q] = s.mrk2[q];
            d.mprop[q] = s.mprop[q];
        } else {
            const int h = q - nM;
            d.hpos[h] = s.hpos[h];
            d.hvel[h] = s.hvel[h];
            d.hid[h] = s.hid[h];
            d.hrad[h] = s.hrad[h];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(done, 1u) == gridDim.x - 1) {  // last block: every record is out
            volatile int* h = d.hdr;
            h[0] = s.hdr[0];
            h[1] = s.hdr[1];
            __threadfence_system();
            h[3] = t + 1;
            *done = 0u;
            s.hdr[0] = 0;  // the local send buffer is empty again for the next step
            s.hdr[1] = 0;
        }
    }
}

// Wait (bounded) until the neighbour's records of this step have arrived (flag hdr[3]).
__device__ __forceinline__ void wait_arrival(const ExBuf& b, int want, int* ctr) {
    volatile const int* f = b.hdr + 3;
    long long spins = 0;
    while (*f < want) {
        __nanosleep(200);
        if (++spins > 50000000ll) {  // ~10 s: a missing neighbour step -> error, never a hang
            atomicOr(&ctr[CT_OVF], OVF_TIMEOUT);
            break;
        }
    }
}

// Append the received emigrants (owned) and halo agents (ghosts) to the work arrays.  wait:
// peer-memory transport (buffers of this step's parity, arrival flags); else the buffers
// were filled in stream order (NCCL / loopback copies) and rL0 / rR0 are used.
__global__ void k_receive(StepArgs a, ExBuf rL0, ExBuf rL1, ExBuf rR0, ExBuf rR1, int wait) {
    const int xt = a.ctr[CT_XSTEP];
    const ExBuf rL = (wait && (xt & 1)) ? rL1 : rL0;
    const ExBuf rR = (wait && (xt & 1)) ? rR1 : rR0;
    if (wait) {
        __shared__ int ok;
        if (threadIdx.x == 0) {
            if (a.g.hasL) wait_arrival(rL, xt + 1, a.ctr);
            if (a.g.hasR) wait_arrival(rR, xt + 1, a.ctr);
            __threadfence_system();
            ok = 1;
        }
        __syncthreads();
        (void)ok;
    }
    const int nOwn = a.ctr[CT_NOWN];
    const int mL = a.g.hasL ? min(rL.hdr[0], rL.capM) : 0, hL = a.g.hasL ? min(rL.hdr[1], rL.capH) : 0;
    const int mR = a.g.hasR ? min(rR.hdr[0], rR.capM) : 0, hR = a.g.hasR ? min(rR.hdr[1], rR.capH) : 0;
    const int tot = mL + hL + mR + hR;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += gridDim.x * blockDim.x) {
        int q = t;
        const ExBuf* x = &rL;
        bool mig = true;
        if (q < mL) {
        } else if ((q -= mL) < hL) {
            mig = false;
        } else if ((q -= hL) < mR) {
            x = &rR;
        } else {
            q -= mR;
            x = &rR;
            mig = false;
        }
        const float2 p = mig ? x->mpos[q] : x->hpos[q];
        const int fx = finecol_coord(p.x, a.g);
        const int sy = subrow_coord(p.y, a.g);
        if (mig)
            append_work(a, nOwn, fx, sy, p, x->mvel[q], x->maux[q], x->mid[q], x->mrk2[q], x->mprop[q]);
        else
            append_work(a, nOwn, fx, sy, p, x->hvel[q], make_float2(0.0f, 0.0f), x->hid[q], INFINITY,
                        make_float4(x->hrad[q], 0.0f, 0.0f, 0.0f));
    }
}

// agents per grid column (strip partition at set_agents)
__global__ void k_colhist(int n, const float2* __restrict__ pos, Grid g, int32_t* __restrict__ hist,
                          const uint8_t* __restrict__ active) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (!active || active[i]) atomicAdd(&hist[cell_coord(pos[i].x, g.ox, g.csD, g.invCs, g.nx)], 1);
}

// Block-partial min/max of the positions and a non-finite count over all input arrays.
// partial[b] = {minx, miny, maxx, maxy, nonfinite}
__global__ void k_minmax(int n, const float2* __restrict__ pos, const float2* __restrict__ vel,
                         const float2* __restrict__ aux, float* __restrict__ partial,
                         const uint8_t* __restrict__ active) {
    float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    int bad = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (active && !active[i]) continue;  // removed at its goal
        const float2 p = pos[i];
        const float2 v = vel[i];
        const float2 q = aux[i];
        bad += !(isfinite(p.x) && isfinite(p.y) && isfinite(v.x) && isfinite(v.y) && isfinite(q.x) &&
                 isfinite(q.y));
        mnx = fminf(mnx, p.x);
        mny = fminf(mny, p.y);
        mxx = fmaxf(mxx, p.x);
        mxy = fmaxf(mxy, p.y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    __shared__ float s[32][5];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        s[wid][0] = mnx;
        s[wid][1] = mny;
        s[wid][2] = mxx;
        s[wid][3] = mxy;
        s[wid][4] = (float)bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float r[5] = {INFINITY, INFINITY, -INFINITY, -INFINITY, 0.0f};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            r[0] = fminf(r[0], s[w][0]);
            r[1] = fminf(r[1], s[w][1]);
            r[2] = fmaxf(r[2], s[w][2]);
            r[3] = fmaxf(r[3], s[w][3]);
            r[4] += s[w][4];
        }
        for (int q = 0; q < 5; ++q) partial[blockIdx.x * 5 + q] = r[q];
    }
}

}  // namespace orca
