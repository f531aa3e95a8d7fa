// orca.cu -- host runtime + C ABI of liborca (include/orca.h).
//
// Owns device buffers, the context stream and the CUDA graph of n step bodies.  Every
// arithmetic step of the ORCA update runs in the kernels of orca_kernels.cuh; this file
// only validates arguments, allocates, copies and launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/orca.h"
#include "orca_kernels.cuh"

using namespace orca;

namespace {

constexpr int kSubRowsLog2 = 3;  // 8 sort sub-rows per cell

int scan_tiles(int64_t C) { return (int)((C + kScanTile - 1) / kScanTile); }
int lp3_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + kStepThreads - 1) / kStepThreads, 148 * 8)); }

thread_local std::string g_last_error;

orca_status fail(orca_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

orca_status cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();  // clear sticky-free errors
    return fail(e == cudaErrorMemoryAllocation ? ORCA_ERR_OUT_OF_MEMORY : ORCA_ERR_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                      \
    do {                                              \
        cudaError_t _e = (expr);                      \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
    } while (0)

bool finite_params(const orca_params* p) {
    return std::isfinite(p->timeStep) && std::isfinite(p->neighborDist) && std::isfinite(p->timeHorizon) &&
           std::isfinite(p->radius) && std::isfinite(p->maxSpeed) && p->timeStep > 0.0f &&
           p->neighborDist > 0.0f && p->timeHorizon > 0.0f && p->radius > 0.0f && p->maxSpeed >= 0.0f &&
           p->maxNeighbors >= 0 && p->maxNeighbors <= ORCA_MAX_K;
}

template <typename T>
void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

int grid_blocks(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

}  // namespace

struct orca_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    orca_params p{};
    int64_t n = 0;
    int64_t cap = 0;     // agent capacity of the buffers
    int64_t cellCap = 0; // cell capacity
    bool ready = false;
    bool goals = false;
    float prefSpeed = 0.0f;
    Grid g{};
    int64_t C = 0;     // sort bins = cells x 2^lgS sub-rows
    // sorted (rest) state and work buffers
    float2 *posS = nullptr, *velS = nullptr, *auxS = nullptr;
    uint32_t* idS = nullptr;
    float2 *posW = nullptr, *velW = nullptr, *auxW = nullptr;
    float *rk2S = nullptr, *rk2W = nullptr;  // previous k-th neighbour d2 (search bound)
    uint32_t *idW = nullptr, *cellW = nullptr, *rankW = nullptr;
    uint32_t *count = nullptr, *binStart = nullptr;
    unsigned long long* scanStatus = nullptr;  // look-back status words + ticket + LP3 queue count
    int4* qEntry = nullptr;                    // LP3 queue (capacity cap)
    float4* qLines = nullptr;                  // cap x k lines
    int lp3Smem = 0;
    unsigned long long* stats = nullptr;
    float* partial = nullptr;  // k_minmax partials
    float2* tmp2 = nullptr;    // id-ordered scratch (get_state / set_goals)
    float2* tmp2b = nullptr;
    int64_t host_steps = 0, host_updates = 0;
    // graph cache: (step count, executable), a few entries
    std::vector<std::pair<int, cudaGraphExec_t>> graphs;
    cudaEvent_t ev[9] = {};
    int smemBytes = 0;
};

namespace {

Model make_model(const orca_ctx* c) {
    Model m{};
    const orca_params& p = c->p;
    m.dt = p.timeStep;
    m.maxSpeed = p.maxSpeed;
    m.R = p.radius + p.radius;
    m.invTauF = 1.0f / p.timeHorizon;
    m.invDtF = 1.0f / p.timeStep;
    m.invTauD = 1.0 / (double)p.timeHorizon;
    m.invDtD = 1.0 / (double)p.timeStep;
    const double R = (double)p.radius + (double)p.radius;
    m.R2D = R * R;
    m.nd2D = (double)p.neighborDist * (double)p.neighborDist;
    // fp32 prefilter bound: nd^2 rounded up, plus relative margin 2^-20 (> fp32 d2 error)
    float nd2f = (float)m.nd2D;
    if ((double)nd2f < m.nd2D) nd2f = std::nextafter(nd2f, INFINITY);
    m.nd2Fup = std::nextafter(nd2f * (1.0f + 0x1p-20f), INFINITY);
    // fp32 d2 below nd2Lo proves kappa < nd^2 (relative error < 2^-22, margin 2^-20)
    float nd2d = (float)m.nd2D;
    if ((double)nd2d > m.nd2D) nd2d = std::nextafter(nd2d, 0.0f);
    m.nd2Lo = std::nextafter(nd2d * (1.0f - 0x1p-20f), 0.0f);
    m.k = p.maxNeighbors;
    m.goals = c->goals ? 1 : 0;
    m.prefSpeed = c->prefSpeed;
    return m;
}

StepArgs make_args(orca_ctx* c) {
    StepArgs a{};
    a.n = (int)c->n;
    a.g = c->g;
    a.m = make_model(c);
    a.posS = c->posS;
    a.velS = c->velS;
    a.auxS = c->auxS;
    a.rk2S = c->rk2S;
    a.rk2W = c->rk2W;
    a.idS = c->idS;
    a.binStart = c->binStart;
    a.posW = c->posW;
    a.velW = c->velW;
    a.auxW = c->auxW;
    a.idW = c->idW;
    a.cellW = c->cellW;
    a.rankW = c->rankW;
    a.count = c->count;
    a.stats = c->stats;
    a.qEntry = c->qEntry;
    a.qLines = c->qLines;
    a.qcap = (int)c->cap;
    a.qCount = reinterpret_cast<unsigned int*>(c->scanStatus + scan_tiles(c->C) + 1);
    return a;
}

orca_status ensure_capacity(orca_ctx* c, int64_t n, int64_t C) {
    if (n > c->cap) {
        const int64_t cap = std::max<int64_t>(n, 1);
        float2** f2[] = {&c->posS, &c->velS, &c->auxS, &c->posW, &c->velW, &c->auxW, &c->tmp2, &c->tmp2b};
        uint32_t** u4[] = {&c->idS, &c->idW, &c->cellW, &c->rankW};
        for (auto pp : f2) dfree(*pp);
        for (auto pp : u4) dfree(*pp);
        for (auto pp : f2) CK(cudaMalloc(pp, cap * sizeof(float2)));
        for (auto pp : u4) CK(cudaMalloc(pp, cap * sizeof(uint32_t)));
        dfree(c->qEntry);
        dfree(c->qLines);
        dfree(c->rk2S);
        dfree(c->rk2W);
        CK(cudaMalloc(&c->rk2S, cap * sizeof(float)));
        CK(cudaMalloc(&c->rk2W, cap * sizeof(float)));
        CK(cudaMalloc(&c->qEntry, cap * sizeof(int4)));
        CK(cudaMalloc(&c->qLines, cap * std::max(1, c->p.maxNeighbors) * sizeof(float4)));
        c->cap = cap;
    }
    if (C > c->cellCap) {
        dfree(c->count);
        dfree(c->binStart);
        dfree(c->scanStatus);
        CK(cudaMalloc(&c->count, (C + 4) * sizeof(uint32_t)));
        CK(cudaMalloc(&c->binStart, (C + 1) * sizeof(uint32_t)));
        CK(cudaMalloc(&c->scanStatus, (scan_tiles(C) + 2) * sizeof(unsigned long long)));
        c->cellCap = C;
    }
    return ORCA_OK;
}

// exclusive scan of the bin counts (memset of the look-back status + one launch)
cudaError_t enqueue_scan(orca_ctx* c) {
    const int tiles = scan_tiles(c->C);
    // status words, tile ticket and the LP3 queue count (consumed by k_lp3 before this point)
    cudaError_t e = cudaMemsetAsync(c->scanStatus, 0, (tiles + 2) * sizeof(unsigned long long), c->stream);
    if (e != cudaSuccess) return e;
    k_scan<<<tiles, 1024, 0, c->stream>>>(c->count, c->binStart, (int)c->C, c->scanStatus,
                                          reinterpret_cast<unsigned int*>(c->scanStatus + tiles));
    return cudaGetLastError();
}

void drop_graph(orca_ctx* c) {
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.second);
    c->graphs.clear();
}

// one step body: fused step kernel -> scan -> scatter (rest state = sorted arrays)
cudaError_t enqueue_step(orca_ctx* c, cudaEvent_t* ev) {
    const int n = (int)c->n;
    StepArgs a = make_args(c);
    if (ev) cudaEventRecord(ev[0], c->stream);
    if (n > 0) {
        const int blocks = (n + kStepThreads - 1) / kStepThreads;
        k_step<false><<<blocks, kStepThreads, c->smemBytes, c->stream>>>(a);
        k_lp3<false><<<lp3_blocks(n), kStepThreads, c->lp3Smem, c->stream>>>(a);
    }
    if (ev) cudaEventRecord(ev[1], c->stream);
    enqueue_scan(c);
    if (ev) cudaEventRecord(ev[2], c->stream);
    if (n > 0)
        k_scatter<<<grid_blocks(n, 256), 256, 0, c->stream>>>(n, c->cellW, c->rankW, c->binStart, c->posW, c->velW,
                                                              c->auxW, c->idW, c->posS, c->velS, c->auxS, c->idS,
                                                              c->rk2W, c->rk2S);
    if (ev) cudaEventRecord(ev[3], c->stream);
    return cudaGetLastError();
}

// The dry (debug) step: same kernels, outputs by id, state untouched; the LP3 queue
// count is zeroed before and after so the next real step starts from an empty queue.
cudaError_t dry_step(orca_ctx* c, StepArgs& a) {
    const int n = (int)c->n;
    cudaError_t e = cudaMemsetAsync(a.qCount, 0, sizeof(unsigned int), c->stream);
    if (e != cudaSuccess) return e;
    k_step<true><<<(n + kStepThreads - 1) / kStepThreads, kStepThreads, c->smemBytes, c->stream>>>(a);
    k_lp3<true><<<lp3_blocks(n), kStepThreads, c->lp3Smem, c->stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(a.qCount, 0, sizeof(unsigned int), c->stream);
}

// Copy a float[2n] user array (host or device) into a device float2 buffer.
cudaError_t copy_in(orca_ctx* c, float2* dst, const float* src, int64_t n) {
    if (n == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->stream);
}

}  // namespace

// =============================================================================== ABI
extern "C" {

const char* orca_status_string(orca_status s) {
    switch (s) {
        case ORCA_OK: return "ok";
        case ORCA_ERR_INVALID_ARGUMENT: return "invalid argument";
        case ORCA_ERR_NOT_READY: return "not ready (call orca_set_agents first)";
        case ORCA_ERR_OUT_OF_MEMORY: return "out of device memory";
        case ORCA_ERR_CUDA: return "CUDA error";
        case ORCA_ERR_NCCL: return "NCCL error";
        case ORCA_ERR_CAPACITY: return "capacity exceeded";
        case ORCA_ERR_INTERNAL: return "internal error";
        default: return "unknown status";
    }
}

const char* orca_last_error(void) { return g_last_error.c_str(); }

orca_status orca_create(const orca_params* params, int32_t device, orca_ctx** out) {
    if (!params || !out) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (!finite_params(params)) return fail(ORCA_ERR_INVALID_ARGUMENT, "parameter out of range or not finite");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(ORCA_ERR_INVALID_ARGUMENT, "no such CUDA device");
    CK(cudaSetDevice(device));
    orca_ctx* c = new (std::nothrow) orca_ctx();
    if (!c) return fail(ORCA_ERR_OUT_OF_MEMORY, "host allocation");
    c->device = device;
    c->p = *params;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&c->stats, ST_COUNT * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(c->stats, 0, ST_COUNT * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&c->partial, 1024 * 5 * sizeof(float));
    for (int q = 0; q < 9 && e == cudaSuccess; ++q) e = cudaEventCreate(&c->ev[q]);
    c->smemBytes = step_smem_per_thread(params->maxNeighbors) * kStepThreads;
    c->lp3Smem = std::max(1, 6 * params->maxNeighbors) * 4 * kStepThreads;
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smemBytes);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smemBytes);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_lp3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->lp3Smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_lp3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->lp3Smem);
    if (e != cudaSuccess) {
        orca_destroy(c);
        return cuda_fail(e, "orca_create");
    }
    *out = c;
    return ORCA_OK;
}

void orca_destroy(orca_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    drop_graph(c);
    float2** f2[] = {&c->posS, &c->velS, &c->auxS, &c->posW, &c->velW, &c->auxW, &c->tmp2, &c->tmp2b};
    uint32_t** u4[] = {&c->idS, &c->idW, &c->cellW, &c->rankW, &c->count, &c->binStart};
    for (auto pp : f2) dfree(*pp);
    for (auto pp : u4) dfree(*pp);
    dfree(c->stats);
    dfree(c->partial);
    dfree(c->scanStatus);
    dfree(c->qEntry);
    dfree(c->qLines);
    dfree(c->rk2S);
    dfree(c->rk2W);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

orca_status orca_set_agents(orca_ctx* c, int64_t n, const float* pos, const float* vel, const float* pref) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (n < 0 || n > (int64_t)1 << 30) return fail(ORCA_ERR_INVALID_ARGUMENT, "n out of range");
    if (n > 0 && (!pos || !vel || !pref)) return fail(ORCA_ERR_INVALID_ARGUMENT, "null array");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->stream));
    drop_graph(c);
    c->ready = false;
    c->goals = false;
    // stage the inputs in the work buffers (capacity first; grid sized after min/max)
    orca_status st = ensure_capacity(c, n, 1);
    if (st) return st;
    CK(copy_in(c, c->posW, pos, n));
    CK(copy_in(c, c->velW, vel, n));
    CK(copy_in(c, c->auxW, pref, n));
    // bounds + finiteness on the device (inputs may be device pointers)
    float mn[2] = {0.0f, 0.0f}, mx[2] = {0.0f, 0.0f};
    if (n > 0) {
        const int blocks = std::min(1024, grid_blocks(n, 256));
        k_minmax<<<blocks, 256, 0, c->stream>>>((int)n, c->posW, c->velW, c->auxW, c->partial);
        CK(cudaGetLastError());
        std::vector<float> h((size_t)blocks * 5);
        CK(cudaMemcpyAsync(h.data(), c->partial, h.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        mn[0] = mn[1] = INFINITY;
        mx[0] = mx[1] = -INFINITY;
        double bad = 0;
        for (int b = 0; b < blocks; ++b) {
            mn[0] = std::min(mn[0], h[b * 5 + 0]);
            mn[1] = std::min(mn[1], h[b * 5 + 1]);
            mx[0] = std::max(mx[0], h[b * 5 + 2]);
            mx[1] = std::max(mx[1], h[b * 5 + 3]);
            bad += h[b * 5 + 4];
        }
        if (bad > 0) return fail(ORCA_ERR_INVALID_ARGUMENT, "NaN/Inf in pos/vel/prefVel");
    }
    // frozen grid (reading Q12)
    const float cs = c->p.neighborDist;
    Grid g{};
    g.cs = cs;
    g.lgS = kSubRowsLog2;
    if (n == 0) {
        g.ox = g.oy = 0.0f;
        g.nx = g.ny = 1;
    } else {
        volatile float ox = mn[0] - cs, oy = mn[1] - cs;
        g.ox = ox;
        g.oy = oy;
        const double tx = std::floor(((double)mx[0] - (double)g.ox) / (double)cs);
        const double ty = std::floor(((double)mx[1] - (double)g.oy) / (double)cs);
        if (tx + 2 > 1e9 || ty + 2 > 1e9 || (tx + 2) * (ty + 2) * (double)(1 << kSubRowsLog2) > (double)(1 << 28))
            return fail(ORCA_ERR_CAPACITY, "grid would exceed 2^28 sort bins");
        g.nx = (int)tx + 2;
        g.ny = (int)ty + 2;
    }
    g.csD = (double)cs;
    g.invCs = 1.0 / (double)cs;
    g.csSub = (double)cs / (double)(1 << g.lgS);
    g.invCsSub = (double)(1 << g.lgS) / (double)cs;
    c->g = g;
    c->C = ((int64_t)g.nx * g.ny) << g.lgS;
    st = ensure_capacity(c, n, c->C);
    if (st) return st;
    c->n = n;
    // ids, initial binning, scan, scatter -> rest state
    CK(cudaMemsetAsync(c->count, 0, c->C * sizeof(uint32_t), c->stream));
    if (n > 0) {
        k_iota<<<grid_blocks(n, 256), 256, 0, c->stream>>>((int)n, c->idW, c->rk2W);
        k_hash<<<grid_blocks(n, 256), 256, 0, c->stream>>>((int)n, c->posW, c->g, c->cellW, c->rankW, c->count);
    }
    CK(enqueue_scan(c));
    if (n > 0)
        k_scatter<<<grid_blocks(n, 256), 256, 0, c->stream>>>((int)n, c->cellW, c->rankW, c->binStart, c->posW,
                                                              c->velW, c->auxW, c->idW, c->posS, c->velS, c->auxS,
                                                              c->idS, c->rk2W, c->rk2S);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    c->ready = true;
    return ORCA_OK;
}

orca_status orca_set_goals(orca_ctx* c, const float* goal, float prefSpeed) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (!(prefSpeed >= 0.0f) || !std::isfinite(prefSpeed)) return fail(ORCA_ERR_INVALID_ARGUMENT, "prefSpeed");
    if (c->n > 0 && !goal) return fail(ORCA_ERR_INVALID_ARGUMENT, "null goal");
    CK(cudaSetDevice(c->device));
    const int n = (int)c->n;
    if (n > 0) {
        // goals arrive in id order: check finiteness, then permute into sorted order
        CK(copy_in(c, c->tmp2, goal, n));
        const int blocks = std::min(1024, grid_blocks(n, 256));
        k_minmax<<<blocks, 256, 0, c->stream>>>(n, c->tmp2, c->tmp2, c->tmp2, c->partial);
        std::vector<float> h((size_t)blocks * 5);
        CK(cudaMemcpyAsync(h.data(), c->partial, h.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int b = 0; b < blocks; ++b)
            if (h[b * 5 + 4] > 0) return fail(ORCA_ERR_INVALID_ARGUMENT, "NaN/Inf in goal");
        // gather by id into the sorted aux array
        k_gather_by_id<<<grid_blocks(n, 256), 256, 0, c->stream>>>(n, c->idS, c->tmp2, c->auxS);
        CK(cudaGetLastError());
    }
    drop_graph(c);
    c->goals = true;
    c->prefSpeed = prefSpeed;
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

orca_status orca_step(orca_ctx* c, int32_t n_steps) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (n_steps < 0) return fail(ORCA_ERR_INVALID_ARGUMENT, "n_steps < 0");
    if (n_steps == 0) return ORCA_OK;
    CK(cudaSetDevice(c->device));
    // one graph of up to kChunk step bodies, replayed
    const int kChunk = 64;
    int remaining = n_steps;
    while (remaining > 0) {
        const int s = std::min(remaining, kChunk);
        cudaGraphExec_t exec = nullptr;
        for (auto& g : c->graphs)
            if (g.first == s) exec = g.second;
        if (!exec) {
            if (c->graphs.size() >= 4) {
                cudaGraphExecDestroy(c->graphs.front().second);
                c->graphs.erase(c->graphs.begin());
            }
            cudaGraph_t gr;
            CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            cudaError_t e = cudaSuccess;
            for (int q = 0; q < s && e == cudaSuccess; ++q) e = enqueue_step(c, nullptr);
            cudaError_t e2 = cudaStreamEndCapture(c->stream, &gr);
            if (e != cudaSuccess) return cuda_fail(e, "capture");
            if (e2 != cudaSuccess) return cuda_fail(e2, "cudaStreamEndCapture");
            e = cudaGraphInstantiate(&exec, gr, 0);
            cudaGraphDestroy(gr);
            if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
            c->graphs.emplace_back(s, exec);
        }
        CK(cudaGraphLaunch(exec, c->stream));
        remaining -= s;
    }
    c->host_steps += n_steps;
    c->host_updates += (int64_t)n_steps * c->n;
    return ORCA_OK;
}

orca_status orca_step_timed(orca_ctx* c, int32_t n_steps, double ms[4]) {
    if (!c || !ms) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (n_steps < 0) return fail(ORCA_ERR_INVALID_ARGUMENT, "n_steps < 0");
    CK(cudaSetDevice(c->device));
    for (int q = 0; q < 4; ++q) ms[q] = 0.0;
    for (int s = 0; s < n_steps; ++s) {
        CK(enqueue_step(c, c->ev));
        CK(cudaEventSynchronize(c->ev[3]));
        float t;
        CK(cudaEventElapsedTime(&t, c->ev[0], c->ev[1]));
        ms[0] += t;
        CK(cudaEventElapsedTime(&t, c->ev[1], c->ev[2]));
        ms[1] += t;
        CK(cudaEventElapsedTime(&t, c->ev[2], c->ev[3]));
        ms[2] += t;
    }
    c->host_steps += n_steps;
    c->host_updates += (int64_t)n_steps * c->n;
    return ORCA_OK;
}

orca_status orca_get_state(orca_ctx* c, float* pos, float* vel) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    const int n = (int)c->n;
    if (n > 0 && (pos || vel)) {
        k_unpermute<<<grid_blocks(n, 256), 256, 0, c->stream>>>(n, c->idS, c->posS, c->velS, c->tmp2, c->tmp2b);
        CK(cudaGetLastError());
        if (pos) CK(cudaMemcpyAsync(pos, c->tmp2, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->stream));
        if (vel) CK(cudaMemcpyAsync(vel, c->tmp2b, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

orca_status orca_get_local_state(orca_ctx* c, int32_t* ids, float* pos, float* vel) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    const size_t n = (size_t)c->n;
    if (n > 0) {
        if (ids) CK(cudaMemcpyAsync(ids, c->idS, n * sizeof(uint32_t), cudaMemcpyDefault, c->stream));
        if (pos) CK(cudaMemcpyAsync(pos, c->posS, n * sizeof(float2), cudaMemcpyDefault, c->stream));
        if (vel) CK(cudaMemcpyAsync(vel, c->velS, n * sizeof(float2), cudaMemcpyDefault, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

orca_status orca_get_count(orca_ctx* c, int64_t* n) {
    if (!c || !n) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    *n = c->n;
    return ORCA_OK;
}

orca_status orca_get_grid(orca_ctx* c, double origin[2], float* cs, int32_t dims[2]) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (origin) {
        origin[0] = c->g.ox;
        origin[1] = c->g.oy;
    }
    if (cs) *cs = c->g.cs;
    if (dims) {
        dims[0] = c->g.nx;
        dims[1] = c->g.ny;
    }
    return ORCA_OK;
}

orca_status orca_debug_cells(orca_ctx* c, int32_t* cx, int32_t* cy) {
    if (!c || !cx || !cy) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    const int n = (int)c->n;
    if (n > 0) {
        int32_t* d = reinterpret_cast<int32_t*>(c->tmp2);  // 2 x int32 per agent
        k_cells<<<grid_blocks(n, 256), 256, 0, c->stream>>>(n, c->idS, c->posS, c->g, d, d + n);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(cx, d, (size_t)n * sizeof(int32_t), cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(cy, d + n, (size_t)n * sizeof(int32_t), cudaMemcpyDefault, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

orca_status orca_debug_step(orca_ctx* c, float* vnew, uint8_t* flags, int32_t* nbr, int32_t* cnt) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    const int n = (int)c->n;
    if (n == 0) return ORCA_OK;
    const int k = c->p.maxNeighbors;
    float2* dV = nullptr;
    uint8_t* dF = nullptr;
    int32_t *dN = nullptr, *dC = nullptr;
    CK(cudaMalloc(&dV, (size_t)n * sizeof(float2)));
    cudaError_t e = cudaMalloc(&dF, (size_t)n);
    if (e == cudaSuccess) e = cudaMalloc(&dC, (size_t)n * sizeof(int32_t));
    if (e == cudaSuccess && k > 0) e = cudaMalloc(&dN, (size_t)n * k * sizeof(int32_t));
    if (e == cudaSuccess) {
        StepArgs a = make_args(c);
        a.dbgV = dV;
        a.dbgFlags = dF;
        a.dbgNbr = dN;
        a.dbgCnt = dC;
        e = dry_step(c, a);
    }
    if (e == cudaSuccess && vnew) e = cudaMemcpyAsync(vnew, dV, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->stream);
    if (e == cudaSuccess && flags) e = cudaMemcpyAsync(flags, dF, (size_t)n, cudaMemcpyDefault, c->stream);
    if (e == cudaSuccess && cnt) e = cudaMemcpyAsync(cnt, dC, (size_t)n * sizeof(int32_t), cudaMemcpyDefault, c->stream);
    if (e == cudaSuccess && nbr && k > 0)
        e = cudaMemcpyAsync(nbr, dN, (size_t)n * k * sizeof(int32_t), cudaMemcpyDefault, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(dV);
    cudaFree(dF);
    cudaFree(dC);
    if (dN) cudaFree(dN);
    if (e != cudaSuccess) return cuda_fail(e, "orca_debug_step");
    return ORCA_OK;
}

orca_status orca_debug_work(orca_ctx* c, int64_t out[5]) {
    if (!c || !out) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    for (int q = 0; q < 5; ++q) out[q] = 0;
    const int n = (int)c->n;
    if (n == 0) return ORCA_OK;
    Work* dW = nullptr;
    CK(cudaMalloc(&dW, sizeof(Work)));
    cudaError_t e = cudaMemsetAsync(dW, 0, sizeof(Work), c->stream);
    if (e == cudaSuccess) {
        StepArgs a = make_args(c);
        a.work = dW;
        e = dry_step(c, a);
    }
    Work h{};
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, dW, sizeof(Work), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(dW);
    if (e != cudaSuccess) return cuda_fail(e, "orca_debug_work");
    out[0] = (int64_t)h.cand;
    out[1] = (int64_t)h.lines;
    out[2] = (int64_t)h.checks;
    out[3] = (int64_t)h.lp1;
    out[4] = (int64_t)h.proj;
    return ORCA_OK;
}

orca_status orca_get_stats(orca_ctx* c, orca_stats* out) {
    if (!c || !out) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    CK(cudaSetDevice(c->device));
    unsigned long long h[ST_COUNT];
    CK(cudaMemcpyAsync(h, c->stats, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    out->steps = c->host_steps;
    out->agent_updates = c->host_updates;
    out->infeasible = (int64_t)h[ST_INFEASIBLE];
    out->degenerate = (int64_t)h[ST_DEGENERATE];
    out->coincident = (int64_t)h[ST_G1];
    out->eps_parallel = (int64_t)h[ST_G2];
    out->marginal = (int64_t)h[ST_G3];
    out->collision_pairs = (int64_t)h[ST_COLLISION];
    return ORCA_OK;
}

orca_status orca_reset_stats(orca_ctx* c) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    CK(cudaSetDevice(c->device));
    CK(cudaMemsetAsync(c->stats, 0, ST_COUNT * sizeof(unsigned long long), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->host_steps = 0;
    c->host_updates = 0;
    return ORCA_OK;
}

orca_status orca_get_stream(orca_ctx* c, void** stream) {
    if (!c || !stream) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    *stream = (void*)c->stream;
    return ORCA_OK;
}

// ---- multi-GPU --------------------------------------------------------
orca_status orca_nccl_unique_id(void* id128) {
    if (!id128) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    return fail(ORCA_ERR_NCCL, "multi-GPU strips not built yet");
}

orca_status orca_create_dist(const orca_params* params, int32_t device, int32_t rank, int32_t world,
                             const void* nccl_id128, orca_ctx** out) {
    if (world == 1 && rank == 0) return orca_create(params, device, out);
    (void)nccl_id128;
    return fail(ORCA_ERR_NCCL, "multi-GPU strips not built yet");
}
}  // extern "C"
