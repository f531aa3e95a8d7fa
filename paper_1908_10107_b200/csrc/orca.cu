// orca.cu -- host runtime + C ABI of liborca (include/orca.h).
//
// Owns device buffers, the context stream, the CUDA graph of n step bodies and the
// strip decomposition.  Every arithmetic step of the ORCA update runs in
// the kernels of orca_kernels.cuh; this file validates arguments, allocates, copies,
// launches and moves exchange buffers (NCCL send/recv between ranks, or device copies
// between the strips of an in-process "loopback" group used to test the decomposition on
// one GPU).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <type_traits>
#include <new>
#include <string>
#include <vector>

#include "../../include/orca.h"
#include "orca_kernels.cuh"
#include "orca_step_group.cuh"
#include "orca_lp3_group.cuh"

using namespace orca;

namespace {

#ifndef ORCA_SUBROWS_LOG2
#define ORCA_SUBROWS_LOG2 3
#endif
constexpr int kSubRowsLog2 = ORCA_SUBROWS_LOG2;  // 2^this sort sub-rows per cell
#ifndef ORCA_SUBCOLS_LOG2
#define ORCA_SUBCOLS_LOG2 2
#endif
constexpr int kSubColsLog2 = ORCA_SUBCOLS_LOG2;  // 2^this fine columns per cell

int scan_tiles(int64_t C) { return (int)((C + kScanTile - 1) / kScanTile); }
int cap_blocks(int64_t n, int threads) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 32));
}
// k_lp3 takes one queue entry per thread (the queue holds at most capW agents), grid-stride
// beyond ORCA_LP3_WAVES waves of resident blocks
#ifndef ORCA_LP3_WAVES
#define ORCA_LP3_WAVES 4
#endif
constexpr int kPushBlocks = 64;  // k_push grid (last-block completion)
#ifndef ORCA_REGRID_REACH
#define ORCA_REGRID_REACH 512.0f  // steps of maxSpeed walking a re-derived grid's margin covers (r01: 128)
#endif
constexpr float kRegridReach = ORCA_REGRID_REACH;
constexpr int kBinMaxGrid = 4096;  // k_bin blocks at most (one resident wave)
// threads per block of the specialised block-queue k_step (LP3 on the block queue, strips of at
// most one wave; r02al: 100k 0.0614 -> 0.0585 ms with 256 instead of 128)
#ifndef ORCA_STEP_BQ_THREADS
#define ORCA_STEP_BQ_THREADS 256
#endif
constexpr int kStepBQ = ORCA_STEP_BQ_THREADS;
// blocks/SM of the larger-register lane-pair k_step used while a strip fits one wave of it (0: off)
#ifndef ORCA_PAIR_MB
#define ORCA_PAIR_MB 6  // r02au: 85 registers; 55k -4 %, 20k / corridor 0-5 % (5 and 7 no better)
#endif
// blocks/SM the k_lp3-placement k_step's register budget is sized for (0: 8 = 64 registers)
#ifndef ORCA_LM0_MB
#define ORCA_LM0_MB 0
#endif
#ifndef ORCA_FUSED_BIN
#define ORCA_FUSED_BIN 0  // 1: single-strip steps bin with the cooperative k_bin (scan + scatter fused); measured neutral/slower (r02ac), off
#endif

int lp3_blocks(int64_t n) {
    const int64_t need = (n + kStepThreads - 1) / kStepThreads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)148 * 7 * ORCA_LP3_WAVES));
}

thread_local std::string g_last_error;

orca_status fail(orca_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

orca_status cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? ORCA_ERR_OUT_OF_MEMORY : ORCA_ERR_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                            \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
    } while (0)

#define CKS(expr)                     \
    do {                              \
        orca_status _s = (expr);      \
        if (_s != ORCA_OK) return _s; \
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

// ---------------------------------------------------------------- NCCL (dlopen'ed)
// liborca does not link NCCL: it binds the libnccl.so.2 already loaded by the process
// (torch's) or the system one, so single-GPU use never needs it.
struct NcclApi {
    bool tried = false, ok = false;
    std::string err;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
    ncclResult_t (*commCount)(ncclComm_t, int*) = nullptr;  // optional
};

NcclApi& nccl() {
    static NcclApi api;
    if (api.tried) return api;
    api.tried = true;
#ifdef ORCA_TEST_HOOKS
    // TEST BUILD ONLY (liborca_test.so, build.py test_hooks=True): ORCA_NCCL_LIB names an
    // alternative implementation of the same API -- the tests' host-staged stand-in
    // tests/fake_nccl, which lets several processes share one GPU.  The product liborca.so
    // always uses the process's libnccl.so.2.
    const char* alt = getenv("ORCA_NCCL_LIB");
#else
    const char* alt = nullptr;
#endif
    void* h = (alt && *alt) ? dlopen(alt, RTLD_NOW | RTLD_LOCAL) : dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h && !(alt && *alt)) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        api.err = std::string("dlopen libnccl.so.2: ") + dlerror();
        return api;
    }
    bool ok = true;
    auto sym = [&](const char* n) {
        void* p = dlsym(h, n);
        if (!p) ok = false;
        return p;
    };
    api.getUniqueId = (decltype(api.getUniqueId))sym("ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))sym("ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))sym("ncclCommDestroy");
    api.send = (decltype(api.send))sym("ncclSend");
    api.recv = (decltype(api.recv))sym("ncclRecv");
    api.groupStart = (decltype(api.groupStart))sym("ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))sym("ncclGroupEnd");
    api.allReduce = (decltype(api.allReduce))sym("ncclAllReduce");
    api.allGather = (decltype(api.allGather))sym("ncclAllGather");
    api.errStr = (decltype(api.errStr))sym("ncclGetErrorString");
    api.ok = ok;
    api.commCount = (decltype(api.commCount))dlsym(h, "ncclCommCount");
    if (!ok) api.err = "libnccl.so.2 lacks a required symbol";
    return api;
}

orca_status nccl_fail(ncclResult_t r, const char* what) {
    NcclApi& N = nccl();
    return fail(ORCA_ERR_NCCL, std::string(what) + ": " + (N.errStr ? N.errStr(r) : "?"));
}

// ------------------------------------------------------------- exchange buffers
struct ExAlloc {
    void* base = nullptr;
    size_t bytes = 0;
    ExBuf b{};
};

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

orca_status ex_alloc(ExAlloc& x, int capM, int capH) {
    if (x.base && x.b.capM == capM && x.b.capH == capH) return ORCA_OK;  // layouts must match exactly
    dfree(x.base);
    size_t sz[11] = {16, (size_t)capM * 8, (size_t)capM * 8, (size_t)capM * 8, (size_t)capM * 4,
                     (size_t)capM * 4, (size_t)capH * 8, (size_t)capH * 8, (size_t)capH * 4,
                     (size_t)capM * 16, (size_t)capH * 4};
    size_t off[11], o = 0;
    for (int q = 0; q < 11; ++q) {
        off[q] = o;
        o = align16(o + sz[q]);
    }
    x.bytes = o;
    CK(cudaMalloc(&x.base, x.bytes));
    CK(cudaMemset(x.base, 0, x.bytes));
    char* p = (char*)x.base;
    x.b.hdr = (int*)(p + off[0]);
    x.b.mpos = (float2*)(p + off[1]);
    x.b.mvel = (float2*)(p + off[2]);
    x.b.maux = (float2*)(p + off[3]);
    x.b.mid = (uint32_t*)(p + off[4]);
    x.b.mrk2 = (float*)(p + off[5]);
    x.b.hpos = (float2*)(p + off[6]);
    x.b.hvel = (float2*)(p + off[7]);
    x.b.hid = (uint32_t*)(p + off[8]);
    x.b.mprop = (float4*)(p + off[9]);
    x.b.hrad = (float*)(p + off[10]);
    x.b.capM = capM;
    x.b.capH = capH;
    return ORCA_OK;
}

// --------------------------------------------------------------------- a strip
struct Domain {
    int strip = 0;  // strip index in [0, world)
    Grid g{};
    int64_t nbins = 0, binCap = 0;
    int capW = 0;
    int64_t popBuild = 0;  // agents of the strip when it was (re)built (auto kernel choice)
    float2 *posS = nullptr, *velS = nullptr, *auxS = nullptr, *posW = nullptr, *velW = nullptr, *auxW = nullptr;
    float *rk2S = nullptr, *rk2W = nullptr;
    float4 *propS = nullptr, *propW = nullptr;  // heterogeneous crowds only
    int propCap = 0;
    uint32_t *idS = nullptr, *idW = nullptr, *cellW = nullptr, *rankW = nullptr;
    uint32_t *count = nullptr, *binStart = nullptr;
    unsigned long long* scanStatus = nullptr;  // look-back status + ticket + LP3 queue count
    uint32_t* binPartial = nullptr;            // k_bin's per-block chunk totals (kBinMaxGrid)
    int4* qEntry = nullptr;
    float4* qLines = nullptr;
    int* ctr = nullptr;
    unsigned long long* stats = nullptr;
    ExAlloc sendL, sendR, recvL, recvR;
    // peer-memory transport: receive buffers of odd steps, the neighbours' receive buffers
    // as seen from here ([parity]), cudaIpc mappings to close, k_push completion counters
    ExAlloc recvL1, recvR1;
    ExBuf peerL[2] = {}, peerR[2] = {};
    void* ipcOpen[4] = {};
    unsigned int* pushDone = nullptr;

    void close_ipc() {
        for (void*& p : ipcOpen)
            if (p) {
                cudaIpcCloseMemHandle(p);
                p = nullptr;
            }
    }

    void release() {
        close_ipc();
        dfree(pushDone);
        for (ExAlloc* x : {&recvL1, &recvR1}) dfree(x->base);
        float2** f2[] = {&posS, &velS, &auxS, &posW, &velW, &auxW};
        uint32_t** u4[] = {&idS, &idW, &cellW, &rankW, &count, &binStart};
        for (auto p : f2) dfree(*p);
        for (auto p : u4) dfree(*p);
        dfree(rk2S);
        dfree(rk2W);
        dfree(propS);
        dfree(propW);
        dfree(scanStatus);
        dfree(binPartial);
        dfree(qEntry);
        dfree(qLines);
        dfree(ctr);
        dfree(stats);
        for (ExAlloc* x : {&sendL, &sendR, &recvL, &recvR}) dfree(x->base);
    }
};

}  // namespace

struct orca_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // strips' halo overlap (orca_set_overlap): the exchange and k_receive run on `side` while
    // the interior columns step on `stream` (fork / join by events, inside the step graphs)
    cudaStream_t side = nullptr;
    cudaEvent_t evFork = nullptr, evJoin = nullptr;
    int overlapMode = -1;  // -1 auto (on for strips), 0 off, 1 on
    // orca_step_io_async left its step's binning undone: the work arrays hold the state, the
    // sorted arrays are stale; flush_deferred() sorts them before anything else reads them
    bool deferred = false;
    // loopback strips: one stream per strip (fork / join by events), so the strips' kernels
    // run concurrently like ranks on their own GPUs (peer-memory transport only)
    std::vector<cudaStream_t> stripStream;
    std::vector<cudaEvent_t> stripDone;
    orca_params p{};
    bool ready = false, goals = false;
    float prefSpeed = 0.0f;
    float removeR = 0.0f;  // > 0: agents within removeR of their goal leave
    bool het = false;      // per-agent radius / maxSpeed / prefSpeed set
    float maxSpeedAll = 0.0f;
    float4* props4 = nullptr;  // id-ordered staging of the per-agent properties
    int64_t props4Cap = 0;
    // orca_step_trace: copy stream + double-buffered id-ordered frames (pos, vel) x 2
    cudaStream_t copyStream = nullptr;
    cudaEvent_t frameReady[2] = {}, frameFree[2] = {};
    float2* traceBuf[4] = {};
    int64_t traceCap = 0;
    int world = 1;  // strips in the whole decomposition
    int rank = 0;   // NCCL rank (= the strip held by this context)
    bool loopback = false;
    ncclComm_t comm = nullptr;
    std::vector<Domain> doms;
    Grid gg{};  // global grid
    int64_t nGlobal = 0;
    int64_t stageCap = 0;
    float2* stage = nullptr;                  // global inputs (pos | vel | aux), 3 x nGlobal
    float2 *outA = nullptr, *outB = nullptr;  // id-ordered outputs
    float* partial = nullptr;
    int32_t* colHist = nullptr;
    int colCap = 0;
    int64_t host_steps = 0, host_updates = 0;
    int64_t steps_total = 0;  // steps since creation (never reset): the LP-order step index
    std::vector<std::pair<int, cudaGraphExec_t>> graphs;
    std::vector<int64_t> graphGen;        // keyGen each cached graph was captured under
    std::vector<unsigned char> graphKey;  // graph_key() of the current generation
    int64_t keyGen = 0;
    cudaEvent_t ev[8] = {};
    cudaEvent_t chunkEv[2] = {};  // after the last two step chunks (orca_step's grid check)
    int smemBytes = 0, lp3Smem = 0, groupSmem = 0;
    int lpMode = 0;  // LP constraint order (orca_set_lp_order): 0 greedy, 1 randomized, 2 neighbour order
    unsigned long long lpSeed = 0;
    int64_t lpStep0 = 0, lpMark = 0;  // step index t = lpStep0 + steps_total - lpMark
    int variant = -1;  // -1: auto (pick_variant)
    int lp3Lanes = -1;  // lanes per queued agent in the LP3 kernel (1 = thread, -1 = auto)
    int lp3InlineMode = -1;  // orca_set_lp3_inline: -1 auto (strips up to inlineBelow agents), 0 queue, 1 inline
    int64_t inlineBelow = 0;  // one wave of k_step blocks with the inline-LP3 shared memory (orca_create)
    int64_t pairBelow = 0;    // one wave of the lane-pair k_step (variant 4) blocks (orca_create)
    int64_t bq3Below = 0;     // one wave of the 3-blocks/SM block-queue k_step (orca_create)
    int64_t pairMBBelow = 0;  // one wave of the lane-pair k_step with the ORCA_PAIR_MB register budget
    int binGrid = 0;          // k_bin blocks that are co-resident (cooperative launch limit)
    // strip rebalance: by-id active flags, all-gather records, fill reports
    uint8_t* activeBuf = nullptr;
    int64_t activeCap = 0;
    float4* gatherBuf = nullptr;
    size_t gatherCap = 0;  // float4 entries
    int* report = nullptr;
    int reportCap = 0;
    int64_t rebalances = 0;
    int transport = 0;  // 0: peer memory (k_push / cudaIpc), 1: NCCL send/recv (loopback: copies);
                        // orca_create_dist defaults to 1, loopback strips to 0
    int commRanks = 1;  // ranks in the NCCL communicator (ncclCommCount; -1 unknown)
    // set (host-mapped, no synchronisation) when an agent enters the grid's outer cell ring:
    // the grid is re-derived before the next chunk of steps (reading Q12)
    int* gridFlagHost = nullptr;
    int* gridFlagDev = nullptr;
    int64_t regrids = 0;
    unsigned char* ipcStage = nullptr;  // device staging of the cudaIpc handles for the all-gather
    // asynchronous per-step I/O (orca_set_state_async / orca_get_state_async / orca_io_wait):
    // uploads on ioIn and read-backs on ioOut overlap the steps on `stream`; two slots each
    cudaStream_t ioIn = nullptr, ioOut = nullptr;
    cudaEvent_t inReady[2] = {}, inFree[2] = {}, outReady[2] = {}, outFree[2] = {};
    float2* inBuf[2] = {};   // pos | vel by id, 2 x nGlobal
    float2* outBuf[2] = {};  // pos | vel by id, 2 x nGlobal
    int64_t ioCap = 0;
    int inSlot = 0, outSlot = 0;
    int* ioBadHost = nullptr;  // host-mapped: a non-finite value in an asynchronous upload
    int* ioBadDev = nullptr;
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
    m.removeR2 = (c->goals && c->removeR > 0.0f) ? c->removeR * c->removeR : 0.0f;
    m.maxSpeedAll = c->het ? std::max(c->maxSpeedAll, p.maxSpeed) : p.maxSpeed;
    m.lpRandom = c->lpMode == 1 ? 1 : 0;
    m.lpGreedy = c->lpMode == 0 ? 1 : 0;
    m.lpSeed = c->lpSeed;
    return m;
}

int pick_lp3_mode(const orca_ctx* c, const Domain& d);

StepArgs make_args(orca_ctx* c, Domain& d) {
    StepArgs a{};
    a.g = d.g;
    a.m = make_model(c);
    a.posS = d.posS;
    a.velS = d.velS;
    a.auxS = d.auxS;
    a.rk2S = d.rk2S;
    a.idS = d.idS;
    a.binStart = d.binStart;
    a.posW = d.posW;
    a.velW = d.velW;
    a.auxW = d.auxW;
    a.rk2W = d.rk2W;
    a.propS = c->het ? d.propS : nullptr;
    a.propW = c->het ? d.propW : nullptr;
    a.idW = d.idW;
    a.cellW = d.cellW;
    a.rankW = d.rankW;
    a.count = d.count;
    a.stats = d.stats;
    a.ctr = d.ctr;
    a.capW = d.capW;
    a.sendL = d.sendL.b;
    a.sendR = d.sendR.b;
    a.qEntry = d.qEntry;
    a.qLines = d.qLines;
    a.qcap = d.capW;
    a.lp3Inline = pick_lp3_mode(c, d);
    a.gridFlag = c->gridFlagDev;
    a.qCount = reinterpret_cast<unsigned int*>(d.scanStatus + scan_tiles(d.nbins) + 1);
    return a;
}

orca_status dom_alloc(orca_ctx* c, Domain& d, int capW, int64_t nbins, int capM, int capH) {
    if (capW > d.capW) {
        float2** f2[] = {&d.posS, &d.velS, &d.auxS, &d.posW, &d.velW, &d.auxW};
        uint32_t** u4[] = {&d.idS, &d.idW, &d.cellW, &d.rankW};
        for (auto p : f2) {  // (+2 spare entries: the staged copies round runs up to 16 bytes)
            dfree(*p);
            CK(cudaMalloc(p, (size_t)(capW + 2) * sizeof(float2)));
        }
        for (auto p : u4) {
            dfree(*p);
            CK(cudaMalloc(p, (size_t)capW * sizeof(uint32_t)));
        }
        dfree(d.rk2S);
        dfree(d.rk2W);
        dfree(d.qEntry);
        dfree(d.qLines);
        CK(cudaMalloc(&d.rk2S, (size_t)capW * sizeof(float)));
        CK(cudaMalloc(&d.rk2W, (size_t)capW * sizeof(float)));
        CK(cudaMalloc(&d.qEntry, (size_t)capW * sizeof(int4)));
        CK(cudaMalloc(&d.qLines, (size_t)capW * std::max(1, c->p.maxNeighbors) * sizeof(float4)));
        d.capW = capW;
    }
    if (nbins > d.binCap) {
        dfree(d.count);
        dfree(d.binStart);
        dfree(d.scanStatus);
        CK(cudaMalloc(&d.count, (nbins + 4) * sizeof(uint32_t)));
        CK(cudaMalloc(&d.binStart, (nbins + 1) * sizeof(uint32_t)));
        CK(cudaMalloc(&d.scanStatus, (scan_tiles(nbins) + 2) * sizeof(unsigned long long)));
        if (!d.binPartial) CK(cudaMalloc(&d.binPartial, kBinMaxGrid * sizeof(uint32_t)));
        d.binCap = nbins;
    }
    if (!d.ctr) {
        CK(cudaMalloc(&d.ctr, CT_COUNT * sizeof(int)));
        CK(cudaMemset(d.ctr, 0, CT_COUNT * sizeof(int)));
        CK(cudaMalloc(&d.stats, ST_COUNT * sizeof(unsigned long long)));
        CK(cudaMemset(d.stats, 0, ST_COUNT * sizeof(unsigned long long)));
    }
    if (d.g.hasL) {
        CKS(ex_alloc(d.sendL, capM, capH));
        CKS(ex_alloc(d.recvL, capM, capH));
        CKS(ex_alloc(d.recvL1, capM, capH));
    }
    if (d.g.hasR) {
        CKS(ex_alloc(d.sendR, capM, capH));
        CKS(ex_alloc(d.recvR, capM, capH));
        CKS(ex_alloc(d.recvR1, capM, capH));
    }
    if (!d.pushDone) {
        CK(cudaMalloc(&d.pushDone, 2 * sizeof(unsigned int)));
        CK(cudaMemset(d.pushDone, 0, 2 * sizeof(unsigned int)));
    }
    // arrival flags restart with the exchange sequence number (CT_XSTEP = 0); send buffers empty
    for (ExAlloc* x : {&d.recvL, &d.recvL1, &d.recvR, &d.recvR1, &d.sendL, &d.sendR})
        if (x->base) CK(cudaMemsetAsync(x->b.hdr, 0, 16, c->stream));
    return ORCA_OK;
}

void drop_graph(orca_ctx* c) {
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.second);
    c->graphs.clear();
    c->graphGen.clear();
    c->graphKey.clear();
}

// auto (-1): while a strip fits one wave of the lane-pair kernel (variant 4: 64 agents per
// block; blocks/SM from the occupancy API x SMs, orca_create) the step is latency bound and
// halving each warp's dependency chain wins; above, one thread per agent (variant 0).
// Measured r02m (whole-step ms, v0 / v1 / v4, block-queue LP3 for v0 and v4): 5k 0.047 /
// 0.047 / 0.041, 10k 0.049 / 0.049 / 0.043, 20k 0.049 / 0.064 / 0.043, 50k 0.055 / 0.095 /
// 0.049, 70k 0.057 / 0.117 / 0.051; 100k v0 0.063 / v4 0.076 (two waves).  The 8-lane group
// (variant 1, r01x's choice below 17k) no longer wins anywhere: explicit only.
#ifndef ORCA_AUTO_GROUP_BELOW
#define ORCA_AUTO_GROUP_BELOW 0
#endif
// variant 4 (two lanes per agent) needs k <= 14 (the merged list in one buffer column) and
// the greedy LP order; elsewhere it runs as variant 0
bool pair_ok(const orca_ctx* c) { return c->p.maxNeighbors <= 14 && c->lpMode == 0; }
int pick_variant(const orca_ctx* c, const Domain& d) {
    int v = c->variant;
    if (v < 0) v = (d.popBuild < ORCA_AUTO_GROUP_BELOW) ? 1 : (d.popBuild <= c->pairBelow) ? 4 : 0;
    if (v == 4 && !pair_ok(c)) v = 0;
    return v;
}

// LP3 lanes, auto (-1): an 8-lane group per queued agent below ORCA_AUTO_LP3_GROUP_BELOW
// agents per strip, one thread per agent above.  With the sequential LP3 the groups won below
// ~250k (100k -3.5 %, r01af); with the greedy LP3 one thread per agent wins at every size
// (100k -10 %, corridor -3 %, r01ap), so the threshold is 0
#ifndef ORCA_AUTO_LP3_GROUP_BELOW
#define ORCA_AUTO_LP3_GROUP_BELOW 0
#endif
int pick_lp3_lanes(const orca_ctx* c, const Domain& d) {
    if (c->lp3Lanes > 0) return c->lp3Lanes;
    return (d.popBuild < ORCA_AUTO_LP3_GROUP_BELOW) ? 8 : 1;
}

// LP3 inside k_step (StepArgs::lp3Inline) for small strips on the thread-per-agent kernels
// (DESIGN.md §12): there the step is latency bound and the separate k_lp3 launch is a serial
// tail; the group kernel always queues.
#ifndef ORCA_AUTO_LP3_INLINE_BELOW
#define ORCA_AUTO_LP3_INLINE_BELOW 1000000000  // cap on top of the measured rule below (no cap)
// The rule (r02h): LP3 on the block-local queue inside k_step (mode 2) while the strip fits ONE
// wave of k_step blocks at the occupancy its shared memory allows (cudaOccupancyMax-
// ActiveBlocksPerMultiprocessor x SMs x block size, computed in orca_create for the context's
// k; 8 blocks/SM -> 151,552 agents at k = 10), else the k_lp3 kernel (mode 0).  Measured at
// k = 10 (scripts/lp3_modes_probe.py, ms/step for modes 0 / 1 / 2): 100k 0.0676 / 0.0778 /
// 0.0595, dense 500k 0.193 / 0.231 / 0.203, 1M 0.309 / 0.410 / 0.338 -- beyond one wave the
// block barrier leaves one busy warp per block during its LP3 phase, while k_lp3 runs full warps.
#endif
// 0: queued for k_lp3, 1: inside k_step per thread, 2: inside k_step on the block's
// compacted queue (orca_set_lp3_inline)
bool overlap_on(const orca_ctx* c, const Domain& d);
bool strip_streams_on(const orca_ctx* c);
int pick_lp3_mode(const orca_ctx* c, const Domain& d) {
    const int v = pick_variant(c, d);
    if (v == 1) return 0;  // the group kernel always queues
    if (overlap_on(c, d)) return 2;  // the boundary agents' LP3 must finish inside their launch
    if (c->lp3InlineMode >= 0) return (v == 4 && c->lp3InlineMode == 1) ? 2 : c->lp3InlineMode;
    // loopback strips on their own streams share ONE GPU: the wave rule applies to the whole crowd
    const int64_t pop = strip_streams_on(c) ? c->nGlobal : d.popBuild;
    return pop <= std::min<int64_t>(c->inlineBelow, ORCA_AUTO_LP3_INLINE_BELOW) ? 2 : 0;
}
bool pick_lp3_inline(const orca_ctx* c, const Domain& d) { return pick_lp3_mode(c, d) != 0; }

// Halo overlap: the strip's boundary columns (two on each side: every agent
// that can end the step in an edge column or leave the strip, since maxSpeed dt < one
// column) step first, then their exchange and k_receive run on the side stream while the
// interior columns step.  Needs >= 4 owned columns and the thread-per-agent kernels.
bool strip_streams_on(const orca_ctx* c);
bool overlap_on(const orca_ctx* c, const Domain& d) {
    if (c->world == 1 || c->overlapMode == 0 || !(d.g.hasL || d.g.hasR)) return false;
    if (pick_variant(c, d) == 1 || d.g.c1 - d.g.c0 < 4) return false;
    if (strip_streams_on(c)) return false;  // loopback strips already overlap on their own streams
    // automatic: only where LP3 runs inside k_step anyway (a strip within one wave of blocks);
    // a bigger strip's k_lp3 placement is faster, and its exchange a small part of its step
    if (c->overlapMode < 0 && d.popBuild > std::min<int64_t>(c->inlineBelow, ORCA_AUTO_LP3_INLINE_BELOW)) return false;
    return true;
}

// Everything a captured step body depends on: the kernel arguments of every strip (device
// pointers, grid, model), launch sizes, the exchange buffers and the kernel selection.  A
// cached graph is replayed only while this is unchanged, so orca_set_agents with the same
// layout (e.g. reloading a checkpoint every step) keeps the graphs.
std::vector<unsigned char> graph_key(orca_ctx* c) {
    std::vector<unsigned char> k;
    auto put = [&k](const void* p, size_t n) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        k.insert(k.end(), b, b + n);
    };
    const int hdr[9] = {c->variant, c->lp3Lanes, c->smemBytes, c->world, c->loopback ? 1 : 0, (int)c->doms.size(),
                        c->transport, c->overlapMode, strip_streams_on(c) ? 1 : 0};
    put(hdr, sizeof hdr);
    for (Domain& d : c->doms) {
        const StepArgs a = make_args(c, d);
        put(&a, sizeof a);
        put(&d.capW, sizeof d.capW);
        put(&d.nbins, sizeof d.nbins);
        const int v = pick_variant(c, d);
        put(&v, sizeof v);
        const int l3 = pick_lp3_lanes(c, d);
        put(&l3, sizeof l3);
        for (const ExAlloc* x : {&d.sendL, &d.sendR, &d.recvL, &d.recvR, &d.recvL1, &d.recvR1}) {
            put(&x->base, sizeof x->base);
            put(&x->bytes, sizeof x->bytes);
        }
        put(d.peerL, sizeof d.peerL);
        put(d.peerR, sizeof d.peerR);
    }
    return k;
}

// Launch of a step-chain kernel with the programmatic-dependent-launch attribute (one strip:
// the chain is k_step -> k_lp3 -> k_scan -> k_scatter -> next k_step, every kernel opens with
// pdl_entry()), so each kernel's launch overlaps its predecessor's tail.  Strips keep plain
// launches (exchange kernels and NCCL calls sit in the chain).  Errors surface through
// cudaGetLastError at the call sites.
template <typename... KArgs, typename... Args>
void launch_k(orca_ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (ORCA_PDL && c->world == 1) ? 1 : 0;
    (void)cudaLaunchKernelEx(&cfg, kern, args...);
}

// LP3 on the queue (same results bit for bit): a GW-lane group per agent on a persistent
// grid (pick_lp3_lanes > 1), else one thread per agent on a capacity grid
template <bool DRY, int GW>
void launch_lp3_grp(orca_ctx* c, Domain& d, StepArgs& a) {
    constexpr int ppb = kStepThreads / GW;
    const int blocks = (int)std::min<int64_t>((d.capW + ppb - 1) / ppb, 148 * 16);
    launch_k(c, k_lp3_grp<DRY, GW>, dim3(std::max(blocks, 1)), dim3(kStepThreads),
             (size_t)lp3_grp_words(c->p.maxNeighbors) * 4 * ppb, a);
}

template <bool DRY>
void launch_lp3(orca_ctx* c, Domain& d, StepArgs& a) {
    if (a.lp3Inline) return;  // k_step finished its infeasible agents
    switch (pick_lp3_lanes(c, d)) {
        case 4: launch_lp3_grp<DRY, 4>(c, d, a); break;
        case 8: launch_lp3_grp<DRY, 8>(c, d, a); break;
        case 16: launch_lp3_grp<DRY, 16>(c, d, a); break;
        default:
            if (!a.g.hasL && !a.g.hasR && !a.propS)  // one strip of homogeneous agents
                launch_k(c, k_lp3<DRY, true>, dim3(lp3_blocks(d.capW)), dim3(kStepThreads), (size_t)c->lp3Smem, a);
            else
                launch_k(c, k_lp3<DRY>, dim3(lp3_blocks(d.capW)), dim3(kStepThreads), (size_t)c->lp3Smem, a);
    }
}

// The k_step instantiation a strip runs (one source of truth for launch_step and
// orca_get_kernel_config): the default configurations -- greedy LP order, LP3 in k_lp3 (LM 0) or
// on the block queue (LM 2), one strip of homogeneous agents (mono) -- run kernels compiled for
// exactly that case, with their block size and register budget (min blocks per SM) chosen by the
// strip's size (DESIGN.md §10, §12 r02ai-au); everything else runs the general instantiation.
struct StepKernelCfg {
    int variant;  // 0 thread per agent (shared-memory list), 1 8-lane group, 2 register list, 3 work units, 4 lane pair
    int lm;       // -1 general; 0 / 2: compiled for that LP3 placement and the greedy order
    int mono;     // compiled for one strip of homogeneous agents
    int threads;  // threads per block
    int mb;       // min blocks per SM of the register budget (0: 1024 threads per SM)
};
StepKernelCfg step_kernel_cfg(const orca_ctx* c, const Domain& d, const StepArgs& a) {
    const int k = c->p.maxNeighbors;
    const int v = pick_variant(c, d);
    const bool spec = a.m.lpGreedy && !a.m.lpRandom;
    const int mono = (!a.g.hasL && !a.g.hasR && !a.propS) ? 1 : 0;
    if (v == 1) return {1, -1, 0, kGroupThreads, 0};
    if (v == 3) return {3, -1, 0, kStepThreads, 0};
    if (v == 4) {
        if (spec && a.lp3Inline == 2) return {4, 2, mono, kStepThreads, d.popBuild <= c->pairMBBelow ? ORCA_PAIR_MB : 0};
        return {4, -1, 0, kStepThreads, 0};
    }
    const bool shared = v != 2 || k < 1 || k > 16;
    if (shared && spec && a.lp3Inline == 0) return {0, 0, mono, kStepThreads, ORCA_LM0_MB};
    if (shared && spec && a.lp3Inline == 2) return {0, 2, mono, kStepBQ, d.popBuild <= c->bq3Below ? 3 : 0};
    return {shared ? 0 : 2, -1, 0, kStepThreads, 0};
}

// fused step kernel of the selected configuration (same results bit for bit)
template <bool DRY>
void launch_step(orca_ctx* c, Domain& d, StepArgs& a) {
    const int blocks = (d.capW + kStepThreads - 1) / kStepThreads;
    const int k = c->p.maxNeighbors;
    const StepKernelCfg kc = step_kernel_cfg(c, d, a);
    // per-thread inline LP3 (mode 1) needs the projected half-planes: 3k more words per thread
    // after the columns; the block queue (mode 2) only its small scratch area
    const size_t smem = (size_t)c->smemBytes +
                        (a.lp3Inline == 1   ? (size_t)3 * k * 4 * kStepThreads
                         : a.lp3Inline == 2 ? (size_t)step_lp3q_scratch_bytes(k)
                                            : 0);
    const bool mono = kc.mono != 0;
    if (kc.variant == 1)  // 8-lane group per agent
        launch_k(c, k_step_group<DRY>, dim3((d.capW + kGroupAgents - 1) / kGroupAgents), dim3(kGroupThreads),
                 (size_t)c->groupSmem, a);
    else if (kc.variant == 3)  // work-unit LP2 (P:84-89 ablation)
        launch_k(c, k_step<DRY, 0, true>, dim3(blocks), dim3(kStepThreads), smem, a);
    else if (kc.variant == 4 && kc.lm == 2)  // two lanes per agent, specialised (LM = 2)
        launch_k(c,
                 kc.mb == ORCA_PAIR_MB && kc.mb > 0
                     ? (mono ? k_step<DRY, 0, false, true, 2, true, kStepThreads, ORCA_PAIR_MB>
                             : k_step<DRY, 0, false, true, 2, false, kStepThreads, ORCA_PAIR_MB>)
                     : (mono ? k_step<DRY, 0, false, true, 2, true> : k_step<DRY, 0, false, true, 2, false>),
                 dim3((d.capW + kStepThreads / 2 - 1) / (kStepThreads / 2)), dim3(kStepThreads), smem, a);
    else if (kc.variant == 4)  // two lanes per agent: 64 agents per block
        launch_k(c, k_step<DRY, 0, false, true>, dim3((d.capW + kStepThreads / 2 - 1) / (kStepThreads / 2)),
                 dim3(kStepThreads), smem, a);
    else if (kc.lm == 0)  // specialised: LM = 0
        launch_k(c, mono ? k_step<DRY, 0, false, false, 0, true, kStepThreads, ORCA_LM0_MB>
                         : k_step<DRY, 0, false, false, 0, false, kStepThreads, ORCA_LM0_MB>,
                 dim3(blocks), dim3(kStepThreads), smem, a);
    else if (kc.lm == 2)  // specialised: LM = 2, 256 threads
        launch_k(c,
                 kc.mb == 3
                     ? (mono ? k_step<DRY, 0, false, false, 2, true, kStepBQ, 3> : k_step<DRY, 0, false, false, 2, false, kStepBQ, 3>)
                     : (mono ? k_step<DRY, 0, false, false, 2, true, kStepBQ> : k_step<DRY, 0, false, false, 2, false, kStepBQ>),
                 dim3((d.capW + kStepBQ - 1) / kStepBQ), dim3(kStepBQ),
                 (size_t)step_smem_per_thread(k) * kStepBQ + (size_t)step_lp3q_scratch_bytes(k), a);
    else if (kc.variant == 0)  // shared-memory top-k list (any k)
        launch_k(c, k_step<DRY, 0, false>, dim3(blocks), dim3(kStepThreads), smem, a);
    else if (k <= 10)  // register top-k list
        launch_k(c, k_step<DRY, 10, false>, dim3(blocks), dim3(kStepThreads), smem, a);
    else
        launch_k(c, k_step<DRY, 16, false>, dim3(blocks), dim3(kStepThreads), smem, a);
}

// zero: clear the status words, tile ticket and LP3 queue count first (at set-up); in the
// step body the previous step's k_scatter has already cleared them
cudaError_t enqueue_scan(orca_ctx* c, Domain& d, bool zero) {
    const int tiles = scan_tiles(d.nbins);
    if (zero) {
        cudaError_t e = cudaMemsetAsync(d.scanStatus, 0, (tiles + 2) * sizeof(unsigned long long), c->stream);
        if (e != cudaSuccess) return e;
    }
    launch_k(c, k_scan, dim3(tiles), dim3(kScanThreads), 0, d.count, d.binStart, (int)d.nbins, d.scanStatus,
             reinterpret_cast<unsigned int*>(d.scanStatus + tiles));
    return cudaGetLastError();
}

// props: move the per-agent properties too (false right after k_select, which does not
// write them: refresh_props then gathers them by id into the new sorted order)
cudaError_t enqueue_scatter(orca_ctx* c, Domain& d, int bump, bool props = true) {
    launch_k(c, k_scatter, dim3(cap_blocks(d.capW, 256)), dim3(256), 0, d.ctr, bump, d.cellW, d.rankW, d.binStart,
             d.posW, d.velW, d.auxW, d.idW, d.rk2W, d.posS, d.velS, d.auxS, d.idS, d.rk2S, d.capW,
             (c->het && props) ? d.propW : nullptr, (c->het && props) ? d.propS : nullptr, d.scanStatus,
             scan_tiles(d.nbins) + 2);
    return cudaGetLastError();
}

// Scan + scatter of one strip as ONE cooperative launch (k_bin); the grid is at most one
// resident wave, sized to the work (~1024 bins or agents per block).  Same result as
// enqueue_scan + enqueue_scatter.
cudaError_t enqueue_bin(orca_ctx* c, Domain& d, int bump) {
    const int64_t work = std::max<int64_t>(d.capW, d.nbins);
    const int G = (int)std::max<int64_t>(1, std::min<int64_t>(c->binGrid, (work + 4 * kBinThreads - 1) / (4 * kBinThreads)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kBinThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_bin, d.ctr, bump, d.count, d.binStart, (int)d.nbins, d.binPartial, d.cellW,
                              d.rankW, d.posW, d.velW, d.auxW, d.idW, d.rk2W, d.posS, d.velS, d.auxS, d.idS, d.rk2S,
                              d.capW, c->het ? d.propW : nullptr, c->het ? d.propS : nullptr, d.scanStatus,
                              scan_tiles(d.nbins) + 2);
}
bool fused_bin(const orca_ctx* c) { return ORCA_FUSED_BIN && c->doms.size() == 1 && c->binGrid > 0; }

// Neighbour exchange of one step: every strip sends its L/R buffers and receives its
// neighbours'.  Loopback: device copies between the strips of this context.  NCCL: one
// group of send/recv with ranks +-1.
// The binning orca_step_io_async skipped: scan + scatter of the work arrays the last step wrote
// (bump: that step is complete).  No-op unless deferred.
cudaError_t flush_deferred(orca_ctx* c) {
    if (!c->deferred) return cudaSuccess;
    c->deferred = false;
    for (Domain& d : c->doms) {
        cudaError_t e = fused_bin(c) ? enqueue_bin(c, d, 1) : enqueue_scan(c, d, false);
        if (e == cudaSuccess && !fused_bin(c)) e = enqueue_scatter(c, d, 1);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

orca_status enqueue_exchange(orca_ctx* c, cudaStream_t st) {
    if (c->world == 1) return ORCA_OK;
    if (c->transport == 0) {  // peer memory: exact-size remote stores + arrival flags
        for (Domain& d : c->doms) {
            if (d.g.hasL)
                k_push<<<kPushBlocks, 256, 0, st>>>(d.sendL.b, d.peerL[0], d.peerL[1], d.ctr, d.pushDone);
            if (d.g.hasR)
                k_push<<<kPushBlocks, 256, 0, st>>>(d.sendR.b, d.peerR[0], d.peerR[1], d.ctr, d.pushDone + 1);
        }
        CK(cudaGetLastError());
        return ORCA_OK;
    }
    if (c->loopback) {
        const int P = (int)c->doms.size();
        for (int s = 0; s < P; ++s) {
            Domain& d = c->doms[s];
            if (d.g.hasR)
                CK(cudaMemcpyAsync(c->doms[s + 1].recvL.base, d.sendR.base, d.sendR.bytes, cudaMemcpyDeviceToDevice,
                                   st));
            if (d.g.hasL)
                CK(cudaMemcpyAsync(c->doms[s - 1].recvR.base, d.sendL.base, d.sendL.bytes, cudaMemcpyDeviceToDevice,
                                   st));
        }
        return ORCA_OK;
    }
    NcclApi& N = nccl();
    Domain& d = c->doms[0];
    ncclResult_t r = N.groupStart();
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    if (d.g.hasL) {
        r = N.send(d.sendL.base, d.sendL.bytes, ncclUint8, c->rank - 1, c->comm, st);
        if (r == ncclSuccess) r = N.recv(d.recvL.base, d.recvL.bytes, ncclUint8, c->rank - 1, c->comm, st);
    }
    if (r == ncclSuccess && d.g.hasR) {
        r = N.send(d.sendR.base, d.sendR.bytes, ncclUint8, c->rank + 1, c->comm, st);
        if (r == ncclSuccess) r = N.recv(d.recvR.base, d.recvR.bytes, ncclUint8, c->rank + 1, c->comm, st);
    }
    ncclResult_t r2 = N.groupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "ncclSend/ncclRecv");
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
    return ORCA_OK;
}

// One step body for every strip: reset per-step counters -> k_step (query, half-planes,
// LP2, integrate, route) -> k_lp3 (queued infeasible agents) -> exchange -> k_receive ->
// scan -> scatter.  ev (nullable): events around the stages for orca_step_timed.
void enqueue_receive(orca_ctx* c, cudaStream_t st) {
    for (Domain& d : c->doms) {
        if (d.g.hasL || d.g.hasR) {
            StepArgs a = make_args(c, d);
            const int capX = (d.g.hasL ? d.recvL.b.capM + d.recvL.b.capH : 0) +
                             (d.g.hasR ? d.recvR.b.capM + d.recvR.b.capH : 0);
            k_receive<<<cap_blocks(capX, 256), 256, 0, st>>>(a, d.recvL.b, d.recvL1.b, d.recvR.b, d.recvR1.b,
                                                             c->transport == 0 ? 1 : 0);
        }
    }
}

// Loopback strips with the peer-memory exchange on one stream per strip: each strip's whole step
// body (k_step, k_lp3, k_push into its neighbours' receive buffers, k_receive waiting on their
// arrival flags, scan, scatter) runs on its own stream, forked from and joined back into the
// context stream, so the strips overlap on the GPU as ranks do on their own GPUs.  The arrival
// flags and the step-parity receive buffers order the exchange across streams exactly as
// across ranks; results are the single-stream ones bit for bit.
bool strip_streams_on(const orca_ctx* c) {
    return c->loopback && c->transport == 0 && c->stripStream.size() == c->doms.size() && c->doms.size() > 1 &&
           !std::getenv("ORCA_ONE_STREAM");
}

orca_status enqueue_step_streams(orca_ctx* c) {
    cudaStream_t main = c->stream;
    CK(cudaEventRecord(c->evFork, main));
    orca_status st = ORCA_OK;
    for (size_t q = 0; q < c->doms.size() && st == ORCA_OK; ++q) {
        Domain& d = c->doms[q];
        cudaStream_t ss = c->stripStream[q];
        cudaError_t e = cudaStreamWaitEvent(ss, c->evFork, 0);
        if (e != cudaSuccess) {
            st = cuda_fail(e, "cudaStreamWaitEvent");
            break;
        }
        c->stream = ss;  // every enqueue below (launch_k, scan, scatter) goes to the strip's stream
        StepArgs a = make_args(c, d);
        launch_step<false>(c, d, a);
        launch_lp3<false>(c, d, a);
        if (d.g.hasL)
            k_push<<<kPushBlocks, 256, 0, ss>>>(d.sendL.b, d.peerL[0], d.peerL[1], d.ctr, d.pushDone);
        if (d.g.hasR)
            k_push<<<kPushBlocks, 256, 0, ss>>>(d.sendR.b, d.peerR[0], d.peerR[1], d.ctr, d.pushDone + 1);
        const int capX = (d.g.hasL ? d.recvL.b.capM + d.recvL.b.capH : 0) + (d.g.hasR ? d.recvR.b.capM + d.recvR.b.capH : 0);
        k_receive<<<cap_blocks(capX, 256), 256, 0, ss>>>(a, d.recvL.b, d.recvL1.b, d.recvR.b, d.recvR1.b, 1);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = enqueue_scan(c, d, false);
        if (e == cudaSuccess) e = enqueue_scatter(c, d, 1);
        if (e == cudaSuccess) e = cudaEventRecord(c->stripDone[q], ss);
        if (e != cudaSuccess) st = cuda_fail(e, "strip step");
    }
    c->stream = main;
    if (st != ORCA_OK) return st;
    for (size_t q = 0; q < c->doms.size(); ++q) CK(cudaStreamWaitEvent(main, c->stripDone[q], 0));
    return ORCA_OK;
}

orca_status enqueue_step(orca_ctx* c, cudaEvent_t* ev) {
    if (!ev && strip_streams_on(c)) return enqueue_step_streams(c);
    if (ev) CK(cudaEventRecord(ev[0], c->stream));
    bool anyOverlap = false;
    for (Domain& d : c->doms) {
        if (c->transport != 0) {  // (the peer-memory k_push empties the send buffers itself)
            if (d.g.hasL) CK(cudaMemsetAsync(d.sendL.b.hdr, 0, 16, c->stream));
            if (d.g.hasR) CK(cudaMemsetAsync(d.sendR.b.hdr, 0, 16, c->stream));
        }
        StepArgs a = make_args(c, d);
        if (overlap_on(c, d)) {  // the boundary columns first
            a.phase = 1;
            anyOverlap = true;
        }
        launch_step<false>(c, d, a);
        launch_lp3<false>(c, d, a);
    }
    CK(cudaGetLastError());
    if (ev) CK(cudaEventRecord(ev[1], c->stream));
    if (anyOverlap) {
        // fork: exchange + k_receive on the side stream, the interior columns here; join
        // before the binning of the next step
        CK(cudaEventRecord(c->evFork, c->stream));
        CK(cudaStreamWaitEvent(c->side, c->evFork, 0));
        CKS(enqueue_exchange(c, c->side));
        enqueue_receive(c, c->side);
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->evJoin, c->side));
        for (Domain& d : c->doms) {
            if (!overlap_on(c, d)) continue;
            StepArgs a = make_args(c, d);
            a.phase = 2;
            launch_step<false>(c, d, a);
        }
        CK(cudaGetLastError());
        CK(cudaStreamWaitEvent(c->stream, c->evJoin, 0));
    } else {
        CKS(enqueue_exchange(c, c->stream));
        enqueue_receive(c, c->stream);
        CK(cudaGetLastError());
    }
    if (ev) CK(cudaEventRecord(ev[2], c->stream));
    if (!ev && fused_bin(c)) {  // (orca_step_timed keeps the two kernels for its stage times)
        CK(enqueue_bin(c, c->doms[0], 1));
        return ORCA_OK;
    }
    for (Domain& d : c->doms) CK(enqueue_scan(c, d, false));
    if (ev) CK(cudaEventRecord(ev[3], c->stream));
    for (Domain& d : c->doms) CK(enqueue_scatter(c, d, 1));
    if (ev) CK(cudaEventRecord(ev[4], c->stream));
    return ORCA_OK;
}

// The dry (debug) step: same kernels, outputs by id, state untouched; the LP3 queue
// count is zeroed before and after so the next real step starts from an empty queue.
cudaError_t dry_step(orca_ctx* c, Domain& d, StepArgs& a) {
    cudaError_t e = cudaMemsetAsync(a.qCount, 0, sizeof(unsigned int), c->stream);
    if (e != cudaSuccess) return e;
    launch_step<true>(c, d, a);
    launch_lp3<true>(c, d, a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(a.qCount, 0, sizeof(unsigned int), c->stream);
}

orca_status check_overflow(orca_ctx* c) {
    int any = 0;
    for (Domain& d : c->doms) {
        if (!d.ctr) continue;
        int f = 0;
        CK(cudaMemcpyAsync(&f, d.ctr + CT_OVF, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        any |= f;
    }
    if (any & OVF_TIMEOUT)
        return fail(ORCA_ERR_INTERNAL, "strip exchange timed out waiting for a neighbour's step (every rank must "
                                       "call orca_step with the same counts)");
    if (any)
        return fail(ORCA_ERR_CAPACITY, std::string("strip buffer overflow (") + ((any & OVF_WORK) ? "work " : "") +
                                           ((any & OVF_MIG) ? "migrants " : "") + ((any & OVF_HALO) ? "halo" : "") +
                                           "); call orca_set_agents again to re-partition");
    return ORCA_OK;
}

// owned range [o0, o1) of a domain (host read; synchronises)
orca_status owned_range_host(orca_ctx* c, Domain& d, int* o0, int* o1) {
    const int64_t cb = d.g.colBins;
    uint32_t v[2];
    CK(cudaMemcpyAsync(&v[0], d.binStart + (d.g.c0 - d.g.e0) * cb, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&v[1], d.binStart + (d.g.c1 - d.g.e0) * cb, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *o0 = (int)v[0];
    *o1 = (int)v[1];
    return ORCA_OK;
}

orca_status ctx_init(const orca_params* params, int32_t device, orca_ctx** out, orca_ctx** cp) {
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
    *cp = c;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->evFork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->evJoin, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&c->partial, 1024 * 5 * sizeof(float));
    if (e == cudaSuccess) e = cudaHostAlloc(&c->gridFlagHost, sizeof(int), cudaHostAllocMapped);
    if (e == cudaSuccess) {
        *c->gridFlagHost = 0;
        e = cudaHostGetDevicePointer(&c->gridFlagDev, c->gridFlagHost, 0);
    }
    for (int q = 0; q < 8 && e == cudaSuccess; ++q) e = cudaEventCreate(&c->ev[q]);
    c->smemBytes = step_smem_per_thread(params->maxNeighbors) * kStepThreads;
    c->lp3Smem = std::max(1, 6 * params->maxNeighbors) * 4 * kStepThreads;
    const void* stepFns[] = {(const void*)k_step<false, 0>,  (const void*)k_step<true, 0>,
                             (const void*)k_step<false, 10>, (const void*)k_step<true, 10>,
                             (const void*)k_step<false, 16>, (const void*)k_step<true, 16>,
                             (const void*)k_step<false, 0, true>, (const void*)k_step<true, 0, true>,
                             (const void*)k_step<false, 0, false, true>, (const void*)k_step<true, 0, false, true>,
                             (const void*)k_step<false, 0, false, false, 0, false, kStepThreads, ORCA_LM0_MB>,
                             (const void*)k_step<true, 0, false, false, 0, false, kStepThreads, ORCA_LM0_MB>,
                             (const void*)k_step<false, 0, false, false, 0, true, kStepThreads, ORCA_LM0_MB>,
                             (const void*)k_step<true, 0, false, false, 0, true, kStepThreads, ORCA_LM0_MB>,
                             (const void*)k_step<false, 0, false, false, 2, false>,
                             (const void*)k_step<true, 0, false, false, 2, false>,
                             (const void*)k_step<false, 0, false, false, 2, true>,
                             (const void*)k_step<true, 0, false, false, 2, true>,
                             (const void*)k_step<false, 0, false, true, 2, false>,
                             (const void*)k_step<true, 0, false, true, 2, false>,
                             (const void*)k_step<false, 0, false, true, 2, true>,
                             (const void*)k_step<true, 0, false, true, 2, true>,
                             (const void*)k_step<false, 0, false, true, 2, false, kStepThreads, ORCA_PAIR_MB>,
                             (const void*)k_step<true, 0, false, true, 2, false, kStepThreads, ORCA_PAIR_MB>,
                             (const void*)k_step<false, 0, false, true, 2, true, kStepThreads, ORCA_PAIR_MB>,
                             (const void*)k_step<true, 0, false, true, 2, true, kStepThreads, ORCA_PAIR_MB>};
    const void* stepFnsBQ[] = {(const void*)k_step<false, 0, false, false, 2, false, kStepBQ>,
                               (const void*)k_step<true, 0, false, false, 2, false, kStepBQ>,
                               (const void*)k_step<false, 0, false, false, 2, true, kStepBQ>,
                               (const void*)k_step<true, 0, false, false, 2, true, kStepBQ>,
                               (const void*)k_step<false, 0, false, false, 2, false, kStepBQ, 3>,
                               (const void*)k_step<true, 0, false, false, 2, false, kStepBQ, 3>,
                               (const void*)k_step<false, 0, false, false, 2, true, kStepBQ, 3>,
                               (const void*)k_step<true, 0, false, false, 2, true, kStepBQ, 3>};
    const int stepSmemMax = c->smemBytes + 3 * std::max(params->maxNeighbors, 1) * 4 * kStepThreads;  // + inline LP3
    for (const void* f : stepFns)
        if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, stepSmemMax);
    const int stepSmemBQ = step_smem_per_thread(params->maxNeighbors) * kStepBQ + step_lp3q_scratch_bytes(params->maxNeighbors);
    for (const void* f : stepFnsBQ)
        if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, stepSmemBQ);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_lp3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->lp3Smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_lp3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->lp3Smem);
    for (const void* f : {(const void*)k_lp3<false, true>, (const void*)k_lp3<true, true>})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, c->lp3Smem);
    c->groupSmem = group_words(params->maxNeighbors) * 4 * kGroupAgents;
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_step_group<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->groupSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_step_group<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->groupSmem);
    if (e == cudaSuccess) {
        // inline-LP3 threshold: one wave of k_step blocks with the inline shared memory
        const int k = params->maxNeighbors;
        const size_t smemInl = (size_t)c->smemBytes + (size_t)step_lp3q_scratch_bytes(k);  // mode 2
        int blocks = 0, sms = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_step<false, 0, false>, kStepThreads, smemInl);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        c->inlineBelow = (int64_t)blocks * sms * kStepThreads;
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_step<false, 0, false, true>, kStepThreads, smemInl);
        c->pairBelow = (int64_t)blocks * sms * (kStepThreads / 2);
        // the 3-blocks/SM block-queue kernel (85 registers) while a strip fits one wave of it (r02ao)
        const size_t smemBQ = (size_t)step_smem_per_thread(k) * kStepBQ + (size_t)step_lp3q_scratch_bytes(k);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_step<false, 0, false, false, 2, true, kStepBQ, 3>,
                                                              kStepBQ, smemBQ);
        c->bq3Below = (int64_t)blocks * sms * kStepBQ;
        // the lane-pair kernel with a larger register budget while a strip fits one wave of it
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &blocks, k_step<false, 0, false, true, 2, true, kStepThreads, ORCA_PAIR_MB>, kStepThreads, smemInl);
        c->pairMBBelow = ORCA_PAIR_MB > 0 ? (int64_t)blocks * sms * (kStepThreads / 2) : 0;
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_bin, kBinThreads, 0);
        c->binGrid = std::min(kBinMaxGrid, blocks * sms);
    }
    if (e != cudaSuccess) return cuda_fail(e, "orca_create");
    return ORCA_OK;
}

// Copy a float[2n] user array (host or device) into a device float2 buffer.
cudaError_t copy_in(orca_ctx* c, float2* dst, const float* src, int64_t n) {
    if (n == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->stream);
}

// min/max of the staged positions + finiteness of the three staged arrays
orca_status stage_bounds(orca_ctx* c, const float2* a, const float2* b, const float2* q, int64_t n, float mn[2],
                         float mx[2], const uint8_t* active = nullptr) {
    const int blocks = std::min(1024, cap_blocks(n, 256));
    k_minmax<<<blocks, 256, 0, c->stream>>>((int)n, a, b, q, c->partial, active);
    CK(cudaGetLastError());
    std::vector<float> h((size_t)blocks * 5);
    CK(cudaMemcpyAsync(h.data(), c->partial, h.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    mn[0] = mn[1] = INFINITY;
    mx[0] = mx[1] = -INFINITY;
    double bad = 0;
    for (int k = 0; k < blocks; ++k) {
        mn[0] = std::min(mn[0], h[k * 5 + 0]);
        mn[1] = std::min(mn[1], h[k * 5 + 1]);
        mx[0] = std::max(mx[0], h[k * 5 + 2]);
        mx[1] = std::max(mx[1], h[k * 5 + 3]);
        bad += h[k * 5 + 4];
    }
    if (bad > 0) return fail(ORCA_ERR_INVALID_ARGUMENT, "NaN/Inf in the input arrays");
    return ORCA_OK;
}

// The frozen grid of reading Q12 from the bounding box [mn, mx] of the agents: origin =
// fl32(min - cs), dims = floor((max - origin) / cs) + 2 (one margin cell on each side).
orca_status derive_grid(orca_ctx* c, int64_t n, const float mn[2], const float mx[2], int margin = 1) {
    const float cs = c->p.neighborDist;
    Grid g{};
    g.cs = cs;
    g.lgS = kSubRowsLog2;
    g.lgC = kSubColsLog2;
    if (n == 0) {
        g.ox = g.oy = 0.0f;
        g.nx = g.ny = 1;
    } else {
        const float mc = cs * (float)margin;
        volatile float ox = mn[0] - mc, oy = mn[1] - mc;
        g.ox = ox;
        g.oy = oy;
        const double tx = std::floor(((double)mx[0] - (double)g.ox) / (double)cs) + margin + 1;
        const double ty = std::floor(((double)mx[1] - (double)g.oy) / (double)cs) + margin + 1;
        if (tx > 1e9 || ty > 1e9 || tx * ty * (double)(1 << (kSubRowsLog2 + kSubColsLog2)) > (double)(1 << 28))
            return fail(ORCA_ERR_CAPACITY, "grid would exceed 2^28 sort bins");
        g.nx = (int)tx;
        g.ny = (int)ty;
    }
    g.csD = (double)cs;
    g.invCs = 1.0 / (double)cs;
    g.csSub = (double)cs / (double)(1 << g.lgS);
    g.invCsSub = (double)(1 << g.lgS) / (double)cs;
    g.csSubX = (double)cs / (double)(1 << g.lgC);
    g.invCsSubX = (double)(1 << g.lgC) / (double)cs;
    g.colBins = (g.ny << g.lgS) << g.lgC;
    c->gg = g;
    return ORCA_OK;
}

// ExBuf of a neighbour's receive buffer mapped at `base`: same layout as the local
// template (exchange capacities are global, so every strip's buffers share one layout).
ExBuf rebase(const ExAlloc& tmpl, void* base) {
    ExBuf b = tmpl.b;
    const char* t = static_cast<const char*>(tmpl.base);
    char* n = static_cast<char*>(base);
    auto mv = [&](auto*& p) {
        using P = std::remove_reference_t<decltype(p)>;
        p = reinterpret_cast<P>(n + (reinterpret_cast<const char*>(p) - t));
    };
    mv(b.hdr);
    mv(b.mpos);
    mv(b.mvel);
    mv(b.maux);
    mv(b.mid);
    mv(b.mrk2);
    mv(b.hpos);
    mv(b.hvel);
    mv(b.hid);
    mv(b.mprop);
    mv(b.hrad);
    return b;
}

// Peer-memory transport: where every strip's k_push writes.  Loopback: the
// neighbour strip's receive buffers.  Ranks: cudaIpc handles of every rank's four receive
// buffers are all-gathered over NCCL (a collective: all ranks call it together, after their
// arrival flags were reset), and the neighbours' buffers are mapped (NVLink peer access).
orca_status setup_peers(orca_ctx* c) {
    if (c->world == 1 || c->transport != 0) return ORCA_OK;
    if (c->loopback) {
        const int P = (int)c->doms.size();
        for (int s = 0; s < P; ++s) {
            Domain& d = c->doms[s];
            if (d.g.hasL) {
                d.peerL[0] = c->doms[s - 1].recvR.b;
                d.peerL[1] = c->doms[s - 1].recvR1.b;
            }
            if (d.g.hasR) {
                d.peerR[0] = c->doms[s + 1].recvL.b;
                d.peerR[1] = c->doms[s + 1].recvL1.b;
            }
        }
        return ORCA_OK;
    }
    Domain& d = c->doms[0];
    struct Handles {
        cudaIpcMemHandle_t h[4];  // recvL (even, odd), recvR (even, odd)
    };
    Handles mine;
    std::memset(&mine, 0, sizeof mine);
    const ExAlloc* xs[4] = {&d.recvL, &d.recvL1, &d.recvR, &d.recvR1};
    for (int q = 0; q < 4; ++q)
        if (xs[q]->base) CK(cudaIpcGetMemHandle(&mine.h[q], xs[q]->base));
    const size_t hb = sizeof(Handles);
    if (!c->ipcStage) CK(cudaMalloc(&c->ipcStage, hb * (c->world + 1)));
    CK(cudaMemcpyAsync(c->ipcStage, &mine, hb, cudaMemcpyHostToDevice, c->stream));
    NcclApi& N = nccl();
    ncclResult_t r = N.allGather(c->ipcStage, c->ipcStage + hb, hb, ncclUint8, c->comm, c->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather (cudaIpc handles)");
    std::vector<Handles> all(c->world);
    CK(cudaMemcpyAsync(all.data(), c->ipcStage + hb, hb * c->world, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    d.close_ipc();
    std::memset(d.peerL, 0, sizeof d.peerL);
    std::memset(d.peerR, 0, sizeof d.peerR);
    int ok = 1;
    for (int p = 0; p < 2 && ok; ++p) {
        if (d.g.hasL) {  // the left neighbour's right-side receive buffers
            if (cudaIpcOpenMemHandle(&d.ipcOpen[p], all[c->rank - 1].h[2 + p], cudaIpcMemLazyEnablePeerAccess) ==
                cudaSuccess)
                d.peerL[p] = rebase(d.recvL, d.ipcOpen[p]);
            else
                ok = 0;
        }
        if (ok && d.g.hasR) {  // the right neighbour's left-side receive buffers
            if (cudaIpcOpenMemHandle(&d.ipcOpen[2 + p], all[c->rank + 1].h[p], cudaIpcMemLazyEnablePeerAccess) ==
                cudaSuccess)
                d.peerR[p] = rebase(d.recvR, d.ipcOpen[2 + p]);
            else
                ok = 0;
        }
    }
    // no peer mapping between some pair of GPUs: every rank falls back to NCCL together
    cudaGetLastError();
    int* flag = reinterpret_cast<int*>(c->ipcStage);
    CK(cudaMemcpyAsync(flag, &ok, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    r = N.allReduce(flag, flag, 1, ncclInt32, ncclMin, c->comm, c->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce (peer mapping)");
    CK(cudaMemcpyAsync(&ok, flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (!ok) {
        d.close_ipc();
        c->transport = 1;
    }
    return ORCA_OK;
}

// Strips from the global by-id arrays (every rank holds the same arrays): column histogram
// of the active agents -> partition -> per-strip capacities, selection, scan, scatter.
// The grid (c->gg) is frozen; hist (nullable) seeds the per-agent search radius; active
// (nullable) excludes agents removed at their goal.  Used by orca_set_agents and by the
// strip rebalance.
orca_status build_domains(orca_ctx* c, int64_t n, const float2* sp, const float2* sv, const float2* sa,
                          const float* hist, const uint8_t* active) {
    const Grid& g = c->gg;
    if (c->world > g.nx) return fail(ORCA_ERR_CAPACITY, "more strips than grid columns");
    // column histogram -> strips (every rank computes the same partition)
    std::vector<int64_t> colCount(g.nx, 0);
    if (c->world > 1 && n > 0) {
        if (g.nx > c->colCap) {
            dfree(c->colHist);
            CK(cudaMalloc(&c->colHist, (size_t)g.nx * sizeof(int32_t)));
            c->colCap = g.nx;
        }
        CK(cudaMemsetAsync(c->colHist, 0, (size_t)g.nx * sizeof(int32_t), c->stream));
        k_colhist<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, sp, g, c->colHist, active);
        CK(cudaGetLastError());
        std::vector<int32_t> h(g.nx);
        CK(cudaMemcpyAsync(h.data(), c->colHist, (size_t)g.nx * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int x = 0; x < g.nx; ++x) colCount[x] = h[x];
    } else {
        colCount[0] = n;
    }
    std::vector<int32_t> bounds(c->world + 1);
    CKS(orca_partition_columns(colCount.data(), g.nx, c->world, bounds.data()));
    // exchange capacities are global (sender and receiver must agree on the layout):
    // 1.5x the largest strip-edge column of the whole partition
    int64_t edgeMax = 0;
    for (int s = 0; s < c->world; ++s)
        edgeMax = std::max(edgeMax, std::max(colCount[bounds[s]], colCount[bounds[s + 1] - 1]));
    const int capH = (int)std::min<int64_t>(edgeMax + edgeMax / 2 + 1024, (int64_t)1 << 28);
    const int capM = std::max(1024, capH / 4);
    const int first = c->loopback ? 0 : c->rank;
    for (size_t q = 0; q < c->doms.size(); ++q) {
        Domain& d = c->doms[q];
        const int s = first + (int)q;
        d.strip = s;
        d.g = g;
        d.g.c0 = bounds[s];
        d.g.c1 = bounds[s + 1];
        d.g.e0 = std::max(d.g.c0 - 1, 0);
        d.g.e1 = std::min(d.g.c1 + 1, g.nx);
        d.g.hasL = s > 0;
        d.g.hasR = s < c->world - 1;
        d.nbins = (int64_t)(d.g.e1 - d.g.e0) * g.colBins;
        int64_t sel = 0;
        for (int x = d.g.e0; x < d.g.e1; ++x) sel += colCount[x];
        d.popBuild = 0;
        for (int x = d.g.c0; x < d.g.c1; ++x) d.popBuild += colCount[x];
        // single strip: exact; strips: headroom for density drift between re-partitions
        const int64_t capW = (c->world == 1) ? std::max<int64_t>(n, 1) : sel + sel / 2 + 4096;
        if (capW > ((int64_t)1 << 30)) return fail(ORCA_ERR_CAPACITY, "strip too large");
        CKS(dom_alloc(c, d, (int)capW, d.nbins, capM, capH));
        CK(cudaMemsetAsync(d.ctr, 0, CT_COUNT * sizeof(int), c->stream));
        {
            const int t = (int)(c->lpStep0 + c->steps_total - c->lpMark);  // LP-order step index
            k_set_int<<<1, 1, 0, c->stream>>>(d.ctr + CT_STEP, t);
        }
        CK(cudaMemsetAsync(d.count, 0, d.nbins * sizeof(uint32_t), c->stream));
        if (n > 0)
            k_select<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, sp, sv, sa, d.g, d.posW, d.velW, d.auxW,
                                                                d.idW, d.rk2W, d.cellW, d.rankW, d.count, d.ctr,
                                                                d.capW, hist, active);
        CK(cudaGetLastError());
        CK(enqueue_scan(c, d, true));
        CK(enqueue_scatter(c, d, 0, false));
    }
    CK(cudaStreamSynchronize(c->stream));
    CKS(check_overflow(c));
    CKS(setup_peers(c));
    c->ready = true;
    return ORCA_OK;
}

// Per-agent properties (heterogeneous crowds) from the by-id copy into every strip's
// sorted order, after the strips were (re)built.
orca_status refresh_props(orca_ctx* c) {
    if (!c->het || !c->props4) return ORCA_OK;
    for (Domain& d : c->doms) {
        if (d.propCap < d.capW) {
            dfree(d.propS);
            dfree(d.propW);
            CK(cudaMalloc(&d.propS, (size_t)d.capW * sizeof(float4)));
            CK(cudaMalloc(&d.propW, (size_t)d.capW * sizeof(float4)));
            d.propCap = d.capW;
        }
        k_gather4_by_id<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, (int)d.nbins, d.idS, c->props4,
                                                                       d.propS);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

// Re-partition the strips from the current state: every strip's owned agents
// go back to by-id arrays (all-gathered between ranks), then build_domains re-runs the
// partition on the frozen grid.  Goals / preferred velocities (aux), per-agent properties,
// removals, search-radius history, counters and the LP-order step index carry over; the
// step results do not depend on the partition (bit-identical to one strip).
orca_status ensure_report(orca_ctx* c) {
    const int need = 3 * (int)c->doms.size() + 4;
    if (c->reportCap < need) {
        dfree(c->report);
        CK(cudaMalloc(&c->report, (size_t)need * sizeof(int)));
        c->reportCap = need;
    }
    return ORCA_OK;
}

// Every strip's owned agents back to by-id arrays in the stage (pos | vel | aux), their
// search-radius hints (outA) and active flags -- all-gathered between ranks (collective).
orca_status gather_state(orca_ctx* c) {
    const int64_t n = c->nGlobal;
    CKS(ensure_report(c));
    if (c->activeCap < n) {
        dfree(c->activeBuf);
        CK(cudaMalloc(&c->activeBuf, (size_t)n));
        c->activeCap = n;
    }
    float2 *sp = c->stage, *sv = c->stage + n, *sa = c->stage + 2 * n;
    float* hist = reinterpret_cast<float*>(c->outA);
    CK(cudaMemsetAsync(c->activeBuf, 0, (size_t)n, c->stream));
    k_fill1<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, hist, INFINITY);
    if (c->loopback || c->world == 1) {
        for (Domain& d : c->doms)
            k_gather_state<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, d.g, d.idS, d.posS, d.velS,
                                                                          d.auxS, d.rk2S, sp, sv, sa, hist,
                                                                          c->activeBuf);
        CK(cudaGetLastError());
    } else {
        NcclApi& N = nccl();
        Domain& d = c->doms[0];
        // records per rank = the largest owned count (all-gather needs equal sizes)
        k_fill_report<<<1, 32, 0, c->stream>>>(d.binStart, d.g, c->report);
        ncclResult_t r = N.allReduce(c->report, c->report + 3, 1, ncclInt32, ncclMax, c->comm, c->stream);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
        int cap = 0;
        CK(cudaMemcpyAsync(&cap, c->report + 3, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        cap = std::max(cap, 1);
        const size_t need = (size_t)2 * cap * (c->world + 1);
        if (c->gatherCap < need) {
            dfree(c->gatherBuf);
            CK(cudaMalloc(&c->gatherBuf, need * sizeof(float4)));
            c->gatherCap = need;
        }
        float4* mine = c->gatherBuf;
        float4* all = c->gatherBuf + (size_t)2 * cap;
        k_pack_owned<<<cap_blocks(cap, 256), 256, 0, c->stream>>>(d.binStart, d.g, d.idS, d.posS, d.velS, d.auxS,
                                                                  d.rk2S, mine, cap);
        r = N.allGather(mine, all, (size_t)8 * cap, ncclFloat32, c->comm, c->stream);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
        k_unpack_gathered<<<cap_blocks((int64_t)cap * c->world, 256), 256, 0, c->stream>>>(
            all, cap * c->world, sp, sv, sa, hist, c->activeBuf);
        CK(cudaGetLastError());
    }
    return ORCA_OK;
}

orca_status rebalance(orca_ctx* c, bool regrid) {
    const int64_t n = c->nGlobal;
    if (n == 0) return ORCA_OK;
    CKS(gather_state(c));
    float2 *sp = c->stage, *sv = c->stage + n, *sa = c->stage + 2 * n;
    float* hist = reinterpret_cast<float*>(c->outA);
    if (regrid) {  // a new frozen grid around the agents still in the simulation
        float mn[2], mx[2];
        CKS(stage_bounds(c, sp, sv, sa, n, mn, mx, c->activeBuf));
        if (!(mn[0] <= mx[0])) {  // nobody left: keep the grid
            mn[0] = mx[0] = c->gg.ox + c->gg.cs;
            mn[1] = mx[1] = c->gg.oy + c->gg.cs;
        }
        // margin: agents move up to 128 maxSpeed dt before the next check sees them (a chunk of
        // <= 64 steps is checked once the chunk after it is queued, orca_step); the margin covers
        // kRegridReach steps of walking, so a spreading crowd re-grids rarely (empty margin bins
        // cost the latency-bound scan next to nothing)
        const float reach = kRegridReach * std::max(c->maxSpeedAll, c->p.maxSpeed) * c->p.timeStep;
        CKS(derive_grid(c, n, mn, mx, 1 + (int)std::ceil(reach / c->p.neighborDist)));
        c->regrids += 1;
    } else {
        c->rebalances += 1;
    }
    c->ready = false;
    CKS(build_domains(c, n, sp, sv, sa, hist, c->activeBuf));
    CKS(refresh_props(c));
    return ORCA_OK;
}

// Before a chunk of up to 64 steps: rebalance if a strip could outgrow its capacities
// within the chunk.  Agents move at most 64 maxSpeed dt < 1.5 columns in a chunk, so a
// strip gains at most ~1.5 edge columns' worth of agents, and an edge column stays within
// its halo buffer while it is below 70 % of it.  One small read-back per chunk (strips only).
orca_status maybe_rebalance(orca_ctx* c) {
    if (c->nGlobal == 0) return ORCA_OK;
    volatile int* outside = c->gridFlagHost;
    if (c->world == 1) {  // no strips: only the grid check, without a synchronisation
        if (!*outside) return ORCA_OK;
        CK(cudaStreamSynchronize(c->stream));
        *outside = 0;
        const auto t0 = std::chrono::steady_clock::now();
        const orca_status st = rebalance(c, true);
        if (std::getenv("ORCA_DEBUG_TIMING"))
            std::fprintf(stderr, "[orca] regrid %.3f ms\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        return st;
    }
    const int nd = (int)c->doms.size();
    if (c->reportCap < 3 * nd + 4) {
        dfree(c->report);
        CK(cudaMalloc(&c->report, (size_t)(3 * nd + 4) * sizeof(int)));
        c->reportCap = 3 * nd + 4;
    }
    int* rep = c->report + 4;  // [0, 4) is scratch for the rebalance all-reduce
    for (int q = 0; q < nd; ++q) k_fill_report<<<1, 32, 0, c->stream>>>(c->doms[q].binStart, c->doms[q].g, rep + 3 * q);
    CK(cudaGetLastError());
    std::vector<int> h(3 * nd);
    CK(cudaMemcpyAsync(h.data(), rep, h.size() * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    int need = 0;
    for (int q = 0; q < nd; ++q) {
        const Domain& d = c->doms[q];
        const int owned = h[3 * q], colL = h[3 * q + 1], colR = h[3 * q + 2];
        const int capH = d.g.hasL ? d.sendL.b.capH : (d.g.hasR ? d.sendR.b.capH : INT32_MAX);
        if ((int64_t)owned + (3 * ((int64_t)colL + colR)) / 2 > (int64_t)d.capW) need = 1;
        if (d.g.hasL && (int64_t)colL * 10 > (int64_t)capH * 7) need = 1;
        if (d.g.hasR && (int64_t)colR * 10 > (int64_t)capH * 7) need = 1;
    }
    if (*outside) need = 2;  // (read after the synchronisation: every earlier step is done)
    if (!c->loopback) {  // every rank must take the same decision (2 = re-grid, 1 = re-partition)
        NcclApi& N = nccl();
        CK(cudaMemcpyAsync(c->report, &need, sizeof(int), cudaMemcpyHostToDevice, c->stream));
        ncclResult_t r = N.allReduce(c->report, c->report, 1, ncclInt32, ncclMax, c->comm, c->stream);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
        CK(cudaMemcpyAsync(&need, c->report, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    if (!need) return ORCA_OK;
    *outside = 0;
    return rebalance(c, need == 2);
}

// Streams, events, the host-mapped error word and the two upload / read-back slots of the
// asynchronous I/O path, sized for the loaded agent count.
orca_status io_init(orca_ctx* c) {
    if (!c->ioIn) {
        CK(cudaStreamCreateWithFlags(&c->ioIn, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->ioOut, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b)
            for (cudaEvent_t* e : {&c->inReady[b], &c->inFree[b], &c->outReady[b], &c->outFree[b]})
                CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CK(cudaHostAlloc(&c->ioBadHost, sizeof(int), cudaHostAllocMapped));
        *c->ioBadHost = 0;
        CK(cudaHostGetDevicePointer(&c->ioBadDev, c->ioBadHost, 0));
    }
    if (c->ioCap < c->nGlobal) {
        CK(cudaStreamSynchronize(c->ioIn));
        CK(cudaStreamSynchronize(c->ioOut));
        CK(cudaStreamSynchronize(c->stream));
        for (int b = 0; b < 2; ++b) {
            dfree(c->inBuf[b]);
            dfree(c->outBuf[b]);
            CK(cudaMalloc(&c->inBuf[b], (size_t)c->nGlobal * 2 * sizeof(float2)));
            CK(cudaMalloc(&c->outBuf[b], (size_t)c->nGlobal * 2 * sizeof(float2)));
        }
        c->ioCap = c->nGlobal;
    }
    return ORCA_OK;
}

}  // namespace

// =============================================================================== ABI

// ------------------------------------------------------------------ ALU peak probe
// Measured denominators of the ALU roofline: kProbeChains independent FMA
// chains per thread (enough ILP to cover the FMA latency), 2048 threads per SM.  Every block
// records its SM id and its first / last clock64(); the host takes, per SM, the span from the
// earliest start to the latest end (the per-SM cycle counter runs at the SM clock), so the
// caller also gets the SM clock the probe ran at.  The results are written so the compiler
// cannot drop the chains.
constexpr int kProbeChains = 8;
template <typename T>
__global__ void __launch_bounds__(256) k_probe_fma(T* out, int iters, T a, T b, long long* cyc) {
    long long c0;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0));
    T x[kProbeChains];
    // the chains start from a value that depends on the first clock read (c0 >> 62 is 0 in
    // practice), so the compiler cannot hoist the FMAs above it
#pragma unroll
    for (int q = 0; q < kProbeChains; ++q) x[q] = (T)(threadIdx.x + q + (int)(c0 >> 62));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int q = 0; q < kProbeChains; ++q) x[q] = x[q] * a + b;
        }
    }
    T acc = 0;
#pragma unroll
    for (int q = 0; q < kProbeChains; ++q) acc += x[q];
    if (acc == (T)-1.2345) out[blockIdx.x] = acc;  // practically never; keeps the chains live
    long long c1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1) : "l"((long long)(acc != acc)));  // after acc
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        cyc[3 * blockIdx.x] = c0;
        cyc[3 * blockIdx.x + 1] = c1;
        cyc[3 * blockIdx.x + 2] = smid;
    }
}

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

orca_status orca_partition_columns(const int64_t* colCount, int32_t nx, int32_t world, int32_t* bounds) {
    if (!colCount || !bounds || nx < 1 || world < 1 || world > nx)
        return fail(ORCA_ERR_INVALID_ARGUMENT, "need 1 <= world <= nx and non-null arrays");
    double total = 0.0;
    for (int c = 0; c < nx; ++c) {
        if (colCount[c] < 0) return fail(ORCA_ERR_INVALID_ARGUMENT, "negative count");
        total += (double)colCount[c];
    }
    bounds[0] = 0;
    double cum = 0.0;
    int c = 0;
    for (int s = 1; s < world; ++s) {
        const double target = total * s / world;
        // at least one column for this strip and for every remaining one
        const int lo = bounds[s - 1] + 1, hi = nx - (world - s);
        while (c < lo) cum += (double)colCount[c++];
        while (c < hi && cum + 0.5 * (double)colCount[c] < target) cum += (double)colCount[c++];
        bounds[s] = c;
    }
    bounds[world] = nx;
    return ORCA_OK;
}

orca_status orca_create(const orca_params* params, int32_t device, orca_ctx** out) {
    orca_ctx* c = nullptr;
    orca_status s = ctx_init(params, device, out, &c);
    if (s != ORCA_OK) {
        orca_destroy(c);
        return s;
    }
    c->doms.resize(1);
    *out = c;
    return ORCA_OK;
}

orca_status orca_create_strips(const orca_params* params, int32_t device, int32_t nstrips, orca_ctx** out) {
    if (nstrips < 1 || nstrips > 64) return fail(ORCA_ERR_INVALID_ARGUMENT, "nstrips out of range");
    if (params && nstrips > 1 && !(params->maxSpeed * params->timeStep < params->neighborDist))
        return fail(ORCA_ERR_INVALID_ARGUMENT, "strips need maxSpeed * timeStep < neighborDist");
    orca_ctx* c = nullptr;
    orca_status s = ctx_init(params, device, out, &c);
    if (s != ORCA_OK) {
        orca_destroy(c);
        return s;
    }
    c->doms.resize(nstrips);
    c->world = nstrips;
    c->loopback = true;
    if (nstrips > 1) {
        c->stripStream.resize(nstrips);
        c->stripDone.resize(nstrips);
        for (int q = 0; q < nstrips; ++q) {
            cudaError_t e = cudaStreamCreateWithFlags(&c->stripStream[q], cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->stripDone[q], cudaEventDisableTiming);
            if (e != cudaSuccess) {
                orca_destroy(c);
                *out = nullptr;
                return cuda_fail(e, "orca_create_strips streams");
            }
        }
    }
    *out = c;
    return ORCA_OK;
}

orca_status orca_nccl_unique_id(void* id128) {
    if (!id128) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    NcclApi& N = nccl();
    if (!N.ok) return fail(ORCA_ERR_NCCL, N.err);
    ncclUniqueId id;
    ncclResult_t r = N.getUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id128, &id, sizeof(id));
    return ORCA_OK;
}

orca_status orca_create_dist(const orca_params* params, int32_t device, int32_t rank, int32_t world,
                             const void* nccl_id128, orca_ctx** out) {
    if (world < 1 || rank < 0 || rank >= world) return fail(ORCA_ERR_INVALID_ARGUMENT, "bad rank/world");
    if (world == 1) return orca_create(params, device, out);
    if (!nccl_id128) return fail(ORCA_ERR_INVALID_ARGUMENT, "null NCCL id");
    if (params && !(params->maxSpeed * params->timeStep < params->neighborDist))
        return fail(ORCA_ERR_INVALID_ARGUMENT, "strips need maxSpeed * timeStep < neighborDist");
    NcclApi& N = nccl();
    if (!N.ok) return fail(ORCA_ERR_NCCL, N.err);
    orca_ctx* c = nullptr;
    orca_status s = ctx_init(params, device, out, &c);
    if (s != ORCA_OK) {
        orca_destroy(c);
        return s;
    }
    ncclUniqueId id;
    std::memcpy(&id, nccl_id128, sizeof(id));
    ncclResult_t r = N.commInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        orca_destroy(c);
        return nccl_fail(r, "ncclCommInitRank");
    }
    c->world = world;
    c->rank = rank;
    // NCCL send/recv is the default exchange between ranks: the fused
    // peer-memory transport (orca_set_transport(0)) is selectable, but no NVLink measurement
    // has shown it faster yet
    c->transport = 1;
    c->commRanks = -1;
    if (N.commCount) {
        int cnt = -1;
        if (N.commCount(c->comm, &cnt) == ncclSuccess) c->commRanks = cnt;
    }
    c->doms.resize(1);
    *out = c;
    return ORCA_OK;
}

void orca_destroy(orca_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->side) cudaStreamSynchronize(c->side);
    for (cudaStream_t st : c->stripStream)
        if (st) cudaStreamSynchronize(st);
    drop_graph(c);
    for (Domain& d : c->doms) d.release();
    dfree(c->stage);
    dfree(c->outA);
    dfree(c->outB);
    dfree(c->partial);
    dfree(c->colHist);
    dfree(c->props4);
    if (c->gridFlagHost) cudaFreeHost(c->gridFlagHost);
    dfree(c->activeBuf);
    dfree(c->gatherBuf);
    dfree(c->ipcStage);
    dfree(c->report);
    for (auto& b : c->traceBuf) dfree(b);
    for (int b = 0; b < 2; ++b) {
        if (c->frameReady[b]) cudaEventDestroy(c->frameReady[b]);
        if (c->frameFree[b]) cudaEventDestroy(c->frameFree[b]);
    }
    if (c->copyStream) {
        cudaStreamSynchronize(c->copyStream);
        cudaStreamDestroy(c->copyStream);
    }
    for (cudaStream_t s : {c->ioIn, c->ioOut})
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    for (int b = 0; b < 2; ++b) {
        for (cudaEvent_t e : {c->inReady[b], c->inFree[b], c->outReady[b], c->outFree[b]})
            if (e) cudaEventDestroy(e);
        dfree(c->inBuf[b]);
        dfree(c->outBuf[b]);
    }
    if (c->ioBadHost) cudaFreeHost(c->ioBadHost);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->chunkEv)
        if (e) cudaEventDestroy(e);
    if (c->comm && nccl().ok) nccl().commDestroy(c->comm);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->side) cudaStreamDestroy(c->side);
    for (cudaStream_t st : c->stripStream)
        if (st) cudaStreamDestroy(st);
    for (cudaEvent_t ev : c->stripDone)
        if (ev) cudaEventDestroy(ev);
    if (c->evFork) cudaEventDestroy(c->evFork);
    if (c->evJoin) cudaEventDestroy(c->evJoin);
    delete c;
}

orca_status orca_set_agents(orca_ctx* c, int64_t n, const float* pos, const float* vel, const float* pref) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (n < 0 || n > ((int64_t)1 << 30)) return fail(ORCA_ERR_INVALID_ARGUMENT, "n out of range");
    if (n > 0 && (!pos || !vel || !pref)) return fail(ORCA_ERR_INVALID_ARGUMENT, "null array");
    CK(cudaSetDevice(c->device));
    if (c->ready) CK(flush_deferred(c));  // (the radius hints below are read in sorted order)
    CK(cudaStreamSynchronize(c->stream));
    if (c->ioBadHost) *c->ioBadHost = 0;  // a refused asynchronous upload is superseded
    *c->gridFlagHost = 0;  // a new grid is derived below
    // same agent count as the loaded state: keep each agent's last k-th neighbour distance
    // as its first search radius (a hint; the selection is exact for any radius)
    const bool keepHist = c->ready && c->nGlobal == n && n > 0;
    // cached step graphs stay: orca_step re-captures only if graph_key() changed
    c->ready = false;
    c->goals = false;
    c->het = false;
    // stage the global inputs (every rank of a decomposition gets the same arrays)
    if (n > c->stageCap) {
        dfree(c->stage);
        dfree(c->outA);
        dfree(c->outB);
        CK(cudaMalloc(&c->stage, (size_t)n * 3 * sizeof(float2)));
        CK(cudaMalloc(&c->outA, (size_t)n * sizeof(float2)));
        CK(cudaMalloc(&c->outB, (size_t)n * sizeof(float2)));
        c->stageCap = n;
    }
    float2 *sp = c->stage, *sv = c->stage + n, *sa = c->stage + 2 * n;
    float* hist = nullptr;
    if (keepHist) {  // before any domain is re-allocated
        hist = reinterpret_cast<float*>(c->outA);
        k_fill1<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, hist, INFINITY);
        for (Domain& d : c->doms)
            k_hist_by_id<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, d.g, d.idS, d.rk2S, hist);
        CK(cudaGetLastError());
    }
    CK(copy_in(c, sp, pos, n));
    CK(copy_in(c, sv, vel, n));
    CK(copy_in(c, sa, pref, n));
    float mn[2] = {0.0f, 0.0f}, mx[2] = {0.0f, 0.0f};
    if (n > 0) CKS(stage_bounds(c, sp, sv, sa, n, mn, mx));
    // frozen global grid (reading Q12)
    CKS(derive_grid(c, n, mn, mx));
    c->nGlobal = n;
    return build_domains(c, n, sp, sv, sa, hist, nullptr);
}

orca_status orca_set_state(orca_ctx* c, const float* pos, const float* vel) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    const int64_t n = c->nGlobal;
    if (n > 0 && (!pos || !vel)) return fail(ORCA_ERR_INVALID_ARGUMENT, "null array");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    CK(cudaStreamSynchronize(c->stream));
    if (n == 0) return ORCA_OK;
    // everything but the kinematic state stays: preferred velocities or goals, per-agent
    // properties, removals, search-radius hints (by id), counters, the LP-order step index
    CKS(gather_state(c));
    float2 *sp = c->stage, *sv = c->stage + n, *sa = c->stage + 2 * n;
    float* hist = reinterpret_cast<float*>(c->outA);
    CK(copy_in(c, sp, pos, n));
    CK(copy_in(c, sv, vel, n));
    float mn[2], mx[2];
    CKS(stage_bounds(c, sp, sv, sa, n, mn, mx, c->activeBuf));  // finiteness of the agents present
    const Grid& g = c->gg;
    const bool inside = !(mn[0] <= mx[0]) ||
                        (mn[0] >= g.ox + g.cs && mn[1] >= g.oy + g.cs && (double)mx[0] < g.ox + (double)g.cs * (g.nx - 1) &&
                         (double)mx[1] < g.oy + (double)g.cs * (g.ny - 1));
    if (!inside) {  // the new state leaves the grid's interior: re-derive it (reading Q12)
        const float reach = kRegridReach * std::max(c->maxSpeedAll, c->p.maxSpeed) * c->p.timeStep;
        CKS(derive_grid(c, n, mn, mx, 1 + (int)std::ceil(reach / c->p.neighborDist)));
        c->regrids += 1;
    }
    *c->gridFlagHost = 0;
    c->ready = false;
    CKS(build_domains(c, n, sp, sv, sa, hist, c->activeBuf));
    CKS(refresh_props(c));
    return ORCA_OK;
}

orca_status orca_set_state_async(orca_ctx* c, const float* pos, const float* vel) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    const int64_t n = c->nGlobal;
    if (n > 0 && (!pos || !vel)) return fail(ORCA_ERR_INVALID_ARGUMENT, "null array");
    if (c->world > 1 || c->doms.size() != 1) return orca_set_state(c, pos, vel);  // strips: synchronous
    if (n == 0) return ORCA_OK;
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    CKS(io_init(c));
    const int b = c->inSlot;
    c->inSlot ^= 1;
    float2* buf = c->inBuf[b];
    // upload (copy stream) once the step that last read this slot is done with it
    CK(cudaStreamWaitEvent(c->ioIn, c->inFree[b], 0));
    CK(cudaMemcpyAsync(buf, pos, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->ioIn));
    CK(cudaMemcpyAsync(buf + n, vel, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->ioIn));
    CK(cudaEventRecord(c->inReady[b], c->ioIn));
    // re-bin on the step stream: k_reload -> scan -> scatter (no host synchronisation)
    CK(cudaStreamWaitEvent(c->stream, c->inReady[b], 0));
    Domain& d = c->doms[0];
    k_reload<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(
        d.binStart, d.g, d.idS, d.auxS, d.rk2S, c->het ? d.propS : nullptr, buf, buf + n, d.posW, d.velW, d.auxW,
        d.idW, d.rk2W, c->het ? d.propW : nullptr, d.cellW, d.rankW, d.count, d.ctr, c->gridFlagDev, c->ioBadDev);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->inFree[b], c->stream));
    CK(enqueue_scan(c, d, false));
    CK(enqueue_scatter(c, d, 0));
    return ORCA_OK;
}

// One frame of the per-frame loop in one call (single strip; strips fall back to the three
// calls): upload pos_in / vel_in (copy stream 1), bin them, one step, and read the stepped state
// back into pos_out / vel_out (copy stream 2), without host synchronisation.  Since the next
// frame uploads a new state anyway, the step's own next-step binning is skipped: the upload is
// binned in place in the work arrays the previous frame's step left (k_reload_work), and the
// read-back un-permutes those work arrays (k_unpermute_work).  Any other call first completes
// the skipped binning (flush_deferred), so results equal orca_set_state_async -> orca_step(1)
// -> orca_get_state_async bit for bit.
orca_status orca_step_io_async(orca_ctx* c, const float* pos_in, const float* vel_in, float* pos_out,
                               float* vel_out) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    const int64_t n = c->nGlobal;
    if (n > 0 && (!pos_in || !vel_in)) return fail(ORCA_ERR_INVALID_ARGUMENT, "null array");
    if (c->world > 1 || c->doms.size() != 1 || n == 0 || *c->gridFlagHost) {
        // strips, an empty crowd, or a pending grid re-derivation: the three calls
        CKS(orca_set_state_async(c, pos_in, vel_in));
        CKS(orca_step(c, 1));
        return orca_get_state_async(c, pos_out, vel_out);
    }
    CK(cudaSetDevice(c->device));
    CKS(io_init(c));
    Domain& d = c->doms[0];
    const int b = c->inSlot;
    c->inSlot ^= 1;
    float2* buf = c->inBuf[b];
    CK(cudaStreamWaitEvent(c->ioIn, c->inFree[b], 0));
    CK(cudaMemcpyAsync(buf, pos_in, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->ioIn));
    CK(cudaMemcpyAsync(buf + n, vel_in, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->ioIn));
    CK(cudaEventRecord(c->inReady[b], c->ioIn));
    CK(cudaStreamWaitEvent(c->stream, c->inReady[b], 0));
    const bool prevStep = c->deferred;  // the previous frame's step is complete once binned
    if (c->deferred) {
        // the previous frame's step left its agents in the work arrays: bin the upload there
        CK(cudaMemsetAsync(d.count, 0, (size_t)d.nbins * sizeof(uint32_t), c->stream));
        k_reload_work<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.ctr, d.capW, d.g, buf, buf + n, d.posW,
                                                                      d.velW, d.idW, d.cellW, d.rankW, d.count,
                                                                      c->gridFlagDev, c->ioBadDev);
    } else {
        k_reload<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(
            d.binStart, d.g, d.idS, d.auxS, d.rk2S, c->het ? d.propS : nullptr, buf, buf + n, d.posW, d.velW, d.auxW,
            d.idW, d.rk2W, c->het ? d.propW : nullptr, d.cellW, d.rankW, d.count, d.ctr, c->gridFlagDev, c->ioBadDev);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->inFree[b], c->stream));
    if (fused_bin(c)) {
        CK(enqueue_bin(c, d, prevStep ? 1 : 0));
    } else {
        CK(enqueue_scan(c, d, false));
        CK(enqueue_scatter(c, d, prevStep ? 1 : 0));
    }
    // the step without its trailing binning
    StepArgs a = make_args(c, d);
    launch_step<false>(c, d, a);
    launch_lp3<false>(c, d, a);
    CK(cudaGetLastError());
    c->deferred = true;
    c->host_steps += 1;
    c->steps_total += 1;
    c->host_updates += n;
    // read-back of the work arrays
    if (pos_out || vel_out) {
        const int ob_i = c->outSlot;
        c->outSlot ^= 1;
        float2* ob = c->outBuf[ob_i];
        CK(cudaStreamWaitEvent(c->stream, c->outFree[ob_i], 0));
        if (c->removeR > 0.0f)  // agents removed at their goal read as NaN
            k_fill2<<<cap_blocks(2 * n, 256), 256, 0, c->stream>>>((int)(2 * n), ob, NAN);
        k_unpermute_work<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.ctr, d.capW, d.cellW, d.idW, d.posW, d.velW,
                                                                         pos_out ? ob : nullptr,
                                                                         vel_out ? ob + n : nullptr);
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->outReady[ob_i], c->stream));
        CK(cudaStreamWaitEvent(c->ioOut, c->outReady[ob_i], 0));
        if (pos_out) CK(cudaMemcpyAsync(pos_out, ob, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->ioOut));
        if (vel_out) CK(cudaMemcpyAsync(vel_out, ob + n, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->ioOut));
        CK(cudaEventRecord(c->outFree[ob_i], c->ioOut));
    }
    return ORCA_OK;
}

orca_status orca_set_goals(orca_ctx* c, const float* goal, float prefSpeed) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (!(prefSpeed >= 0.0f) || !std::isfinite(prefSpeed)) return fail(ORCA_ERR_INVALID_ARGUMENT, "prefSpeed");
    if (c->nGlobal > 0 && !goal) return fail(ORCA_ERR_INVALID_ARGUMENT, "null goal");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    const int64_t n = c->nGlobal;
    if (n > 0) {
        // goals arrive in id order (global): check finiteness, gather into sorted order
        CK(copy_in(c, c->outA, goal, n));
        float mn[2], mx[2];
        CKS(stage_bounds(c, c->outA, c->outA, c->outA, n, mn, mx));
        for (Domain& d : c->doms) {
            k_gather_by_id<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, (int)d.nbins, d.idS, c->outA,
                                                                          d.auxS);
            CK(cudaGetLastError());
        }
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
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    // one graph of up to kChunk step bodies, replayed
    const int kChunk = 64;
    int remaining = n_steps;
    if (c->world == 1 && !c->chunkEv[0])
        for (auto& e : c->chunkEv) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int q = 0; remaining > 0; ++q) {
        const int s = std::min(remaining, kChunk);
        // one strip: the outer-ring flag of chunk q-2 is final once that chunk is done, so a long
        // call re-derives the grid while it runs (chunk q-1 keeps the GPU busy meanwhile); the
        // first two chunks of a call only read the flag (no synchronisation for short calls)
        if (c->world == 1 && q >= 2) CK(cudaEventSynchronize(c->chunkEv[q & 1]));
        CKS(maybe_rebalance(c));  // grid check; strips: capacities for the next chunk
        {
            std::vector<unsigned char> key = graph_key(c);
            if (key != c->graphKey) {  // new arguments: cached graphs are updated on next use
                c->graphKey = std::move(key);
                c->keyGen += 1;
            }
        }
        int slot = -1;
        for (size_t g = 0; g < c->graphs.size(); ++g)
            if (c->graphs[g].first == s) slot = (int)g;
        if (slot < 0 || c->graphGen[slot] != c->keyGen) {
            const auto tg0 = std::chrono::steady_clock::now();
            cudaGraph_t gr;
            CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            orca_status st = ORCA_OK;
            for (int t = 0; t < s && st == ORCA_OK; ++t) st = enqueue_step(c, nullptr);
            cudaError_t e2 = cudaStreamEndCapture(c->stream, &gr);
            if (st != ORCA_OK) return st;
            if (e2 != cudaSuccess) return cuda_fail(e2, "cudaStreamEndCapture");
            bool updated = false;
            if (slot >= 0) {
                // same step body with new arguments (a re-grid, a rebalance, a reload): update
                // the instantiated graph in place -- much cheaper than instantiating it again
                cudaGraphExecUpdateResultInfo info;
                updated = cudaGraphExecUpdate(c->graphs[slot].second, gr, &info) == cudaSuccess;
                if (!updated) {
                    (void)cudaGetLastError();
                    cudaGraphExecDestroy(c->graphs[slot].second);
                    c->graphs.erase(c->graphs.begin() + slot);
                    c->graphGen.erase(c->graphGen.begin() + slot);
                    slot = -1;
                }
            }
            if (!updated) {
                if (c->graphs.size() >= 4) {
                    cudaGraphExecDestroy(c->graphs.front().second);
                    c->graphs.erase(c->graphs.begin());
                    c->graphGen.erase(c->graphGen.begin());
                }
                cudaGraphExec_t ex = nullptr;
                cudaError_t e = cudaGraphInstantiate(&ex, gr, 0);
                if (e != cudaSuccess) {
                    cudaGraphDestroy(gr);
                    return cuda_fail(e, "cudaGraphInstantiate");
                }
                c->graphs.emplace_back(s, ex);
                c->graphGen.push_back(c->keyGen);
                slot = (int)c->graphs.size() - 1;
            }
            c->graphGen[slot] = c->keyGen;
            cudaGraphDestroy(gr);
            if (std::getenv("ORCA_DEBUG_TIMING"))
                std::fprintf(stderr, "[orca] graph %d steps %s %.3f ms\n", s, updated ? "updated" : "instantiated",
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tg0).count());
        }
        cudaGraphExec_t exec = c->graphs[slot].second;
        CK(cudaGraphLaunch(exec, c->stream));
        if (c->world == 1) CK(cudaEventRecord(c->chunkEv[q & 1], c->stream));
        remaining -= s;
    }
    c->host_steps += n_steps;
    c->steps_total += n_steps;
    c->host_updates += (int64_t)n_steps * c->nGlobal;
    return ORCA_OK;
}

orca_status orca_step_timed(orca_ctx* c, int32_t n_steps, double ms[4]) {
    if (!c || !ms) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (n_steps < 0) return fail(ORCA_ERR_INVALID_ARGUMENT, "n_steps < 0");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    for (int q = 0; q < 4; ++q) ms[q] = 0.0;
    for (int s = 0; s < n_steps; ++s) {
        if (s % 64 == 0) CKS(maybe_rebalance(c));
        CKS(enqueue_step(c, c->ev));
        CK(cudaEventSynchronize(c->ev[4]));
        float t;
        CK(cudaEventElapsedTime(&t, c->ev[0], c->ev[1]));
        ms[0] += t;  // k_step + k_lp3
        CK(cudaEventElapsedTime(&t, c->ev[2], c->ev[3]));
        ms[1] += t;  // scan
        CK(cudaEventElapsedTime(&t, c->ev[3], c->ev[4]));
        ms[2] += t;  // scatter
        CK(cudaEventElapsedTime(&t, c->ev[1], c->ev[2]));
        ms[3] += t;  // exchange + receive
    }
    c->host_steps += n_steps;
    c->steps_total += n_steps;
    c->host_updates += (int64_t)n_steps * c->nGlobal;
    return ORCA_OK;
}

orca_status orca_get_state(orca_ctx* c, float* pos, float* vel) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (c->world > 1 && !c->loopback)
        return fail(ORCA_ERR_INVALID_ARGUMENT, "multi-rank context: use orca_get_local_state");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    CKS(check_overflow(c));
    const int64_t n = c->nGlobal;
    if (n > 0 && (pos || vel)) {
        if (c->removeR > 0.0f) {  // agents removed at their goal read as NaN
            k_fill2<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, c->outA, NAN);
            k_fill2<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, c->outB, NAN);
        }
        for (Domain& d : c->doms)
            k_unpermute<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, d.g, d.idS, d.posS, d.velS,
                                                                       pos ? c->outA : nullptr,
                                                                       vel ? c->outB : nullptr);
        CK(cudaGetLastError());
        if (pos) CK(cudaMemcpyAsync(pos, c->outA, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->stream));
        if (vel) CK(cudaMemcpyAsync(vel, c->outB, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

orca_status orca_get_state_async(orca_ctx* c, float* pos, float* vel) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (c->world > 1 && !c->loopback)
        return fail(ORCA_ERR_INVALID_ARGUMENT, "multi-rank context: use orca_get_local_state");
    if (c->doms.size() != 1) return orca_get_state(c, pos, vel);  // loopback strips: synchronous
    const int64_t n = c->nGlobal;
    if (n == 0 || (!pos && !vel)) return ORCA_OK;
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    CKS(io_init(c));
    const int b = c->outSlot;
    c->outSlot ^= 1;
    float2* ob = c->outBuf[b];
    Domain& d = c->doms[0];
    // un-permute on the step stream once the read-back that last used this slot is done
    CK(cudaStreamWaitEvent(c->stream, c->outFree[b], 0));
    if (c->removeR > 0.0f)  // agents removed at their goal read as NaN
        k_fill2<<<cap_blocks(2 * n, 256), 256, 0, c->stream>>>((int)(2 * n), ob, NAN);
    k_unpermute<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, d.g, d.idS, d.posS, d.velS,
                                                               pos ? ob : nullptr, vel ? ob + n : nullptr);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->outReady[b], c->stream));
    // read back on the copy stream
    CK(cudaStreamWaitEvent(c->ioOut, c->outReady[b], 0));
    if (pos) CK(cudaMemcpyAsync(pos, ob, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->ioOut));
    if (vel) CK(cudaMemcpyAsync(vel, ob + n, (size_t)n * sizeof(float2), cudaMemcpyDefault, c->ioOut));
    CK(cudaEventRecord(c->outFree[b], c->ioOut));
    return ORCA_OK;
}

orca_status orca_io_wait(orca_ctx* c) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    CK(cudaSetDevice(c->device));
    if (c->ioIn) CK(cudaStreamSynchronize(c->ioIn));
    CK(cudaStreamSynchronize(c->stream));
    if (c->ioOut) CK(cudaStreamSynchronize(c->ioOut));
    if (c->ioBadHost && *(volatile int*)c->ioBadHost) {
        *c->ioBadHost = 0;
        c->ready = false;
        return fail(ORCA_ERR_INVALID_ARGUMENT,
                    "NaN/Inf in an orca_set_state_async upload; load the agents again with orca_set_agents");
    }
    return ORCA_OK;
}

orca_status orca_get_count(orca_ctx* c, int64_t* n) {
    if (!c || !n) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready) {
        *n = 0;
        return ORCA_OK;
    }
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    int64_t t = 0;
    for (Domain& d : c->doms) {
        int o0, o1;
        CKS(owned_range_host(c, d, &o0, &o1));
        t += o1 - o0;
    }
    *n = t;
    return ORCA_OK;
}

orca_status orca_get_local_state(orca_ctx* c, int32_t* ids, float* pos, float* vel) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    CKS(check_overflow(c));
    size_t off = 0;
    for (Domain& d : c->doms) {
        int o0, o1;
        CKS(owned_range_host(c, d, &o0, &o1));
        const size_t m = (size_t)(o1 - o0);
        if (m > 0) {
            if (ids) CK(cudaMemcpyAsync(ids + off, d.idS + o0, m * 4, cudaMemcpyDefault, c->stream));
            if (pos) CK(cudaMemcpyAsync(pos + 2 * off, d.posS + o0, m * 8, cudaMemcpyDefault, c->stream));
            if (vel) CK(cudaMemcpyAsync(vel + 2 * off, d.velS + o0, m * 8, cudaMemcpyDefault, c->stream));
        }
        off += m;
    }
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

orca_status orca_get_grid(orca_ctx* c, double origin[2], float* cs, int32_t dims[2]) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (origin) {
        origin[0] = c->gg.ox;
        origin[1] = c->gg.oy;
    }
    if (cs) *cs = c->gg.cs;
    if (dims) {
        dims[0] = c->gg.nx;
        dims[1] = c->gg.ny;
    }
    return ORCA_OK;
}

orca_status orca_get_strips(orca_ctx* c, int32_t* bounds) {
    if (!c || !bounds) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    for (size_t q = 0; q < c->doms.size(); ++q) {
        bounds[2 * q] = c->doms[q].g.c0;
        bounds[2 * q + 1] = c->doms[q].g.c1;
    }
    return ORCA_OK;
}

orca_status orca_debug_cells(orca_ctx* c, int32_t* cx, int32_t* cy) {
    if (!c || !cx || !cy) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    const int64_t n = c->nGlobal;
    if (n > 0) {
        int32_t* d0 = reinterpret_cast<int32_t*>(c->outA);  // 2 x int32 per agent
        CK(cudaMemsetAsync(d0, 0xff, (size_t)n * 2 * sizeof(int32_t), c->stream));  // removed: -1
        for (Domain& d : c->doms)
            k_cells<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, d.g, d.idS, d.posS, d0, d0 + n);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(cx, d0, (size_t)n * sizeof(int32_t), cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(cy, d0 + n, (size_t)n * sizeof(int32_t), cudaMemcpyDefault, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

orca_status orca_debug_step(orca_ctx* c, float* vnew, uint8_t* flags, int32_t* nbr, int32_t* cnt) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    const int64_t n = c->nGlobal;
    if (n == 0) return ORCA_OK;
    const int k = c->p.maxNeighbors;
    float2* dV = nullptr;
    uint8_t* dF = nullptr;
    int32_t *dN = nullptr, *dC = nullptr;
    CK(cudaMalloc(&dV, (size_t)n * sizeof(float2)));
    cudaError_t e = cudaMalloc(&dF, (size_t)n);
    if (e == cudaSuccess) e = cudaMalloc(&dC, (size_t)n * sizeof(int32_t));
    if (e == cudaSuccess && k > 0) e = cudaMalloc(&dN, (size_t)n * k * sizeof(int32_t));
    // agents no longer in the simulation (removed at their goal): NaN, flags 0, cnt -1
    if (e == cudaSuccess) {
        k_fill2<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, dV, NAN);
        e = cudaMemsetAsync(dF, 0, (size_t)n, c->stream);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(dC, 0xff, (size_t)n * sizeof(int32_t), c->stream);
    if (e == cudaSuccess && k > 0) e = cudaMemsetAsync(dN, 0xff, (size_t)n * k * sizeof(int32_t), c->stream);
    for (Domain& d : c->doms) {
        if (e != cudaSuccess) break;
        StepArgs a = make_args(c, d);
        a.dbgV = dV;
        a.dbgFlags = dF;
        a.dbgNbr = dN;
        a.dbgCnt = dC;
        e = dry_step(c, d, a);
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

orca_status orca_debug_work(orca_ctx* c, int64_t out[6]) {
    if (!c || !out) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    for (int q = 0; q < 6; ++q) out[q] = 0;
    if (c->nGlobal == 0) return ORCA_OK;
    Work* dW = nullptr;
    CK(cudaMalloc(&dW, sizeof(Work)));
    cudaError_t e = cudaMemsetAsync(dW, 0, sizeof(Work), c->stream);
    for (Domain& d : c->doms) {
        if (e != cudaSuccess) break;
        StepArgs a = make_args(c, d);
        a.work = dW;
        e = dry_step(c, d, a);
        if (e == cudaSuccess) {
            k_stencil_count<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, d.g, d.posS, &dW->stencil);
            e = cudaGetLastError();
        }
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
    out[5] = (int64_t)h.stencil;
    return ORCA_OK;
}

orca_status orca_get_stats(orca_ctx* c, orca_stats* out) {
    if (!c || !out) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    CK(cudaSetDevice(c->device));
    unsigned long long t[ST_COUNT] = {};
    for (Domain& d : c->doms) {
        if (!d.stats) continue;
        unsigned long long h[ST_COUNT];
        CK(cudaMemcpyAsync(h, d.stats, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int q = 0; q < ST_COUNT; ++q) t[q] += h[q];
    }
    out->steps = c->host_steps;
    out->agent_updates = c->host_updates;
    out->infeasible = (int64_t)t[ST_INFEASIBLE];
    out->degenerate = (int64_t)t[ST_DEGENERATE];
    out->coincident = (int64_t)t[ST_G1];
    out->eps_parallel = (int64_t)t[ST_G2];
    out->marginal = (int64_t)t[ST_G3];
    out->collision_pairs = (int64_t)t[ST_COLLISION];
    out->removed = (int64_t)t[ST_REMOVED];
    out->rebalances = c->rebalances;
    out->regrids = c->regrids;
    if (c->ready) CKS(check_overflow(c));
    return ORCA_OK;
}

orca_status orca_reset_stats(orca_ctx* c) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    CK(cudaSetDevice(c->device));
    for (Domain& d : c->doms)
        if (d.stats) CK(cudaMemsetAsync(d.stats, 0, ST_COUNT * sizeof(unsigned long long), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->host_steps = 0;
    c->host_updates = 0;
    return ORCA_OK;
}

orca_status orca_set_agent_props(orca_ctx* c, const float* radius, const float* maxSpeed, const float* prefSpeed) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    CK(cudaStreamSynchronize(c->stream));
    const int64_t n = c->nGlobal;
    drop_graph(c);
    if (!radius && !maxSpeed && !prefSpeed) {  // back to the global parameters
        c->het = false;
        return ORCA_OK;
    }
    if (n == 0) return ORCA_OK;
    // stage the three arrays (NULL -> global value) as float4 by id in the input stage
    float* st = reinterpret_cast<float*>(c->stage);  // >= 6n floats
    const float* src[3] = {radius, maxSpeed, prefSpeed};
    // prefSpeed -1: use the orca_set_goals speed
    const float def[3] = {c->p.radius, c->p.maxSpeed, -1.0f};
    for (int q = 0; q < 3; ++q) {
        if (src[q])
            CK(cudaMemcpyAsync(st + q * n, src[q], (size_t)n * sizeof(float), cudaMemcpyDefault, c->stream));
        else
            k_fill1<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, st + q * n, def[q]);
    }
    if (c->props4Cap < n) {
        dfree(c->props4);
        CK(cudaMalloc(&c->props4, (size_t)n * sizeof(float4)));
        c->props4Cap = n;
    }
    float4* props = c->props4;
    const int blocks = std::min(1024, cap_blocks(n, 256));
    k_pack_props<<<blocks, 256, 0, c->stream>>>((int)n, st, props, c->partial);
    CK(cudaGetLastError());
    std::vector<float> h((size_t)blocks * 5);
    CK(cudaMemcpyAsync(h.data(), c->partial, h.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float vmax = 0.0f;
    double bad = 0.0;
    for (int b = 0; b < blocks; ++b) {
        vmax = std::max(vmax, h[b * 5 + 0]);
        bad += h[b * 5 + 4];
    }
    if (bad > 0) return fail(ORCA_ERR_INVALID_ARGUMENT, "radius must be > 0 and speeds >= 0, finite");
    if (c->world > 1 && !(vmax * c->p.timeStep < c->p.neighborDist))
        return fail(ORCA_ERR_INVALID_ARGUMENT, "strips need maxSpeed * timeStep < neighborDist");
    for (Domain& d : c->doms) {
        if (d.propCap < d.capW) {
            dfree(d.propS);
            dfree(d.propW);
            CK(cudaMalloc(&d.propS, (size_t)d.capW * sizeof(float4)));
            CK(cudaMalloc(&d.propW, (size_t)d.capW * sizeof(float4)));
            d.propCap = d.capW;
        }
        k_gather4_by_id<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, (int)d.nbins, d.idS, props,
                                                                       d.propS);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(c->stream));
    c->het = true;
    c->maxSpeedAll = vmax;
    return ORCA_OK;
}

orca_status orca_step_trace(orca_ctx* c, int32_t n_steps, float* frames, float* vframes) {
    if (!c || !frames || n_steps < 0) return fail(ORCA_ERR_INVALID_ARGUMENT, "null frames or n_steps < 0");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (c->world > 1 && !c->loopback)
        return fail(ORCA_ERR_INVALID_ARGUMENT, "multi-rank context: trace each rank with orca_get_local_state");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    const int64_t n = c->nGlobal;
    if (n == 0 || n_steps == 0) return orca_step(c, n_steps);
    if (!c->copyStream) {
        CK(cudaStreamCreateWithFlags(&c->copyStream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            CK(cudaEventCreateWithFlags(&c->frameReady[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->frameFree[b], cudaEventDisableTiming));
        }
    }
    if (c->traceCap < n) {
        for (int b = 0; b < 4; ++b) dfree(c->traceBuf[b]);
        for (int b = 0; b < 4; ++b) CK(cudaMalloc(&c->traceBuf[b], (size_t)n * sizeof(float2)));
        c->traceCap = n;
    }
    const size_t fb = (size_t)n * sizeof(float2);
    for (int s = 0; s < n_steps; ++s) {
        const int b = s & 1;
        CKS(orca_step(c, 1));
        if (s >= 2) CK(cudaStreamWaitEvent(c->stream, c->frameFree[b], 0));  // frame buffer b copied out
        float2* fp = c->traceBuf[2 * b];
        float2* fv = vframes ? c->traceBuf[2 * b + 1] : nullptr;
        if (c->removeR > 0.0f) {
            k_fill2<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, fp, NAN);
            if (fv) k_fill2<<<cap_blocks(n, 256), 256, 0, c->stream>>>((int)n, fv, NAN);
        }
        for (Domain& d : c->doms)
            k_unpermute<<<cap_blocks(d.capW, 256), 256, 0, c->stream>>>(d.binStart, d.g, d.idS, d.posS, d.velS, fp, fv);
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->frameReady[b], c->stream));
        CK(cudaStreamWaitEvent(c->copyStream, c->frameReady[b], 0));
        CK(cudaMemcpyAsync(frames + (size_t)s * 2 * n, fp, fb, cudaMemcpyDefault, c->copyStream));
        if (vframes) CK(cudaMemcpyAsync(vframes + (size_t)s * 2 * n, fv, fb, cudaMemcpyDefault, c->copyStream));
        CK(cudaEventRecord(c->frameFree[b], c->copyStream));
    }
    CK(cudaStreamSynchronize(c->copyStream));
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

orca_status orca_set_goal_removal(orca_ctx* c, float radius) {
    if (!c || !(radius >= 0.0f) || !std::isfinite(radius)) return fail(ORCA_ERR_INVALID_ARGUMENT, "radius");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    CK(cudaStreamSynchronize(c->stream));
    drop_graph(c);
    c->removeR = radius;
    return ORCA_OK;
}

// device step counters of every domain := the current LP-order step index
cudaError_t write_lp_step(orca_ctx* c) {
    const int t = (int)(c->lpStep0 + c->steps_total - c->lpMark);
    for (Domain& d : c->doms) {
        if (!d.ctr) continue;
        k_set_int<<<1, 1, 0, c->stream>>>(d.ctr + CT_STEP, t);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaStreamSynchronize(c->stream);
}

orca_status orca_set_transport(orca_ctx* c, int32_t mode) {
    if (!c || (mode != 0 && mode != 1)) return fail(ORCA_ERR_INVALID_ARGUMENT, "mode must be 0 or 1");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    CK(cudaStreamSynchronize(c->stream));
    if (mode == c->transport) return ORCA_OK;
    c->transport = mode;
    if (c->ready && c->world > 1) {
        // a new exchange sequence on every strip: counters and arrival flags from zero
        for (Domain& d : c->doms) {
            k_set_int<<<1, 1, 0, c->stream>>>(d.ctr + CT_XSTEP, 0);
            for (ExAlloc* x : {&d.recvL, &d.recvL1, &d.recvR, &d.recvR1, &d.sendL, &d.sendR})
                if (x->base) CK(cudaMemsetAsync(x->b.hdr, 0, 16, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
        CKS(setup_peers(c));
    }
    return ORCA_OK;
}

orca_status orca_get_transport(orca_ctx* c, int32_t* mode) {
    if (!c || !mode) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    *mode = c->transport;
    return ORCA_OK;
}

orca_status orca_get_launch_info(orca_ctx* c, int32_t info[4]) {
    if (!c || !info) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready || c->doms.empty()) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    // summed over the context's strips (each strip launches its own chain; strips may differ in
    // the inline-LP3 choice); NCCL's own kernels (transport 1) are not ours and not counted
    int n = 0;
    for (const Domain& d : c->doms) {
        n += (pick_lp3_inline(c, d) ? 3 : 4) - (fused_bin(c) ? 1 : 0);  // (k_bin = k_scan + k_scatter)
        if (overlap_on(c, d)) n += 1;  // the step kernel twice: boundary, then interior columns
        if (d.g.hasL || d.g.hasR) {  // strips: k_receive, and k_push per neighbour (peer memory)
            n += 1;
            if (c->transport == 0) n += (d.g.hasL ? 1 : 0) + (d.g.hasR ? 1 : 0);
        }
    }
    const Domain& d = c->doms[0];
    info[0] = pick_variant(c, d);
    info[1] = pick_lp3_inline(c, d) ? 0 : pick_lp3_lanes(c, d);
    info[2] = n;
    info[3] = c->transport;
    return ORCA_OK;
}

orca_status orca_get_kernel_config(orca_ctx* c, int32_t cfg[6]) {
    if (!c || !cfg) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready || c->doms.empty()) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    Domain& d = c->doms[0];
    const StepArgs a = make_args(c, d);
    const StepKernelCfg kc = step_kernel_cfg(c, d, a);
    cfg[0] = kc.variant;
    cfg[1] = a.lp3Inline;
    cfg[2] = kc.lm;
    cfg[3] = kc.mono;
    cfg[4] = kc.threads;
    cfg[5] = kc.mb;
    return ORCA_OK;
}

orca_status orca_get_comm_info(orca_ctx* c, int32_t info[3]) {
    if (!c || !info) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    info[0] = c->world;
    info[1] = c->rank;
    info[2] = c->world > 1 ? c->commRanks : 1;
    return ORCA_OK;
}

orca_status orca_set_overlap(orca_ctx* c, int32_t mode) {
    if (!c || mode < -1 || mode > 1) return fail(ORCA_ERR_INVALID_ARGUMENT, "mode must be -1 (auto), 0 or 1");
    CK(cudaSetDevice(c->device));
    if (c->ready && c->deferred) {  // a pending step completes before the change
        CK(cudaSetDevice(c->device));
        CK(flush_deferred(c));
    }
    CK(cudaStreamSynchronize(c->stream));
    drop_graph(c);
    c->overlapMode = mode;
    return ORCA_OK;
}

orca_status orca_set_lp3_inline(orca_ctx* c, int32_t mode) {
    if (!c || mode < -1 || mode > 2) return fail(ORCA_ERR_INVALID_ARGUMENT, "mode must be -1 (auto), 0, 1 or 2");
    CK(cudaSetDevice(c->device));
    if (c->ready && c->deferred) {  // a pending step completes before the change
        CK(cudaSetDevice(c->device));
        CK(flush_deferred(c));
    }
    CK(cudaStreamSynchronize(c->stream));
    drop_graph(c);
    c->lp3InlineMode = mode;
    return ORCA_OK;
}

orca_status orca_rebalance(orca_ctx* c) {
    if (!c) return fail(ORCA_ERR_INVALID_ARGUMENT, "null context");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    if (c->world == 1) return ORCA_OK;
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    CK(cudaStreamSynchronize(c->stream));
    CKS(check_overflow(c));
    if (c->reportCap < 3 * (int)c->doms.size() + 4) {
        dfree(c->report);
        CK(cudaMalloc(&c->report, (size_t)(3 * c->doms.size() + 4) * sizeof(int)));
        c->reportCap = 3 * (int)c->doms.size() + 4;
    }
    return rebalance(c, false);
}

orca_status orca_set_lp3_lanes(orca_ctx* c, int32_t lanes) {
    if (!c || (lanes != -1 && lanes != 1 && lanes != 4 && lanes != 8 && lanes != 16))
        return fail(ORCA_ERR_INVALID_ARGUMENT, "lanes must be -1 (auto), 1, 4, 8 or 16");
    CK(cudaSetDevice(c->device));
    if (c->ready && c->deferred) {  // a pending step completes before the change
        CK(cudaSetDevice(c->device));
        CK(flush_deferred(c));
    }
    CK(cudaStreamSynchronize(c->stream));
    drop_graph(c);
    c->lp3Lanes = lanes;
    return ORCA_OK;
}

orca_status orca_set_lp_order(orca_ctx* c, int32_t mode, uint64_t seed, int64_t first_step) {
    if (!c || mode < 0 || mode > 2) return fail(ORCA_ERR_INVALID_ARGUMENT, "mode must be 0, 1 or 2");
    if (first_step < 0 || first_step >= ((int64_t)1 << 31) - ((int64_t)1 << 24))
        return fail(ORCA_ERR_INVALID_ARGUMENT, "first_step out of range");
    CK(cudaSetDevice(c->device));
    if (c->ready && c->deferred) {  // a pending step completes before the change
        CK(cudaSetDevice(c->device));
        CK(flush_deferred(c));
    }
    CK(cudaStreamSynchronize(c->stream));
    drop_graph(c);
    c->lpMode = mode;
    c->lpSeed = seed;
    c->lpStep0 = first_step;
    c->lpMark = c->steps_total;
    CK(write_lp_step(c));
    return ORCA_OK;
}

orca_status orca_get_active(orca_ctx* c, uint8_t* active) {
    if (!c || !active) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->ready) return fail(ORCA_ERR_NOT_READY, "set_agents first");
    CK(cudaSetDevice(c->device));
    CK(flush_deferred(c));  // (orca_step_io_async left the binning to the next reader)
    const int64_t n = c->nGlobal;
    if (n > 0) {
        uint8_t* d = reinterpret_cast<uint8_t*>(c->outA);
        CK(cudaMemsetAsync(d, 0, (size_t)n, c->stream));
        for (Domain& dm : c->doms)
            k_mark_active<<<cap_blocks(dm.capW, 256), 256, 0, c->stream>>>(dm.binStart, dm.g, dm.idS, d);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(active, d, (size_t)n, cudaMemcpyDefault, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return ORCA_OK;
}

orca_status orca_set_variant(orca_ctx* c, int32_t variant) {
    if (!c || variant < -1 || variant > 4) return fail(ORCA_ERR_INVALID_ARGUMENT, "variant must be -1, 0, 1, 2, 3 or 4");
    if (c->ready && c->deferred) {  // a pending step completes before the change
        CK(cudaSetDevice(c->device));
        CK(flush_deferred(c));
    }
    CK(cudaStreamSynchronize(c->stream));
    drop_graph(c);
    c->variant = variant;
    return ORCA_OK;
}

orca_status orca_get_stream(orca_ctx* c, void** stream) {
    if (!c || !stream) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    *stream = (void*)c->stream;
    return ORCA_OK;
}

orca_status orca_probe_alu(int32_t device, double out[4]) {
    if (!out) return fail(ORCA_ERR_INVALID_ARGUMENT, "null argument");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(ORCA_ERR_INVALID_ARGUMENT, "no such CUDA device");
    CK(cudaSetDevice(device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int blocks = sms * 8, threads = 256;
    void* buf = nullptr;
    long long* cyc = nullptr;
    CK(cudaMalloc(&buf, (size_t)blocks * sizeof(double)));
    CK(cudaMalloc(&cyc, (size_t)blocks * 3 * sizeof(long long)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double best32 = 0.0, best64 = 0.0, mhz = 0.0;
    std::vector<long long> h((size_t)blocks * 3);
    for (int pass = 0; pass < 4; ++pass) {
        const bool f64 = pass & 1;
        const int iters = f64 ? 256 : 1024;
        CK(cudaEventRecord(e0, 0));
        if (f64)
            k_probe_fma<double><<<blocks, threads>>>((double*)buf, iters, 0.999999, 1e-7, cyc);
        else
            k_probe_fma<float><<<blocks, threads>>>((float*)buf, iters, 0.999999f, 1e-7f, cyc);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1, 0));
        CK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double ops = (double)blocks * threads * iters * 16.0 * kProbeChains;  // FMA lane-ops
        const double rate = ops / (ms * 1e-3);
        if (f64) {
            best64 = std::max(best64, rate);
        } else if (rate > best32) {
            best32 = rate;
            CK(cudaMemcpy(h.data(), cyc, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
            std::vector<long long> lo(1024, LLONG_MAX), hi(1024, LLONG_MIN);
            for (int q = 0; q < blocks; ++q) {
                const int sm = (int)(h[3 * q + 2] & 1023);
                lo[sm] = std::min(lo[sm], h[3 * q]);
                hi[sm] = std::max(hi[sm], h[3 * q + 1]);
            }
            long long span = 0;  // the busiest SM's cycles from its first block start to last end
            for (int q = 0; q < 1024; ++q)
                if (hi[q] > lo[q]) span = std::max(span, hi[q] - lo[q]);
            mhz = (double)span / (ms * 1e-3) / 1e6;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(cyc);
    out[0] = best32;
    out[1] = best64;
    out[2] = mhz;
    out[3] = (mhz > 0.0) ? best32 / (mhz * 1e6 * sms) : 0.0;  // FP32 FMA lanes per SM per clock
    return ORCA_OK;
}

}  // extern "C"
