// fake_nccl.cu -- TEST INFRASTRUCTURE: a host-staged stand-in for the subset of NCCL that
// liborca uses (GetUniqueId, CommInitRank/Destroy, Send/Recv in groups, AllReduce,
// AllGather, GetErrorString), so that several processes can share ONE GPU and drive the
// strips' multi-rank code path end to end (real NCCL refuses two ranks on one device).
//
// liborca loads it instead of libnccl.so.2 when ORCA_NCCL_LIB names it.  Every operation is
// enqueued on the caller's stream as async copies through a POSIX shared-memory segment
// (cudaHostRegister'ed) plus host-function nodes that wait on / publish counters in that
// segment, so the whole thing is stream-ordered and capturable into CUDA graphs like NCCL.
// All waiting happens at execution time on counters, so graph replays stay consistent.
// Message sizes are checked: a send/recv byte-count mismatch aborts the process.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

namespace {

constexpr int kMaxRanks = 8;
constexpr size_t kSlot = 2u << 20;  // bytes per mailbox / gather slot (test-sized crowds)

struct Shared {
    std::atomic<uint64_t> seq[kMaxRanks][kMaxRanks];  // messages published src -> dst
    std::atomic<uint64_t> ack[kMaxRanks][kMaxRanks];  // messages consumed
    uint64_t len[kMaxRanks][kMaxRanks];               // bytes of the pending message
    std::atomic<uint64_t> barCount;                   // sense-reversing barrier
    std::atomic<uint64_t> barGen;
    std::atomic<int> joined;
};

size_t seg_bytes(int n) { return sizeof(Shared) + (size_t)n * n * kSlot + (size_t)n * kSlot + (size_t)n * kSlot; }

}  // namespace

struct ncclComm {
    int rank = 0, n = 1;
    char name[64] = {};
    Shared* sh = nullptr;
    unsigned char* base = nullptr;
    size_t bytes = 0;
    bool inGroup = false;
    struct Op {
        bool send;
        void* buf;
        size_t bytes;
        int peer;
        cudaStream_t st;
    };
    std::vector<Op> pending;
    unsigned char* box(int src, int dst) { return base + sizeof(Shared) + ((size_t)src * n + dst) * kSlot; }
    unsigned char* gslot(int r) { return base + sizeof(Shared) + (size_t)n * n * kSlot + (size_t)r * kSlot; }
    unsigned char* rslot(int r) { return base + sizeof(Shared) + (size_t)n * n * kSlot + (size_t)n * kSlot + r * kSlot; }
};

namespace {

std::vector<ncclComm*> g_group_comms;  // comms with ops queued in the current group

struct WaitArg {
    ncclComm* c;
    int src, dst;
    size_t bytes;
};

void CUDART_CB h_wait_free(void* p) {  // sender: previous message src->dst consumed
    WaitArg* a = static_cast<WaitArg*>(p);
    Shared* s = a->c->sh;
    while (s->ack[a->src][a->dst].load(std::memory_order_acquire) != s->seq[a->src][a->dst].load()) usleep(5);
}
void CUDART_CB h_publish(void* p) {
    WaitArg* a = static_cast<WaitArg*>(p);
    Shared* s = a->c->sh;
    s->len[a->src][a->dst] = a->bytes;
    s->seq[a->src][a->dst].fetch_add(1, std::memory_order_acq_rel);
}
void CUDART_CB h_wait_msg(void* p) {  // receiver: a message src->dst pending, of the right size
    WaitArg* a = static_cast<WaitArg*>(p);
    Shared* s = a->c->sh;
    while (s->seq[a->src][a->dst].load(std::memory_order_acquire) == s->ack[a->src][a->dst].load()) usleep(5);
    if (s->len[a->src][a->dst] != a->bytes) {
        fprintf(stderr, "fake_nccl: rank %d recv %zu bytes from %d but %llu were sent\n", a->dst, a->bytes, a->src,
                (unsigned long long)s->len[a->src][a->dst]);
        abort();
    }
}
void CUDART_CB h_consumed(void* p) {
    WaitArg* a = static_cast<WaitArg*>(p);
    a->c->sh->ack[a->src][a->dst].fetch_add(1, std::memory_order_acq_rel);
}
void CUDART_CB h_barrier(void* p) {
    ncclComm* c = static_cast<ncclComm*>(p);
    Shared* s = c->sh;
    const uint64_t gen = s->barGen.load(std::memory_order_acquire);
    if (s->barCount.fetch_add(1, std::memory_order_acq_rel) + 1 == (uint64_t)c->n) {
        s->barCount.store(0, std::memory_order_release);
        s->barGen.fetch_add(1, std::memory_order_acq_rel);
    } else {
        while (s->barGen.load(std::memory_order_acquire) == gen) usleep(5);
    }
}

struct RedArg {
    ncclComm* c;
    size_t count;
    ncclDataType_t dt;
    ncclRedOp_t op;
};
template <typename T>
void reduce_into(ncclComm* c, size_t count, ncclRedOp_t op) {
    T* out = reinterpret_cast<T*>(c->rslot(c->rank) + kSlot / 2);
    for (size_t i = 0; i < count; ++i) {
        T v = reinterpret_cast<T*>(c->rslot(0))[i];
        for (int r = 1; r < c->n; ++r) {
            const T x = reinterpret_cast<T*>(c->rslot(r))[i];
            v = (op == ncclMax) ? (x > v ? x : v) : (op == ncclMin) ? (x < v ? x : v) : (T)(v + x);
        }
        out[i] = v;
    }
}
void CUDART_CB h_reduce(void* p) {
    RedArg* a = static_cast<RedArg*>(p);
    if (a->dt == ncclInt32)
        reduce_into<int32_t>(a->c, a->count, a->op);
    else if (a->dt == ncclFloat32)
        reduce_into<float>(a->c, a->count, a->op);
    else if (a->dt == ncclUint64 || a->dt == ncclInt64)
        reduce_into<int64_t>(a->c, a->count, a->op);
    else {
        fprintf(stderr, "fake_nccl: unsupported reduction dtype %d\n", (int)a->dt);
        abort();
    }
}

size_t dt_bytes(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;
    }
}

// host-function arguments live as long as the process (graphs may replay them)
template <typename T>
T* keep(const T& v) {
    static std::vector<void*> pool;
    T* p = new T(v);
    pool.push_back(p);
    return p;
}

ncclResult_t do_send(ncclComm* c, const void* buf, size_t bytes, int peer, cudaStream_t st) {
    if (bytes > kSlot) return ncclInvalidUsage;
    WaitArg* a = keep(WaitArg{c, c->rank, peer, bytes});
    if (cudaLaunchHostFunc(st, h_wait_free, a) != cudaSuccess) return ncclUnhandledCudaError;
    if (bytes && cudaMemcpyAsync(c->box(c->rank, peer), buf, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return ncclUnhandledCudaError;
    if (cudaLaunchHostFunc(st, h_publish, a) != cudaSuccess) return ncclUnhandledCudaError;
    return ncclSuccess;
}

ncclResult_t do_recv(ncclComm* c, void* buf, size_t bytes, int peer, cudaStream_t st) {
    if (bytes > kSlot) return ncclInvalidUsage;
    WaitArg* a = keep(WaitArg{c, peer, c->rank, bytes});
    if (cudaLaunchHostFunc(st, h_wait_msg, a) != cudaSuccess) return ncclUnhandledCudaError;
    if (bytes && cudaMemcpyAsync(buf, c->box(peer, c->rank), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return ncclUnhandledCudaError;
    if (cudaLaunchHostFunc(st, h_consumed, a) != cudaSuccess) return ncclUnhandledCudaError;
    return ncclSuccess;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    memset(id, 0, sizeof(*id));
    std::random_device rd;
    snprintf(id->internal, sizeof(id->internal), "/orca_fake_nccl_%08x%08x", rd(), rd());
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    ncclComm* c = new ncclComm;
    c->rank = rank;
    c->n = nranks;
    memcpy(c->name, id.internal, sizeof(c->name) - 1);  // NUL-terminated by the zeroed id
    c->bytes = seg_bytes(nranks);
    int fd = shm_open(c->name, O_RDWR | O_CREAT, 0600);
    if (fd < 0 || ftruncate(fd, (off_t)c->bytes) != 0) return ncclSystemError;
    void* m = mmap(nullptr, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return ncclSystemError;
    c->base = static_cast<unsigned char*>(m);
    c->sh = reinterpret_cast<Shared*>(m);  // zero-filled by ftruncate
    if (cudaHostRegister(c->base, c->bytes, cudaHostRegisterPortable) != cudaSuccess) return ncclUnhandledCudaError;
    c->sh->joined.fetch_add(1);
    while (c->sh->joined.load() < nranks) usleep(100);  // all ranks attached
    *out = c;
    return ncclSuccess;
}

ncclResult_t ncclCommCount(const ncclComm_t c, int* count) {
    if (!c || !count) return ncclInvalidArgument;
    *count = c->n;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
    if (!c) return ncclSuccess;
    cudaDeviceSynchronize();
    cudaHostUnregister(c->base);
    munmap(c->base, c->bytes);
    if (c->rank == 0) shm_unlink(c->name);
    delete c;
    return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
    g_group_comms.clear();
    return ncclSuccess;
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t c, cudaStream_t st) {
    c->pending.push_back({true, const_cast<void*>(buf), count * dt_bytes(dt), peer, st});
    g_group_comms.push_back(c);
    return ncclSuccess;
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t c, cudaStream_t st) {
    c->pending.push_back({false, buf, count * dt_bytes(dt), peer, st});
    g_group_comms.push_back(c);
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
    // all sends of the group first, then the receives: no rank waits before it has sent
    for (ncclComm* c : g_group_comms) {
        for (auto& o : c->pending)
            if (o.send) {
                ncclResult_t r = do_send(c, o.buf, o.bytes, o.peer, o.st);
                if (r != ncclSuccess) return r;
            }
        for (auto& o : c->pending)
            if (!o.send) {
                ncclResult_t r = do_recv(c, o.buf, o.bytes, o.peer, o.st);
                if (r != ncclSuccess) return r;
            }
        c->pending.clear();
    }
    g_group_comms.clear();
    return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                           ncclComm_t c, cudaStream_t st) {
    const size_t b = count * dt_bytes(dt);
    if (b > kSlot / 2) return ncclInvalidUsage;
    if (cudaMemcpyAsync(c->rslot(c->rank), send, b, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return ncclUnhandledCudaError;
    cudaLaunchHostFunc(st, h_barrier, c);
    cudaLaunchHostFunc(st, h_reduce, keep(RedArg{c, count, dt, op}));
    if (cudaMemcpyAsync(recv, c->rslot(c->rank) + kSlot / 2, b, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return ncclUnhandledCudaError;
    cudaLaunchHostFunc(st, h_barrier, c);  // slots reusable
    return ncclSuccess;
}

ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t dt, ncclComm_t c,
                           cudaStream_t st) {
    const size_t b = count * dt_bytes(dt);
    if (b > kSlot) return ncclInvalidUsage;
    if (cudaMemcpyAsync(c->gslot(c->rank), send, b, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return ncclUnhandledCudaError;
    cudaLaunchHostFunc(st, h_barrier, c);
    for (int r = 0; r < c->n; ++r)
        if (cudaMemcpyAsync(static_cast<unsigned char*>(recv) + (size_t)r * b, c->gslot(r), b, cudaMemcpyHostToDevice,
                            st) != cudaSuccess)
            return ncclUnhandledCudaError;
    cudaLaunchHostFunc(st, h_barrier, c);
    return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
    static char buf[64];
    snprintf(buf, sizeof(buf), "fake_nccl error %d", (int)r);
    return buf;
}

}  // extern "C"
