// TEST INFRASTRUCTURE ONLY: a stand-in for the NCCL entry points spp_create_dist uses
// (csrc/dist.cu nccl_api), so that the one-strip-per-PROCESS path can be exercised on a box with a
// single GPU, where the real NCCL refuses two ranks on one device.  The library loads it only when
// SPP_NCCL_LIB points at it (tests/test_gpu_dist_proc.py); nothing in the product links it.
//
// Transport: one file-backed shared mapping per communicator with a byte FIFO per ordered pair of
// ranks.  A group of sends / receives is executed at ncclGroupEnd: the send buffers are copied to
// the host after the stream's earlier work, all FIFOs are progressed together (no send blocks a
// receive, so any message size is deadlock-free), and the received bytes are copied back on the
// stream before the call returns.  Messages between two ranks match in list order, as NCCL's do.
// This is stricter than NCCL (synchronous at group end) and holds none of the method's
// arithmetic.  It is a functional check, never a measurement: the ranks share one device, and no
// kernel of one rank waits on another's (all waiting is on the host).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

extern "C" {
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;       // 0 success, 2 system error, 4 invalid argument, 5 invalid usage
typedef int ncclDataType_t;
typedef struct MockComm *ncclComm_t;
}

namespace {
constexpr size_t CAP = 4u << 20;            // bytes per FIFO
struct Fifo {
    std::atomic<uint64_t> head;             // bytes written
    std::atomic<uint64_t> tail;             // bytes consumed
    char pad[48];
    char data[CAP];
};
struct Op { int send; void *buf; size_t bytes; int peer; cudaStream_t st; size_t done; std::vector<char> host; };
}  // namespace

struct MockComm {
    int nranks, rank;
    Fifo *f;                                // nranks * nranks, index src * nranks + dst
    size_t map_bytes;
    char path[128];
};

static thread_local int g_depth = 0;
static thread_local std::vector<Op> g_ops;
static thread_local MockComm *g_comm = nullptr;

static size_t dtype_size(ncclDataType_t t)
{
    switch (t) {
    case 0: case 1: return 1;
    case 2: case 3: case 7: return 4;
    case 4: case 5: case 8: return 8;
    default: return 2;
    }
}

static ncclResult_t run_ops(MockComm *c, std::vector<Op> &ops)
{
    // stage the send buffers on the host, after everything already queued on their streams
    for (Op &o : ops) {
        o.host.resize(o.bytes);
        o.done = 0;
        if (o.send && o.bytes && cudaMemcpyAsync(o.host.data(), o.buf, o.bytes, cudaMemcpyDeviceToHost, o.st) != cudaSuccess)
            return 2;
    }
    for (Op &o : ops)
        if (cudaStreamSynchronize(o.st) != cudaSuccess) return 2;
    const int P = c->nranks;
    auto t_last = std::chrono::steady_clock::now();
    const char *te = getenv("SPP_MOCK_NCCL_TIMEOUT_S");
    const double limit = te && atof(te) > 0.0 ? atof(te) : 120.0;
    for (;;) {
        bool all = true, moved = false;
        std::vector<char> busy_s(P, 0), busy_r(P, 0);   // an earlier unfinished op of the same pair goes first
        for (Op &o : ops) {
            if (o.done == o.bytes) continue;
            all = false;
            char &busy = o.send ? busy_s[o.peer] : busy_r[o.peer];
            if (busy) continue;
            busy = 1;
            Fifo &q = o.send ? c->f[(size_t)c->rank * P + o.peer] : c->f[(size_t)o.peer * P + c->rank];
            const uint64_t h = q.head.load(std::memory_order_acquire), t = q.tail.load(std::memory_order_acquire);
            size_t n = o.send ? (size_t)(CAP - (h - t)) : (size_t)(h - t);
            if (n > o.bytes - o.done) n = o.bytes - o.done;
            if (!n) continue;
            size_t pos = (size_t)((o.send ? h : t) % CAP);
            size_t first = n < CAP - pos ? n : CAP - pos;
            if (o.send) {
                memcpy(q.data + pos, o.host.data() + o.done, first);
                memcpy(q.data, o.host.data() + o.done + first, n - first);
                q.head.store(h + n, std::memory_order_release);
            } else {
                memcpy(o.host.data() + o.done, q.data + pos, first);
                memcpy(o.host.data() + o.done + first, q.data, n - first);
                q.tail.store(t + n, std::memory_order_release);
            }
            o.done += n;
            moved = true;
        }
        if (all) break;
        const auto now = std::chrono::steady_clock::now();
        if (moved) t_last = now;
        else {
            if (std::chrono::duration<double>(now - t_last).count() > limit) {
                fprintf(stderr, "[mock_nccl] rank %d: no progress for %.0f s (unmatched send/recv?)\n", c->rank, limit);
                return 2;
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
    for (Op &o : ops)
        if (!o.send && o.bytes && cudaMemcpyAsync(o.buf, o.host.data(), o.bytes, cudaMemcpyHostToDevice, o.st) != cudaSuccess)
            return 2;
    for (Op &o : ops)
        if (cudaStreamSynchronize(o.st) != cudaSuccess) return 2;
    return 0;
}

static ncclResult_t enqueue(int send, void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st)
{
    if (!c || peer < 0 || peer >= c->nranks) return 4;
    if (g_comm && g_comm != c && !g_ops.empty()) return 5;     // one communicator per group
    g_comm = c;
    g_ops.push_back(Op{send, buf, count * dtype_size(t), peer, st, 0, {}});
    if (g_depth > 0) return 0;
    std::vector<Op> ops;
    ops.swap(g_ops);
    return run_ops(c, ops);
}

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId *id)
{
    if (!id) return 4;
    memset(id, 0, sizeof(*id));
    const char *dir = getenv("SPP_MOCK_NCCL_DIR");
    snprintf(id->internal, sizeof(id->internal), "%s/spp_mock_nccl_%d_%lld", dir && *dir ? dir : "/tmp", (int)getpid(),
             (long long)std::chrono::steady_clock::now().time_since_epoch().count());
    return 0;
}

ncclResult_t ncclCommInitRank(ncclComm_t *comm, int nranks, ncclUniqueId id, int rank)
{
    if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return 4;
    id.internal[sizeof(id.internal) - 1] = 0;
    const size_t bytes = sizeof(Fifo) * (size_t)nranks * nranks;
    const int fd = open(id.internal, O_CREAT | O_RDWR, 0600);
    if (fd < 0) return 2;
    if (ftruncate(fd, (off_t)bytes) != 0) { close(fd); return 2; }     // same size on every rank; new pages read as zero
    void *p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return 2;
    MockComm *c = new MockComm;
    c->nranks = nranks; c->rank = rank; c->f = (Fifo *)p; c->map_bytes = bytes;
    memcpy(c->path, id.internal, sizeof(c->path));
    *comm = c;
    return 0;
}

ncclResult_t ncclCommDestroy(ncclComm_t c)
{
    if (!c) return 0;
    munmap(c->f, c->map_bytes);
    if (c->rank == 0) unlink(c->path);
    delete c;
    return 0;
}

ncclResult_t ncclCommCount(const ncclComm_t c, int *n) { if (!c || !n) return 4; *n = c->nranks; return 0; }
ncclResult_t ncclCommUserRank(const ncclComm_t c, int *r) { if (!c || !r) return 4; *r = c->rank; return 0; }

ncclResult_t ncclCommGetAsyncError(ncclComm_t c, ncclResult_t *e) { if (!c || !e) return 4; *e = 0; return 0; }

const char *ncclGetErrorString(ncclResult_t r)
{
    switch (r) {
    case 0: return "mock: success";
    case 2: return "mock: system error (CUDA copy, shared file, or a send/recv that never matched)";
    case 4: return "mock: invalid argument";
    case 5: return "mock: invalid usage";
    default: return "mock: error";
    }
}

ncclResult_t ncclGroupStart() { g_depth++; return 0; }

ncclResult_t ncclGroupEnd()
{
    if (g_depth <= 0) return 5;
    if (--g_depth > 0) return 0;
    std::vector<Op> ops;
    ops.swap(g_ops);
    MockComm *c = g_comm;
    g_comm = nullptr;
    if (ops.empty()) return 0;
    return run_ops(c, ops);
}

ncclResult_t ncclSend(const void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st)
{
    return enqueue(1, const_cast<void *>(buf), count, t, peer, c, st);
}

ncclResult_t ncclRecv(void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st)
{
    return enqueue(0, buf, count, t, peer, c, st);
}

}  // extern "C"
