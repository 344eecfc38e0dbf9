// comm.cuh -- communication layer of the slab-decomposed (multi-GPU) path.
//
// Every exchange the hot path needs is a *group* of point-to-point transfers issued on the context
// stream: the ghost-plane exchange before each semi-Lagrangian gather (the slab analogue of the
// paper's ghost layers) and the all-to-all transposes around the x3 FFT pass (the slab
// analogue of AccFFT's alltoall).  Two backends implement the same group semantics:
//
//  * NcclComm     -- one process per GPU; NCCL 2.28 (the torch-bundled libnccl.so.2, loaded with dlopen
//                    so single-GPU users never need it) grouped ncclSend/ncclRecv over NVLink/NVSwitch.
//  * LoopbackComm -- P virtual ranks in ONE process on one GPU (one host thread and one stream per
//                    rank), for testing the slab logic without P GPUs.  Transfers are device-to-device
//                    copies ordered with CUDA events; ranks rendezvous on a host barrier.  No kernel
//                    ever waits on another rank's kernel.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace dr {

struct P2P {
    bool send;        // true: send `bytes` from buf to peer; false: receive into buf from peer
    int peer;
    const void* sbuf; // send buffer (send ops)
    void* rbuf;       // receive buffer (recv ops)
    size_t bytes;
};

struct Comm {
    int rank = 0, size = 1;
    virtual ~Comm() = default;
    // Execute a group of transfers stream-ordered on s.  Sends and receives between a pair of ranks are
    // matched in the order they appear in the two ranks' lists (NCCL semantics).
    virtual void group(const std::vector<P2P>& ops, cudaStream_t s) = 0;
    virtual std::string check() { return ""; }  // asynchronous error, empty if none
    virtual bool capturable() const { return false; }  // group() may be recorded into a CUDA graph
};

// ----------------------------------------------------------------------------------------------- NCCL
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
enum { nccl_uint8 = 1 };  // ncclDataType_t ncclUint8 (= ncclChar + 1)

struct NcclApi {
    void* h = nullptr;
    int (*GetUniqueId)(ncclUniqueId*) = nullptr;
    int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*CommGetAsyncError)(ncclComm_t, int*) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;

    static NcclApi& get() {
        static NcclApi api;
        static std::once_flag once;
        std::call_once(once, [] { api.load(); });
        if (!api.h) throw std::runtime_error("libnccl.so.2 could not be loaded");
        return api;
    }
    void load() {
        const char* env = getenv("DR_NCCL_LIB");
        const char* cands[] = {env, "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
                               "libnccl.so.2", "libnccl.so"};
        for (const char* c : cands) {
            if (!c) continue;
            h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return;
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + n);
            return p;
        };
        GetUniqueId = (decltype(GetUniqueId))sym("ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))sym("ncclCommInitRank");
        CommDestroy = (decltype(CommDestroy))sym("ncclCommDestroy");
        CommGetAsyncError = (decltype(CommGetAsyncError))sym("ncclCommGetAsyncError");
        GetErrorString = (decltype(GetErrorString))sym("ncclGetErrorString");
        GroupStart = (decltype(GroupStart))sym("ncclGroupStart");
        GroupEnd = (decltype(GroupEnd))sym("ncclGroupEnd");
        Send = (decltype(Send))sym("ncclSend");
        Recv = (decltype(Recv))sym("ncclRecv");
    }
};

struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void nccl_ck(int r, const char* what) {
    if (r != 0) throw NcclError(std::string(what) + ": " + NcclApi::get().GetErrorString(r));
}

struct NcclComm : Comm {
    ncclComm_t comm = nullptr;
    NcclComm(const uint8_t uid[128], int r, int n) {
        NcclApi& A = NcclApi::get();
        ncclUniqueId id;
        std::memcpy(id.internal, uid, 128);
        rank = r;
        size = n;
        nccl_ck(A.CommInitRank(&comm, n, id, r), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm) NcclApi::get().CommDestroy(comm);
    }
    void group(const std::vector<P2P>& ops, cudaStream_t s) override {
        NcclApi& A = NcclApi::get();
        nccl_ck(A.GroupStart(), "ncclGroupStart");
        for (const P2P& o : ops) {
            if (o.bytes == 0) continue;
            if (o.send) nccl_ck(A.Send(o.sbuf, o.bytes, nccl_uint8, o.peer, comm, s), "ncclSend");
            else nccl_ck(A.Recv(o.rbuf, o.bytes, nccl_uint8, o.peer, comm, s), "ncclRecv");
        }
        nccl_ck(A.GroupEnd(), "ncclGroupEnd");
    }
    bool capturable() const override { return true; }  // NCCL kernels under stream capture
    std::string check() override {
        int e = 0;
        NcclApi& A = NcclApi::get();
        A.CommGetAsyncError(comm, &e);
        return e ? std::string("NCCL async error: ") + A.GetErrorString(e) : std::string();
    }
};

// ------------------------------------------------------------------------------------------ loopback
struct Hub {
    explicit Hub(int n) : size(n), posts(n), done(n), ready(n), fin(n) {
        for (int i = 0; i < n; ++i) {
            cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&fin[i], cudaEventDisableTiming);
        }
    }
    ~Hub() {
        for (int i = 0; i < size; ++i) {
            cudaEventDestroy(ready[i]);
            cudaEventDestroy(fin[i]);
        }
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const long g = gen;
        if (++arrived == size) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
    int size;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<std::vector<P2P>> posts;
    std::vector<int> done;
    std::vector<cudaEvent_t> ready, fin;
};

struct LoopbackComm : Comm {
    Hub* hub;
    LoopbackComm(Hub* h, int r) : hub(h) {
        rank = r;
        size = h->size;
    }
    void group(const std::vector<P2P>& ops, cudaStream_t s) override {
        Hub& H = *hub;
        // 1. publish this rank's ops and the point after which its send buffers are ready
        if (cudaEventRecord(H.ready[rank], s) != cudaSuccess) throw std::runtime_error("loopback: event record");
        H.posts[rank] = ops;
        H.barrier();
        // 2. pull every receive from the matching send of the peer (k-th recv from q <-> k-th send of q to me)
        std::vector<int> seen(size, 0);
        std::vector<char> waited(size, 0);
        for (const P2P& o : ops) {
            if (o.send) continue;
            const int q = o.peer;
            int k = seen[q]++, idx = -1;
            for (size_t i = 0; i < H.posts[q].size(); ++i) {
                const P2P& p = H.posts[q][i];
                if (p.send && p.peer == rank && k-- == 0) {
                    idx = (int)i;
                    break;
                }
            }
            if (idx < 0) throw std::runtime_error("loopback: unmatched receive");
            const P2P& p = H.posts[q][idx];
            if (p.bytes != o.bytes) throw std::runtime_error("loopback: size mismatch");
            if (!waited[q]) {
                cudaStreamWaitEvent(s, H.ready[q], 0);
                waited[q] = 1;
            }
            if (o.bytes && cudaMemcpyAsync(o.rbuf, p.sbuf, o.bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                throw std::runtime_error("loopback: copy failed");
        }
        if (cudaEventRecord(H.fin[rank], s) != cudaSuccess) throw std::runtime_error("loopback: event record");
        H.barrier();
        // 3. later writes to this rank's send buffers wait until every peer has pulled them
        for (int q = 0; q < size; ++q)
            if (q != rank) cudaStreamWaitEvent(s, H.fin[q], 0);
        H.barrier();  // posts may be overwritten by the next group
    }
};

}  // namespace dr
