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
    // Peer memory (fused ghost exchange, EpiPeer): rank q's workspace mapped in this process, or null.
    virtual char* peer_ws(int) { return nullptr; }
    virtual void set_ws(char*) {}
    // Stream-ordered neighbour barrier: work issued on s after peer_sync starts only when both x3
    // neighbours (rank +- 1, periodic) have issued everything before their matching peer_sync -- i.e.
    // their peer stores into this rank's ghosts are complete, and their reads of earlier fields are done.
    // pflags: this rank's flag words in its workspace (NCCL backend).
    virtual void peer_sync(cudaStream_t, uint64_t*) {}
    // Stream-ordered barrier of all ranks (the fused all-to-all transposes): work after it starts only
    // when every rank has issued everything before its matching call.  pws: device table of every rank's
    // mapped workspace (NCCL backend), pf_off: byte offset of the flag words in a workspace.
    virtual void peer_barrier_all(cudaStream_t, uint64_t*, char* const*, int64_t) {}
};

// pf[3]: epoch of the all-rank barrier; pf[8 + q]: flag written by rank q.
__global__ void k_peer_sync_all(uint64_t* pf, char* const* pws, int64_t pf_off, int rank, int P) {
    if (threadIdx.x != 0) return;
    const uint64_t e = pf[3] + 1;
    pf[3] = e;
    __threadfence_system();
    for (int q = 0; q < P; ++q) {
        uint64_t* f = reinterpret_cast<uint64_t*>(pws[q] + pf_off) + 8 + rank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
    }
    for (int q = 0; q < P; ++q) {
        uint64_t v = 0;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(pf + 8 + q) : "memory");
        } while (v < e);
    }
}

// Flag protocol of peer_sync for one process per GPU: each rank keeps an epoch counter and two flag
// words (written by its lower / upper neighbour) in its own workspace; one thread bumps the epoch,
// publishes it into both neighbours' flags (release at system scope, after a system fence that orders
// this rank's preceding peer stores) and waits until both of its own flags reach it (acquire).  The
// epoch lives in device memory, so a CUDA graph that captured the kernel stays correct on replay.
// pf: [0] epoch, [1] flag from the lower neighbour, [2] flag from the upper neighbour.
__global__ void k_peer_sync(uint64_t* pf, uint64_t* dn_from_up, uint64_t* up_from_dn) {
    if (threadIdx.x != 0) return;
    const uint64_t e = pf[0] + 1;
    pf[0] = e;
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dn_from_up), "l"(e) : "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(up_from_dn), "l"(e) : "memory");
    for (int w = 1; w <= 2; ++w) {
        uint64_t v = 0;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(pf + w) : "memory");
        } while (v < e);
    }
}

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
        // DR_NCCL_LIB (the Python binding points it at torch's bundled libnccl.so.2 when unset), then the
        // dynamic loader's search path
        const char* env = getenv("DR_NCCL_LIB");
        const char* cands[] = {env, "libnccl.so.2", "libnccl.so"};
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
        for (void* p : opened) cudaIpcCloseMemHandle(p);
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
    // NCCL kernels under stream capture (the matvec / preconditioner call graphs): opt-in with
    // DR_NCCL_GRAPHS=1 -- never exercised with more than one GPU in this build's tests, so the eager
    // path stays the default for multi-process runs
    bool capturable() const override {
        const char* e = getenv("DR_NCCL_GRAPHS");
        return e && e[0] == '1';
    }
    // CUDA IPC mappings of the neighbours' workspaces (dr_peer_import); index = rank, null if unmapped
    std::vector<char*> peers;
    std::vector<void*> opened;
    char* peer_ws(int q) override { return q >= 0 && q < (int)peers.size() ? peers[q] : nullptr; }
    void peer_sync(cudaStream_t s, uint64_t* pf) override {
        const int dn = (rank + size - 1) % size, up = (rank + 1) % size;
        // my flag words sit at the same workspace offset in every rank
        auto far = [&](int q, int w) {
            return reinterpret_cast<uint64_t*>(peers[q] + ((char*)(pf + w) - peers[rank]));
        };
        k_peer_sync<<<1, 32, 0, s>>>(pf, far(dn, 2), far(up, 1));
    }
    void peer_barrier_all(cudaStream_t s, uint64_t* pf, char* const* pws, int64_t pf_off) override {
        k_peer_sync_all<<<1, 32, 0, s>>>(pf, pws, pf_off, rank, size);
    }
    std::string check() override {
        int e = 0;
        NcclApi& A = NcclApi::get();
        A.CommGetAsyncError(comm, &e);
        return e ? std::string("NCCL async error: ") + A.GetErrorString(e) : std::string();
    }
};

// ------------------------------------------------------------------------------------------ loopback
struct Hub {
    explicit Hub(int n) : size(n), posts(n), done(n), ready(n), fin(n), ws(n, nullptr) {
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
    std::vector<char*> ws;  // each rank's workspace (peer stores of the fused ghost exchange)
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
    char* peer_ws(int q) override { return hub->ws[q]; }
    void set_ws(char* w) override { hub->ws[rank] = w; }
    // every rank records the point its stream has reached; each waits for its neighbours' (all ranks
    // here: the host barrier is global anyway) -- events only, no kernel waits on another rank's kernel
    void peer_sync(cudaStream_t s, uint64_t*) override {
        Hub& H = *hub;
        if (cudaEventRecord(H.ready[rank], s) != cudaSuccess) throw std::runtime_error("loopback: event record");
        H.barrier();
        const int dn = (rank + size - 1) % size, up = (rank + 1) % size;
        cudaStreamWaitEvent(s, H.ready[dn], 0);
        if (up != dn) cudaStreamWaitEvent(s, H.ready[up], 0);
        H.barrier();  // the events may be re-recorded by the next sync
    }
    void peer_barrier_all(cudaStream_t s, uint64_t*, char* const*, int64_t) override {
        Hub& H = *hub;
        if (cudaEventRecord(H.ready[rank], s) != cudaSuccess) throw std::runtime_error("loopback: event record");
        H.barrier();
        for (int q = 0; q < size; ++q)
            if (q != rank) cudaStreamWaitEvent(s, H.ready[q], 0);
        H.barrier();
    }
};

}  // namespace dr
