// diffreg.cu -- C-ABI implementation (include/diffreg.h) of the B200 Gauss-Newton Hessian matvec of
// arXiv 1608.03630.  Host orchestration of the CUDA kernels in fft.cuh / sl.cuh / pointwise.cuh and
// of the slab exchanges in comm.cuh: every step of the hot path runs in those kernels; this file
// sizes the workspace, validates arguments and call order, and launches.  See DESIGN.md for the data
// layout and the dataflow.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <type_traits>
#include <string>
#include <vector>

#include "diffreg.h"
#include "common.cuh"
#include "fft.cuh"
#include "pointwise.cuh"
#include "sl.cuh"
#include "plane2d.cuh"
#include "comm.cuh"

using namespace dr;

namespace {

struct DrError {
    dr_status s;
    std::string msg;
};

[[noreturn]] void fail(dr_status s, const std::string& m) { throw DrError{s, m}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear the non-sticky error so the next call starts clean
        fail(DR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define CK(x) ck((x), #x)
#define CKL(name) ck(cudaGetLastError(), name)
// launch bracketing: PB(tag) before a kernel launch, PE(tag) after it (error check + accounting + profiling)

int ilog2(int n) {
    int l = 0;
    while ((1 << l) < n) ++l;
    return l;
}
bool pow2_in_range(int n) { return n >= 4 && n <= 1024 && (n & (n - 1)) == 0; }
// x2 extents that are not powers of two (one rank): even, 6 .. 510, transformed by Bluestein's chirp-z
// form through power-of-two FFTs of length M >= 2 N2 - 1 <= 1024 (fft.cuh ColBlue*)
bool blue_len(int n) { return n >= 6 && n <= 510 && n % 2 == 0 && (n & (n - 1)) != 0; }
// x1 (one rank): N1 = 2L with L not a power of two, N1 % 4 == 0 (16-byte box chunks and TMA row strides
// of the gathers), L <= 510; the half-length complex row transforms run in Bluestein form
bool blue1_len(int n) { return n >= 12 && n <= 1020 && n % 4 == 0 && ((n / 2) & (n / 2 - 1)) != 0; }
int blue_m(int n) {
    int m = 1;
    while (m < 2 * n - 1) m <<= 1;
    return m;
}

// Ghost planes of a slab: the stencil of a departure point s3 spans floor(s3)-1 ..
// floor(s3)+2, so (g, g + 1) planes cover x3 displacements |d3| <= g - 1 cells.  Default (4, 5).
constexpr int GHOST_LO = 4, GHOST_HI = 5;
int ghost_lo(const dr_config* c) { return c->ghost_lo > 0 ? c->ghost_lo : GHOST_LO; }
int ghost_hi(const dr_config* c) { return c->ghost_hi > 0 ? c->ghost_hi : GHOST_HI; }

dr_status validate(const dr_config* c, int nranks = 1) {
    if (!c) return DR_ERR_ARG;
    for (int a = 0; a < 3; ++a)
        if (!pow2_in_range(c->n[a]) && !(nranks == 1 && (a >= 1 ? blue_len(c->n[a]) : blue1_len(c->n[a]))))
            return DR_ERR_GRID;
    if (c->nt < 1 || c->nt > 64) return DR_ERR_PARAM;
    if (c->reg != DR_REG_H1 && c->reg != DR_REG_H2) return DR_ERR_PARAM;
    if (!(c->beta > 0.0) || !std::isfinite(c->beta)) return DR_ERR_PARAM;
    if (c->flags & ~(uint32_t)(DR_ISOCHORIC | DR_FP64 | DR_FULL_NEWTON | DR_CHECK_FINITE)) return DR_ERR_PARAM;
    if (nranks < 1) return DR_ERR_ARG;
    if (nranks > 1) {  // slabs: P | N3 and P | N2 (x2 blocks of the transposes), slab >= ghost width
        if (c->n[2] % nranks || c->n[1] % nranks) return DR_ERR_GRID;
        if (c->ghost_lo < 0 || c->ghost_hi < 0) return DR_ERR_PARAM;
        // a stencil spans floor(s3) - 1 .. floor(s3) + 2: even an owner serving an off-rank point at
        // its own slab edge reads one plane below and two above (ghost widths (g, g + 1), g >= 1)
        if (ghost_lo(c) < 1 || ghost_hi(c) < 2) return DR_ERR_PARAM;
        if (c->n[2] / nranks < ghost_lo(c) || c->n[2] / nranks < ghost_hi(c)) return DR_ERR_GRID;
    }
    return DR_OK;
}

Grid make_grid(const dr_config* c, int rank = 0, int nranks = 1) {
    Grid g{};
    g.n1 = c->n[0];
    g.n2 = c->n[1];
    g.n3 = c->n[2] / nranks;
    g.l1 = ilog2(g.n1);
    g.l2 = ilog2(g.n2);
    g.l3 = ilog2(g.n3);
    g.M = (int64_t)g.n1 * g.n2 * g.n3;
    g.n1c = g.n1 / 2 + 1;
    g.n1p = ((g.n1c + 15) / 16) * 16;
    g.S = (int64_t)g.n3 * g.n2 * g.n1p;
    g.z0 = rank * g.n3;
    g.n3g = c->n[2];
    g.ghost = nranks > 1;
    g.zg = g.ghost ? ghost_lo(c) : 0;
    g.zgh = g.ghost ? ghost_hi(c) : 0;
    return g;
}

bool is_device_ptr(const void* p);  // (defined with the C ABI below)

int64_t n_tiles(const Grid& g) {
    return (int64_t)((g.n1 + SL_TX - 1) / SL_TX) * ((g.n2 + SL_TY - 1) / SL_TY) * ((g.n3 + SL_TZ - 1) / SL_TZ);
}

// Workspace layout (byte offsets, 256-aligned).  "Ghosted" slots (the fields semi-Lagrangian gathers
// read: rho_j, lambda_j, lambda~_j / g_j, rho~(1), div v, and each velocity component) hold
// zg + n3 + zgh planes; every other slot holds the slab's n3 planes.
struct Layout {
    size_t F, GF, vstride;
    int64_t rcap = 0;
    size_t rem = 0;
    size_t kry, sN, bN, sc, rhoT, rhoR, v, vin, dp, dm, m, D, rho, G, lam, lt, rt1, bt, tmp3, stin, stout, specD, specF, xs, xr, plan_p,
        plan_m, plan_t, maxext, red, pflags, twx, twy, twz, twxd, twyd, twzd, blue, blue3, blue1, total;
};

Layout layout(const dr_config* c, int nranks = 1) {
    const Grid g = make_grid(c, 0, nranks);
    const size_t es = (c->flags & DR_FP64) ? 8 : 4;
    const size_t plane = (size_t)g.n1 * g.n2;
    const int nt = c->nt;
    const bool dist = nranks > 1;
    Layout L{};
    L.F = (size_t)g.M * es;
    L.GF = ((size_t)(g.n3 + g.zg + g.zgh) * plane * es + 255) & ~(size_t)255;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    L.rhoT = take(L.GF);                      // rho_0 = rho_T (ghosted)
    L.rhoR = take(L.F);
    L.v = take(3 * L.GF);                     // velocity components (ghosted)
    L.vin = (c->flags & DR_ISOCHORIC) ? take(3 * L.F) : 0;  // the caller's v before projection
    L.vstride = L.GF / es;
    L.dp = take(3 * L.F);
    L.dm = take(3 * L.F);
    L.m = take(L.F);
    L.D = take(L.GF);
    L.rho = take((size_t)nt * L.GF);          // rho_1..rho_nt
    L.G = take((size_t)(nt + 1) * 3 * L.F);   // grad rho_j
    L.lam = take((size_t)(nt + 1) * L.GF);    // lambda_j
    L.lt = take((size_t)nt * L.GF);           // lambda~_0..lambda~_{nt-1} (also the g_j of the inc-state sweep)
    L.rt1 = take(L.GF);                       // rho~(1)
    L.bt = take(3 * L.F);                     // b~
    L.tmp3 = take(3 * L.F);                   // d* and scratch
    L.stin = take(3 * L.F);                   // host staging in
    L.stout = take(3 * L.F);                  // host staging out
    L.kry = take(5 * 3 * L.F);                // PCG work vectors r, z, p, q, dv (NEXT-2)
    const bool newton = c->flags & DR_FULL_NEWTON;
    L.sN = newton ? take((size_t)(nt + 1) * L.GF) : 0;  // NEXT-3: s_k = div(lam_k vt) (gathered: ghosted)
    L.bN = newton ? take(3 * L.F) : 0;                   // NEXT-3: int lam grad rho~ dt
    L.sc = newton ? take(L.F) : 0;                       // NEXT-3: rho~_j scratch
    // forward half spectra (complex<double>): 6 (+2 transpose buffers with slabs); inverse-direction
    // (complex<T>): 3 (+2)
    L.specD = take((size_t)(dist ? 8 : 6) * g.S * 16);
    L.specF = take((size_t)(dist ? 5 : 3) * g.S * 2 * es);
    // off-rank departure points (dist only): per displacement field (d*, d+, d-) ids + records out and in,
    // values out and in (3 components), capacity M / 8 points each way
    L.rcap = dist ? std::max<int64_t>(1024, g.M / 8) : 0;
    const size_t es2 = es;
    L.rem = dist ? take(3 * (size_t)L.rcap * (2 * 4 + 2 * (12 + 3 * es2) + 2 * 3 * es2) + 3 * 4 * 4 * 64) : 0;
    L.xs = dist ? take(L.F) : 0;              // real-field transpose buffers (x3 derivatives)
    L.xr = dist ? take(L.F) : 0;
    const size_t pb = (size_t)n_tiles(g) * PLAN_INTS * sizeof(int);
    L.plan_p = take(pb);
    L.plan_m = take(pb);
    L.plan_t = take(pb);
    L.maxext = take(16 * sizeof(int));
    L.red = take(4096 * sizeof(double));  // reduction partials + per-rank gather slots
    L.pflags = take(2048);                // peer barriers: epochs + flags (bytes 0..1023), rank workspace table (1024..)
    L.twx = take((size_t)g.n1 * 2 * es);
    L.twy = take((size_t)g.n2 * 2 * es);
    L.twz = take((size_t)g.n3g * 2 * es);
    L.twxd = take((size_t)g.n1 * 16);
    L.twyd = take((size_t)g.n2 * 16);
    L.twzd = take((size_t)g.n3g * 16);
    // Bluestein tables of a non-power-of-two x2 extent, fp32 then fp64: twM[M], w_fwd[N], w_inv[N],
    // bhat_fwd[M], bhat_inv[M]
    L.blue = blue_len(g.n2) ? take((size_t)(3 * blue_m(g.n2) + 2 * g.n2) * (8 + 16)) : 0;
    L.blue3 = blue_len(g.n3g) ? take((size_t)(3 * blue_m(g.n3g) + 2 * g.n3g) * (8 + 16)) : 0;  // the same for x3
    L.blue1 = blue1_len(g.n1) ? take((size_t)(3 * blue_m(g.n1 / 2) + g.n1) * (8 + 16)) : 0;  // x1 rows: L = N1 / 2
    L.total = off;
    return L;
}

}  // namespace

struct dr_comm {
    std::unique_ptr<dr::Comm> impl;
};
struct dr_hub {
    std::unique_ptr<dr::Hub> impl;
};

struct dr_ctx {
    dr_config cfg;
    Grid g;
    Layout L;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;               // second stream: spectral work that overlaps the gathers
    cudaStream_t hi = nullptr;                // high-priority stream: the gather sweeps while aux runs
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_hi = nullptr;
    bool overlap = false;                     // DR_OVERLAP=1 in the environment at dr_create
    bool window = false;                      // DR_WINDOW=1: sliding-window fp32 gathers (sl.cuh k_sl_window)
    bool pairs = false;                       // DR_PAIRS=1: x3-adjacent shared-plane pair gathers (sl.cuh k_sl_pairs)
    bool gather_tma = true;                   // DR_GATHER_TMA=0: gather boxes staged by cp.async only
    bool plane2d = false;                     // DR_PLANE2D=1: fused x1/x2 cluster plane transforms (plane2d.cuh)
    int ring = 0;                             // DR_RING=P: x1/x2 pass pairs per P planes through an L2-resident scratch
    bool peer_ghosts = false;                 // DR_PEER_GHOSTS=1 (slabs): gathers store boundary planes into the
                                              // neighbours' ghosts (EpiPeer); consumers peer_sync instead of exchanging
    const void* last_peer_out = nullptr;      // the field whose ghosts the last peer-storing gather filled
    bool peer_inv_fresh = false;              // the last middle pass stored its transpose chunks into the ranks' specF(3)
    bool pws_ready = false;                   // the device table of mapped rank workspaces is filled
    bool tma_middle = true;                   // DR_TMA_MIDDLE=0 at dr_create: the unstaged fp32 middle pass
    bool graphs = true;                       // DR_GRAPHS=0 disables the CUDA-graph PCG iteration
    int chunk = 0;                            // DR_CHUNK=P: x1/x2 pass pairs run per P planes (L2 reuse)
    cudaGraphExec_t pcg_graph = nullptr;      // one captured PCG iteration (single rank), reused
    double* pinned = nullptr;                 // pinned host scalar the graph reports |r|^2 into
    struct RemotePlanH {                      // host side of an off-rank plan (per displacement field)
        bool any = false;                     // some rank has remote points for this field
        std::vector<int> out_cnt, out_off, in_cnt, in_off;
        int n_out = 0, n_in = 0;
    } rp[3];
    int num_sms = 148;
    int dev = 0;                              // CUDA device the context was created on
    int rank = 0, nranks = 1;
    dr::Comm* comm = nullptr;  // not owned; NULL with one rank
    char* ws = nullptr;
    bool own_ws = false;
    bool have_images = false, have_velocity = false, have_state = false, have_adjoint = false, have_matvec = false;
    std::string err;
    // launch accounting and optional per-kernel CUDA-event profiling (dr_profile_*)
    int64_t launches = 0;
    bool prof = false;
    std::string prof_only;  // non-empty: time only the launches with this tag (dr_profile_only)
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Pending { const char* tag; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    // Captured matvec / preconditioner calls (dr_hessian_matvec, dr_precond_apply), keyed by their
    // argument pointers; the CUDA graph holds every launch of the call (and, with NCCL slabs, its
    // send/recv), replayed with one cudaGraphLaunch.  Invalidated by set_images / set_velocity (the
    // off-rank plans' host counts are baked into the launches) and by profiler changes.
    struct CallGraph {
        int kind = 0;
        const void* a = nullptr;
        const void* b = nullptr;
        uint64_t epoch = 0;
        std::string prof_sig;
        cudaGraph_t graph = nullptr;          // kept: its event-record nodes are retargeted per replay
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;                 // kernel launches one replay performs
        struct EvNode { const char* tag; cudaGraphNode_t a, b; };
        std::vector<EvNode> ev;               // profiled launches: start / end event-record nodes
        std::vector<cudaEvent_t> own;         // the events recorded at capture (identify the nodes)
    };
    std::vector<CallGraph> call_graphs;
    uint64_t graph_epoch = 1;
    bool capturing = false;                   // profiler events go to cap_ev, not the pending list
    std::vector<Pending> cap_ev;
    std::vector<cudaEvent_t> graph_events;    // events recorded by the PCG graph's nodes
    struct Acc { std::string tag; int64_t n = 0; double ms = 0; };
    std::vector<Acc> acc;
    cudaEvent_t cur_start = nullptr;
    bool dist() const { return nranks > 1; }
    cudaEvent_t take_event() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
    bool prof_on(const char* tag) const { return prof && (prof_only.empty() || prof_only == tag); }
    void prof_begin(const char* tag, cudaStream_t st) {
        if (prof_on(tag)) {
            if (capturing) {  // a dedicated event, recorded as a graph node (retargeted at every replay)
                cudaEventCreate(&cur_start);
                cudaEventRecordWithFlags(cur_start, st, cudaEventRecordExternal);
            } else {
                cur_start = take_event();
                cudaEventRecord(cur_start, st);
            }
        }
    }
    void prof_end(const char* tag, cudaStream_t st);
    void prof_flush();
    template <typename T>
    T* at(size_t off) const { return reinterpret_cast<T*>(ws + off); }
};

void dr_ctx::prof_end(const char* tag, cudaStream_t st) {
    ck(cudaGetLastError(), tag);
    ++launches;
    if (prof_on(tag)) {
        cudaEvent_t e;
        if (capturing) {
            cudaEventCreate(&e);
            cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
        } else {
            e = take_event();
            cudaEventRecord(e, st);
        }
        (capturing ? cap_ev : pending).push_back(Pending{tag, cur_start, e});
    }
}

void dr_ctx::prof_flush() {
    if (pending.empty()) return;
    for (const Pending& p : pending) CK(cudaEventSynchronize(p.b));
    for (const Pending& p : pending) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, p.a, p.b));
        auto it = std::find_if(acc.begin(), acc.end(), [&](const Acc& a) { return a.tag == p.tag; });
        if (it == acc.end()) {
            acc.push_back(Acc{p.tag, 0, 0});
            it = acc.end() - 1;
        }
        it->n += 1;
        it->ms += ms;
    }
    pending.clear();
    ev_used = 0;
}

namespace {

template <typename T>
struct V3 {  // a vector field as three component pointers
    T* c[3];
};
template <typename T>
V3<T> vec(T* base, size_t stride) { return V3<T>{{base, base + stride, base + 2 * stride}}; }
template <typename T>
V3<const T> cvec(const V3<T>& v) { return V3<const T>{{v.c[0], v.c[1], v.c[2]}}; }

template <typename T>
__global__ void k_pack_split(Grid g, const T* __restrict__ f, T* __restrict__ out, int nb) {
    // [i3][i2][i1] -> [i2 / nb][i3][i2 % nb][i1]
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.M; e += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(e % g.n1);
        const int64_t r = e / g.n1;
        const int y = (int)(r % g.n2), z = (int)(r / g.n2);
        out[((((int64_t)(y / nb) * g.n3 + z) * nb) + (y % nb)) * g.n1 + x] = f[e];
    }
}
template <typename T>
__global__ void k_unpack_split(Grid g, const T* __restrict__ in, T* __restrict__ f, int nb, int accumulate) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.M; e += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(e % g.n1);
        const int64_t r = e / g.n1;
        const int y = (int)(r % g.n2), z = (int)(r / g.n2);
        const T v = in[((((int64_t)(y / nb) * g.n3 + z) * nb) + (y % nb)) * g.n1 + x];
        f[e] = accumulate ? f[e] + v : v;
    }
}

template <typename T>
struct Impl {
    dr_ctx& c;
    const Grid& g;
    cudaStream_t s;
    explicit Impl(dr_ctx& cc) : c(cc), g(cc.g), s(cc.stream) {}
    Impl(dr_ctx& cc, const Grid& gg, cudaStream_t st) : c(cc), g(gg), s(st) {}  // a plane range of the grid
    void PB(const char* tag) { c.prof_begin(tag, s); }
    void PE(const char* tag) { c.prof_end(tag, s); }

    size_t plane() const { return (size_t)g.n1 * g.n2; }
    T* gf(size_t off) { return c.at<T>(off) + (size_t)g.zg * plane(); }  // interior of a ghosted slot
    size_t gstride() const { return c.L.GF / sizeof(T); }
    T dt() const { return T(1) / T(c.cfg.nt); }
    T* rhoT() { return gf(c.L.rhoT); }
    T* rhoR() { return c.at<T>(c.L.rhoR); }
    T* vc(int a) { return gf(c.L.v) + (size_t)a * gstride(); }
    V3<T> v3() { return V3<T>{{vc(0), vc(1), vc(2)}}; }
    T* vraw() { return c.at<T>(c.L.vin); }
    T* sN(int k) { return gf(c.L.sN) + (size_t)k * gstride(); }
    T* bN() { return c.at<T>(c.L.bN); }
    T* sc() { return c.at<T>(c.L.sc); }
    bool newton() const { return c.cfg.flags & DR_FULL_NEWTON; }
    T* dplus() { return c.at<T>(c.L.dp); }
    T* dminus() { return c.at<T>(c.L.dm); }
    T* mult() { return c.at<T>(c.L.m); }
    T* Dv() { return gf(c.L.D); }
    T* rho(int j) { return j == 0 ? rhoT() : gf(c.L.rho) + (size_t)(j - 1) * gstride(); }
    T* G(int j) { return c.at<T>(c.L.G) + (size_t)j * 3 * g.M; }
    V3<T> G3(int j) { return vec(G(j), (size_t)g.M); }
    T* lam(int j) { return gf(c.L.lam) + (size_t)j * gstride(); }
    T* lt(int j) { return gf(c.L.lt) + (size_t)j * gstride(); }
    T* rt1() { return gf(c.L.rt1); }
    T* bt() { return c.at<T>(c.L.bt); }
    T* tmp3() { return c.at<T>(c.L.tmp3); }
    T* stin() { return c.at<T>(c.L.stin); }
    T* stout() { return c.at<T>(c.L.stout); }
    T* xs() { return c.at<T>(c.L.xs); }
    T* xr() { return c.at<T>(c.L.xr); }
    Cx<double>* specD(int i) { return c.at<Cx<double>>(c.L.specD) + (size_t)i * g.S; }
    Cx<T>* specF(int i) { return c.at<Cx<T>>(c.L.specF) + (size_t)i * g.S; }
    const Cx<T>* twx() { return c.at<Cx<T>>(c.L.twx); }
    const Cx<T>* twy() { return c.at<Cx<T>>(c.L.twy); }
    const Cx<T>* twz() { return c.at<Cx<T>>(c.L.twz); }
    const Cx<double>* twxd() { return c.at<Cx<double>>(c.L.twxd); }
    const Cx<double>* twyd() { return c.at<Cx<double>>(c.L.twyd); }
    const Cx<double>* twzd() { return c.at<Cx<double>>(c.L.twzd); }
    T* mult_or_null() { return (c.cfg.flags & DR_ISOCHORIC) ? nullptr : mult(); }

    int grid_1d(int64_t n, int block = 256) const {
        int64_t b = (n + block - 1) / block;
        return (int)std::min<int64_t>(b, 148 * 16);
    }

    // -------------------------------------------------------------------- slab exchanges
    int nb() const { return g.n2 / c.nranks; }  // x2 block of one rank in the transposed layout
    void exchange(const std::vector<P2P>& ops) {
        PB("exchange");
        try {
            c.comm->group(ops, s);
        } catch (const NcclError& e) {
            fail(DR_ERR_NCCL, e.what());
        } catch (const std::exception& e) {
            fail(DR_ERR_NCCL, e.what());
        }
        PE("exchange");
    }
    // ghost planes of a ghosted scalar field (interior pointer f): my top zg planes go to rank + 1 (its
    // lower ghosts), my bottom zgh planes to rank - 1 (its upper ghosts); periodic in rank.
    // fused ghost exchange: every rank's peer-storing gathers run in the same order, so all ranks agree
    // on whether a field's ghosts were filled by its producer (then only the neighbour barrier remains)
    bool peer_on() const {
        if (!c.dist() || !c.peer_ghosts) return false;
        const int P = c.nranks;
        return c.comm->peer_ws((c.rank + 1) % P) && c.comm->peer_ws((c.rank + P - 1) % P);
    }
    void peer_sync() {
        PB("peer_sync");
        c.comm->peer_sync(s, c.at<uint64_t>(c.L.pflags));
        PE("peer_sync");
    }
    // fused all-to-all transposes: every rank's workspace mapped (loopback: all contexts; NCCL: all IPC
    // handles imported), at most 64 ranks
    bool peer_a2a_on() {
        if (!c.dist() || !c.peer_ghosts || c.nranks > 64) return false;
        for (int q = 0; q < c.nranks; ++q)
            if (!c.comm->peer_ws(q)) return false;
        if (!c.pws_ready) {  // the device table of rank workspaces, read by the peer-storing passes
            std::vector<char*> h(c.nranks);
            for (int q = 0; q < c.nranks; ++q) h[q] = c.comm->peer_ws(q);
            CK(cudaMemcpyAsync(pws(), h.data(), h.size() * sizeof(char*), cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));
            c.pws_ready = true;
        }
        return true;
    }
    char** pws() { return reinterpret_cast<char**>(c.ws + c.L.pflags + 1024); }
    void peer_barrier_all() {
        PB("peer_barrier");
        c.comm->peer_barrier_all(s, c.at<uint64_t>(c.L.pflags), pws(), (int64_t)c.L.pflags);
        PE("peer_barrier");
    }
    void ghosts(T* f) {
        if (!c.dist()) return;
        if (f == c.last_peer_out) {  // the producing gather already stored them (EpiPeer)
            c.last_peer_out = nullptr;
            peer_sync();
            return;
        }
        c.last_peer_out = nullptr;
        const int P = c.nranks, up = (c.rank + 1) % P, dn = (c.rank + P - 1) % P;
        const size_t pl = plane() * sizeof(T);
        std::vector<P2P> ops = {
            P2P{true, up, f + (size_t)(g.n3 - g.zg) * plane(), nullptr, g.zg * pl},
            P2P{false, dn, nullptr, f - (size_t)g.zg * plane(), g.zg * pl},
            P2P{true, dn, f, nullptr, g.zgh * pl},
            P2P{false, up, nullptr, f + (size_t)g.n3 * plane(), g.zgh * pl},
        };
        exchange(ops);
    }
    // all-to-all of P equal contiguous chunks: chunk q of send goes to rank q, chunk q of recv comes
    // from rank q
    void alltoall(const void* send, void* recv, size_t chunk_bytes) {
        std::vector<P2P> ops;
        for (int q = 0; q < c.nranks; ++q) {
            ops.push_back(P2P{true, q, static_cast<const char*>(send) + q * chunk_bytes, nullptr, chunk_bytes});
            ops.push_back(P2P{false, q, nullptr, static_cast<char*>(recv) + q * chunk_bytes, chunk_bytes});
        }
        exchange(ops);
    }

    // -------------------------------------------------------------------- twiddle tables
    template <typename U>
    void fill_twiddles(int n, size_t off) {
        std::vector<Cx<U>> h(n);
        for (int m = 0; m < n; ++m) {
            const long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)n;
            h[m].re = (U)std::cos(a);
            h[m].im = (U)std::sin(a);
        }
        CK(cudaMemcpyAsync(c.ws + off, h.data(), sizeof(Cx<U>) * n, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    // Bluestein tables (fft.cuh ColBlue*), fp32 then fp64, from long double: w_j = e^{D i pi (j^2 mod 2N) / N},
    // b_j = conj(w_j) for |j| < N placed circularly in M, bhat = DFT_M(b) / M (direct sum: M <= 1024)
    static size_t blue_bytes_f(int n) { return (size_t)(3 * blue_m(n) + 2 * n) * sizeof(Cx<float>); }
    void fill_blue(size_t off, int n) {
        const int M = blue_m(n);
        const long double pi = 3.141592653589793238462643383279502884L;
        std::vector<long double> re((size_t)3 * M + 2 * n), im((size_t)3 * M + 2 * n);
        for (int m = 0; m < M; ++m) {
            const long double a = -2.0L * pi * (long double)m / (long double)M;
            re[m] = std::cos(a);
            im[m] = std::sin(a);
        }
        for (int d = 0; d < 2; ++d) {
            const long double sg = d == 0 ? -1.0L : 1.0L;
            std::vector<long double> br(M, 0.0L), bi(M, 0.0L);
            for (int j = 0; j < n; ++j) {
                const long long q = ((long long)j * j) % (2LL * n);
                const long double a = sg * pi * (long double)q / (long double)n;
                re[(size_t)M + (size_t)d * n + j] = std::cos(a);
                im[(size_t)M + (size_t)d * n + j] = std::sin(a);
                br[j] = std::cos(a);
                bi[j] = -std::sin(a);
                if (j > 0) {
                    br[M - j] = br[j];
                    bi[M - j] = bi[j];
                }
            }
            for (int k = 0; k < M; ++k) {
                long double sr = 0.0L, si = 0.0L;
                for (int j = 0; j < M; ++j) {
                    if (br[j] == 0.0L && bi[j] == 0.0L) continue;
                    const long double a = -2.0L * pi * (long double)(((long long)j * k) % M) / (long double)M;
                    const long double cr = std::cos(a), ci = std::sin(a);
                    sr += br[j] * cr - bi[j] * ci;
                    si += br[j] * ci + bi[j] * cr;
                }
                re[(size_t)M + 2 * n + (size_t)d * M + k] = sr / M;
                im[(size_t)M + 2 * n + (size_t)d * M + k] = si / M;
            }
        }
        std::vector<Cx<float>> hf(re.size());
        std::vector<Cx<double>> hd(re.size());
        for (size_t i = 0; i < re.size(); ++i) {
            hf[i] = Cx<float>{(float)re[i], (float)im[i]};
            hd[i] = Cx<double>{(double)re[i], (double)im[i]};
        }
        CK(cudaMemcpyAsync(c.ws + off, hf.data(), hf.size() * sizeof(Cx<float>), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(c.ws + off + blue_bytes_f(n), hd.data(), hd.size() * sizeof(Cx<double>), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    template <typename U>
    BlueTab<U> bluetab_at(size_t base, int n) {
        const int M = blue_m(n);
        const Cx<U>* t = reinterpret_cast<const Cx<U>*>(c.ws + base + (sizeof(U) == 8 ? blue_bytes_f(n) : 0));
        return BlueTab<U>{t, {t + M, t + M + n}, {t + M + 2 * n, t + 2 * M + 2 * n}, n};
    }
    template <typename U>
    BlueTab<U> bluetab() { return bluetab_at<U>(c.L.blue, g.n2); }
    BlueTab<double> bluetab3() { return bluetab_at<double>(c.L.blue3, g.n3g); }
    template <typename U>
    BlueTab<U> bluetab1() { return bluetab_at<U>(c.L.blue1, g.n1 / 2); }
    bool blue1() const { return blue1_len(g.n1); }
    bool blue3() const { return blue_len(g.n3g); }
    bool blue2() const { return blue_len(g.n2); }
    void init_twiddles() {
        if (blue2()) fill_blue(c.L.blue, g.n2);
        if (blue3()) fill_blue(c.L.blue3, g.n3g);
        if (blue1()) fill_blue(c.L.blue1, g.n1 / 2);
        fill_twiddles<T>(g.n1, c.L.twx);
        fill_twiddles<T>(g.n2, c.L.twy);
        fill_twiddles<T>(g.n3g, c.L.twz);
        fill_twiddles<double>(g.n1, c.L.twxd);
        fill_twiddles<double>(g.n2, c.L.twyd);
        fill_twiddles<double>(g.n3g, c.L.twzd);
    }

    // -------------------------------------------------------------------- FFT pass launchers
    template <typename K>
    static void set_smem(K kernel, size_t bytes) {
        if (bytes > 48 * 1024) CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    }

    // Launch of an FFT pass: one CTA per tile.
    // Batched launches (nc > 1, blockIdx.y = component) carry the tag suffix "_x<nc>".
    static const char* tag_n(const char* tag, int nc) {
        if (nc == 1) return tag;
        static std::mutex mu;               // contexts may be driven from several host threads
        static std::set<std::string> pool;  // stable storage for composed tags
        std::lock_guard<std::mutex> lock(mu);
        return pool.insert(std::string(tag) + "_x" + std::to_string(nc)).first->c_str();
    }
    // resident CTAs per SM of a kernel with `smem` dynamic shared memory (sets the smem attribute)
    template <class K>
    static int occupancy(K k, int nt, size_t smem) {
        set_smem(k, smem);
        int n = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, nt, smem));
        return std::max(n, 1);
    }
    // Function attributes belong to the device context: cache the occupancy (and the smem attribute set
    // by occupancy()) per kernel instantiation AND device (a process may drive contexts on several GPUs).
    static constexpr int MAX_DEV = 64;
    template <class K>
    int per_device_occupancy(K k, int nt, size_t smem) {
        static std::atomic<int> cache[MAX_DEV];  // 0: not yet queried on that device
        const int d = c.dev < MAX_DEV ? c.dev : MAX_DEV - 1;
        int v = cache[d].load(std::memory_order_relaxed);
        if (v == 0 || c.dev >= MAX_DEV) {
            v = occupancy(k, nt, smem);
            cache[d].store(v, std::memory_order_relaxed);
        }
        return v;
    }
    template <class PassT>
    void stream(const char* tag, const PassT& pass, int64_t ntiles, int nc = 1) {
        auto k = k_stream<PassT>;
        per_device_occupancy(k, PassT::NT, PassT::BUF);  // sets the smem attribute on this device once
        tag = tag_n(tag, nc);
        PB(tag);
        k<<<dim3((unsigned)ntiles, (unsigned)nc), PassT::NT, PassT::BUF, s>>>(pass);
        PE(tag);
    }
    template <int RB>
    int64_t row_tiles() const { return ((int64_t)g.n2 * g.n3 + RB - 1) / RB; }
    // Launch of a staged row pass (fft.cuh k_rows): persistent, one wave of resident CTAs.
    template <class PassT>
    void stream_rows(const char* tag, const PassT& pass, int nc = 1) {
        auto k = k_rows<PassT>;
        const int per_sm = per_device_occupancy(k, PassT::NT, PassT::BUF);
        const int64_t nt = row_tiles<PassT::RB>();
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nt, (int64_t)per_sm * c.num_sms / nc));
        tag = tag_n(tag, nc);
        PB(tag);
        k<<<dim3(grid, nc), PassT::NT, PassT::BUF, s>>>(pass, (int)nt);
        PE(tag);
    }
    // the bulk-copy engine needs 16-byte aligned rows (all workspace fields are; caller buffers may not be)
    static bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

    template <int L>
    void row_deriv_L(const T* f, T* out, int acc, int nf = 1, int64_t fs = 0, int64_t os = 0) {
        using PT = RowDerivPass<T, L>;  // (a staged variant measured 46 -> 50 us: fewer warps for the compute)
        stream("row_deriv", PT{g, f, out, acc, twx(), fs, os}, row_tiles<PT::RB>(), nf);
    }
    // twiddle tables by compute type (the forward spectral passes run in double, or in T for symbols that
    // damp high wavenumbers -- see spec_forward)
    template <typename U> const Cx<U>* twx_t() { if constexpr (sizeof(U) == sizeof(double)) return reinterpret_cast<const Cx<U>*>(twxd()); else return reinterpret_cast<const Cx<U>*>(twx()); }
    template <typename U> const Cx<U>* twy_t() { if constexpr (sizeof(U) == sizeof(double)) return reinterpret_cast<const Cx<U>*>(twyd()); else return reinterpret_cast<const Cx<U>*>(twy()); }
    template <typename U> const Cx<U>* twz_t() { if constexpr (sizeof(U) == sizeof(double)) return reinterpret_cast<const Cx<U>*>(twzd()); else return reinterpret_cast<const Cx<U>*>(twz()); }
    template <typename U> Cx<U>* specD_t(int i) { return reinterpret_cast<Cx<U>*>(c.ws + c.L.specD) + (size_t)i * g.S; }

    // (nc components at element strides csf (real fields) / css (spectra) in one launch)
    template <int L, typename Tc>
    void row_r2c_L(const T* f, Cx<Tc>* sp, int nc, int64_t csf, int64_t css) {
        const char* tag = sizeof(Tc) == 8 ? "row_r2c_f64" : "row_r2c_f32";
        // staged (bulk-copy prefetch, shared stage-major twiddles) in either precision: fp32 101 -> 79 us,
        // fp64 148 -> 129 us for three components at 256^3 once the twiddle reads stopped conflicting
        if (al16(f)) {
            stream_rows(tag, RowR2cStaged<T, Tc, L>{g, f, sp, twx_t<Tc>(), csf, css}, nc);
            return;
        }
        using PT = RowR2cPass<T, Tc, L>;
        stream(tag, PT{g, f, sp, twx_t<Tc>(), csf, css}, row_tiles<PT::RB>(), nc);
    }
    template <int L>
    void row_c2r_L(const Cx<T>* sp, T* out, const T* add, int nc, int64_t csf, int64_t css) {
        if (al16(sp) && al16(add)) {
            if (add) stream_rows("row_c2r_add", RowC2rStaged<T, L, true>{g, sp, RowOut<T>{out, add}, twx(), csf, css}, nc);
            else stream_rows("row_c2r", RowC2rStaged<T, L, false>{g, sp, RowOut<T>{out, nullptr}, twx(), csf, css}, nc);
            return;
        }
        using PT = RowC2rPass<T, L>;
        stream(add ? "row_c2r_add" : "row_c2r", PT{g, sp, RowOut<T>{out, add}, twx(), csf, css}, row_tiles<PT::RB>(), nc);
    }

    // Fused x1/x2 plane transforms (plane2d.cuh): one rank, fp32 fields, N1 = N2 = 256.  Persistent
    // clusters of 8 CTAs (one per SM), as many as can be co-resident.
    // scratch ring of 3 components x c.ring planes of half spectra (after the 3 batched spectrum slots;
    // the forward (Tc) and inverse (T) rings share the same bytes, so the lines stay L2-resident)
    bool ring_ok() const { return c.ring > 0 && !c.dist() && c.ring < g.n3 && g.n3 % c.ring == 0; }
    template <typename U>
    Cx<U>* ring_scratch() { return reinterpret_cast<Cx<U>*>(specD(3)); }
    bool plane2d_ok(const void* a, const void* b) const {
        return c.plane2d && !c.dist() && std::is_same<T, float>::value && g.n1 == 256 && g.n2 == 256 && al16(a) && al16(b);
    }
    template <class K>
    int plane_clusters(K k, size_t smem, int nitems) {
        set_smem(k, smem);
        static std::atomic<int> cache[MAX_DEV];
        const int d = c.dev < MAX_DEV ? c.dev : MAX_DEV - 1;
        int n = cache[d].load(std::memory_order_relaxed);
        if (n == 0) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(8 * 16);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 8;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CK(cudaOccupancyMaxActiveClusters(&n, k, &cfg));
            n = std::max(n, 1);
            cache[d].store(n, std::memory_order_relaxed);
        }
        return std::min(n, nitems);
    }
    template <typename Tc>
    void fwd2d(const T* f, Cx<Tc>* sp, int nc, int64_t csf, int64_t css) {
        if constexpr (std::is_same<T, float>::value) {
            auto k = k_plane_fwd<float, Tc>;
            constexpr size_t sm = plane_fwd_smem<float, Tc>();
            const int nitems = nc * g.n3;
            const int ncl = plane_clusters(k, sm, nitems);
            const char* tag = tag_n(sizeof(Tc) == 8 ? "plane_fwd_f64" : "plane_fwd_f32", nc);
            PB(tag);
            k<<<8 * ncl, 256, sm, s>>>(f, sp, g.n3, nitems, csf, css, g.n1p, twx_t<Tc>(), twy_t<Tc>());
            PE(tag);
        }
    }
    void inv2d(const Cx<T>* sp, T* out, const T* add, int nc, int64_t csf, int64_t css) {
        if constexpr (std::is_same<T, float>::value) {
            auto k = k_plane_inv<float>;
            constexpr size_t sm = plane_inv_smem<float>();
            const int nitems = nc * g.n3;
            const int ncl = plane_clusters(k, sm, nitems);
            const char* tag = tag_n(add ? "plane_inv_add" : "plane_inv", nc);
            PB(tag);
            k<<<8 * ncl, 256, sm, s>>>(sp, out, add, g.n3, nitems, csf, css, g.n1p, twx(), twy());
            PE(tag);
        }
    }

#define DR_SWITCH_ROW(Lval, call)                          \
    switch (Lval) {                                        \
        case 2: call(2); break;                            \
        case 4: call(4); break;                            \
        case 8: call(8); break;                            \
        case 16: call(16); break;                          \
        case 32: call(32); break;                          \
        case 64: call(64); break;                          \
        case 128: call(128); break;                        \
        case 256: call(256); break;                        \
        case 512: call(512); break;                        \
        default: fail(DR_ERR_GRID, "unsupported row length"); \
    }
// Bluestein convolution lengths M (non-power-of-two extents, one rank)
#define DR_SWITCH_BLUE(Mval, call)                          \
    switch (Mval) {                                         \
        case 16: call(16); break;                           \
        case 32: call(32); break;                           \
        case 64: call(64); break;                           \
        case 128: call(128); break;                         \
        case 256: call(256); break;                         \
        case 512: call(512); break;                         \
        case 1024: call(1024); break;                       \
        default: fail(DR_ERR_GRID, "unsupported Bluestein length"); \
    }
#define DR_SWITCH_COL(Lval, call)                          \
    switch (Lval) {                                        \
        case 4: call(4); break;                            \
        case 8: call(8); break;                            \
        case 16: call(16); break;                          \
        case 32: call(32); break;                          \
        case 64: call(64); break;                          \
        case 128: call(128); break;                        \
        case 256: call(256); break;                        \
        case 512: call(512); break;                        \
        case 1024: call(1024); break;                      \
        default: fail(DR_ERR_GRID, "unsupported column length"); \
    }

    // ---- x1 rows of a non-power-of-two extent (Bluestein, fft.cuh RowBlue*; one rank)
    template <int M>
    void blue_row_deriv_M(const T* f, T* out, int acc, int nf, int64_t fs, int64_t os) {
        using PT = RowBlueDerivPass<T, M>;
        stream("row_deriv", PT{g, f, out, acc, twxd(), bluetab1<double>(), fs, os}, row_tiles<PT::RB>(), nf);
    }
    void blue_row_deriv(const T* f, T* out, int acc, int nf = 1, int64_t fs = 0, int64_t os = 0) {
#define CALL(MM) blue_row_deriv_M<MM>(f, out, acc, nf, fs, os)
        DR_SWITCH_BLUE(blue_m(g.n1 / 2), CALL)
#undef CALL
    }
    template <typename Tc, int M>
    void blue_row_r2c_M(const T* f, Cx<Tc>* sp, int nc, int64_t csf, int64_t css) {
        using PT = RowBlueR2cPass<T, Tc, M>;
        stream(sizeof(Tc) == 8 ? "row_r2c_f64" : "row_r2c_f32", PT{g, f, sp, twx_t<Tc>(), bluetab1<Tc>(), csf, css},
               row_tiles<PT::RB>(), nc);
    }
    template <int M>
    void blue_row_c2r_M(const Cx<T>* sp, T* out, const T* add, int nc, int64_t csf, int64_t css) {
        using PT = RowBlueC2rPass<T, M>;
        stream(add ? "row_c2r_add" : "row_c2r", PT{g, sp, RowOut<T>{out, add}, twx(), bluetab1<T>(), csf, css},
               row_tiles<PT::RB>(), nc);
    }
    void row_deriv(const T* f, T* out, int acc) {
        if (blue1()) {
            blue_row_deriv(f, out, acc);
            return;
        }
#define CALL(LL) row_deriv_L<LL>(f, out, acc)
        DR_SWITCH_ROW(g.n1 / 2, CALL)
#undef CALL
    }
    template <typename Tc>
    void row_r2c(const T* f, Cx<Tc>* sp, int nc = 1, int64_t csf = 0, int64_t css = 0) {
        if (blue1()) {
#define CALL(MM) blue_row_r2c_M<Tc, MM>(f, sp, nc, csf, css)
            DR_SWITCH_BLUE(blue_m(g.n1 / 2), CALL)
#undef CALL
            return;
        }
#define CALL(LL) row_r2c_L<LL, Tc>(f, sp, nc, csf, css)
        DR_SWITCH_ROW(g.n1 / 2, CALL)
#undef CALL
    }
    void row_c2r(const Cx<T>* sp, T* out, const T* add, int nc = 1, int64_t csf = 0, int64_t css = 0) {
        if (blue1()) {
#define CALL(MM) blue_row_c2r_M<MM>(sp, out, add, nc, csf, css)
            DR_SWITCH_BLUE(blue_m(g.n1 / 2), CALL)
#undef CALL
            return;
        }
#define CALL(LL) row_c2r_L<LL>(sp, out, add, nc, csf, css)
        DR_SWITCH_ROW(g.n1 / 2, CALL)
#undef CALL
    }

    template <class PT>
    static int64_t col_tiles(const ColGeom& cg, int nother) {
        return (int64_t)((cg.nx + PT::XC - 1) / PT::XC) * ((nother + PT::OL - 1) / PT::OL);
    }
    ColGeom spec_geom() const { return ColGeom{g.n1p, g.n1c, g.n2, g.n3}; }
    ColGeom pair_geom() const { return ColGeom{g.n1 / 2, g.n1 / 2, g.n2, g.n3}; }
    // the transposed slab: all N3 planes of this rank's x2 block
    ColGeom spec_geom_t() const { return ColGeom{g.n1p, g.n1c, nb(), g.n3g, c.rank * nb(), g.n2}; }
    ColGeom pair_geom_t() const { return ColGeom{g.n1 / 2, g.n1 / 2, nb(), g.n3g, c.rank * nb(), g.n2}; }

    // ---- x2 passes of a non-power-of-two extent (Bluestein, fft.cuh ColBlue*; one rank)
    template <typename U, int M, int DIR>
    void blue_fft_M(const Cx<U>* src, Cx<U>* dst, int nc, int64_t cs, int64_t csd) {
        using PT = ColBlueFftPass<U, M, DIR>;
        const ColGeom cg = spec_geom();
        const char* tag = DIR > 0 ? "col_fft_inv" : sizeof(U) == 8 ? "col_fft_fwd_f64" : "col_fft_fwd_f32";
        stream(tag, PT{cg, src, dst, bluetab<U>(), cs, csd}, col_tiles<PT>(cg, g.n3), nc);
    }
    template <typename U, int DIR>
    void blue_fft(const Cx<U>* src, Cx<U>* dst, int nc, int64_t cs, int64_t csd) {
#define CALL(MM) blue_fft_M<U, MM, DIR>(src, dst, nc, cs, csd)
        DR_SWITCH_BLUE(blue_m(g.n2), CALL)
#undef CALL
    }
    template <int M>
    void blue_deriv_M(const T* f, T* out, int acc, int nf, int64_t fs, int64_t os) {
        using PT = ColBlueDerivPass<T, M>;
        const ColGeom cg = pair_geom();
        stream("col_deriv", PT{cg, reinterpret_cast<const Cx<T>*>(f), reinterpret_cast<Cx<T>*>(out), acc, bluetab<double>(),
                               fs / 2, os / 2},
               col_tiles<PT>(cg, cg.n3), nf);
    }
    template <int M>
    void blue_deriv3_M(const T* f, T* out, int acc, int nf, int64_t fs, int64_t os) {
        using PT = ColBlueDerivPass<T, M, 3>;
        const ColGeom cg = pair_geom();
        stream("col_deriv", PT{cg, reinterpret_cast<const Cx<T>*>(f), reinterpret_cast<Cx<T>*>(out), acc, bluetab3(),
                               fs / 2, os / 2},
               col_tiles<PT>(cg, cg.n2), nf);
    }
    void blue_deriv3(const T* f, T* out, int acc, int nf = 1, int64_t fs = 0, int64_t os = 0) {
#define CALL(MM) blue_deriv3_M<MM>(f, out, acc, nf, fs, os)
        DR_SWITCH_BLUE(blue_m(g.n3g), CALL)
#undef CALL
    }
    // x3 middle pass of a non-power-of-two x3 extent (fft.cuh BlueMiddlePass; one rank)
    template <int KIND, typename Tc, int M>
    void blue_middle_M(Cx<Tc>* const* in, Cx<T>* const* out, int comp, int nc, int64_t cs, Cx<T>* const* inq) {
        using PT = BlueMiddlePass<Tc, T, M, KIND>;
        PT pt;
        pt.c = spec_geom();
        for (int i = 0; i < PT::NCI; ++i) pt.in.p[i] = in[i];
        for (int i = 0; i < PT::NCO; ++i) pt.out.p[i] = out[i];
        if (inq) pt.inq = SpecPtrs<T, 2>{{inq[0], inq[1]}};
        pt.s = SymInfo{c.cfg.reg, c.cfg.beta, 2.0 / ((double)g.n1 * g.n2 * g.n3g), comp};
        pt.bt = bluetab3();
        pt.cs = cs;
        stream(sizeof(Tc) == 8 ? "col_middle_f64" : "col_middle_f32", pt, col_tiles<PT>(pt.c, pt.c.n2), nc);
    }
    template <int KIND, typename Tc>
    void blue_middle(Cx<Tc>* const* in, Cx<T>* const* out, int comp, int nc, int64_t cs, Cx<T>* const* inq) {
        if constexpr (KIND == 6 || KIND == 7 || KIND == 9) {
            fail(DR_ERR_GRID, "non-power-of-two x3 extents run on one rank only");
        } else {
#define CALL(MM) blue_middle_M<KIND, Tc, MM>(in, out, comp, nc, cs, inq)
            DR_SWITCH_BLUE(blue_m(g.n3g), CALL)
#undef CALL
        }
    }
    void blue_deriv(const T* f, T* out, int acc, int nf = 1, int64_t fs = 0, int64_t os = 0) {
#define CALL(MM) blue_deriv_M<MM>(f, out, acc, nf, fs, os)
        DR_SWITCH_BLUE(blue_m(g.n2), CALL)
#undef CALL
    }
    template <int M>
    void blue_div_M(const Cx<T>* p1, const Cx<T>* p2, const Cx<T>* p3, Cx<T>* q, Cx<T>* r) {
        using PT = ColBlueDivPass<T, M>;
        const ColGeom cg = spec_geom();
        stream("col_div", PT{cg, p1, p2, p3, q, r, bluetab<double>(), g.n1}, col_tiles<PT>(cg, g.n3));
    }

    template <int L, int AX>
    void col_deriv_L(const ColGeom& cg, const T* f, T* out, int acc, int nf = 1, int64_t fs = 0, int64_t os = 0) {
        using PT = ColDerivPass<T, L, AX>;
        stream("col_deriv", PT{cg, reinterpret_cast<const Cx<T>*>(f), reinterpret_cast<Cx<T>*>(out), acc, AX == 2 ? twy() : twz(),
                               fs / 2, os / 2},
               col_tiles<PT>(cg, AX == 2 ? cg.n3 : cg.n2), nf);
    }
    // out (+)= d f / dx_ax (1-D transforms along the axis only); x3 on slabs transposes first
    void col_deriv(int ax, const T* f, T* out, int acc) {
        if (ax == 2 && blue2()) {
            blue_deriv(f, out, acc);
            return;
        }
        if (ax == 2) {
#define CALL(LL) col_deriv_L<LL, 2>(pair_geom(), f, out, acc)
            DR_SWITCH_COL(g.n2, CALL)
#undef CALL
            return;
        }
        if (!c.dist() && blue3()) {
            blue_deriv3(f, out, acc);
            return;
        }
        if (!c.dist()) {
#define CALL(LL) col_deriv_L<LL, 3>(pair_geom(), f, out, acc)
            DR_SWITCH_COL(g.n3, CALL)
#undef CALL
            return;
        }
        const size_t chunk = (size_t)g.n3 * nb() * g.n1 * sizeof(T);
        PB("pack");
        k_pack_split<T><<<grid_1d(g.M), 256, 0, s>>>(g, f, xs(), nb());
        PE("pack");
        alltoall(xs(), xr(), chunk);
#define CALL(LL) col_deriv_L<LL, 3>(pair_geom_t(), xr(), xr(), 0)
        DR_SWITCH_COL(g.n3g, CALL)
#undef CALL
        alltoall(xr(), xs(), chunk);
        PB("unpack");
        k_unpack_split<T><<<grid_1d(g.M), 256, 0, s>>>(g, xs(), out, nb(), acc);
        PE("unpack");
    }

    template <typename U, int L, int DIR, bool SI, bool SO>
    void col_fft_LS(const Cx<U>* src, Cx<U>* dst, const Cx<U>* tw, int nb_in, int nb_out, int nc, int64_t cs, int64_t csd) {
        const ColGeom cg = spec_geom();
        const char* tag = DIR > 0 ? "col_fft_inv" : sizeof(U) == 8 ? "col_fft_fwd_f64" : "col_fft_fwd_f32";
        if (csd >= 0 && csd != cs && !SI && !SO) {
            using PT = ColFftPass<U, L, DIR, false, false, false, true>;
            stream(tag, PT{cg, src, dst, tw, nb_in, nb_out, cs, csd}, col_tiles<PT>(cg, g.n3), nc);
            return;
        }
        using PT = ColFftPass<U, L, DIR, SI, SO>;
        stream(tag, PT{cg, src, dst, tw, nb_in, nb_out, cs, csd}, col_tiles<PT>(cg, g.n3), nc);
    }
    template <typename U, int L, int DIR>
    void col_fft_L(const Cx<U>* src, Cx<U>* dst, const Cx<U>* tw, int nb_in, int nb_out, int nc, int64_t cs, int64_t csd) {
        // the split layouts only occur on the side facing an all-to-all: out of the forward, into the inverse
        if (DIR < 0 && nb_out) col_fft_LS<U, L, DIR, false, true>(src, dst, tw, nb_in, nb_out, nc, cs, csd);
        else if (DIR > 0 && nb_in) col_fft_LS<U, L, DIR, true, false>(src, dst, tw, nb_in, nb_out, nc, cs, csd);
        else col_fft_LS<U, L, DIR, false, false>(src, dst, tw, nb_in, nb_out, nc, cs, csd);
    }
    // (csd: component stride of dst when it differs from src's cs)
    template <typename Tc>
    void col_fft_fwd(const Cx<Tc>* src, Cx<Tc>* dst, int nb_out, int nc = 1, int64_t cs = 0, int64_t csd = -1) {  // forward along x2, in Tc
        if (blue2()) {  // one rank: nb_out == 0
            blue_fft<Tc, -1>(src, dst, nc, cs, csd);
            return;
        }
#define CALL(LL) col_fft_L<Tc, LL, -1>(src, dst, twy_t<Tc>(), 0, nb_out, nc, cs, csd)
        DR_SWITCH_COL(g.n2, CALL)
#undef CALL
    }
    template <typename Tc, int L>
    void col_fft_fwd_peer(const Cx<Tc>* src, const PeerDst& pd) {
        using PT = ColFftPass<Tc, L, -1, false, true, true>;
        const ColGeom cg = spec_geom();
        PT pt{cg, src, nullptr, twy_t<Tc>(), 0, nb(), 0, -1};
        pt.pd = pd;
        stream(sizeof(Tc) == 8 ? "col_fft_fwd_f64" : "col_fft_fwd_f32", pt, col_tiles<PT>(cg, g.n3), 1);
    }
    void col_fft_inv(const Cx<T>* src, Cx<T>* dst, int nb_in, int nc = 1, int64_t cs = 0, int64_t csd = -1) {  // inverse along x2, in T
        if (blue2()) {  // one rank: nb_in == 0
            blue_fft<T, +1>(src, dst, nc, cs, csd);
            return;
        }
#define CALL(LL) col_fft_L<T, LL, +1>(src, dst, twy(), nb_in, 0, nc, cs, csd)
        DR_SWITCH_COL(g.n2, CALL)
#undef CALL
    }

    // isochoric data term, x2 stage (fft.cuh ColDivPass): Q = i (k1' F2 P1 + k2' F2 P2), R = F2 P3 from the x1
    // half spectra P_a of b~'s components; nb_out != 0: the split layout of the slab transposes
    template <int L, bool SO>
    void col_div_L(const Cx<T>* p1, const Cx<T>* p2, const Cx<T>* p3, Cx<T>* q, Cx<T>* r, int nb_out) {
        using PT = ColDivPass<T, L, SO>;
        const ColGeom cg = spec_geom();
        stream("col_div", PT{cg, p1, p2, p3, q, r, twy_t<T>(), nb_out, g.n1}, col_tiles<PT>(cg, g.n3));
    }
    void col_div(const Cx<T>* p1, const Cx<T>* p2, const Cx<T>* p3, Cx<T>* q, Cx<T>* r, int nb_out) {
        if (blue2()) {  // one rank
#define CALL(MM) blue_div_M<MM>(p1, p2, p3, q, r)
            DR_SWITCH_BLUE(blue_m(g.n2), CALL)
#undef CALL
            return;
        }
#define CALL(LL) (nb_out ? col_div_L<LL, true>(p1, p2, p3, q, r, nb_out) : col_div_L<LL, false>(p1, p2, p3, q, r, 0))
        DR_SWITCH_COL(g.n2, CALL)
#undef CALL
    }

    template <int L, int KIND, typename Tc>
    void middle_L(const ColGeom& cg, Cx<Tc>* const* in, Cx<T>* const* out, int comp, int nc, int64_t cs,
                  Cx<T>* const* inq) {
        if constexpr (MiddlePass<Tc, T, L, KIND>::NCO == 1) {
            if (c.dist() && nc == 1 && peer_a2a_on()) {  // store the transpose chunks into the ranks' specF(3)
                using PQ = MiddlePass<Tc, T, L, KIND, true>;
                PQ pt;
                pt.c = cg;
                for (int i = 0; i < PQ::NCI; ++i) pt.in.p[i] = in[i];
                pt.out.p[0] = out[0];
                if (inq) pt.inq = SpecPtrs<T, 2>{{inq[0], inq[1]}};
                pt.s = SymInfo{c.cfg.reg, c.cfg.beta, 2.0 / ((double)g.n1 * g.n2 * g.n3g), comp};
                pt.tw = twz_t<Tc>();
                pt.two = twz();
                pt.cs = cs;
                const size_t chunk = (size_t)g.n3 * nb() * g.n1p * sizeof(Cx<T>);
                pt.pd = PeerDst{pws(), (int64_t)((char*)specF(3) - c.ws) + (int64_t)(c.rank * chunk), ilog2c(g.n3)};
                peer_barrier_all();  // every rank finished reading its specF(3)
                stream(sizeof(Tc) == 8 ? "col_middle_f64" : "col_middle_f32", pt, col_tiles<PQ>(cg, cg.n2), nc);
                c.peer_inv_fresh = true;
                return;
            }
        }
        using PT = MiddlePass<Tc, T, L, KIND>;
        PT pt;
        pt.c = cg;
        for (int i = 0; i < PT::NCI; ++i) pt.in.p[i] = in[i];
        for (int i = 0; i < PT::NCO; ++i) pt.out.p[i] = out[i];
        if (inq) pt.inq = SpecPtrs<T, 2>{{inq[0], inq[1]}};
        pt.s = SymInfo{c.cfg.reg, c.cfg.beta, 2.0 / ((double)g.n1 * g.n2 * g.n3g), comp};
        pt.tw = twz_t<Tc>();
        pt.two = twz();
        pt.cs = cs;
        stream(sizeof(Tc) == 8 ? "col_middle_f64" : "col_middle_f32", pt, col_tiles<PT>(cg, cg.n2), nc);
    }
    template <int KIND, typename Tc = double>
    void middle(Cx<Tc>* const* in, Cx<T>* const* out, int comp = 0, int nc = 1, int64_t cs = 0,
                Cx<T>* const* inq = nullptr) {
        if (blue3()) {
            blue_middle<KIND, Tc>(in, out, comp, nc, cs, inq);
            return;
        }
        const ColGeom cg = c.dist() ? spec_geom_t() : spec_geom();
#define CALL(LL) middle_L<LL, KIND, Tc>(cg, in, out, comp, nc, cs, inq)
        DR_SWITCH_COL(g.n3g, CALL)
#undef CALL
    }

    // -------------------------------------------------------------------- spectral operators
    // Forward half spectrum of a real slab field into spectrum slot `slot`: x1 r2c, x2 forward FFT and,
    // with slabs, the all-to-all into the transposed layout the x3 middle pass reads.
    // Tc = double for symbols that amplify high wavenumbers (beta A, reading A20); Tc = T for symbols that
    // damp them ((beta A)^-1, Leray), where the fp32 rounding noise of the forward passes is harmless.
    template <typename Tc = double>
    void spec_forward(const T* f, int slot) {
        if (!c.dist()) {
            if (plane2d_ok(f, specD_t<Tc>(slot))) {
                fwd2d<Tc>(f, specD_t<Tc>(slot), 1, 0, 0);
                return;
            }
            row_r2c<Tc>(f, specD_t<Tc>(slot));
            col_fft_fwd<Tc>(specD_t<Tc>(slot), specD_t<Tc>(slot), 0);
            return;
        }
        row_r2c<Tc>(f, specD_t<Tc>(6));
        if (peer_a2a_on()) {  // the x2 pass stores each rank's chunk straight into its spectrum slot
            const size_t chunk = (size_t)g.n3 * nb() * g.n1p * sizeof(Cx<Tc>);
            peer_barrier_all();  // every rank finished reading the slot (its previous middle pass)
#define CALL(LL) col_fft_fwd_peer<Tc, LL>(specD_t<Tc>(6), PeerDst{pws(), (int64_t)((char*)specD_t<Tc>(slot) - c.ws) + (int64_t)(c.rank * chunk), ilog2c(nb())})
            DR_SWITCH_COL(g.n2, CALL)
#undef CALL
            peer_barrier_all();  // every chunk arrived
            return;
        }
        col_fft_fwd<Tc>(specD_t<Tc>(6), specD_t<Tc>(7), nb());  // the split layout: one contiguous chunk per rank
        alltoall(specD_t<Tc>(7), specD_t<Tc>(slot), (size_t)g.n3 * nb() * g.n1p * sizeof(Cx<Tc>));
    }
    // Back from the middle pass's output slot to a real slab field (+ add).
    void spec_inverse(int slot, T* out, const T* add) {
        if (!c.dist()) {
            if (plane2d_ok(out, add)) {
                inv2d(specF(slot), out, add, 1, 0, 0);
                return;
            }
            col_fft_inv(specF(slot), specF(slot), 0);
            row_c2r(specF(slot), out, add);
            return;
        }
        if (c.peer_inv_fresh) {  // the middle pass stored the chunks into every rank's specF(3)
            c.peer_inv_fresh = false;
            peer_barrier_all();
        } else {
            alltoall(specF(slot), specF(3), (size_t)g.n3 * nb() * g.n1p * sizeof(Cx<T>));
        }
        col_fft_inv(specF(3), specF(4), nb());
        row_c2r(specF(4), out, add);
    }

    // gradients of nf fields f + i fs into out + i os (components M apart) with one launch per axis
    // (one rank; the x3 derivative of slabs transposes, so they take grad() per field)
    void grad_batch(const T* f, int64_t fs, T* out, int64_t os, int nf) {
        if (c.dist() || (fs & 1) || (os & 1)) {
            for (int i = 0; i < nf; ++i) grad(f + i * fs, vec(out + i * os, (size_t)g.M));
            return;
        }
        if (blue1()) {
            blue_row_deriv(f, out, 0, nf, fs, os);
        } else {
#define CALL(LL) row_deriv_L<LL>(f, out, 0, nf, fs, os)
            DR_SWITCH_ROW(g.n1 / 2, CALL)
#undef CALL
        }
        if (blue2()) {
            blue_deriv(f, out + g.M, 0, nf, fs, os);
        } else {
#define CALL(LL) col_deriv_L<LL, 2>(pair_geom(), f, out + g.M, 0, nf, fs, os)
            DR_SWITCH_COL(g.n2, CALL)
#undef CALL
        }
        if (blue3()) {
            blue_deriv3(f, out + 2 * g.M, 0, nf, fs, os);
        } else {
#define CALL(LL) col_deriv_L<LL, 3>(pair_geom(), f, out + 2 * g.M, 0, nf, fs, os)
            DR_SWITCH_COL(g.n3, CALL)
#undef CALL
        }
    }
    void grad(const T* f, V3<T> out) {
        row_deriv(f, out.c[0], 0);
        col_deriv(2, f, out.c[1], 0);
        col_deriv(3, f, out.c[2], 0);
    }
    void div(V3<const T> u, T* out) {
        row_deriv(u.c[0], out, 0);
        col_deriv(2, u.c[1], out, 1);
        col_deriv(3, u.c[2], out, 1);
    }
    // out_c = F^-1[sym F in_c] (+ add_c), componentwise symbol KIND 0/1.  Forward passes (x1 r2c, x2)
    // and the x3 forward transform run in double; the inverse x3 / x2 / x1 passes in T.
    template <typename P>
    static int64_t uniform_stride(const P* const* c3) {  // element stride of 3 components, or 0
        const int64_t a = c3[1] - c3[0], b = c3[2] - c3[1];
        return (a == b && a > 0) ? a : 0;
    }
    // Tensor-map TMA tiles (fft.cuh MiddleTma): a 4-D map (2 W scalars, n2, n3, components)
    // over spectrum slots `base` .. (component stride S); false if the driver entry point is missing.
    static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
        static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
            cudaDriverEntryPointQueryResult q;
            void* fn = nullptr;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) {
                cudaGetLastError();
                fn = nullptr;
            }
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        }();
        return encode;
    }
    // 3-D map over a gather source's slot (x1, x2, slot planes) with the staged box's extents
    GatherTma gather_tma(const T* slot_base) {
        GatherTma gt;
        std::memset(&gt, 0, sizeof(gt));
        if constexpr (std::is_same<T, float>::value) {
            const auto encode = tma_encoder();
            if (!c.gather_tma || !encode || ((uintptr_t)slot_base & 15)) return gt;
            using BG = BoxGeom<float, 1>;
            const cuuint64_t dims[3] = {(cuuint64_t)g.n1, (cuuint64_t)g.n2, (cuuint64_t)(g.n3 + g.zg + g.zgh)};
            const cuuint64_t strides[2] = {(cuuint64_t)g.n1 * 4, (cuuint64_t)g.n1 * g.n2 * 4};
            const cuuint32_t box[3] = {(cuuint32_t)BG::BX, (cuuint32_t)BG::BY, (cuuint32_t)BG::BZ};
            const cuuint32_t el[3] = {1, 1, 1};
            if (box[0] > 256 || box[1] > 256 || box[2] > 256) return gt;
            gt.use = encode(&gt.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<T*>(slot_base), dims, strides, box, el,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        return gt;
    }
    template <typename U>
    bool tensor_map(CUtensorMap* tm, const void* base, int nc, cuuint32_t box0, cuuint32_t box1, cuuint32_t box2) {
        const auto encode = tma_encoder();
        if (!encode) return false;
        const ColGeom cg = spec_geom();
        const cuuint64_t es = sizeof(U);
        const cuuint64_t dims[4] = {(cuuint64_t)2 * cg.W, (cuuint64_t)cg.n2, (cuuint64_t)cg.n3, (cuuint64_t)nc};
        const cuuint64_t strides[3] = {(cuuint64_t)cg.W * 2 * es, (cuuint64_t)cg.n2 * cg.W * 2 * es, (cuuint64_t)g.S * 2 * es};
        const cuuint32_t box[4] = {box0, box1, box2, 1};
        const cuuint32_t el[4] = {1, 1, 1, 1};
        return encode(tm, TmaType<U>::V, 4, const_cast<void*>(base), dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    int persistent_grid(int per_sm, int64_t ntiles, int nc) const {
        return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)per_sm * c.num_sms / nc));
    }
    // x3 middle pass of a scalar symbol over nc spectra (one 256-plane line per tile)
    template <typename Ti, int L, int KIND>
    bool middle_tma(Cx<Ti>* in, Cx<float>* out, int nc) {
        using P = MiddleTma<Ti, L, KIND>;
        CUtensorMap tm;
        if (!tensor_map<Ti>(&tm, in, nc, 2 * P::XC, 1, L)) return false;
        const ColGeom cg = spec_geom();
        const int64_t nt = (int64_t)((cg.nx + P::XC - 1) / P::XC) * cg.n2;
        auto k = k_middle_tma<Ti, L, KIND>;
        const int per_sm = per_device_occupancy(k, P::NT, P::BUF);
        const int grid = persistent_grid(per_sm, nt, nc);
        P pass{cg, out, g.S, SymInfo{c.cfg.reg, c.cfg.beta, 2.0 / ((double)g.n1 * g.n2 * g.n3g), 0}, twz_t<Ti>(),
               reinterpret_cast<const Cx<float>*>(twz())};
        const char* tag = tag_n(sizeof(Ti) == 8 ? "col_middle_f64" : "col_middle_f32", nc);
        PB(tag);
        k<<<dim3(grid, nc), P::NT, P::BUF, s>>>(tm, pass, (int)nt);
        PE(tag);
        return true;
    }

    template <int KIND>
    void scalar_symbol3(V3<const T> in, V3<T> out, const V3<const T>* add) {
        using Tc = std::conditional_t<KIND == 1, T, double>;  // preconditioner: damping symbol
        // one rank, components at one stride (every SoA vector field): the 3 components go through
        // each pass in one launch (blockIdx.y), three times the CTAs per wave-quantised launch
        const int64_t si = uniform_stride(in.c), so = uniform_stride(out.c);
        if (!c.dist() && si && so && (!add || uniform_stride(add->c) == so)) {
            if (c.chunk > 0 && g.n3 % c.chunk == 0 && c.chunk < g.n3) {
                // plane chunks: each chunk's x1 output is still in L2 when its x2 pass reads it
                Grid gc = g;
                gc.n3 = c.chunk;
                gc.M = (int64_t)g.n1 * g.n2 * gc.n3;
                Impl sub(c, gc, s);
                for (int z = 0; z < g.n3; z += c.chunk) {
                    Cx<Tc>* sp = specD_t<Tc>(0) + (size_t)z * g.n2 * g.n1p;
                    sub.template row_r2c<Tc>(in.c[0] + (size_t)z * plane(), sp, 3, si, g.S);
                    sub.template col_fft_fwd<Tc>(sp, sp, 0, 3, g.S);
                }
            } else if (plane2d_ok(in.c[0], specD_t<Tc>(0))) {
                fwd2d<Tc>(in.c[0], specD_t<Tc>(0), 3, si, g.S);
            } else if (ring_ok()) {
                // plane chunks through one scratch ring: the x1 half spectra of a chunk are written to the
                // same (L2-resident) scratch lines every chunk and read back by the chunk's x2 pass
                Grid gc = g;
                gc.n3 = c.ring;
                gc.M = (int64_t)g.n1 * g.n2 * gc.n3;
                Impl sub(c, gc, s);
                const int64_t rs = (int64_t)c.ring * g.n2 * g.n1p;
                Cx<Tc>* sc = ring_scratch<Tc>();
                for (int z = 0; z < g.n3; z += c.ring) {
                    sub.template row_r2c<Tc>(in.c[0] + (size_t)z * plane(), sc, 3, si, rs);
                    sub.template col_fft_fwd<Tc>(sc, specD_t<Tc>(0) + (size_t)z * g.n2 * g.n1p, 0, 3, rs, g.S);
                }
            } else {
                row_r2c<Tc>(in.c[0], specD_t<Tc>(0), 3, si, g.S);
                col_fft_fwd<Tc>(specD_t<Tc>(0), specD_t<Tc>(0), 0, 3, g.S);
            }
            Cx<Tc>* sd = specD_t<Tc>(0);
            Cx<T>* sf = specF(0);
            // fp32 spectra: the TMA-tile middle pass (152 -> 118 us for three components at 256^3); the
            // fp64-input middle and the x2 passes through TMA tiles measured no gain / slower
            bool done = false;
            if constexpr (std::is_same_v<Tc, float> && std::is_same_v<T, float>) {
                done = c.tma_middle && g.n3g == 256 && middle_tma<Tc, 256, KIND>(sd, sf, 3);
            }
            if (!done) middle<KIND, Tc>(&sd, &sf, 0, 3, g.S);
            if (c.chunk > 0 && g.n3 % c.chunk == 0 && c.chunk < g.n3) {
                Grid gc = g;
                gc.n3 = c.chunk;
                gc.M = (int64_t)g.n1 * g.n2 * gc.n3;
                Impl sub(c, gc, s);
                for (int z = 0; z < g.n3; z += c.chunk) {
                    Cx<T>* sp = specF(0) + (size_t)z * g.n2 * g.n1p;
                    const size_t off = (size_t)z * plane();
                    sub.col_fft_inv(sp, sp, 0, 3, g.S);
                    sub.row_c2r(sp, out.c[0] + off, add ? add->c[0] + off : nullptr, 3, so, g.S);
                }
                return;
            }
            if (plane2d_ok(out.c[0], add ? add->c[0] : nullptr)) {
                inv2d(specF(0), out.c[0], add ? add->c[0] : nullptr, 3, so, g.S);
                return;
            }
            if (ring_ok()) {
                Grid gc = g;
                gc.n3 = c.ring;
                gc.M = (int64_t)g.n1 * g.n2 * gc.n3;
                Impl sub(c, gc, s);
                const int64_t rs = (int64_t)c.ring * g.n2 * g.n1p;
                Cx<T>* sc = ring_scratch<T>();
                for (int z = 0; z < g.n3; z += c.ring) {
                    const size_t off = (size_t)z * plane();
                    sub.col_fft_inv(specF(0) + (size_t)z * g.n2 * g.n1p, sc, 0, 3, g.S, rs);
                    sub.row_c2r(sc, out.c[0] + off, add ? add->c[0] + off : nullptr, 3, so, rs);
                }
                return;
            }
            col_fft_inv(specF(0), specF(0), 0, 3, g.S);
            row_c2r(specF(0), out.c[0], add ? add->c[0] : nullptr, 3, so, g.S);
            return;
        }
        for (int cc = 0; cc < 3; ++cc) {
            spec_forward<Tc>(in.c[cc], 0);
            Cx<Tc>* sd = specD_t<Tc>(0);
            Cx<T>* sf = specF(0);
            middle<KIND, Tc>(&sd, &sf);
            spec_inverse(0, out.c[cc], add ? add->c[cc] : nullptr);
        }
    }
    // coupled 3-component symbol (KIND 2 Leray, 3 Leray / (beta A)): out = F^-1[sym F in]; both damp or
    // keep the magnitude of every mode, so the forward passes run in T
    template <int KIND>
    void vector_symbol3(V3<const T> in, V3<T> out) {
        Cx<T>* sd[3] = {specD_t<T>(0), specD_t<T>(1), specD_t<T>(2)};
        Cx<T>* sf[3] = {specF(0), specF(1), specF(2)};
        for (int cc = 0; cc < 3; ++cc) spec_forward<T>(in.c[cc], cc);
        middle<KIND, T>(sd, sf);
        for (int cc = 0; cc < 3; ++cc) spec_inverse(cc, out.c[cc], nullptr);
    }
    void reg_apply(V3<const T> in, V3<T> out) { scalar_symbol3<0>(in, out, nullptr); }
    void leray(V3<const T> in, V3<T> out) { vector_symbol3<2>(in, out); }
    void precond(V3<const T> r, V3<T> z) {
        if (c.cfg.flags & DR_ISOCHORIC) vector_symbol3<3>(r, z);
        else scalar_symbol3<1>(r, z, nullptr);
    }

    // -------------------------------------------------------------------- semi-Lagrangian
    // Per-tile gather plan of a displacement field (once per velocity and direction).
    void plan(const T* d, int* plan_buf) {
        int* mx = c.at<int>(c.L.maxext);
        PB("sl_plan");
        k_sl_plan<T><<<(unsigned)n_tiles(g), SL_THREADS, 0, s>>>(g, d, plan_buf, mx);
        PE("sl_plan");
    }
    // d = (c0 v0, c1 v1, c2 v2) written while its plan is taken (the first stage of Eq. 6)
    void dstar_plan(T* d, int* plan_buf, T c0, T c1, T c2) {
        int* mx = c.at<int>(c.L.maxext);
        PB("dstar_plan");
        k_sl_plan<T, true><<<(unsigned)n_tiles(g), SL_THREADS, 0, s>>>(g, d, plan_buf, mx,
                                                                        DstarIn<T>{{vc(0), vc(1), vc(2)}, {c0, c1, c2}});
        PE("dstar_plan");
    }

    // ---------------------------------------------------------------- off-rank departure points
    // device arrays of remote plan f (0: d*, 1: d+, 2: d-): [ids_out][ids_in][rec_out][rec_in][val_out][val_in]
    // then 4 int arrays of 64 (cnt, off, cursor, scratch)
    struct RP {
        int *ids_out;
        RemoteRec<T> *rec_out, *rec_in;
        T *val_out, *val_in;
        int *cnt, *off, *cur;
    };
    RP rp(int f) {
        const size_t cap = (size_t)c.L.rcap;
        char* b = c.ws + c.L.rem + (size_t)f * cap * (2 * 4 + 2 * sizeof(RemoteRec<T>) + 2 * 3 * sizeof(T));
        RP r;
        r.ids_out = reinterpret_cast<int*>(b);
        b += 2 * cap * 4;
        r.rec_out = reinterpret_cast<RemoteRec<T>*>(b);
        r.rec_in = r.rec_out + cap;
        b += 2 * cap * sizeof(RemoteRec<T>);
        r.val_out = reinterpret_cast<T*>(b);
        r.val_in = r.val_out + 3 * cap;
        int* ints = reinterpret_cast<int*>(c.ws + c.L.rem + 3 * cap * (2 * 4 + 2 * sizeof(RemoteRec<T>) + 2 * 3 * sizeof(T)));
        r.cnt = ints + f * 192;
        r.off = r.cnt + 64;
        r.cur = r.cnt + 128;
        return r;
    }
    int field_of(const int* plan_buf) { return plan_buf == plan_t() ? 0 : plan_buf == plan_p() ? 1 : 2; }
    // classify the points of displacement field d whose stencil leaves the slab + ghosts, send their
    // cells to the owners (counts, then records), once per velocity
    void remote_plan(int f, const T* d) {
        auto& H = c.rp[f];
        H = dr_ctx::RemotePlanH{};
        if (!c.dist()) return;
        const int P = c.nranks;
        RP r = rp(f);
        const Disp<T> dp{{d, d + g.M, d + 2 * g.M}};
        CK(cudaMemsetAsync(r.cnt, 0, 192 * sizeof(int), s));
        PB("remote_plan");
        k_remote_classify<T><<<grid_1d(g.M), 256, 0, s>>>(g, dp, 0, r.cnt, r.off, r.cur, r.ids_out, r.rec_out, 0);
        PE("remote_plan");
        H.out_cnt.assign(P, 0);
        CK(cudaMemcpyAsync(H.out_cnt.data(), r.cnt, P * sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        H.out_off.assign(P, 0);
        for (int q = 1; q < P; ++q) H.out_off[q] = H.out_off[q - 1] + H.out_cnt[q - 1];
        H.n_out = H.out_off[P - 1] + H.out_cnt[P - 1];
        // counts to the owners (the receiving side learns its in-counts)
        int* cnt_in = r.cnt + 64 * 0 + 32;  // scratch inside cnt's 64 slots (P <= 32)
        if (P > 32) fail(DR_ERR_PLAN, "remote plans support at most 32 ranks");
        {
            std::vector<P2P> ops;
            for (int q = 0; q < P; ++q) {
                ops.push_back(P2P{true, q, r.cnt + q, nullptr, sizeof(int)});
                ops.push_back(P2P{false, q, nullptr, cnt_in + q, sizeof(int)});
            }
            exchange(ops);
        }
        H.in_cnt.assign(P, 0);
        CK(cudaMemcpyAsync(H.in_cnt.data(), cnt_in, P * sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        H.in_off.assign(P, 0);
        for (int q = 1; q < P; ++q) H.in_off[q] = H.in_off[q - 1] + H.in_cnt[q - 1];
        H.n_in = H.in_off[P - 1] + H.in_cnt[P - 1];
        if (H.n_out > c.L.rcap || H.n_in > c.L.rcap)
            fail(DR_ERR_PLAN, "off-rank departure points exceed the scatter capacity (M/8 per rank)");
        CK(cudaMemcpyAsync(r.off, H.out_off.data(), P * sizeof(int), cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(r.cur, 0, 64 * sizeof(int), s));
        if (H.n_out > 0) {
            PB("remote_plan");
            k_remote_classify<T><<<grid_1d(g.M), 256, 0, s>>>(g, dp, 1, r.cnt, r.off, r.cur, r.ids_out, r.rec_out,
                                                                (int)c.L.rcap);
            PE("remote_plan");
        }
        {  // records to the owners
            std::vector<P2P> ops;
            for (int q = 0; q < P; ++q) {
                ops.push_back(P2P{true, q, r.rec_out + H.out_off[q], nullptr, H.out_cnt[q] * sizeof(RemoteRec<T>)});
                ops.push_back(P2P{false, q, nullptr, r.rec_in + H.in_off[q], H.in_cnt[q] * sizeof(RemoteRec<T>)});
            }
            exchange(ops);
        }
        // does any rank have remote points for this field?  (every rank must join the per-gather exchange)
        double* tot = c.at<double>(c.L.red) + 4000;
        const double mine = (double)H.n_out;
        CK(cudaMemcpyAsync(tot, &mine, sizeof(double), cudaMemcpyHostToDevice, s));
        H.any = allsum(tot) > 0;
    }
    // per gather: owners interpolate the incoming cells, values go back to the requesters
    template <int NC>
    void remote_serve(int f, const Src<T, NC>& base_src) {
        auto& H = c.rp[f];
        RP r = rp(f);
        if (H.n_in > 0) {
            PB("remote_eval");
            k_remote_eval<T, NC><<<grid_1d(H.n_in), 256, 0, s>>>(g, base_src, r.rec_in, H.n_in, r.val_in);
            PE("remote_eval");
        }
        std::vector<P2P> ops;
        for (int q = 0; q < c.nranks; ++q) {
            ops.push_back(P2P{true, q, r.val_in + (size_t)H.in_off[q] * NC, nullptr, (size_t)H.in_cnt[q] * NC * sizeof(T)});
            ops.push_back(P2P{false, q, nullptr, r.val_out + (size_t)H.out_off[q] * NC, (size_t)H.out_cnt[q] * NC * sizeof(T)});
        }
        exchange(ops);
    }

    // gather sources are ghosted fields: the kernel indexes x3 from the slot base (zg planes below).
    // pout: the ghosted output slot when the next gather reads it -- with the fused ghost exchange the
    // epilogue also stores the boundary planes into the neighbours' ghosts (EpiPeer).
    template <int NC, class Epi>
    void gather(const char* tag, Src<T, NC> src, const T* d, const int* plan_buf, Epi epi, T* pout = nullptr) {
        for (int cc = 0; cc < NC; ++cc) {
            ghosts(const_cast<T*>(src.p[cc]));
            src.p[cc] -= (size_t)g.zg * plane();
        }
        if (pout && peer_on()) {
            const int P = c.nranks, up = (c.rank + 1) % P, dn = (c.rank + P - 1) % P;
            const size_t off = (size_t)((char*)pout - c.ws);
            const int64_t pl = (int64_t)plane();
            EpiPeer<T, Epi> pe{epi, reinterpret_cast<T*>(c.comm->peer_ws(dn) + off) + g.n3 * pl,
                               reinterpret_cast<T*>(c.comm->peer_ws(up) + off) - g.n3 * pl, (uint32_t)(g.zgh * pl),
                               (uint32_t)((g.n3 - g.zg) * pl)};
            launch_gather<NC>(tag, src, d, plan_buf, pe);
            c.last_peer_out = pout;
            return;
        }
        launch_gather<NC>(tag, src, d, plan_buf, epi);
    }
    template <class Epi>
    struct IsPeer : std::false_type {};
    template <class E>
    struct IsPeer<EpiPeer<T, E>> : std::true_type {};
    template <int NC, class Epi>
    void launch_gather(const char* tag, const Src<T, NC>& src, const T* d, const int* plan_buf, const Epi& epi) {
        const int f = field_of(plan_buf);
        const bool remote = c.dist() && c.rp[f].any;
        if (remote) remote_serve<NC>(f, src);
        const Disp<T> dp{{d, d + g.M, d + 2 * g.M}};
        const int nt = (int)n_tiles(g);  // one CTA per tile
        if constexpr (std::is_same<T, float>::value && NC == 1 && !IsPeer<Epi>::value) {
            if (c.window) {  // sliding-window gather (sl.cuh k_sl_window)
                constexpr size_t sm = win_box_bytes();
                auto k = k_sl_window<Epi>;
                set_smem(k, sm);
                PB(tag);
                k<<<(unsigned)nt, SL_THREADS, sm, s>>>(g, src, dp, plan_buf, nt, epi);
                PE(tag);
                goto launched;
            }
            if (c.pairs) {  // shared-plane pair gather (sl.cuh k_sl_pairs)
                constexpr size_t sm = pairs_smem_bytes();
                auto k = k_sl_pairs<Epi>;
                set_smem(k, sm);
                PB(tag);
                k<<<(unsigned)nt, SL_THREADS, sm, s>>>(g, src, dp, plan_buf, nt, epi);
                PE(tag);
                goto launched;
            }
        }
        if constexpr (std::is_same<T, float>::value && NC == 1) {
            const GatherTma gt = gather_tma(src.p[0]);
            if (gt.use) {  // box staged by the TMA engine (sl.cuh k_sl_gather_tma)
                constexpr size_t sm = box_bytes<T, NC>();
                auto k = k_sl_gather_tma<Epi>;
                set_smem(k, sm);
                PB(tag);
                k<<<(unsigned)nt, SL_THREADS, sm, s>>>(g, src, dp, plan_buf, nt, epi, gt);
                PE(tag);
                goto launched;
            }
        }
        {
            constexpr size_t sm = box_bytes<T, NC>();
            auto k = k_sl_gather<T, NC, Epi>;
            set_smem(k, sm);
            PB(tag);
            k<<<(unsigned)nt, SL_THREADS, sm, s>>>(g, src, dp, plan_buf, nt, epi);
            PE(tag);
        }
    launched:
        if (remote && c.rp[f].n_out > 0) {
            RP r = rp(f);
            PB("remote_fixup");
            k_remote_fixup<T, NC, Epi><<<grid_1d(c.rp[f].n_out), 256, 0, s>>>(r.ids_out, r.val_out, c.rp[f].n_out, epi);
            PE("remote_fixup");
        }
    }
    int* plan_p() { return c.at<int>(c.L.plan_p); }
    int* plan_m() { return c.at<int>(c.L.plan_m); }
    int* plan_t() { return c.at<int>(c.L.plan_t); }

    void gather_scalar_p(T* f, T* out, bool next_gathered = false) {
        gather<1>("sl_state", Src<T, 1>{{f}}, dplus(), plan_p(), EpiStore<T>{out}, next_gathered ? out : nullptr);
    }

    // -------------------------------------------------------------------- API steps
    void set_velocity(const T* vin) {
        if (c.cfg.flags & DR_ISOCHORIC) {  // keep the caller's v: the gradient projects beta A v + b at once
            CK(cudaMemcpyAsync(vraw(), vin, 3 * g.M * sizeof(T), cudaMemcpyDefault, s));
            leray(cvec(vec(vraw(), (size_t)g.M)), v3());
        } else {
            for (int a = 0; a < 3; ++a)
                CK(cudaMemcpyAsync(vc(a), vin + (size_t)a * g.M, g.M * sizeof(T), cudaMemcpyDefault, s));
        }
        CK(cudaMemsetAsync(c.at<int>(c.L.maxext), 0, 16 * sizeof(int), s));
        const double h[3] = {2.0 * M_PI / g.n1, 2.0 * M_PI / g.n2, 2.0 * M_PI / g.n3g};
        const double dtt = 1.0 / c.cfg.nt;
        for (int sg = 1; sg >= -1; sg -= 2) {
            T* dout = sg > 0 ? dplus() : dminus();
            dstar_plan(tmp3(), plan_t(), (T)(sg * dtt / h[0]), (T)(sg * dtt / h[1]), (T)(sg * dtt / h[2]));
            remote_plan(0, tmp3());
            for (int a = 0; a < 3; ++a) {
                EpiDeparture1<T> e{dout + (size_t)a * g.M, vc(a), (T)(sg * 0.5 * dtt / h[a])};
                gather<1>("sl_departure", Src<T, 1>{{vc(a)}}, tmp3(), plan_t(), e);
            }
            plan(dout, sg > 0 ? plan_p() : plan_m());
            remote_plan(sg > 0 ? 1 : 2, dout);
        }
        if (!(c.cfg.flags & DR_ISOCHORIC)) {
            div(cvec(v3()), Dv());
            gather<1>("sl_multiplier", Src<T, 1>{{Dv()}}, dminus(), plan_m(), EpiMultiplier<T>{mult(), Dv(), dt()});
        }
    }
    void forward_solve() {
        for (int j = 0; j < c.cfg.nt; ++j) gather_scalar_p(rho(j), rho(j + 1), j + 1 < c.cfg.nt);
        // grad rho_0 alone (rho_T has its own slot), rho_1..rho_nt batched (one stride apart)
        grad(rho(0), G3(0));
        grad_batch(rho(1), (int64_t)gstride(), G(1), 3 * g.M, c.cfg.nt);
    }

    void adjoint_solve() {
        const int nt = c.cfg.nt;
        PB("sub");
        k_sub<T><<<grid_1d(g.M), 256, 0, s>>>(g.M, rhoR(), rho(nt), lam(nt));
        PE("sub");
        for (int k = nt; k >= 1; --k)
            gather<1>("sl_adjoint", Src<T, 1>{{lam(k)}}, dminus(), plan_m(), EpiAdjoint<T>{lam(k - 1), mult_or_null(), T(1)},
                      k > 1 ? lam(k - 1) : nullptr);
    }

    // out = beta A u + P b (P = Leray when isochoric, else I): the tail of Eq. 5e and of Eq. 4
    void reg_plus_data(V3<const T> u, V3<const T> b, V3<T> out) {
        if (c.cfg.flags & DR_ISOCHORIC) {
            // L b = b - grad Lap^-1 div b with F[div b] = F3 Q + i k3' F3 R formed in the x3 middle pass from
            // b's x1 half spectra (r2c in T: the projection damps their rounding) through the x2 stage
            // ColDivPass -- no real-space derivative passes, no transform of div b; then per component the
            // kind-6 symbol beta a(k) u_c + i k'_c D/|k'|^2 (middle kind 8 / 9) and the c2r adds b_c
            constexpr int F = (int)(sizeof(Cx<double>) / sizeof(Cx<T>));  // T spectrum slots per complex128 slot
            const int64_t su = uniform_stride(u.c), sb = uniform_stride(b.c), so = uniform_stride(out.c);
            if (!c.dist() && su && sb == so && so) {
                // one rank: the components batched per pass, D formed once per line (kind 8), Q / R in
                // place of P1 / P3 (T slots of complex128 slots 3..5; u's spectra fill slots 0..2)
                row_r2c<double>(u.c[0], specD(0), 3, su, g.S);
                col_fft_fwd<double>(specD(0), specD(0), 0, 3, g.S);
                Cx<T>* P0 = specD_t<T>(3 * F);
                row_r2c<T>(b.c[0], P0, 3, sb, g.S);
                col_div(P0, P0 + g.S, P0 + 2 * g.S, P0, P0 + 2 * g.S, 0);
                Cx<double>* sd[3] = {specD(0), specD(1), specD(2)};
                Cx<T>* sf[3] = {specF(0), specF(1), specF(2)};
                Cx<T>* sq[2] = {P0, P0 + 2 * g.S};
                middle<8>(sd, sf, 0, 1, 0, sq);
                col_fft_inv(specF(0), specF(0), 0, 3, g.S);
                row_c2r(specF(0), out.c[0], b.c[0], 3, so, g.S);
                return;
            }
            // slabs: P_a in T slots from complex128 slot 1 (spec_forward keeps slot 0 and scratch slots 6, 7),
            // Q / R in the split layout, transposed into P1 / P2's slots; kind 9 per component (same bits)
            Cx<T>* P0 = specD_t<T>(1 * F);
            for (int cc = 0; cc < 3; ++cc) row_r2c<T>(b.c[cc], P0 + (size_t)cc * g.S);
            col_div(P0, P0 + g.S, P0 + 2 * g.S, P0 + 3 * g.S, P0 + 4 * g.S, nb());
            const size_t chunk = (size_t)g.n3 * nb() * g.n1p * sizeof(Cx<T>);
            alltoall(P0 + 3 * g.S, P0, chunk);
            alltoall(P0 + 4 * g.S, P0 + g.S, chunk);
            Cx<T>* sq[2] = {P0, P0 + g.S};
            for (int cc = 0; cc < 3; ++cc) {
                spec_forward(u.c[cc], 0);
                Cx<double>* sd[1] = {specD(0)};
                Cx<T>* sf = specF(0);
                middle<9>(sd, &sf, cc, 1, 0, sq);
                spec_inverse(0, out.c[cc], b.c[cc]);
            }
        } else {
            scalar_symbol3<0>(u, out, &b);
        }
    }

    // NEXT-1: reduced gradient g = beta A v + P b, b = dt sum_j w_j lambda_j G_j (Eq. 4)
    void gradient(V3<T> gout) {
        PB("quadrature");
        k_quadrature<T><<<grid_1d(g.M), 256, 0, s>>>(g.M, c.cfg.nt, lam(0), gstride(), G(0), tmp3(), dt());
        PE("quadrature");
        if (c.cfg.flags & DR_ISOCHORIC) {
            // g = L(beta A v_in + b): beta A L v_in = L beta A v_in, so the fp32 rounding of the stored
            // projected v never meets the |k|^4 amplification (reading A20)
            Cx<double>* sd[6] = {specD(0), specD(1), specD(2), specD(3), specD(4), specD(5)};
            Cx<T>* sf[3] = {specF(0), specF(1), specF(2)};
            for (int cc = 0; cc < 3; ++cc) {
                spec_forward(vraw() + (size_t)cc * g.M, cc);
                spec_forward(tmp3() + (size_t)cc * g.M, 3 + cc);
            }
            middle<5>(sd, sf);
            for (int cc = 0; cc < 3; ++cc) spec_inverse(cc, gout.c[cc], nullptr);
        } else {
            reg_plus_data(cvec(v3()), cvec(vec(tmp3(), (size_t)g.M)), gout);
        }
    }

    // sum over all ranks of one double per rank (device scalar at `val`), identical on every rank
    // DR_CHECK_FINITE: any NaN / Inf among n values of p (device or host) on any rank -> DR_ERR_NONFINITE
    // (every rank takes the same decision: the flags are summed over ranks)
    void check_finite(const void* p, int64_t n, const char* what) {
        double* flag = c.at<double>(c.L.red) + 4001;
        double bad = 0.0;
        if (is_device_ptr(p)) {
            CK(cudaMemsetAsync(flag, 0, sizeof(double), s));
            PB("nonfinite");
            k_nonfinite<T><<<grid_1d(n), 256, 0, s>>>(n, static_cast<const T*>(p), flag);
            PE("nonfinite");
        } else {
            CK(cudaStreamSynchronize(s));
            const T* h = static_cast<const T*>(p);
            for (int64_t i = 0; i < n; ++i)
                if (!std::isfinite(h[i])) { bad = 1.0; break; }
            CK(cudaMemcpyAsync(flag, &bad, sizeof(double), cudaMemcpyHostToDevice, s));
        }
        if (allsum(flag) > 0) fail(DR_ERR_NONFINITE, std::string(what) + " holds NaN or Inf values");
    }
    double allsum(double* val) {
        double* slots = c.at<double>(c.L.red) + 3072;
        const int P = c.nranks;
        CK(cudaMemcpyAsync(slots + c.rank, val, sizeof(double), cudaMemcpyDeviceToDevice, s));
        if (c.dist()) {
            std::vector<P2P> ops;
            for (int q = 0; q < P; ++q) {
                if (q == c.rank) continue;
                ops.push_back(P2P{true, q, val, nullptr, sizeof(double)});
                ops.push_back(P2P{false, q, nullptr, slots + q, sizeof(double)});
            }
            exchange(ops);
        }
        std::vector<double> h(P);
        CK(cudaMemcpyAsync(h.data(), slots, P * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double t = 0;
        for (int q = 0; q < P; ++q) t += h[q];  // rank order: the same on every rank
        return t;
    }
    double reduce(const T* a, const T* b, const T* a2, int mode, int64_t n) {
        double* part = c.at<double>(c.L.red);
        const int nb = (int)std::min<int64_t>(2048, (n + 255) / 256);
        PB("reduce");
        k_dot_parts<T><<<nb, 256, 0, s>>>(n, a, b, a2, nullptr, part, mode);
        PE("reduce");
        PB("reduce");
        k_sum_parts<<<1, 256, 0, s>>>(part, nb, part + 2048);
        PE("reduce");
        return allsum(part + 2048);
    }
    // J = 1/2 <rho(1) - rho_R, rho(1) - rho_R> + beta/2 <v, A v>  (Eq. 2a; S:L53 inner product)
    void objective(double* J, double* misfit) {
        const double hv = (2.0 * M_PI / g.n1) * (2.0 * M_PI / g.n2) * (2.0 * M_PI / g.n3g);
        const double mis = 0.5 * hv * reduce(rho(c.cfg.nt), nullptr, rhoR(), 1, g.M);
        reg_apply(cvec(v3()), vec(tmp3(), (size_t)g.M));  // beta A v
        double vav = 0;
        for (int a = 0; a < 3; ++a) vav += reduce(vc(a), tmp3() + (size_t)a * g.M, nullptr, 0, g.M);
        if (misfit) *misfit = mis;
        if (J) *J = mis + 0.5 * hv * vav;
    }

    // ---------------------------------------------------------------- NEXT-2: inexact PCG
    T* kry(int i) { return c.at<T>(c.L.kry) + (size_t)i * 3 * g.M; }
    double dot3(const T* a, const T* b) {  // <a, b> over all ranks (D1 without the h^3 factor)
        return reduce(a, b, nullptr, 0, 3 * g.M);
    }
    void axpby(double a, const T* x, double b, T* y) {
        PB("axpby");
        k_axpby<T><<<grid_1d(3 * g.M), 256, 0, s>>>(3 * g.M, a, x, b, y);
        PE("axpby");
    }
    // H dv = -g from dv = 0, preconditioner (beta A)^-1 (+ Leray when isochoric); stop when
    // |r| <= eta |g| or after maxit matvecs.  One rank: the iteration (matvec, preconditioner, inner
    // products into device scalars, vector updates) is one CUDA graph, captured once per context and
    // replayed, with one small device-to-host read of |r|^2 per iteration -- small grids are launch-
    // bound otherwise.  Slabs (or profiling): host-scalar loop, one synchronisation per inner product.
    void pcg(const T* gin, T* dv, double eta, int maxit, int* iters, double* relres) {
        if (!c.dist() && c.graphs && !c.prof) {
            pcg_graph(gin, dv, eta, maxit, iters, relres);
            return;
        }
        T *r = kry(0), *z = kry(1), *p = kry(2), *q = kry(3);
        const size_t V = 3 * g.M;
        CK(cudaMemsetAsync(dv, 0, V * sizeof(T), s));
        axpby(-1.0, gin, 0.0, r);  // r = -g
        const double gnorm = std::sqrt(dot3(gin, gin));
        double rnorm = gnorm;
        int it = 0;
        if (gnorm > 0) {
            precond(cvec(vec(r, (size_t)g.M)), vec(z, (size_t)g.M));
            CK(cudaMemcpyAsync(p, z, V * sizeof(T), cudaMemcpyDeviceToDevice, s));
            double rz = dot3(r, z);
            while (it < maxit && rnorm > eta * gnorm) {
                hessian_matvec(p, q);
                const double alpha = rz / dot3(p, q);
                axpby(alpha, p, 1.0, dv);
                axpby(-alpha, q, 1.0, r);
                ++it;
                rnorm = std::sqrt(dot3(r, r));
                if (rnorm <= eta * gnorm) break;
                precond(cvec(vec(r, (size_t)g.M)), vec(z, (size_t)g.M));
                const double rzn = dot3(r, z);
                axpby(1.0, z, rzn / rz, p);  // p = z + (rz_new / rz) p
                rz = rzn;
            }
        }
        if (iters) *iters = it;
        if (relres) *relres = gnorm > 0 ? rnorm / gnorm : 0.0;
    }

    // device scalars of the graph PCG: [0] rz, [1] pq, [2] rr, [3] rz_new, [4] alpha, [5] beta
    double* psc() { return c.at<double>(c.L.red) + 3840; }
    void dot_dev(const T* a, const T* b, double* out, int64_t n) {
        double* part = c.at<double>(c.L.red);
        const int nb = (int)std::min<int64_t>(2048, (n + 255) / 256);
        PB("reduce");
        k_dot_parts<T><<<nb, 256, 0, s>>>(n, a, b, nullptr, nullptr, part, 0);
        PE("reduce");
        PB("reduce");
        k_sum_parts<<<1, 256, 0, s>>>(part, nb, out);
        PE("reduce");
    }
    void axpby_dev(const double* pa, double sa, const T* x, const double* pb, double cb, T* y) {
        PB("axpby");
        k_axpby_dev<T><<<grid_1d(3 * g.M), 256, 0, s>>>(3 * g.M, pa, sa, x, pb, cb, y);
        PE("axpby");
    }
    void pcg_iteration_body() {
        T *r = kry(0), *z = kry(1), *p = kry(2), *q = kry(3), *dv = kry(4);
        double* sc = psc();
        const int64_t n = 3 * g.M;
        hessian_matvec(p, q);
        dot_dev(p, q, sc + 1, n);
        PB("pcg_scalar");
        k_scalar_ratio<<<1, 32, 0, s>>>(sc, 0, 1, 4, 0);  // alpha = rz / pq
        PE("pcg_scalar");
        axpby_dev(sc + 4, 1.0, p, nullptr, 1.0, dv);   // dv += alpha p
        axpby_dev(sc + 4, -1.0, q, nullptr, 1.0, r);   // r -= alpha q
        dot_dev(r, r, sc + 2, n);
        CK(cudaMemcpyAsync(c.pinned, sc + 2, sizeof(double), cudaMemcpyDeviceToHost, s));
        precond(cvec(vec(r, (size_t)g.M)), vec(z, (size_t)g.M));
        dot_dev(r, z, sc + 3, n);
        PB("pcg_scalar");
        k_scalar_ratio<<<1, 32, 0, s>>>(sc, 3, 0, 5, 1);  // beta = rz_new / rz; rz = rz_new
        PE("pcg_scalar");
        axpby_dev(nullptr, 1.0, z, sc + 5, 0.0, p);    // p = z + beta p
    }
    void pcg_graph(const T* gin, T* dvout, double eta, int maxit, int* iters, double* relres) {
        T *r = kry(0), *z = kry(1), *p = kry(2), *dv = kry(4);
        const size_t V = 3 * g.M;
        double* sc = psc();
        if (!c.pinned) CK(cudaMallocHost(&c.pinned, sizeof(double)));
        CK(cudaMemsetAsync(dv, 0, V * sizeof(T), s));
        axpby(-1.0, gin, 0.0, r);  // r = -g
        const double gnorm = std::sqrt(dot3(gin, gin));
        double rnorm = gnorm;
        int it = 0;
        if (gnorm > 0 && maxit > 0 && rnorm > eta * gnorm) {
            precond(cvec(vec(r, (size_t)g.M)), vec(z, (size_t)g.M));
            CK(cudaMemcpyAsync(p, z, V * sizeof(T), cudaMemcpyDeviceToDevice, s));
            dot_dev(r, z, sc + 0, 3 * g.M);
            if (!c.pcg_graph) {  // capture on an internal stream (the caller's may be the legacy stream)
                const cudaStream_t user = s;
                cudaGraph_t gr = nullptr;
                s = c.hi;
                CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
                c.capturing = true;
                c.cap_ev.clear();
                try {
                    pcg_iteration_body();
                } catch (...) {
                    c.capturing = false;
                    cudaStreamEndCapture(s, &gr);
                    if (gr) cudaGraphDestroy(gr);
                    s = user;
                    throw;
                }
                c.capturing = false;
                for (const auto& p : c.cap_ev) {  // profiled launches inside the PCG graph are not retargeted
                    c.graph_events.push_back(p.a);
                    c.graph_events.push_back(p.b);
                }
                c.cap_ev.clear();
                CK(cudaStreamEndCapture(s, &gr));
                s = user;
                CK(cudaGraphInstantiate(&c.pcg_graph, gr, 0));
                CK(cudaGraphDestroy(gr));
            }
            while (it < maxit && rnorm > eta * gnorm) {
                CK(cudaGraphLaunch(c.pcg_graph, s));
                CK(cudaStreamSynchronize(s));
                ++it;
                rnorm = std::sqrt(*c.pinned);
            }
        }
        CK(cudaMemcpyAsync(dvout, dv, V * sizeof(T), cudaMemcpyDeviceToDevice, s));
        if (iters) *iters = it;
        if (relres) *relres = gnorm > 0 ? rnorm / gnorm : 0.0;
    }

    template <int QUAD>
    EpiAdjoint<T, QUAD> adjoint_epi(int k, const T* Gk, T wk, T) {
        EpiAdjoint<T, QUAD> e{};
        e.out = lt(k - 1);
        e.m = mult_or_null();
        e.b0 = bt(); e.b1 = bt() + g.M; e.b2 = bt() + 2 * g.M;
        e.G0 = Gk; e.G1 = Gk + g.M; e.G2 = Gk + 2 * g.M;
        e.w = wk;
        return e;
    }
    template <int QUAD>
    EpiAdjoint<T, QUAD, true> to_newton(const EpiAdjoint<T, QUAD>& a, int k, T dtt) {
        EpiAdjoint<T, QUAD, true> e{};
        e.out = a.out; e.m = a.m; e.scale = a.scale;
        e.b0 = a.b0; e.b1 = a.b1; e.b2 = a.b2;
        e.G0 = a.G0; e.G1 = a.G1; e.G2 = a.G2;
        e.w = a.w; e.nu = a.nu; e.snu = a.snu;
        e.H0 = a.H0; e.H1 = a.H1; e.H2 = a.H2; e.wn = a.wn;
        e.D = (c.cfg.flags & DR_ISOCHORIC) ? nullptr : Dv();
        e.snew = sN(k - 1);
        e.hdt = T(0.5) * dtt;
        e.dtt = dtt;
        return e;
    }
    // NEXT-3: the two lambda terms of the full-Newton matvec.  Needs the adjoint slices.
    //   bN = dt sum_j w_j lam_j grad rho~_j   (rho~_j recovered from the inc-state sweep's g_j)
    //   s_k = div(lam_k vt), k = 0..nt        (sources of Eq. 5c, gathered by the adjoint sweep)
    void newton_terms(const T* vt) {
        const int nt = c.cfg.nt;
        const T dtt = dt();
        V3<T> gr = vec(tmp3(), (size_t)g.M);
        bool first = true;
        for (int j = 1; j <= nt; ++j) {
            const T* rtj = rt1();
            if (j < nt) {
                PB("newton_rt");
                k_rt_from_g<T><<<grid_1d(g.M), 256, 0, s>>>(g.M, lt(j), vt, G(j), T(0.5) * dtt, sc());
                PE("newton_rt");
                rtj = sc();
            }
            grad(rtj, gr);
            const T w = (j == nt) ? T(0.5) * dtt : dtt;
            PB("newton_b");
            k_acc_lam_grad<T><<<grid_1d(g.M), 256, 0, s>>>(g.M, lam(j), tmp3(), w, bN(), first ? 1 : 0);
            PE("newton_b");
            first = false;
        }
        if (first) CK(cudaMemsetAsync(bN(), 0, 3 * g.M * sizeof(T), s));
        for (int k = 0; k <= nt; ++k) {
            PB("newton_flux");
            k_lam_vt<T><<<grid_1d(g.M), 256, 0, s>>>(g.M, lam(k), vt, tmp3());
            PE("newton_flux");
            div(cvec(gr), sN(k));
        }
    }

    // ---------------------------------------------------------------- NEXT-4: deformation map
    // u_1 = y_1 - x (Eq. 1): d_t u + v.grad u = -v, u(0) = 0, Eq. 7 with the stationary source
    // f = -v merged into the gather like Algorithm 2: w_0 = -dt/2 v, w_{j+1} = I[w_j](X+) - dt v(x),
    // u_1 = I[w_{nt-1}](X+) - dt/2 v(x).  Ping-pongs through two ghosted slots (lt(0), rho~(1)).
    void deformation(V3<T> u) {
        const int nt = c.cfg.nt;
        const T dtt = dt();
        for (int a = 0; a < 3; ++a) {
            T* w[2] = {lt(0), rt1()};
            PB("deform_init");
            k_scale<T><<<grid_1d(g.M), 256, 0, s>>>(g.M, vc(a), w[0], T(-0.5) * dtt);
            PE("deform_init");
            for (int j = 0; j < nt; ++j) {
                const bool last = (j == nt - 1);
                T* out = last ? u.c[a] : w[(j + 1) & 1];
                gather<1>("sl_deform", Src<T, 1>{{w[j & 1]}}, dplus(), plan_p(),
                          EpiAddScaled<T>{out, vc(a), last ? T(-0.5) * dtt : -dtt}, last ? nullptr : out);
            }
        }
    }
    // det grad y_1 = det(I + grad u_1) and its extrema over all ranks
    void det_grad_y(V3<const T> u, T* det, double* mn, double* mx) {
        for (int a = 0; a < 3; ++a) grad(u.c[a], vec(kry(a), (size_t)g.M));
        PB("det");
        k_det<T><<<grid_1d(g.M), 256, 0, s>>>(g.M, kry(0), kry(1), kry(2), det);
        PE("det");
        double* part = c.at<double>(c.L.red);
        const int nb = (int)std::min<int64_t>(1024, (g.M + 255) / 256);
        PB("reduce");
        k_minmax_parts<T><<<nb, 256, 0, s>>>(g.M, det, part);
        PE("reduce");
        PB("reduce");
        k_minmax_final<<<1, 256, 0, s>>>(part, nb, part + 2048);
        PE("reduce");
        // extrema over ranks: min = -max(-x); gather both per rank through allsum's slots
        double loc[2];
        CK(cudaMemcpyAsync(loc, part + 2048, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double lo = loc[0], hi = loc[1];
        if (c.dist()) {
            double* slots = c.at<double>(c.L.red) + 3072;  // [P] lows, then [P] highs
            const int P = c.nranks;
            CK(cudaMemcpyAsync(slots + c.rank, part + 2048, sizeof(double), cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(slots + 512 + c.rank, part + 2049, sizeof(double), cudaMemcpyDeviceToDevice, s));
            std::vector<P2P> ops;
            for (int q = 0; q < P; ++q) {
                if (q == c.rank) continue;
                ops.push_back(P2P{true, q, part + 2048, nullptr, sizeof(double)});
                ops.push_back(P2P{true, q, part + 2049, nullptr, sizeof(double)});
                ops.push_back(P2P{false, q, nullptr, slots + q, sizeof(double)});
                ops.push_back(P2P{false, q, nullptr, slots + 512 + q, sizeof(double)});
            }
            exchange(ops);
            std::vector<double> h(2 * 512);
            CK(cudaMemcpyAsync(h.data(), slots, 1024 * sizeof(double), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            lo = h[0];
            hi = h[512];
            for (int q = 1; q < P; ++q) {
                lo = std::min(lo, h[q]);
                hi = std::max(hi, h[512 + q]);
            }
        }
        if (mn) *mn = lo;
        if (mx) *mx = hi;
    }

    // ---------------------------------------------------------------- NEXT-4: Armijo (G)N-Krylov solver
    // g_k = g(v_k); stop at |g_k| <= gtol |g_0|; PCG on H dv = -g_k with the quadratic
    // forcing eta = min(0.5, |g_k| / |g_0|); alpha = 1, shrink until J(v + alpha dv) <= J + c1 alpha <g, dv>.
    // v: the current velocity (device, the rank's slab) -- input the initial guess, output the solution.
    void solve(T* v, const dr_solve_opts& o, dr_solve_report* rep) {
        const size_t V = 3 * g.M;
        const double hv = (2.0 * M_PI / g.n1) * (2.0 * M_PI / g.n2) * (2.0 * M_PI / g.n3g);
        T* gk = stout();  // gradient
        T* dv = stin();   // Newton step
        T* vtry = kry(0) + 0;  // trial velocity lives in the PCG's r slot only between PCG calls
        auto set_and_solve = [&](const T* vel) {
            set_velocity(vel);
            c.have_velocity = true;
            forward_solve();
            c.have_state = true;
            c.have_adjoint = false;
        };
        set_and_solve(v);
        double J = 0;
        objective(&J, nullptr);
        adjoint_solve();
        c.have_adjoint = true;
        gradient(vec(gk, (size_t)g.M));
        const double g0 = std::sqrt(hv * dot3(gk, gk));
        double gn = g0;
        int it = 0, matvecs = 0, reason = DR_SOLVE_MAX_NEWTON;
        if (rep) {
            rep->J0 = J;
            rep->g0 = g0;
        }
        for (; it < o.max_newton; ++it) {
            if (gn <= o.gtol * g0) {
                reason = DR_SOLVE_CONVERGED;
                break;
            }
            int pit = 0;
            double rr = 0;
            const double eta = std::min(0.5, gn / g0);
            pcg(gk, dv, eta, o.max_krylov, &pit, &rr);
            matvecs += pit;
            const double slope = hv * dot3(gk, dv);
            double alpha = 1.0, Jt = 0;
            bool ok = false;
            for (int b = 0; b <= o.max_backtracks; ++b) {
                CK(cudaMemcpyAsync(vtry, v, V * sizeof(T), cudaMemcpyDeviceToDevice, s));
                axpby(alpha, dv, 1.0, vtry);
                set_and_solve(vtry);
                objective(&Jt, nullptr);
                if (Jt <= J + o.c1 * alpha * slope) {
                    ok = true;
                    break;
                }
                alpha *= o.shrink;
            }
            if (!ok) {
                reason = DR_SOLVE_LINESEARCH_FAILED;
                set_and_solve(v);  // restore the state of the last accepted iterate
                break;
            }
            CK(cudaMemcpyAsync(v, vtry, V * sizeof(T), cudaMemcpyDeviceToDevice, s));
            J = Jt;
            adjoint_solve();
            c.have_adjoint = true;
            gradient(vec(gk, (size_t)g.M));
            gn = std::sqrt(hv * dot3(gk, gk));
            if (rep && rep->history && it < rep->history_len) {
                double* h = rep->history + 5 * it;
                h[0] = J;
                h[1] = gn / g0;
                h[2] = pit;
                h[3] = alpha;
                h[4] = matvecs;
            }
        }
        if (it == o.max_newton && gn <= o.gtol * g0) reason = DR_SOLVE_CONVERGED;
        if (rep) {
            rep->iterations = it;
            rep->matvecs = matvecs;
            rep->reason = reason;
            rep->J = J;
            rep->g = gn;
        }
    }

    void hessian_matvec(const T* vt, T* Hvt) {
        const int nt = c.cfg.nt;
        const T dtt = dt();
        // Optional (DR_OVERLAP=1), non-isochoric, one rank: beta A vt does not depend on the transport
        // sweeps, so its x1/x2/x3 transforms run on a low-priority stream while the gathers (bound by the
        // shared-memory datapath, HBM ~40 % busy) run on a high-priority one; only the final c2r (+ b~)
        // waits for both.  Off by default: with the three components batched per pass the overlap is
        // slower (bench step 278.8 -> 274 matvecs/s at 256^3: the gathers fill every SM, so the spectral
        // CTAs only slow their tail); it measured 2.97 -> 2.89 ms per matvec before the batching.
        const bool overlap = c.overlap && !(c.cfg.flags & DR_ISOCHORIC) && !c.dist();
        // the entry stream: the context stream, or the capture stream of the PCG graph -- the fork and
        // the join both use it, so a captured matvec stays inside its capture
        const cudaStream_t s0 = s;
        if (overlap) {
            CK(cudaEventRecord(c.ev_fork, s));
            CK(cudaStreamWaitEvent(c.aux, c.ev_fork, 0));
            s = c.aux;
            row_r2c<double>(vt, specD(0), 3, (int64_t)g.M, g.S);
            col_fft_fwd<double>(specD(0), specD(0), 0, 3, g.S);
            Cx<double>* sd = specD(0);
            Cx<T>* sf = specF(0);
            middle<0>(&sd, &sf, 0, 3, g.S);
            col_fft_inv(specF(0), specF(0), 0, 3, g.S);
            CK(cudaEventRecord(c.ev_join, s));
            // the sweeps go to the high-priority stream so their CTAs are scheduled first and the
            // spectral CTAs fill the remaining SM resources
            CK(cudaStreamWaitEvent(c.hi, c.ev_fork, 0));
            s = c.hi;
        }

        // incremental state (Algorithm 2, merged gather g_j = rho~_j + dt/2 f_j)
        PB("inc_init");
        k_inc_init<T><<<grid_1d(g.M), 256, 0, s>>>(g.M, vt, G(0), lt(0), T(0.5) * dtt);
        PE("inc_init");
        for (int j = 0; j < nt; ++j) {
            const bool last = (j == nt - 1);
            const T* Gj = G(j + 1);
            EpiIncState<T> e{last ? rt1() : lt(j + 1), vt, vt + g.M, vt + 2 * g.M, Gj, Gj + g.M, Gj + 2 * g.M,
                             last ? T(0.5) * dtt : dtt};
            if (last && !newton()) {  // GN: the last step also writes b~'s k = nt term (EpiIncState WB)
                EpiIncState<T, true> eb{e.out, e.vt0, e.vt1, e.vt2, e.G0, e.G1, e.G2, e.c,
                                        bt(), bt() + g.M, bt() + 2 * g.M, T(0.5) * dtt * T(-1)};
                gather<1>("sl_inc_state_b", Src<T, 1>{{lt(j)}}, dplus(), plan_p(), eb, e.out);
            } else {
                gather<1>("sl_inc_state", Src<T, 1>{{lt(j)}}, dplus(), plan_p(), e, e.out);
            }
        }
        if (newton()) newton_terms(vt);
        // incremental adjoint (GN): lambda~_nt = -rho~(1), lambda~_{k-1} = m I[lambda~_k](X-); every step
        // also accumulates its term of the b~ trapezoid quadrature in its epilogue
        for (int k = nt; k >= 1; --k) {
            T* src = (k == nt) ? rt1() : lt(k);
            const T* Gk = G(k - 1);
            const T wk = (k - 1 == 0) ? T(0.5) * dtt : dtt;
            if (k == nt && !newton()) {  // b~ already holds the k = nt term (sl_inc_state_b)
                auto e = adjoint_epi<2>(k, Gk, wk, dtt);
                e.scale = T(-1);
                gather<1>("sl_inc_adjoint_q2", Src<T, 1>{{src}}, dminus(), plan_m(), e, k > 1 ? e.out : nullptr);
            } else if (k == nt) {
                auto e = adjoint_epi<1>(k, Gk, wk, dtt);
                e.scale = T(-1);
                e.nu = rt1(); e.snu = T(-1);
                const T* Gn = G(nt);
                e.H0 = Gn; e.H1 = Gn + g.M; e.H2 = Gn + 2 * g.M;
                e.wn = T(0.5) * dtt;
                gather<2>("sl_inc_adjoint_n1", Src<T, 2>{{src, sN(k)}}, dminus(), plan_m(), to_newton(e, k, dtt),
                          k > 1 ? e.out : nullptr);
            } else {
                auto e = adjoint_epi<2>(k, Gk, wk, dtt);
                e.scale = T(1);
                if (newton()) gather<2>("sl_inc_adjoint_n2", Src<T, 2>{{src, sN(k)}}, dminus(), plan_m(), to_newton(e, k, dtt),
                                        k > 1 ? e.out : nullptr);
                else gather<1>("sl_inc_adjoint_q2", Src<T, 1>{{src}}, dminus(), plan_m(), e, k > 1 ? e.out : nullptr);
            }
        }
        if (newton()) axpby(1.0, bN(), 1.0, bt());  // b~ += int lam grad rho~ dt
        // spectral tail: H vt = beta A vt + P b~
        if (overlap) {  // beta A vt was transformed on the aux stream; only the c2r + b~ remains
            CK(cudaEventRecord(c.ev_hi, s));
            s = s0;
            CK(cudaStreamWaitEvent(s, c.ev_hi, 0));
            CK(cudaStreamWaitEvent(s, c.ev_join, 0));
            row_c2r(specF(0), Hvt, bt(), 3, (int64_t)g.M, g.S);
        } else {
            reg_plus_data(cvec(vec(const_cast<T*>(vt), (size_t)g.M)), cvec(vec(bt(), (size_t)g.M)),
                          vec(Hvt, (size_t)g.M));
        }
    }
};

template <typename F>
dr_status run(dr_ctx* c, F&& f) {
    if (!c) return DR_ERR_ARG;
    try {
        f();
        c->err.clear();
        return DR_OK;
    } catch (const DrError& e) {
        c->err = e.msg;
        return e.s;
    } catch (const NcclError& e) {
        c->err = e.what();
        return DR_ERR_NCCL;
    } catch (const std::exception& e) {
        c->err = e.what();
        return DR_ERR_CUDA;
    }
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

size_t elem_size(const dr_ctx* c) { return (c->cfg.flags & DR_FP64) ? 8 : 4; }

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// input: 16-byte aligned device pointers are used in place; host pointers and unaligned device
// pointers (the kernels' bulk copies and vector loads need 16 bytes) are staged into `stage`
const void* stage_in(dr_ctx* c, const void* p, size_t bytes, void* stage) {
    if (is_device_ptr(p) && aligned16(p)) return p;
    CK(cudaMemcpyAsync(stage, p, bytes, cudaMemcpyDefault, c->stream));
    return stage;
}

template <typename F>
void with_output(dr_ctx* c, void* out, size_t bytes, void* stage, F&& f) {
    const bool dev = is_device_ptr(out);
    if (dev && aligned16(out)) {
        f(out);
        return;
    }
    f(stage);
    CK(cudaMemcpyAsync(out, stage, bytes, cudaMemcpyDefault, c->stream));
    if (!dev) CK(cudaStreamSynchronize(c->stream));
}

template <typename F>
void dispatch(dr_ctx* c, F&& f) {
    if (c->cfg.flags & DR_FP64) {
        Impl<double> im(*c);
        f(im);
    } else {
        Impl<float> im(*c);
        f(im);
    }
}
template <typename F>
void dispatch_on(dr_ctx* c, cudaStream_t st, F&& f) {  // the work issued on stream st
    if (c->cfg.flags & DR_FP64) {
        Impl<double> im(*c, c->g, st);
        f(im);
    } else {
        Impl<float> im(*c, c->g, st);
        f(im);
    }
}

void destroy_graph(dr_ctx::CallGraph& e) {
    if (e.exec) cudaGraphExecDestroy(e.exec);
    if (e.graph) cudaGraphDestroy(e.graph);
    for (cudaEvent_t ev : e.own) cudaEventDestroy(ev);
    e = dr_ctx::CallGraph{};
}

std::string prof_signature(const dr_ctx* c) { return c->prof ? "on:" + c->prof_only : "off"; }

// Run body(stream) as a cached CUDA graph keyed by (kind, a, b): captured on the internal stream c->hi
// the first time, then replayed on the context stream.  Profiled launches (dr_profile_*) are event-
// record nodes in the graph; every replay points them at fresh pool events, so the per-kernel
// accounting is the same as in eager execution.  Loopback slabs (host barriers) run eagerly.
template <typename F>
void run_graph(dr_ctx* c, int kind, const void* a, const void* b, F&& body) {
    if (!c->graphs || (c->dist() && !c->comm->capturable())) {
        body(c->stream);
        return;
    }
    const std::string sig = prof_signature(c);
    dr_ctx::CallGraph* e = nullptr;
    for (auto& x : c->call_graphs)
        if (x.kind == kind && x.a == a && x.b == b && x.epoch == c->graph_epoch && x.prof_sig == sig) e = &x;
    if (!e) {
        // drop stale entries; cap the cache (distinct argument pointers each capture once)
        std::vector<dr_ctx::CallGraph> keep;
        for (auto& x : c->call_graphs) {
            if (x.epoch == c->graph_epoch && x.prof_sig == sig && keep.size() < 31) keep.push_back(x);
            else destroy_graph(x);
        }
        c->call_graphs.swap(keep);
        dr_ctx::CallGraph ng;
        ng.kind = kind;
        ng.a = a;
        ng.b = b;
        ng.epoch = c->graph_epoch;
        ng.prof_sig = sig;
        const int64_t l0 = c->launches;
        cudaStream_t cs = c->hi;
        CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        c->capturing = true;
        c->cap_ev.clear();
        try {
            body(cs);
        } catch (...) {
            c->capturing = false;
            cudaGraph_t gr = nullptr;
            cudaStreamEndCapture(cs, &gr);
            if (gr) cudaGraphDestroy(gr);
            for (const auto& p : c->cap_ev) {
                cudaEventDestroy(p.a);
                cudaEventDestroy(p.b);
            }
            c->cap_ev.clear();
            c->launches = l0;
            throw;
        }
        c->capturing = false;
        CK(cudaStreamEndCapture(cs, &ng.graph));
        ng.launches = c->launches - l0;
        c->launches = l0;
        // map the profiler's events to their record nodes
        size_t nn = 0;
        CK(cudaGraphGetNodes(ng.graph, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) CK(cudaGraphGetNodes(ng.graph, nodes.data(), &nn));
        auto node_of = [&](cudaEvent_t ev) -> cudaGraphNode_t {
            for (cudaGraphNode_t n : nodes) {
                cudaGraphNodeType t;
                CK(cudaGraphNodeGetType(n, &t));
                if (t != cudaGraphNodeTypeEventRecord) continue;
                cudaEvent_t x = nullptr;
                CK(cudaGraphEventRecordNodeGetEvent(n, &x));
                if (x == ev) return n;
            }
            fail(DR_ERR_CUDA, "profiler event node missing from the captured graph");
        };
        for (const auto& p : c->cap_ev) {
            ng.ev.push_back(dr_ctx::CallGraph::EvNode{p.tag, node_of(p.a), node_of(p.b)});
            ng.own.push_back(p.a);
            ng.own.push_back(p.b);
        }
        c->cap_ev.clear();
        CK(cudaGraphInstantiate(&ng.exec, ng.graph, 0));
        c->call_graphs.push_back(ng);
        e = &c->call_graphs.back();
    }
    for (const auto& en : e->ev) {
        cudaEvent_t x = c->take_event(), y = c->take_event();
        CK(cudaGraphExecEventRecordNodeSetEvent(e->exec, en.a, x));
        CK(cudaGraphExecEventRecordNodeSetEvent(e->exec, en.b, y));
        c->pending.push_back(dr_ctx::Pending{en.tag, x, y});
    }
    CK(cudaGraphLaunch(e->exec, c->stream));
    c->launches += e->launches;
}

bool graphable(const void* a, const void* b) {  // device buffers the kernels use in place
    return is_device_ptr(a) && aligned16(a) && is_device_ptr(b) && aligned16(b);
}

template <typename F>
dr_status comm_run(F&& f) {
    try {
        f();
        return DR_OK;
    } catch (const NcclError&) {
        return DR_ERR_NCCL;
    } catch (const std::exception&) {
        return DR_ERR_NCCL;
    }
}

}  // namespace

extern "C" {

size_t dr_workspace_bytes(const dr_config* cfg) { return dr_workspace_bytes_dist(cfg, 1); }

size_t dr_workspace_bytes_dist(const dr_config* cfg, int nranks) {
    if (validate(cfg, nranks) != DR_OK) return 0;
    return layout(cfg, nranks).total;
}

dr_status dr_slab(const dr_config* cfg, int nranks, int rank, int* z0, int* nz) {
    const dr_status v = validate(cfg, nranks);
    if (v != DR_OK) return v;
    if (rank < 0 || rank >= nranks || !z0 || !nz) return DR_ERR_ARG;
    const Grid g = make_grid(cfg, rank, nranks);
    *z0 = g.z0;
    *nz = g.n3;
    return DR_OK;
}

dr_status dr_nccl_get_unique_id(uint8_t out[128]) {
    if (!out) return DR_ERR_ARG;
    return comm_run([&] {
        ncclUniqueId id;
        nccl_ck(NcclApi::get().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, id.internal, 128);
    });
}

dr_status dr_comm_create_nccl(const uint8_t uid[128], int rank, int nranks, dr_comm** out) {
    if (!uid || !out || nranks < 1 || rank < 0 || rank >= nranks) return DR_ERR_ARG;
    *out = nullptr;
    return comm_run([&] {
        auto* c = new dr_comm();
        try {
            c->impl.reset(new NcclComm(uid, rank, nranks));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

dr_status dr_peer_export(dr_ctx* c, uint8_t handle[64], uint64_t* offset) {
    if (!c || !handle || !offset) return DR_ERR_ARG;
    return run(c, [&] {
        static const auto range = [] {
            cudaDriverEntryPointQueryResult q;
            void* fn = nullptr;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess) {
                cudaGetLastError();
                fn = nullptr;
            }
            return reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(fn);
        }();
        if (!range) fail(DR_ERR_CUDA, "cuMemGetAddressRange unavailable");
        CUdeviceptr base = 0;
        size_t size = 0;
        if (range(&base, &size, (CUdeviceptr)c->ws) != CUDA_SUCCESS) fail(DR_ERR_CUDA, "cuMemGetAddressRange failed");
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, (void*)base));
        static_assert(sizeof(h) == 64, "IPC handle size");
        std::memcpy(handle, &h, 64);
        *offset = (uint64_t)((CUdeviceptr)c->ws - base);
    });
}

dr_status dr_peer_import(dr_ctx* c, const uint8_t* handles, const uint64_t* offsets) {
    if (!c || !handles || !offsets) return DR_ERR_ARG;
    auto* nc = dynamic_cast<NcclComm*>(c->comm);
    if (!nc) return DR_ERR_ARG;
    return run(c, [&] {
        const int P = nc->size, r = nc->rank;
        nc->peers.assign(P, nullptr);
        nc->peers[r] = c->ws;
        for (int q = 0; q < P; ++q) {  // every rank: neighbours for the ghosts, all for the transposes
            if (q == r) continue;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles + (size_t)q * 64, 64);
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            nc->opened.push_back(p);
            nc->peers[q] = static_cast<char*>(p) + offsets[q];
        }
        if (P <= 64) {  // the device table of rank workspaces (filled here, outside any graph capture)
            CK(cudaMemcpyAsync(c->ws + c->L.pflags + 1024, nc->peers.data(), P * sizeof(char*), cudaMemcpyHostToDevice,
                               c->stream));
            CK(cudaStreamSynchronize(c->stream));
            c->pws_ready = true;
        }
    });
}

dr_status dr_hub_create(int nranks, dr_hub** out) {
    if (!out || nranks < 1) return DR_ERR_ARG;
    auto* h = new dr_hub();
    h->impl.reset(new Hub(nranks));
    *out = h;
    return DR_OK;
}

dr_status dr_hub_destroy(dr_hub* h) {
    if (!h) return DR_ERR_ARG;
    delete h;
    return DR_OK;
}

dr_status dr_comm_create_loopback(dr_hub* hub, int rank, dr_comm** out) {
    if (!hub || !out || rank < 0 || rank >= hub->impl->size) return DR_ERR_ARG;
    auto* c = new dr_comm();
    c->impl.reset(new LoopbackComm(hub->impl.get(), rank));
    *out = c;
    return DR_OK;
}

dr_status dr_comm_destroy(dr_comm* c) {
    if (!c) return DR_ERR_ARG;
    delete c;
    return DR_OK;
}

namespace {
__global__ void k_fill_rank(int* buf, int n, int value) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = value * 1000 + i;
}
}  // namespace

dr_status dr_comm_selftest(dr_comm* comm, void* stream, int* ok) {
    if (!comm || !ok) return DR_ERR_ARG;
    *ok = 0;
    Comm& C = *comm->impl;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int P = C.size, n = 256;
    int *send = nullptr, *recv = nullptr;
    if (cudaMalloc(&send, (size_t)P * n * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&recv, (size_t)P * n * sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        if (send) cudaFree(send);
        return DR_ERR_OOM;
    }
    dr_status st = DR_OK;
    try {
        for (int q = 0; q < P; ++q) k_fill_rank<<<1, 256, 0, s>>>(send + q * n, n, C.rank);
        cudaMemsetAsync(recv, 0xff, (size_t)P * n * sizeof(int), s);
        std::vector<P2P> ops;
        for (int q = 0; q < P; ++q) {  // an all-to-all of rank-stamped chunks, self included
            ops.push_back(P2P{true, q, send + q * n, nullptr, n * sizeof(int)});
            ops.push_back(P2P{false, q, nullptr, recv + q * n, n * sizeof(int)});
        }
        C.group(ops, s);
        std::vector<int> h((size_t)P * n);
        if (cudaMemcpyAsync(h.data(), recv, h.size() * sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            st = DR_ERR_CUDA;
        bool good = st == DR_OK;
        for (int q = 0; q < P && good; ++q)
            for (int i = 0; i < n; ++i)
                if (h[(size_t)q * n + i] != q * 1000 + i) good = false;
        *ok = good ? 1 : 0;
        if (!C.check().empty()) st = DR_ERR_NCCL;
    } catch (const std::exception&) {
        st = DR_ERR_NCCL;
    }
    cudaFree(send);
    cudaFree(recv);
    cudaGetLastError();
    return st;
}

dr_status dr_create(const dr_config* cfg, void* workspace, size_t workspace_bytes, void* stream, dr_ctx** out) {
    return dr_create_dist(cfg, nullptr, workspace, workspace_bytes, stream, out);
}

dr_status dr_create_dist(const dr_config* cfg, dr_comm* comm, void* workspace, size_t workspace_bytes, void* stream,
                         dr_ctx** out) {
    if (!out) return DR_ERR_ARG;
    *out = nullptr;
    const int nranks = comm ? comm->impl->size : 1;
    const int rank = comm ? comm->impl->rank : 0;
    const dr_status v = validate(cfg, nranks);
    if (v != DR_OK) return v;
    dr_ctx* c = new dr_ctx();
    c->cfg = *cfg;
    c->rank = rank;
    c->nranks = nranks;
    c->comm = comm ? comm->impl.get() : nullptr;
    c->g = make_grid(cfg, rank, nranks);
    c->L = layout(cfg, nranks);
    c->stream = reinterpret_cast<cudaStream_t>(stream);
    {
        int dev = 0, nsm = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && nsm > 0)
            c->num_sms = nsm;
        c->dev = dev;
        cudaGetLastError();
    }
    if (workspace) {
        if (workspace_bytes < c->L.total) {
            delete c;
            return DR_ERR_OOM;
        }
        c->ws = static_cast<char*>(workspace);
    } else {
        if (cudaMalloc(&c->ws, c->L.total) != cudaSuccess) {
            cudaGetLastError();
            delete c;
            return DR_ERR_OOM;
        }
        c->own_ws = true;
    }
    {
        const char* ov = getenv("DR_OVERLAP");
        c->overlap = ov && ov[0] == '1';
        const char* tm = getenv("DR_TMA_MIDDLE");
        c->tma_middle = !(tm && tm[0] == '0');
        const char* gr = getenv("DR_GRAPHS");
        c->graphs = !(gr && gr[0] == '0');
        const char* ch = getenv("DR_CHUNK");
        c->chunk = ch ? atoi(ch) : 0;
        const char* wi = getenv("DR_WINDOW");
        c->window = wi && wi[0] == '1';
        const char* gtm = getenv("DR_GATHER_TMA");
        c->gather_tma = !(gtm && gtm[0] == '0');
        const char* pa = getenv("DR_PAIRS");
        c->pairs = pa && pa[0] == '1';
        const char* p2 = getenv("DR_PLANE2D");
        c->plane2d = p2 && p2[0] == '1';
        const char* rg = getenv("DR_RING");
        c->ring = rg ? atoi(rg) : 0;
        const char* pg = getenv("DR_PEER_GHOSTS");
        c->peer_ghosts = pg && pg[0] == '1' && nranks > 1;
    }
    if (c->comm) c->comm->set_ws(c->ws);
    if (cudaMemsetAsync(c->ws + c->L.pflags, 0, 2048, c->stream) != cudaSuccess) {
        cudaGetLastError();
        if (c->own_ws) cudaFree(c->ws);
        delete c;
        return DR_ERR_CUDA;
    }
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_hi, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        if (c->own_ws) cudaFree(c->ws);
        delete c;
        return DR_ERR_CUDA;
    }
    const dr_status st = run(c, [&] { dispatch(c, [](auto& im) { im.init_twiddles(); }); });
    if (st != DR_OK) {
        if (c->own_ws) cudaFree(c->ws);
        delete c;
        return st;
    }
    *out = c;
    return DR_OK;
}

dr_status dr_destroy(dr_ctx* c) {
    if (!c) return DR_ERR_ARG;
    cudaStreamSynchronize(c->stream);
    if (c->aux) {
        cudaStreamSynchronize(c->aux);
        cudaStreamDestroy(c->aux);
    }
    if (c->hi) {
        cudaStreamSynchronize(c->hi);
        cudaStreamDestroy(c->hi);
    }
    if (c->ev_hi) cudaEventDestroy(c->ev_hi);
    if (c->comm) c->comm->set_ws(nullptr);
    if (c->pcg_graph) cudaGraphExecDestroy(c->pcg_graph);
    for (auto& e : c->call_graphs) destroy_graph(e);
    for (cudaEvent_t e : c->graph_events) cudaEventDestroy(e);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    if (c->own_ws) {
        cudaStreamSynchronize(c->stream);
        cudaFree(c->ws);
    }
    delete c;
    return DR_OK;
}

dr_status dr_set_images(dr_ctx* c, const void* rho_T, const void* rho_R) {
    return run(c, [&] {
        // (captured matvec / preconditioner graphs stay valid: they read the images' fixed workspace slots)
        if (!rho_T || !rho_R) fail(DR_ERR_ARG, "rho_T and rho_R must be non-NULL");
        dispatch(c, [&](auto& im) {
            if (c->cfg.flags & DR_CHECK_FINITE) {
                im.check_finite(rho_T, c->g.M, "rho_T");
                im.check_finite(rho_R, c->g.M, "rho_R");
            }
            const size_t F = c->g.M * elem_size(c);
            CK(cudaMemcpyAsync(im.rhoT(), rho_T, F, cudaMemcpyDefault, c->stream));
            CK(cudaMemcpyAsync(im.rhoR(), rho_R, F, cudaMemcpyDefault, c->stream));
        });
        c->have_images = true;
        c->have_state = c->have_adjoint = c->have_matvec = false;
    });
}

dr_status dr_set_velocity(dr_ctx* c, const void* v) {
    return run(c, [&] {
        // One rank: the captured matvec / preconditioner graphs read the velocity's products (displacements,
        // tile plans, multiplier, state gradients) from fixed workspace slots and take no host-side decision
        // on them, so they stay valid.  Slabs: the off-rank plans' host counts are baked into the launches.
        if (c->dist()) ++c->graph_epoch;
        if (!v) fail(DR_ERR_ARG, "v must be non-NULL");
        c->have_velocity = false;
        c->have_state = c->have_adjoint = c->have_matvec = false;
        dispatch(c, [&](auto& im) {
            using T = std::remove_pointer_t<decltype(im.rhoR())>;
            if (c->cfg.flags & DR_CHECK_FINITE) im.check_finite(v, 3 * c->g.M, "v");
            im.set_velocity(static_cast<const T*>(v));
        });
        c->have_velocity = true;
    });
}

dr_status dr_forward_solve(dr_ctx* c, void* rho1_out) {
    return run(c, [&] {
        if (!c->have_images || !c->have_velocity) fail(DR_ERR_ORDER, "forward_solve needs set_images and set_velocity");
        dispatch(c, [&](auto& im) {
            im.forward_solve();
            c->have_state = true;
            c->have_adjoint = c->have_matvec = false;
            if (rho1_out) {
                CK(cudaMemcpyAsync(rho1_out, im.rho(c->cfg.nt), c->g.M * elem_size(c), cudaMemcpyDefault, c->stream));
                if (!is_device_ptr(rho1_out)) CK(cudaStreamSynchronize(c->stream));
            }
        });
    });
}

dr_status dr_adjoint_solve(dr_ctx* c, void* lambda0_out) {
    return run(c, [&] {
        if (!c->have_state) fail(DR_ERR_ORDER, "adjoint_solve needs forward_solve");
        dispatch(c, [&](auto& im) {
            im.adjoint_solve();
            c->have_adjoint = true;
            if (lambda0_out) {
                CK(cudaMemcpyAsync(lambda0_out, im.lam(0), c->g.M * elem_size(c), cudaMemcpyDefault, c->stream));
                if (!is_device_ptr(lambda0_out)) CK(cudaStreamSynchronize(c->stream));
            }
        });
    });
}

dr_status dr_hessian_matvec(dr_ctx* c, const void* vt, void* Hvt) {
    return run(c, [&] {
        if (!vt || !Hvt) fail(DR_ERR_ARG, "vt and Hvt must be non-NULL");
        if (vt == Hvt) fail(DR_ERR_ARG, "vt and Hvt must not alias");
        if (!c->have_state) fail(DR_ERR_ORDER, "hessian_matvec needs forward_solve");
        const size_t V = 3 * c->g.M * elem_size(c);
        if (c->cfg.flags & DR_CHECK_FINITE) dispatch(c, [&](auto& im) { im.check_finite(vt, 3 * c->g.M, "vt"); });
        if ((c->cfg.flags & DR_FULL_NEWTON) && !c->have_adjoint) {  // the lambda terms need the adjoint slices
            dispatch(c, [&](auto& im) { im.adjoint_solve(); });
            c->have_adjoint = true;
        }
        auto body = [&](const void* in, void* out, cudaStream_t st) {
            dispatch_on(c, st, [&](auto& im) {
                using T = std::remove_pointer_t<decltype(im.rhoR())>;
                im.hessian_matvec(static_cast<const T*>(in), static_cast<T*>(out));
            });
        };
        if (graphable(vt, Hvt)) {
            run_graph(c, 1, vt, Hvt, [&](cudaStream_t st) { body(vt, Hvt, st); });
        } else {
            const void* in = stage_in(c, vt, V, c->ws + c->L.stin);
            with_output(c, Hvt, V, c->ws + c->L.stout, [&](void* out) { body(in, out, c->stream); });
        }
        c->have_matvec = true;
    });
}

dr_status dr_precond_apply(dr_ctx* c, const void* r, void* z) {
    return run(c, [&] {
        if (!r || !z) fail(DR_ERR_ARG, "r and z must be non-NULL");
        const size_t V = 3 * c->g.M * elem_size(c);
        if (c->cfg.flags & DR_CHECK_FINITE) dispatch(c, [&](auto& im) { im.check_finite(r, 3 * c->g.M, "r"); });
        auto body = [&](const void* in, void* out, cudaStream_t st) {
            dispatch_on(c, st, [&](auto& im) {
                using T = std::remove_pointer_t<decltype(im.rhoR())>;
                const T* i = static_cast<const T*>(in);
                im.precond(cvec(vec(const_cast<T*>(i), (size_t)c->g.M)), vec(static_cast<T*>(out), (size_t)c->g.M));
            });
        };
        if (graphable(r, z)) {
            run_graph(c, 2, r, z, [&](cudaStream_t st) { body(r, z, st); });
        } else {
            const void* in = stage_in(c, r, V, c->ws + c->L.stin);
            with_output(c, z, V, c->ws + c->L.stout, [&](void* out) { body(in, out, c->stream); });
        }
    });
}
dr_status dr_gradient(dr_ctx* c, void* gout) {
    return run(c, [&] {
        if (!gout) fail(DR_ERR_ARG, "g must be non-NULL");
        if (!c->have_state) fail(DR_ERR_ORDER, "gradient needs forward_solve");
        const size_t V = 3 * c->g.M * elem_size(c);
        with_output(c, gout, V, c->ws + c->L.stout, [&](void* out) {
            dispatch(c, [&](auto& im) {
                using T = std::remove_pointer_t<decltype(im.rhoR())>;
                if (!c->have_adjoint) {
                    im.adjoint_solve();
                    c->have_adjoint = true;
                }
                im.gradient(vec(static_cast<T*>(out), (size_t)c->g.M));
            });
        });
    });
}

dr_status dr_objective(dr_ctx* c, double* J, double* misfit) {
    return run(c, [&] {
        if (!c->have_state) fail(DR_ERR_ORDER, "objective needs forward_solve");
        dispatch(c, [&](auto& im) { im.objective(J, misfit); });
    });
}

dr_status dr_pcg(dr_ctx* c, const void* g, void* dv, double eta, int maxit, int* iters, double* relres) {
    return run(c, [&] {
        if (!g || !dv) fail(DR_ERR_ARG, "g and dv must be non-NULL");
        if (g == dv) fail(DR_ERR_ARG, "g and dv must not alias");
        if (!(eta >= 0.0) || maxit < 0) fail(DR_ERR_ARG, "eta >= 0 and maxit >= 0 required");
        if (!c->have_state) fail(DR_ERR_ORDER, "pcg needs forward_solve");
        const size_t V = 3 * c->g.M * elem_size(c);
        const void* in = stage_in(c, g, V, c->ws + c->L.stin);
        with_output(c, dv, V, c->ws + c->L.stout, [&](void* out) {
            dispatch(c, [&](auto& im) {
                using T = std::remove_pointer_t<decltype(im.rhoR())>;
                if (im.newton() && !c->have_adjoint) {
                    im.adjoint_solve();
                    c->have_adjoint = true;
                }
                im.pcg(static_cast<const T*>(in), static_cast<T*>(out), eta, maxit, iters, relres);
            });
        });
        c->have_matvec = false;  // the matvec test hooks would show the last Krylov matvec
    });
}

dr_status dr_deformation(dr_ctx* c, void* u, void* det, double* det_min, double* det_max) {
    return run(c, [&] {
        if (!c->have_velocity) fail(DR_ERR_ORDER, "deformation needs set_velocity");
        const size_t V = 3 * c->g.M * elem_size(c), F = c->g.M * elem_size(c);
        dispatch(c, [&](auto& im) {
            using T = std::remove_pointer_t<decltype(im.rhoR())>;
            T* uo = im.tmp3();
            im.deformation(vec(uo, (size_t)c->g.M));
            c->have_matvec = false;  // the deformation reuses the matvec's scratch slices
            if (det || det_min || det_max) {
                T* d = im.bt();  // scratch scalar (b~ is not needed afterwards)
                im.det_grad_y(cvec(vec(uo, (size_t)c->g.M)), d, det_min, det_max);
                if (det) CK(cudaMemcpyAsync(det, d, F, cudaMemcpyDefault, c->stream));
            }
            if (u) CK(cudaMemcpyAsync(u, uo, V, cudaMemcpyDefault, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        });
    });
}

dr_status dr_solve(dr_ctx* c, void* v, const dr_solve_opts* opts, dr_solve_report* rep) {
    return run(c, [&] {
        if (!v) fail(DR_ERR_ARG, "v must be non-NULL");
        if (!c->have_images) fail(DR_ERR_ORDER, "solve needs set_images");
        dr_solve_opts o{1e-2, 50, 100, 1e-4, 0.5, 20};
        if (opts) o = *opts;
        if (!(o.gtol > 0) || o.max_newton < 0 || o.max_krylov < 1 || !(o.c1 > 0 && o.c1 < 1) ||
            !(o.shrink > 0 && o.shrink < 1) || o.max_backtracks < 0)
            fail(DR_ERR_PARAM, "invalid solver options");
        if (!is_device_ptr(v)) fail(DR_ERR_ARG, "dr_solve takes a device velocity");
        dispatch(c, [&](auto& im) {
            using T = std::remove_pointer_t<decltype(im.rhoR())>;
            im.solve(static_cast<T*>(v), o, rep);
        });
        c->have_matvec = false;
        CK(cudaStreamSynchronize(c->stream));
    });
}

dr_status dr_profile_enable(dr_ctx* c, int enable) {
    return run(c, [&] {
        c->prof_flush();
        c->prof = enable != 0;
    });
}

dr_status dr_profile_only(dr_ctx* c, const char* tag) {
    if (!c) return DR_ERR_ARG;
    c->prof_only = tag ? tag : "";
    return DR_OK;
}

dr_status dr_profile_reset(dr_ctx* c) {
    return run(c, [&] {
        c->prof_flush();
        c->acc.clear();
        c->launches = 0;
    });
}

dr_status dr_profile_count(dr_ctx* c, int* n_entries, int64_t* launches) {
    return run(c, [&] {
        c->prof_flush();
        if (n_entries) *n_entries = (int)c->acc.size();
        if (launches) *launches = c->launches;
    });
}

dr_status dr_profile_entry(dr_ctx* c, int i, char* name, int name_len, int64_t* launches, double* total_ms) {
    return run(c, [&] {
        c->prof_flush();
        if (i < 0 || i >= (int)c->acc.size()) fail(DR_ERR_ARG, "profile entry out of range");
        const auto& a = c->acc[i];
        if (name && name_len > 0) {
            std::strncpy(name, a.tag.c_str(), name_len - 1);
            name[name_len - 1] = 0;
        }
        if (launches) *launches = a.n;
        if (total_ms) *total_ms = a.ms;
    });
}

dr_status dr_sync(dr_ctx* c) {
    return run(c, [&] {
        CK(cudaStreamSynchronize(c->stream));
        if (c->comm) {
            const std::string e = c->comm->check();
            if (!e.empty()) fail(DR_ERR_NCCL, e);
        }
    });
}

const char* dr_last_error(const dr_ctx* c) { return c ? c->err.c_str() : "null context"; }

const char* dr_status_string(dr_status s) {
    switch (s) {
        case DR_OK: return "DR_OK";
        case DR_ERR_ARG: return "DR_ERR_ARG";
        case DR_ERR_GRID: return "DR_ERR_GRID";
        case DR_ERR_PARAM: return "DR_ERR_PARAM";
        case DR_ERR_ORDER: return "DR_ERR_ORDER";
        case DR_ERR_CUDA: return "DR_ERR_CUDA";
        case DR_ERR_NCCL: return "DR_ERR_NCCL";
        case DR_ERR_OOM: return "DR_ERR_OOM";
        case DR_ERR_NONFINITE: return "DR_ERR_NONFINITE";
        case DR_ERR_PLAN: return "DR_ERR_PLAN";
    }
    return "unknown";
}

dr_status dr_op_spectral(dr_ctx* c, int op, const void* in, void* out) {
    return run(c, [&] {
        if (!in || !out) fail(DR_ERR_ARG, "in/out must be non-NULL");
        if (op < DR_OP_GRAD || op > DR_OP_LERAY) fail(DR_ERR_ARG, "unknown spectral op");
        const size_t F = c->g.M * elem_size(c);
        const void* ip = stage_in(c, in, op == DR_OP_GRAD ? F : 3 * F, c->ws + c->L.stin);
        with_output(c, out, op == DR_OP_DIV ? F : 3 * F, c->ws + c->L.stout, [&](void* op_out) {
            dispatch(c, [&](auto& im) {
                using T = std::remove_pointer_t<decltype(im.rhoR())>;
                const T* i = static_cast<const T*>(ip);
                T* o = static_cast<T*>(op_out);
                const size_t M = c->g.M;
                const V3<const T> i3 = cvec(vec(const_cast<T*>(i), M));
                const V3<T> o3 = vec(o, M);
                switch (op) {
                    case DR_OP_GRAD: im.grad(i, o3); break;
                    case DR_OP_DIV: im.div(i3, o); break;
                    case DR_OP_REG: im.reg_apply(i3, o3); break;
                    case DR_OP_PRECOND: im.precond(i3, o3); break;
                    case DR_OP_LERAY: im.leray(i3, o3); break;
                }
            });
        });
    });
}

dr_status dr_op_interp(dr_ctx* c, const void* f, int64_t npts, const void* s, void* out) {
    return run(c, [&] {
        if (npts < 0) fail(DR_ERR_ARG, "bad interp arguments");
        if (c->dist()) fail(DR_ERR_ARG, "dr_op_interp is a single-rank test hook");
        if (npts == 0) return;
        if (!f || !s || !out) fail(DR_ERR_ARG, "bad interp arguments");
        dispatch(c, [&](auto& im) {
            using T = std::remove_pointer_t<decltype(im.rhoR())>;
            im.PB("interp_points");
            k_interp_points<T><<<im.grid_1d(npts), 256, 0, c->stream>>>(c->g, static_cast<const T*>(f), npts,
                                                                          static_cast<const T*>(s), static_cast<T*>(out));
            im.PE("interp_points");
        });
    });
}

dr_status dr_get_departure(dr_ctx* c, int sigma, void* d_out) {
    return run(c, [&] {
        if (!d_out || (sigma != 1 && sigma != -1)) fail(DR_ERR_ARG, "bad departure arguments");
        if (!c->have_velocity) fail(DR_ERR_ORDER, "get_departure needs set_velocity");
        CK(cudaMemcpyAsync(d_out, c->ws + (sigma > 0 ? c->L.dp : c->L.dm), 3 * c->g.M * elem_size(c),
                           cudaMemcpyDeviceToDevice, c->stream));
    });
}

dr_status dr_get_field(dr_ctx* c, int which, int j, void* out) {
    return run(c, [&] {
        if (!out) fail(DR_ERR_ARG, "out must be non-NULL");
        const int nt = c->cfg.nt;
        auto need = [&](bool ok, const char* m) {
            if (!ok) fail(DR_ERR_ORDER, m);
        };
        auto jrange = [&]() {
            if (j < 0 || j > nt) fail(DR_ERR_ARG, "slice index out of range");
        };
        dispatch(c, [&](auto& im) {
            using T = std::remove_pointer_t<decltype(im.rhoR())>;
            const size_t F = c->g.M * sizeof(T);
            T* o = static_cast<T*>(out);
            auto copy = [&](const T* src, size_t bytes, T* dst) {
                CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
            };
            switch (which) {
                case DR_FIELD_STATE:
                    need(c->have_state, "needs forward_solve");
                    jrange();
                    copy(im.rho(j), F, o);
                    break;
                case DR_FIELD_STATE_GRAD:
                    need(c->have_state, "needs forward_solve");
                    jrange();
                    copy(im.G(j), 3 * F, o);
                    break;
                case DR_FIELD_ADJOINT:
                    need(c->have_adjoint, "needs adjoint_solve");
                    jrange();
                    copy(im.lam(j), F, o);
                    break;
                case DR_FIELD_INC_STATE:
                    need(c->have_matvec, "needs hessian_matvec");
                    copy(im.rt1(), F, o);
                    break;
                case DR_FIELD_INC_ADJOINT:
                    need(c->have_matvec, "needs hessian_matvec");
                    jrange();
                    if (j == nt) {  // lambda~(1) = -rho~(1) (Eq. 5d); materialise it
                        im.PB("scale");
                        k_scale<T><<<im.grid_1d(c->g.M), 256, 0, c->stream>>>(c->g.M, im.rt1(), o, T(-1));
                        im.PE("scale");
                    } else {
                        copy(im.lt(j), F, o);
                    }
                    break;
                case DR_FIELD_BTILDE:
                    need(c->have_matvec, "needs hessian_matvec");
                    copy(im.bt(), 3 * F, o);
                    break;
                case DR_FIELD_MULTIPLIER:
                    need(c->have_velocity, "needs set_velocity");
                    if (c->cfg.flags & DR_ISOCHORIC) fail(DR_ERR_ARG, "isochoric contexts have m == 1");
                    copy(im.mult(), F, o);
                    break;
                case DR_FIELD_VELOCITY:
                    need(c->have_velocity, "needs set_velocity");
                    for (int a = 0; a < 3; ++a) copy(im.vc(a), F, o + (size_t)a * c->g.M);
                    break;
                default:
                    fail(DR_ERR_ARG, "unknown field");
            }
        });
    });
}

}  // extern "C"
