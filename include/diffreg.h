/*
 * diffreg.h -- C ABI of the B200 Gauss-Newton Hessian-matvec library (paper_1608_03630_b200).
 *
 * The library implements the data-parallel hot path of the Gauss-Newton-Krylov diffeomorphic
 * registration solver of arXiv 1608.03630 ("the paper"; citations "P:Lnnn" are lines of
 * /root/reference/PAPER.md with the section / equation they fall in):
 *
 *   - RK2 semi-Lagrangian departure points along the characteristics of +v and -v
 *     (Eq. 6), computed once per velocity;
 *   - tricubic (cubic Lagrange, 4x4x4 stencil) interpolation at those points;
 *   - the state / adjoint / incremental-state / incremental-adjoint transport solves
 *     (Eq. 2b-c, Eq. 3, Eqs. 5a-5d; Eq. 7; Algorithm 2);
 *   - FFT spectral operators: gradient, divergence, regularisation beta*A with A = Laplacian^2
 *     (H2) or -Laplacian (H1), its inverse as preconditioner, and the Leray
 *     projection for the isochoric variant;
 *   - the Gauss-Newton Hessian matvec H(v) vt = beta A vt + P b~ (Eq. 5e).
 *
 * The exact discrete operator every call computes is SURVEY.md §8(c) D0-D14 (listed in DESIGN.md);
 * an fp64 CPU oracle under oracle/ computes the same quantities for the parity tests.
 *
 * DATA LAYOUT (all calls).  Grid n = (N1, N2, N3), periodic on [0, 2pi)^3, x_a = 2 pi i_a / N_a.
 *   scalar field : N3*N2*N1 values, index i1 + N1*(i2 + N2*i3)  (x1 fastest)
 *   vector field : 3 consecutive scalar fields (SoA): component a at offset a*N1*N2*N3
 *   value type   : float, or double when the context was created with DR_FP64.
 * GPU grid restriction (this build): every N_a is a power of two in [4, 1024] or, on one rank, N2 and
 * N3 any even extent in [6, 510] and N1 any multiple of 4 in [12, 1020] (the paper's 256 x 300 x 256
 * grid): those lines are transformed by Bluestein's chirp-z form through power-of-two FFTs
 * of length M >= 2 N - 1 (x1: of the half-length complex row; slower: two M-point FFTs per DFT).
 *
 * POINTERS.  Every field pointer of the main path (set_images, set_velocity, forward_solve,
 * adjoint_solve, hessian_matvec, precond_apply) may be a device pointer or a host pointer
 * (pinned or pageable); the library detects which with cudaPointerGetAttributes.  Host inputs
 * are copied into the workspace on the context stream; host outputs are copied back and the call
 * synchronises the stream before it returns.  Device-pointer calls are asynchronous w.r.t. the
 * host and ordered on the context stream (like cuBLAS).  Kernels read device fields with 16-byte
 * bulk copies and vector loads: a device pointer that is not 16-byte aligned (e.g. a tensor view at
 * an odd element offset) is staged through the workspace like a host pointer (one extra device copy)
 * by the main-path calls and dr_op_spectral.  The other dr_op_* / dr_get_* test hooks take 16-byte
 * aligned device pointers only.
 *
 * ENVIRONMENT (read by dr_create / dr_create_dist; A/B switches, defaults are the measured best):
 * DR_OVERLAP=1 transforms beta A vt on a second stream concurrently with the transport sweeps
 * (measured slower, off); DR_TMA_MIDDLE=0 replaces the tensor-map TMA fp32 x3 middle pass by the
 * one-tile-per-CTA pass; DR_PEER_GHOSTS=1 (slabs) fuses the ghost exchange into the producing gathers
 * (dr_peer_export); DR_GRAPHS=0 runs matvec / preconditioner calls eagerly instead of replaying the
 * context's captured CUDA graphs; DR_NCCL_GRAPHS=1 also captures NCCL contexts' calls (default eager);
 * DR_NCCL_LIB names the libnccl.so.2 to dlopen (the Python binding sets torch's bundled one).  Opt-in experiments (measured slower on one B200): DR_PAIRS=1
 * (shared-plane pair gathers), DR_WINDOW=1 (sliding-window gathers), DR_PLANE2D=1 (x1/x2 plane
 * transforms through cluster shared memory), DR_RING=P (plane chunks through an L2 scratch ring).
 * Results are bit-identical either way (DR_PLANE2D: within rounding).
 *
 * OWNERSHIP.  The caller owns every input, output and the workspace.  Inputs are only read;
 * images and the velocity are copied into the workspace (retained).  Outputs are fully
 * overwritten.  The library allocates no device memory after dr_create (and none at all when a
 * workspace is passed in).
 *
 * ERRORS.  Every call returns a dr_status; no exception crosses the ABI.  On error, outputs are
 * unspecified and dr_last_error(ctx) describes the failure.  Calls made out of order (e.g. a matvec
 * before dr_forward_solve) return DR_ERR_ORDER.  A context is bound to one device and one stream
 * and is not thread-safe.
 */
#ifndef DIFFREG_H
#define DIFFREG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dr_status {
    DR_OK = 0,
    DR_ERR_ARG = 1,        /* NULL / aliasing / bad enum argument                                */
    DR_ERR_GRID = 2,       /* N_a neither a power of two in [4, 1024] nor (one rank) N2 / N3 even */
                           /* in [6, 510], N1 % 4 == 0 in [12, 1020]; slabs: P | N2, P | N3       */
    DR_ERR_PARAM = 3,      /* beta <= 0, nt < 1 or nt > 64, reg not H1/H2                        */
    DR_ERR_ORDER = 4,      /* call sequence violated (see each function)                         */
    DR_ERR_CUDA = 5,       /* CUDA runtime error (message in dr_last_error)                      */
    DR_ERR_NCCL = 6,       /* multi-GPU communicator error (NCCL, or libnccl.so.2 not loadable)   */
    DR_ERR_OOM = 7,        /* workspace smaller than dr_workspace_bytes / cudaMalloc failed       */
    DR_ERR_NONFINITE = 8,  /* DR_CHECK_FINITE contexts: an input field holds NaN / Inf  */
    DR_ERR_PLAN = 9        /* multi-GPU: off-rank departure points exceed the scatter capacity    */
} dr_status;

enum { DR_REG_H1 = 1,      /* A = -Laplacian   (H1 seminorm, beta/2 |grad v|^2), a(k) = |k|^2   */
       DR_REG_H2 = 2 };    /* A = Laplacian^2  (H2 seminorm, beta/2 |Lap v|^2), |k|^4   */

enum { DR_ISOCHORIC = 1u,  /* incompressible variant: v Leray-projected, P = Leray  */
       DR_FP64 = 2u,       /* all fields are double instead of float                             */
       DR_FULL_NEWTON = 4u,  /* NEXT-3: dr_hessian_matvec keeps the two lambda terms of Eq. 5c /
                                  b~; default is Gauss-Newton          */
       DR_CHECK_FINITE = 8u };  /* dr_set_images, dr_set_velocity, dr_hessian_matvec and
                                  dr_precond_apply scan their inputs first and return
                                  DR_ERR_NONFINITE (on every rank) if any value is NaN or Inf; the
                                  scan synchronises the stream (one pass over the input), so these
                                  calls are no longer asynchronous and are not graph-replayed faster */

typedef struct dr_config {
    int32_t n[3];   /* N1 (x1, fastest), N2, N3                                                   */
    int32_t nt;     /* number of time steps n_t, dt = 1/n_t; 1 <= nt <= 64          */
    int32_t reg;    /* DR_REG_H1 or DR_REG_H2                                                     */
    uint32_t flags; /* DR_ISOCHORIC | DR_FP64 | DR_FULL_NEWTON | DR_CHECK_FINITE                  */
    double beta;    /* regularisation parameter beta > 0 (Eq. 2a)                      */
    int32_t ghost_lo, ghost_hi; /* slab ghost planes below / above (multi-GPU only; 0 -> 4 / 5).  A
                                   gather stencil spans floor(s3)-1 .. floor(s3)+2, so (g, g+1) planes
                                   cover x3 displacements |d3| <= g - 1 cells; 1 <= g <= N3/P.
                                   Set explicitly: ghost_lo >= 1 and ghost_hi >= 2, else DR_ERR_PARAM
                                   (an owner serving an off-rank point reads one plane below its
                                   slab and two above).                                               */
} dr_config;

typedef struct dr_ctx dr_ctx;

/* Bytes of device workspace a context for cfg needs (0 if cfg is invalid). */
size_t dr_workspace_bytes(const dr_config* cfg);

/* Create a context on the current CUDA device.  workspace: device buffer of >= dr_workspace_bytes
 * bytes, or NULL to let dr_create cudaMalloc it (freed by dr_destroy).  stream: a cudaStream_t
 * (NULL = legacy default stream).  Errors: DR_ERR_ARG, DR_ERR_GRID, DR_ERR_PARAM, DR_ERR_OOM. */
dr_status dr_create(const dr_config* cfg, void* workspace, size_t workspace_bytes, void* stream,
                    dr_ctx** out);
dr_status dr_destroy(dr_ctx* ctx);

/* ---------------------------------------------------------------------------------------------
 * Slab decomposition over P GPUs (the B200 replacement of the paper's pencil
 * decomposition, and of its ghost-layer interpolation, Algorithm 1).
 * Rank r owns the x3 planes [r N3/P, (r+1) N3/P) of every field; all field arguments of a
 * distributed context are that rank's slab: scalar [N3/P][N2][N1], vector [3][N3/P][N2][N1].
 * Requirements: P | N3, P | N2, P <= 32, N3/P >= ghost_hi.  Ghost planes (default (4, 5), widened
 * with dr_config.ghost_lo/hi) serve departure points up to ghost_lo - 1 cells away along x3; points
 * farther out (any distance, several slabs included) are served by the off-rank scatter of the
 * paper's Algorithm 1: their cells go to the owning rank once per velocity, and every
 * gather the owners interpolate and return the values.  dr_set_velocity returns DR_ERR_PLAN only if
 * a rank's remote points exceed the scatter capacity (M/8 per displacement field).  Exchanges:
 * ghost planes before every semi-Lagrangian gather and all-to-all transposes around the x3 FFT pass,
 * stream-ordered on the context stream.  Every rank must make the same sequence of calls (collective
 * semantics).
 *
 * Communicators (owned by the caller, must outlive the contexts that use them):
 *   NCCL     -- one process per GPU: rank 0 calls dr_nccl_get_unique_id, the id is broadcast by the
 *               caller (e.g. torch.distributed), every rank calls dr_comm_create_nccl.
 *   loopback -- P virtual ranks inside one process on one GPU (testing): dr_hub_create(P), then one
 *               dr_comm_create_loopback(hub, r) per rank; each rank's calls must run on its own host
 *               thread and its own stream (ranks rendezvous on host barriers inside every exchange).
 * Errors: DR_ERR_NCCL (NCCL failure, or libnccl.so.2 not loadable), DR_ERR_ARG (bad rank/size). */
typedef struct dr_comm dr_comm;
typedef struct dr_hub dr_hub;
dr_status dr_nccl_get_unique_id(uint8_t out[128]);
dr_status dr_comm_create_nccl(const uint8_t uid[128], int rank, int nranks, dr_comm** out);
dr_status dr_hub_create(int nranks, dr_hub** out);
dr_status dr_hub_destroy(dr_hub* hub);
dr_status dr_comm_create_loopback(dr_hub* hub, int rank, dr_comm** out);
dr_status dr_comm_destroy(dr_comm* comm);
/* Communicator self-test: an all-to-all of rank-stamped 1 KiB chunks (self included) through the same
 * grouped send/recv path the slab exchanges use, on `stream`; *ok = 1 when every chunk arrived intact.
 * Collective.  Allocates (and frees) 2 P KiB of device memory. */
dr_status dr_comm_selftest(dr_comm* comm, void* stream, int* ok);

/* Host-only partition query: the slab [z0, z0 + nz) of `rank` (no GPU needed). */
dr_status dr_slab(const dr_config* cfg, int nranks, int rank, int* z0, int* nz);

/* Workspace of one rank's context (0 if the configuration is invalid for nranks). */
size_t dr_workspace_bytes_dist(const dr_config* cfg, int nranks);

/* Create a rank's context; comm = NULL is exactly dr_create (one rank).  Same workspace / stream
 * rules as dr_create. */
dr_status dr_create_dist(const dr_config* cfg, dr_comm* comm, void* workspace, size_t workspace_bytes,
                         void* stream, dr_ctx** out);

/* Fused ghost exchange (SURVEY §8(e) "fuse the collectives"; the ghost layers of P:L314 / Alg. 1
 * P:L326-337).  With DR_PEER_GHOSTS=1 in the environment at dr_create_dist (P > 1), every
 * semi-Lagrangian gather whose output is the next gather's source (state, adjoint, incremental
 * state / adjoint, deformation steps) also stores the slab's boundary planes straight into the x3
 * neighbours' ghost planes of the same workspace slot -- the transfer rides in the gather's epilogue
 * instead of a send/recv before the next gather, which then only waits for its two neighbours (a
 * stream-ordered barrier; host events for loopback ranks, an epoch flag in peer memory for one
 * process per GPU).  Ghosts of fields produced by other kernels are still exchanged with send/recv.
 * The same switch fuses the all-to-all transposes of the spectral operators with one output
 * component: the forward x2 pass stores each rank's chunk straight into that rank's spectrum slot and
 * the x3 middle pass stores its planes straight into the owning ranks' receive buffer (P <= 64), each
 * between two all-rank stream barriers instead of a send/recv all-to-all.
 * Results are bit-identical to the send/recv path and to one rank.  Loopback communicators map the
 * other ranks' workspaces directly.  NCCL communicators need the neighbours' workspaces mapped:
 *   dr_peer_export  -- this context's CUDA IPC handle (64 bytes, of the allocation holding the
 *                      workspace) and the workspace's byte offset in that allocation;
 *   dr_peer_import  -- all ranks' handles [nranks][64] and offsets [nranks] (gathered by the caller,
 *                      e.g. torch.distributed.all_gather_object); opens every other rank's.
 * Collective (import).  Errors: DR_ERR_ARG (NULL, or not an NCCL context for import), DR_ERR_CUDA
 * (IPC failure: e.g. peers on different nodes or without peer access).  Until imported, an NCCL
 * context keeps the send/recv exchange. */
dr_status dr_peer_export(dr_ctx* ctx, uint8_t handle[64], uint64_t* offset);
dr_status dr_peer_import(dr_ctx* ctx, const uint8_t* handles, const uint64_t* offsets);


/* Template rho_T and reference rho_R images (scalar fields).  Copied.  Invalidates the
 * adjoint solve (and the forward solve, whose initial condition is rho_T). */
dr_status dr_set_images(dr_ctx* ctx, const void* rho_T, const void* rho_R);

/* Velocity v (vector field, stationary).  Copied.  Isochoric contexts replace v by L v
 * (P:L157).  Builds, once per velocity (the "interpolation planner"): the RK2
 * departure displacements for +v and -v (Eq. 6), their per-tile gather plans, and (non-isochoric)
 * div v and the adjoint multiplier m (Eq. 7 with f = nu div v).  Invalidates all solves. */
dr_status dr_set_velocity(dr_ctx* ctx, const void* v);

/* State solve (Eqs. 2b-2c): rho_0 = rho_T, rho_{j+1} = I[rho_j](X+), all n_t+1 slices
 * kept, plus the state gradients grad rho_j cached for the matvec.  rho1_out (nullable) receives
 * rho(1) = rho_{n_t}.  Requires dr_set_images and dr_set_velocity, else DR_ERR_ORDER. */
dr_status dr_forward_solve(dr_ctx* ctx, void* rho1_out);

/* Adjoint solve (Eq. 3): lambda(1) = rho_R - rho(1), transported backward with -v
 * (P:L275); lambda0_out (nullable) receives lambda(0).  Requires dr_forward_solve. */
dr_status dr_adjoint_solve(dr_ctx* ctx, void* lambda0_out);

/* Gauss-Newton Hessian matvec Hvt = H(v) vt (Eqs. 5a-5e with the lambda terms
 * dropped): incremental state forward (Algorithm 2), incremental adjoint backward,
 * b~ = int lambda~ grad rho dt (trapezoid), Hvt = beta A vt + P b~.  With DR_FULL_NEWTON the two
 * lambda terms are kept (NEXT-3; runs dr_adjoint_solve first if needed).  vt, Hvt: vector fields,
 * must not alias.  Requires dr_forward_solve. */
dr_status dr_hessian_matvec(dr_ctx* ctx, const void* vt, void* Hvt);

/* Spectral preconditioner z = (beta A)^{-1} r with a_hat(0) = 1, followed by the Leray
 * projection in isochoric contexts.  r, z: vector fields, may alias.  Requires only the context. */
dr_status dr_precond_apply(dr_ctx* ctx, const void* r, void* z);

/* NEXT-1: reduced gradient g = beta A v + P b, b = int_0^1 lambda grad rho dt
 * (Eq. 4; trapezoid in time, reading A12; P = Leray when isochoric).  Requires
 * dr_forward_solve; runs dr_adjoint_solve first if it has not run since.  g: vector field, device or
 * host pointer (host: the call synchronises). */
dr_status dr_gradient(dr_ctx* ctx, void* g);

/* Objective J = 1/2 <rho(1) - rho_R, rho(1) - rho_R> + beta/2 <v, A v> (Eq. 2a) with the
 * inner product h1 h2 h3 sum, accumulated in fp64 deterministically; with slabs the sum runs
 * over all ranks (collective) and every rank gets the same value.  Requires dr_forward_solve.  J and
 * misfit (the first term) are host pointers, either may be NULL.  Synchronises the stream. */
dr_status dr_objective(dr_ctx* ctx, double* J, double* misfit);

/* NEXT-2: inexact preconditioned CG for the Newton step H dv = -g (PCG with
 * the inverse-regulariser preconditioner, Leray-projected when isochoric; relative tolerance from the
 * gradient norm, e.g. the quadratic forcing eta = min(0.5, |g| / |g_0|) of P:L433).  Starts from
 * dv = 0; stops when |r| <= eta |g| (discrete L2 norms, fp64 accumulation, summed over all ranks) or
 * after maxit Hessian matvecs.  g, dv: vector fields (device or host), must not alias.  iters /
 * relres (nullable, host): matvecs used and |r| / |g|.  Requires dr_forward_solve.  One rank: each
 * iteration is a CUDA graph (captured once per context; DR_GRAPHS=0 in the environment at dr_create
 * disables it) with one 8-byte read-back; slabs: one synchronisation per inner product. */
dr_status dr_pcg(dr_ctx* ctx, const void* g, void* dv, double eta, int maxit, int* iters, double* relres);

/* NEXT-4: deformation map and its Jacobian determinant.  u = y_1 - x where
 * d_t y + v.grad y = 0, y(0) = x (Eq. 1; transported like the state, Eq. 7 with the
 * stationary source -v) and det = det(grad y_1) = det(I + grad u) (Fig. 7 caption, P:L537;
 * det > 0 everywhere <=> diffeomorphism).  u (vector), det (scalar): nullable, device or host;
 * det_min / det_max (host, nullable): extrema over all ranks.  Requires dr_set_velocity; clobbers
 * the incremental fields of the last matvec (dr_get_field INC_* / BTILDE need a new matvec).
 * Synchronises. */
dr_status dr_deformation(dr_ctx* ctx, void* u, void* det, double* det_min, double* det_max);

/* NEXT-4: Armijo-globalised inexact (Gauss-)Newton-Krylov registration.
 * Iterates g_k = g(v_k) (dr_gradient); stops when |g_k| <= gtol |g_0|; Newton step by dr_pcg with the
 * quadratic forcing eta = min(0.5, |g_k| / |g_0|) (reading A22) and at most max_krylov matvecs;
 * backtracking alpha = 1, alpha *= shrink until J(v + alpha dv) <= J(v) + c1 alpha <g, dv>.  Uses
 * the full-Newton matvec when the context has DR_FULL_NEWTON, else Gauss-Newton.
 * v: DEVICE vector field, in: initial velocity, out: the last accepted iterate (with its state
 * solved: dr_get_field / dr_deformation apply to it).  opts NULL: {1e-2, 50, 100, 1e-4, 0.5, 20}.
 * rep (nullable): summary and, if history != NULL, history_len rows of (J, |g|/|g0|, PCG matvecs,
 * alpha, cumulative matvecs) per Newton iteration.  Requires dr_set_images.  Collective. */
typedef struct dr_solve_opts {
    double gtol;         /* relative gradient tolerance g_tol (1e-2)   */
    int32_t max_newton;  /* Newton iterations                                   */
    int32_t max_krylov;  /* PCG matvecs per Newton step                         */
    double c1;           /* Armijo sufficient-decrease constant                 */
    double shrink;       /* backtracking factor                                 */
    int32_t max_backtracks;
} dr_solve_opts;
enum { DR_SOLVE_CONVERGED = 0, DR_SOLVE_MAX_NEWTON = 1, DR_SOLVE_LINESEARCH_FAILED = 2 };
typedef struct dr_solve_report {
    int32_t iterations, matvecs, reason;
    double J0, J, g0, g;  /* objective and |g| (discrete L2) at the start / end */
    double* history;      /* caller-owned, 5 * history_len doubles, nullable */
    int32_t history_len;
} dr_solve_report;
dr_status dr_solve(dr_ctx* ctx, void* v, const dr_solve_opts* opts, dr_solve_report* rep);

/* Wait for all work of the context; surfaces asynchronous CUDA errors. */
dr_status dr_sync(dr_ctx* ctx);

/* Human-readable description of the last error of ctx (owned by ctx, valid until the next call). */
const char* dr_last_error(const dr_ctx* ctx);
const char* dr_status_string(dr_status s);

/* ---------------------------------------------------------------- tracing
 * Launch accounting is always on: every kernel launch of the context is counted.  With profiling
 * enabled, each launch is additionally bracketed by two CUDA events on the context stream and the
 * elapsed GPU time is accumulated per kernel tag (e.g. "sl_inc_state", "col_middle").  Reading the
 * profile synchronises the stream.  dr_profile_reset clears the tags and the launch counter. */
dr_status dr_profile_enable(dr_ctx* ctx, int enable);
dr_status dr_profile_reset(dr_ctx* ctx);
/* Restrict the event timing to the launches whose tag equals `tag` (NULL or "": all launches).  Each
 * timed launch is bracketed by two events on its stream, which costs ~2 us of GPU idle per launch
 * (6 % of the 256^3 bench step when every launch is timed); bench.py times one tag in its timed
 * region and takes the full table from an untimed pass. */
dr_status dr_profile_only(dr_ctx* ctx, const char* tag);
/* number of distinct tags so far, and the total number of kernel launches since the last reset */
dr_status dr_profile_count(dr_ctx* ctx, int* n_entries, int64_t* launches);
/* entry i: tag (copied into name[name_len], NUL-terminated), launches and summed GPU milliseconds */
dr_status dr_profile_entry(dr_ctx* ctx, int i, char* name, int name_len, int64_t* launches, double* total_ms);

/* ---------------------------------------------------------------- per-operator test hooks
 * Device pointers only.  They run the same kernels as the main path. */
enum { DR_OP_GRAD = 0,    /* in: scalar   out: vector   grad f  (i k' per axis)       */
       DR_OP_DIV = 1,     /* in: vector   out: scalar   div u                                  */
       DR_OP_REG = 2,     /* in: vector   out: vector   beta A u                               */
       DR_OP_PRECOND = 3, /* in: vector   out: vector   same as dr_precond_apply               */
       DR_OP_LERAY = 4 }; /* in: vector   out: vector   L u = u - grad Lap^{-1} div u          */
dr_status dr_op_spectral(dr_ctx* ctx, int op, const void* in, void* out);

/* out[p] = I[f](s_p): tricubic interpolation of the scalar field f at npts points given
 * in CELL coordinates s (x = h*s), laid out as s[0..npts) = s1, s[npts..2npts) = s2, then s3. */
dr_status dr_op_interp(dr_ctx* ctx, const void* f, int64_t npts, const void* s, void* out);

/* Copy of the departure displacement field d^sigma (sigma = +1 or -1), cell units: the departure
 * point of node i is s_i = i - d_i.  Requires dr_set_velocity. */
dr_status dr_get_departure(dr_ctx* ctx, int sigma, void* d_out);

enum { DR_FIELD_STATE = 0,       /* scalar rho_j, j = 0..nt           (after forward_solve)    */
       DR_FIELD_STATE_GRAD = 1,  /* vector grad rho_j, j = 0..nt      (after forward_solve)    */
       DR_FIELD_ADJOINT = 2,     /* scalar lambda_j, j = 0..nt        (after adjoint_solve)    */
       DR_FIELD_INC_STATE = 3,   /* scalar rho~(1), j ignored         (after hessian_matvec)   */
       DR_FIELD_INC_ADJOINT = 4, /* scalar lambda~_j, j = 0..nt       (after hessian_matvec)   */
       DR_FIELD_BTILDE = 5,      /* vector b~, j ignored              (after hessian_matvec)   */
       DR_FIELD_MULTIPLIER = 6,  /* scalar m (1 when isochoric)       (after set_velocity)     */
       DR_FIELD_VELOCITY = 7 };  /* vector v as used (projected if isochoric)                   */
dr_status dr_get_field(dr_ctx* ctx, int which, int j, void* out);

#ifdef __cplusplus
}
#endif
#endif /* DIFFREG_H */
