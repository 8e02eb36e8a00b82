/*
 * cem.h -- C ABI of libcem.so, the B200 (sm_100a) explicit step of the 3D Crack Element
 * Method (arXiv 2508.04076, "A GPU-Accelerated Three-Dimensional Crack Element Method
 * for Transient Dynamic Fracture Simulation").
 *
 * One explicit step n -> n+1 (§2.2-§3):
 *   u_{n+1} = u_n + dt v_n + dt^2/2 a_n
 *   eps~_s  = sum_{j in inc(s)} w_j B_j u,  w_j = V_j / sum V           (L268-L281, eq:strain_discretization)
 *   sigma_s = D eps~_s                                                  (L197-L202)
 *   f_int   = A_j(A_k B_k^T w_j sigma) (1/6) sum_j V_j                  (L340-L367, eq:fint_discretization)
 *   a_{n+1} = M^-1 (f_ext - f_int(u_{n+1})),  M lumped                   (L392-L416)
 *   v_{n+1} = v_n + dt [(1-gamma) a_n + gamma a_{n+1}]                  (L417)
 *   crack criterion G = max(G_I, G_II) > Gc on every active tet          (L426-L476, eq:G-I, eq:G-II)
 *   split pass: the element is deactivated and excluded from subsequent computations (L151)
 *
 * Conventions
 *  - All floating point is IEEE fp64; indices int32 (meshes up to 2^31-1 entities); one context
 *    holds at most 357M tets (32-bit device offsets; about 520 B of device memory per tet) --
 *    larger meshes are partitioned over ranks (nranks > 1).
 *  - Host pointers passed to cem_init_mesh are read during the call only (copied);
 *    the caller keeps ownership and may free them afterwards.
 *  - Device memory: either the caller hands a device workspace (opts.workspace, at least
 *    cem_workspace_size bytes), or an allocation callback (opts.dev_alloc, e.g. a torch
 *    allocator), or neither, in which case the library uses cudaMalloc and frees on
 *    cem_destroy.
 *  - Asynchrony: the library runs its work on a private non-blocking stream of its own (CUDA
 *    graphs and the L2 access-policy window live there).  Every call that enqueues work first
 *    makes that stream wait for opts.stream (NULL = the legacy default stream) and, on return,
 *    makes opts.stream wait for the library's work, so work on opts.stream is ordered with the
 *    library's in both directions.  cem_step returns without waiting; cem_get_state,
 *    cem_crack_update and cem_energy synchronise.
 *  - Errors: every call returns a cem_status; cem_last_error(ctx) gives a message (also for
 *    a NULL ctx: the last error of cem_init_mesh in this thread).  No exception crosses the
 *    ABI.  A ctx is not thread-safe.
 *  - Determinism: results are bitwise reproducible run to run (fixed association order,
 *    no floating-point atomics) and equal to the CPU oracle's (tests/test_gpu_parity.py).
 */
#ifndef CEM_H
#define CEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CEM_ABI_VERSION 2

#if defined(__GNUC__)
#define CEM_API __attribute__((visibility("default")))
#else
#define CEM_API
#endif

typedef struct cem_ctx cem_ctx; /* opaque; one per rank / GPU */

typedef enum {
    CEM_OK = 0,
    CEM_EINVAL = 1,      /* bad argument: nu >= 0.5, E <= 0, rho <= 0, dt/cfl/gamma out of range, NULL array */
    CEM_EDEGENERATE = 2, /* |V_e| < 1e-14 * bbox^3 */
    CEM_ENEGVOL = 3,     /* a tet with negative orientation (det[X1-X0, X2-X0, X3-X0] < 0) */
    CEM_ETOPOLOGY = 4,   /* node index out of range, repeated node in a tet, duplicate tets */
    CEM_ENONFINITE = 5,  /* a non-finite u, v or a appeared (see cem_state_out.nonfinite_node) */
    CEM_ECUDA = 6,       /* a CUDA runtime error (message in cem_last_error) */
    CEM_ENCCL = 7,       /* multi-GPU communication error */
    CEM_ESTATE = 8,      /* call not valid in the current state */
    CEM_ENOMEM = 9       /* workspace too small / allocation failed */
} cem_status;

/* Isotropic linear elastic material with a Griffith threshold. */
typedef struct {
    double E;   /* Young's modulus (Pa), > 0 */
    double nu;  /* Poisson ratio, -1 < nu < 0.5 */
    double rho; /* density (kg/m^3), > 0 */
    double Gc;  /* default critical energy release rate (J/m^2) for tets without tet_gc */
} cem_material;

/* Tetrahedral mesh (PAPER.md:L264 notation). */
typedef struct {
    int64_t n_nodes;
    const double *X;          /* [n_nodes][3] reference coordinates (m), row-major */
    int64_t n_tets;
    const int32_t *tets;      /* [n_tets][4] node ids, positive orientation required */
    const uint8_t *tet_state; /* NULL | [n_tets]: 0 inactive from the start (notch), 1 active */
    const double *tet_gc;     /* NULL | [n_tets] per-element Gc (J/m^2); 0 = pre-damaged */
    int32_t nodes_per_elem;   /* (ABI >= 2) 0 or 4: linear tets (ES-T-FEM, the default); 8: trilinear
                                 hexahedra (ES-H-FEM; `tets` then holds [n][8]
                                 node ids, nodes 0-3 one face counter-clockwise seen from outside...
                                 i.e. a right-handed (xi, eta) order, 4-7 the opposite face in the same
                                 order; element strain = the volume-averaged strain, R23-R26).
                                 Hexahedral contexts crack by patterns III-VI (PAPER.md:L478-L540,
                                 DESIGN.md R28-R29): cem_step with crack_every > 0 evaluates 84
                                 candidates per active hex (record cand k: III 2f+j, IV 12+4f+2j+t,
                                 V 36+4f+i, VI 60+4f+i); IV-VI leave a half-hex prism of three tets
                                 recorded as elements n_tets + 3e + i when they split (tet criterion,
                                 cand 0..23), so the record arrays need up to 4 n_tets entries and
                                 tet_state reports the hexes only.  cem_crack_update returns
                                 CEM_ESTATE; cem_energy uses the smoothing-domain volume sum V/12
                                 (hex) + V/6 (tet); one GPU (nranks = 1). */
} cem_mesh_in;

/* Loads (PAPER.md:L191 Dirichlet/Neumann boundaries; L408-L412 external force;
 * L572-L579 velocity ramp; L1119 constant traction).  The external force is assembled once at
 * init and is constant from t = 0 (R4, R4b), in this order per node and component:
 * body force b (V_e/4) over the active incident tets (ascending tet id; PAPER.md:L410
 * "A_e [N^e] b A_e"), then the traction triangles in the given order (t A/3 per node), then
 * f_nodal. */
typedef struct {
    int64_t n_tfaces;
    const int32_t *tface;     /* [n_tfaces][3] boundary triangles carrying a traction */
    const double *tface_t;    /* [n_tfaces][3] traction vector (Pa), constant from t = 0 */
    int64_t n_vbc;
    const int32_t *vbc_node;  /* [n_vbc] prescribed-velocity nodes */
    const uint8_t *vbc_mask;  /* [n_vbc] bit0 = x, bit1 = y, bit2 = z */
    const double *vbc_v0;     /* [n_vbc][3] target velocity (m/s) */
    double vbc_t0;            /* ramp time (s): v = (t/t0) v0 for t <= t0, else v0; 0 = step */
    const double *f_nodal;    /* NULL | [n_nodes][3] constant nodal point forces (N) (ABI >= 2) */
    double body[3];           /* uniform body force density b (N/m^3), e.g. rho g; 0 = none (ABI >= 2) */
} cem_load_in;

/* flags */
#define CEM_F_NO_EARLY_OUT 0x1u /* evaluate all 24 crack candidates on every active tet (all 84 on every
                                 * active hexahedron) instead of skipping the elements whose conservative
                                 * bound max g * max |du| (1 + 1e-6) <= Gc_e rules a split out; same results */
#define CEM_F_STAGED 0x2u       /* one kernel per stage (the default; kept for explicitness) */
#define CEM_F_NO_DISCARD 0x4u   /* persistent kernel: keep consumed intermediates in L2 (no discard) */
#define CEM_F_PERSISTENT 0x8u   /* one persistent wavefront kernel per cem_step call */
#define CEM_F_LOOPBACK 0x10u    /* nranks > 1 emulated in one process (cem_step_group, device copies) */
#define CEM_F_P2P 0x20u         /* loopback: the P2P halo path (stage D stores into the peers' buffers).
                                 * Multi-GPU (NCCL) contexts use the P2P halo whenever every rank can
                                 * map its peers' buffers (CUDA IPC over NVLink) and a self-check at
                                 * init passes; CEM_NO_P2P=1 in the environment keeps NCCL send/recv. */
#define CEM_F_FRONT_BOTH_STRETCHED 0x40u /* criterion variant (R11, "whose
                                 * tensile stretches at two edges"): a candidate whose front edges c-p,
                                 * c-q are not both stretched has G = 0 (default: no such condition) */

typedef int (*cem_alloc_fn)(size_t bytes, void *user, void **dev_ptr); /* returns 0 on success */
/* Host all-gather over the ranks (blocking; rank-ordered concatenation of `bytes` from every
 * rank into recv, which holds nranks * bytes); returns 0 on success.  Also used as a barrier. */
typedef int (*cem_allgather_fn)(const void *send, void *recv, size_t bytes, void *user);

typedef struct {
    double dt;           /* time step (s); <= 0 -> cfl * min_e altitude_e / c_d (R12) */
    double cfl;          /* default 0.5 */
    double gamma;        /* Newmark gamma, default 0.5 (central difference) */
    uint32_t flags;      /* CEM_F_* */
    int device;          /* CUDA device ordinal */
    void *stream;        /* cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL = default */
    void *workspace;     /* optional caller-owned device buffer (>= cem_workspace_size bytes) */
    size_t workspace_bytes;
    cem_alloc_fn dev_alloc; /* optional device allocator used when workspace == NULL */
    void *alloc_user;
    int rank, nranks;    /* multi-GPU: rank in [0, nranks); nranks <= 1 -> single GPU */
    const void *nccl_id; /* nranks > 1 without CEM_F_LOOPBACK: the 128-byte ncclUniqueId that rank 0
                            obtained from cem_nccl_unique_id and broadcast to all ranks */
    cem_allgather_fn host_allgather; /* (ABI >= 2) nranks > 1, nccl_id NULL: host-ordered CUDA-IPC halo --
                            the receive buffers are mapped over CUDA IPC (handles exchanged with this
                            callback), stage D and the split pass store into the peers' buffers as in
                            the NVLink P2P halo, and every step the ranks meet in this callback
                            (after their stores completed) before the flag wait and the unpack, so no
                            kernel ever waits for another process's kernel.  For ranks sharing one GPU
                            (tests) or hosts without NCCL; one host round trip per step. */
    void *host_user;     /* passed to host_allgather */
} cem_opts;

/* Domain decomposition of a rank; library-owned arrays,
 * released by cem_partition_free.  Local tets/nodes are in ascending global id. */
typedef struct {
    int64_t n_tets, n_nodes;
    int32_t *tet_global;      /* [n_tets] global tet id of each local tet */
    uint8_t *tet_flag;        /* [n_tets] bit0: layer 1 (criterion evaluated here), bit1: owned (recorded here) */
    int32_t *node_global;     /* [n_nodes] */
    uint8_t *node_owned;      /* [n_nodes] 1 if this rank updates the node */
    int32_t n_peers;
    int32_t *peers;           /* [n_peers] */
    int64_t *send_node_off, *recv_node_off, *send_tet_off, *recv_tet_off; /* [n_peers + 1] CSR */
    int32_t *send_nodes, *recv_nodes, *send_tets, *recv_tets;             /* local ids */
    int32_t *tet_owner;       /* [global n_tets] owning rank of every tet */
    int32_t *node_owner;      /* [global n_nodes] */
} cem_part_out;

/* State snapshot, always in the caller's numbering (node / tet ids of cem_init_mesh) and the
 * layouts below.  where = CEM_HOST: every non-NULL array pointer is caller-owned HOST memory of
 * the stated size and is filled.  where = CEM_DEVICE: every non-NULL array pointer is caller-owned
 * DEVICE memory (same sizes and layouts, e.g. torch tensors on the ctx device) and is filled by
 * kernels / copies on the ctx stream; the call returns after that stream has synchronised.  In
 * both cases records come sorted by (step, element). */
#define CEM_HOST 0
#define CEM_DEVICE 1
typedef struct {
    double *u, *v, *a;        /* [n_nodes][3] at t_n (u_n, v_n, a_n) */
    uint8_t *tet_state;       /* [n_tets] 1 active, 0 inactive */
    double *mass;             /* [n_nodes] lumped mass (0 = frozen node) */
    int64_t *rec_step;        /* [rec_capacity] records of split tets, in split order */
    int32_t *rec_elem;        /*   (step ascending, element id ascending within a step) */
    int32_t *rec_cand;        /*   candidate k = 6c + 2f + t (R7) */
    double *rec_G;            /*   energy release rate at the split (J/m^2) */
    double *rec_area;         /*   crack-surface area (m^2) */
    int64_t rec_capacity;     /* in: size of the record arrays (n_tets; 4 n_tets for hexahedra) */
    /* scalars (always filled) */
    int64_t step;             /* n */
    double time;              /* n dt */
    double dt;
    int64_t n_active;         /* active tets */
    int64_t n_records;        /* total split tets so far */
    double dissipated;        /* U_d = sum Gc_e * area_e over split tets */
    int32_t nonfinite;        /* 1 if a non-finite value was produced */
    int32_t nonfinite_node;   /* lowest offending node id, -1 if none */
} cem_state_out;

/* Device bytes cem_init_mesh will need for this mesh (builds the edge set to count it). */
CEM_API cem_status cem_workspace_size(const cem_mesh_in *mesh, const cem_opts *opts, size_t *bytes);

/* Validate the mesh, build the topology (unique edges, edge->tet and node->tet CSR in
 * ascending tet id), geometry, lumped mass (row sum rho V/4),
 * nodal traction force (t A/3 per triangle node), the time step, upload to the device
 * and set u_0 = v_0 = 0, a_0 = M^-1 f_ext (prescribed dofs: v(0), v'(0)).
 * On failure *ctx is NULL and cem_last_error(NULL) explains. */
CEM_API cem_status cem_init_mesh(const cem_mesh_in *mesh, const cem_material *mat, const cem_load_in *load,
                         const cem_opts *opts, cem_ctx **ctx);

/* Enqueue nsteps explicit steps.  crack_every > 0: evaluate the crack criterion and run
 * the split pass after every crack_every-th step (criterion on u_{n+1} and the same
 * sigma(u_{n+1}) used for f_int, R16); 0 = pure elastodynamics.
 * Asynchronous on the context's stream.  The criterion kernels are chosen per step from the
 * list length of a recent step (long lists, >= 1024 tets or env CEM_CRITB_MIN at init, use the
 * filtered, batched kernels); the choice never changes results.  Multi-GPU contexts: a halo
 * wait that exceeds 60 s (a dead peer) is reported by the next cem_get_state (CEM_ENCCL). */
CEM_API cem_status cem_step(cem_ctx *ctx, int64_t nsteps, int32_t crack_every);

/* Criterion + split pass on the current state (u_n, sigma(u_n)) without advancing time;
 * synchronises; *n_split_out = number of tets split by this call. */
CEM_API cem_status cem_crack_update(cem_ctx *ctx, int64_t *n_split_out);

/* Synchronise and fill *out (see cem_state_out). Returns CEM_ENONFINITE if flagged. */
CEM_API cem_status cem_get_state(cem_ctx *ctx, cem_state_out *out, int where);

/* Checkpoint / resume (SURVEY.md §5 "Checkpoint / resume"): overwrite the state of a
 * single-GPU tetrahedral context with a snapshot taken by cem_get_state(CEM_HOST) -- possibly
 * of another context built from the same mesh, material and loads.  `in` uses cem_state_out's
 * layouts in the caller's numbering, HOST memory, all read-only:
 *   u, v, a [n_nodes][3], tet_state [n_tets], mass [n_nodes]   required (non-NULL)
 *   rec_step/rec_elem/rec_cand/rec_G/rec_area [n_records]       required when n_records > 0
 *   step                                                        the step index n of the snapshot
 * Everything the next step reads is rebuilt from these: the predictor u_{n+1} = (u_n + dt v_n)
 * + (dt^2/2) a_n (the stage kernels' expression), the smoothing-domain volumes
 * Vhat_s from the active flags (ascending original tet id), the split records (U_d follows from
 * them).  Continuing from the snapshot is then bitwise identical to never having stopped.
 * Not part of the checkpoint: the energy ledger's reaction work of prescribed dofs, which reads
 * NaN after this call.  Synchronises.  CEM_ESTATE for multi-rank and hexahedral contexts,
 * CEM_EINVAL for a NULL required array or n_records < 0 / > n_tets. */
CEM_API cem_status cem_set_state(cem_ctx *ctx, const cem_state_out *in);

/* Energy ledger at the current step n (SPEC.md update_energy_ledger;
 * oracle/cem_oracle.c orc_energy defines each quantity and its association order):
 *   kinetic        T   = 1/2 sum_k m_k |v_k|^2
 *   strain         U   = sum_s psi(eps~_s) Vhat_s / 6, psi = 1/2 lam tr(eps~)^2 + mu eps~:eps~
 *                        (L197-L202; Vhat_s / 6 = the smoothing-domain volume)
 *   external_work  W   = sum_k f_ext,k . u_k  (tractions constant from t = 0 and u_0 = 0: the
 *                        f_ext . du sum telescoped, R22)
 *   reaction_work  W_R = sum over steps of 1/2 (R_n + R_{n+1}) (u_{n+1} - u_n) on prescribed
 *                        dofs, R = m a - (f_ext - f_int) the support force (R22)
 *   dissipated     U_d = sum Gc_e A_e over the split records                 (L206)
 * Per-element terms are the oracle's bit for bit; the sums run over per-block partials in a
 * fixed order (run-to-run deterministic, equal to the oracle's sequential sums to rounding).
 * Synchronises the ctx stream; launches two kernels.  Multi-rank: the rank's share (its owned
 * nodes, the edges whose lowest-id incident tet it owns, its records); the sum over ranks is
 * the ledger of the whole mesh. */
typedef struct {
    int64_t step;
    double time;
    double kinetic, strain, external_work, reaction_work, dissipated;
} cem_energy_out;
CEM_API cem_status cem_energy(cem_ctx *ctx, cem_energy_out *out);

/* Host-only: the partition plan rank `rank` of `nranks` uses (no device work). */
CEM_API cem_status cem_partition(const cem_mesh_in *mesh, int nranks, int rank, cem_part_out *out);
CEM_API void cem_partition_free(cem_part_out *out);

/* Multi-GPU: 128-byte NCCL unique id for rank 0 to broadcast (opts.nccl_id).  NCCL is loaded at
 * run time (libnccl.so.2, the one torch uses); CEM_ENCCL if unavailable. */
CEM_API cem_status cem_nccl_unique_id(void *id128);

/* Loopback multi-rank emulation on one device: step n contexts created with nranks = n,
 * rank = i and CEM_F_LOOPBACK; the halo exchange runs as device copies in rank order. */
CEM_API cem_status cem_step_group(cem_ctx **ctxs, int32_t n, int64_t nsteps, int32_t crack_every);

/* Order records by (step, element) and sum U_d = sum Gc_e * area_e in that order (merging
 * the records of several ranks).  gc is indexed by element id; outputs the permutation. */
CEM_API cem_status cem_merge_records(int64_t n, const int64_t *step, const int32_t *elem, const double *area,
                                     const double *gc, int64_t *order_out, double *dissipated_out);

/* Mesh sizes after init. */
CEM_API cem_status cem_sizes(const cem_ctx *ctx, int64_t *n_nodes, int64_t *n_tets, int64_t *n_edges);

/* Total number of kernels this context has launched so far (launch accounting). */
CEM_API int64_t cem_launch_count(const cem_ctx *ctx);

/* Profiling: with cem_set_profiling(ctx, 1) cem_step runs one kernel per stage and brackets
 * each with CUDA events on the ctx stream; cem_kernel_times returns the accumulated ms per
 * stage since profiling was switched on (names[i] are static strings). */
CEM_API cem_status cem_set_profiling(cem_ctx *ctx, int on);
CEM_API cem_status cem_kernel_times(const cem_ctx *ctx, int32_t *n, const char **names, double *ms, int32_t cap);

CEM_API const char *cem_last_error(const cem_ctx *ctx);
CEM_API void cem_destroy(cem_ctx *ctx);
CEM_API int32_t cem_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CEM_H */
