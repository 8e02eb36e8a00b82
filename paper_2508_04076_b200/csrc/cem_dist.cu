// cem_dist.cu -- halo exchange of the multi-GPU step.
//
// After stage D of every step, each rank sends the predicted displacement u_{s+2} of the
// nodes it owns to the ranks that hold them, and the state byte of the tets it owns to the
// ranks that hold them as ghosts.  Pack/unpack are device kernels; transport is NCCL
// point-to-point (grouped send/recv on the step stream, loaded at run time) or, for the
// one-device loopback emulation, device-to-device copies issued in rank order.
#include <dlfcn.h>

#include <cstring>
#include <string>

#include "cem_dist.h"

namespace cem {

namespace {

__global__ void k_pack(const double4 *__restrict__ u, const uint8_t *__restrict__ state, const int32_t *__restrict__ nidx,
                       int64_t nn, const int64_t *__restrict__ ndst, const int32_t *__restrict__ tidx, int64_t nt,
                       const int64_t *__restrict__ tdst, uint8_t *__restrict__ buf) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nn) {
        const double4 w = u[nidx[i]];
        double *o = reinterpret_cast<double *>(buf + ndst[i]);
        o[0] = w.x;
        o[1] = w.y;
        o[2] = w.z;
    } else if (i < nn + nt) {
        buf[tdst[i - nn]] = state[tidx[i - nn]];
    }
}

__global__ void k_unpack(double4 *__restrict__ u, uint8_t *__restrict__ state, const int32_t *__restrict__ nidx,
                         int64_t nn, const int64_t *__restrict__ nsrc, const int32_t *__restrict__ tidx, int64_t nt,
                         const int64_t *__restrict__ tsrc, const uint8_t *__restrict__ buf,
                         const int32_t *__restrict__ eedge, int64_t E, uint8_t *__restrict__ edge_dirty) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nn) {
        const double *o = reinterpret_cast<const double *>(buf + nsrc[i]);
        u[nidx[i]] = make_double4(o[0], o[1], o[2], 0.0);
    } else if (i < nn + nt) {
        // states only go 1 -> 0 (splits are irreversible): apply the transition, never revert
        // (the P2P buffers carry a state byte only in the step it changes)
        const int32_t e = tidx[i - nn];
        if (state[e] && !buf[tsrc[i - nn]]) {  // a ghost tet split on its owner: its edges' Vhat change
            for (int l = 0; l < 6; ++l) edge_dirty[eedge[(int64_t)l * E + e]] = 1;
            state[e] = 0;
        }
    }
}

__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
    asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// one warp: lane j signals peer j (after a system fence: the stage kernels' remote stores,
// complete by stream order, are ordered before the flag), then waits for peer j's flag
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// (watchdog: a peer that stops signalling -- a dead rank -- ends the wait after 60 s with the
// timeout word set, which cem_get_state reports, instead of hanging the GPU)
__global__ void k_p2p_sync(int64_t *flags, int64_t *const *peer_flag, const int32_t *peer_rank, int np, int64_t target,
                           int wait, int64_t *timeout) {
    __threadfence_system();
    for (int j = threadIdx.x; j < np; j += blockDim.x) st_release_sys(peer_flag[j], target);
    if (wait) {
        const uint64_t t0 = globaltimer_ns();
        for (int j = threadIdx.x; j < np; j += blockDim.x)
            while (ld_acquire_sys(flags + peer_rank[j]) < target) {
                __nanosleep(100);
                if (globaltimer_ns() - t0 > 60000000000ull) {
                    atomicExch(reinterpret_cast<unsigned long long *>(timeout), 1ull);
                    break;
                }
            }
    }
    __syncwarp();
    __threadfence_system();
}

__global__ void k_p2p_push(const double4 *__restrict__ u, int64_t N, const int32_t *__restrict__ off,
                           const int32_t *__restrict__ peer, const int32_t *__restrict__ byte, uint8_t *const *recv, int np,
                           int par) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N) return;
    for (int32_t i = off[k]; i < off[k + 1]; ++i) {
        const double4 w = u[k];
        double *o = reinterpret_cast<double *>(recv[par * np + peer[i]] + byte[i]);
        o[0] = w.x;
        o[1] = w.y;
        o[2] = w.z;
    }
}

__global__ void k_mismatch(const uint8_t *a, const uint8_t *b, const int64_t *pos, int64_t n, int64_t width, int64_t *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int64_t j = 0; j < width; ++j)
        if (a[pos[i] + j] != b[pos[i] + j]) {
            atomicAdd(reinterpret_cast<unsigned long long *>(out), 1ull);
            return;
        }
}

// ---------------------------------------------------------------- NCCL, loaded at run time
typedef struct {
    char internal[128];
} ncclUniqueId_t;
typedef void *ncclComm_t;
typedef int (*fn_getid)(ncclUniqueId_t *);
typedef int (*fn_init)(ncclComm_t *, int, ncclUniqueId_t, int);
typedef int (*fn_destroy)(ncclComm_t);
typedef int (*fn_sendrecv)(void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*fn_group)();
typedef const char *(*fn_err)(int);
typedef int (*fn_allgather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t);
typedef int (*fn_allreduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*fn_asyncerr)(ncclComm_t, int *);
struct Nccl {
    void *h = nullptr;
    fn_getid getid;
    fn_init init;
    fn_destroy destroy;
    fn_sendrecv send, recv;
    fn_group gstart, gend;
    fn_err err;
    fn_allgather allgather;
    fn_allreduce allreduce;
    fn_asyncerr asyncerr;
};
Nccl &nccl() {
    static Nccl n;
    if (!n.h) {
        n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!n.h) return n;
        n.getid = (fn_getid)dlsym(n.h, "ncclGetUniqueId");
        n.init = (fn_init)dlsym(n.h, "ncclCommInitRank");
        n.destroy = (fn_destroy)dlsym(n.h, "ncclCommDestroy");
        n.send = (fn_sendrecv)dlsym(n.h, "ncclSend");
        n.recv = (fn_sendrecv)dlsym(n.h, "ncclRecv");
        n.gstart = (fn_group)dlsym(n.h, "ncclGroupStart");
        n.gend = (fn_group)dlsym(n.h, "ncclGroupEnd");
        n.err = (fn_err)dlsym(n.h, "ncclGetErrorString");
        n.allgather = (fn_allgather)dlsym(n.h, "ncclAllGather");
        n.allreduce = (fn_allreduce)dlsym(n.h, "ncclAllReduce");
        n.asyncerr = (fn_asyncerr)dlsym(n.h, "ncclCommGetAsyncError");
        if (!n.getid || !n.init || !n.send || !n.recv || !n.gstart || !n.gend) {
            dlclose(n.h);
            n.h = nullptr;
        }
    }
    return n;
}
constexpr int kNcclUint8 = 1;

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

bool nccl_unique_id(void *id128, std::string &err) {
    Nccl &n = nccl();
    if (!n.h) {
        err = "libnccl.so.2 not loadable";
        return false;
    }
    ncclUniqueId_t id;
    int rc = n.getid(&id);
    if (rc) {
        err = std::string("ncclGetUniqueId: ") + (n.err ? n.err(rc) : "error");
        return false;
    }
    std::memcpy(id128, &id, 128);
    return true;
}

bool nccl_comm_init(void **comm, int nranks, int rank, const void *id128, std::string &err) {
    Nccl &n = nccl();
    if (!n.h) {
        err = "libnccl.so.2 not loadable";
        return false;
    }
    ncclUniqueId_t id;
    std::memcpy(&id, id128, 128);
    ncclComm_t c = nullptr;
    int rc = n.init(&c, nranks, id, rank);
    if (rc) {
        err = std::string("ncclCommInitRank: ") + (n.err ? n.err(rc) : "error");
        return false;
    }
    *comm = c;
    return true;
}

bool nccl_async_error(void *comm, std::string &err) {
    Nccl &n = nccl();
    if (!n.h || !n.asyncerr || !comm) return false;
    int res = 0;
    const int rc = n.asyncerr(static_cast<ncclComm_t>(comm), &res);
    if (rc == 0 && res == 0) return false;
    err = std::string("NCCL asynchronous error: ") + (n.err ? n.err(rc ? rc : res) : "error");
    return true;
}

void nccl_comm_destroy(void *comm) {
    Nccl &n = nccl();
    if (n.h && comm && n.destroy) n.destroy((ncclComm_t)comm);
}

void exchange_pack(const Exchange &x, const double4 *u, const uint8_t *state, cudaStream_t st) {
    const int64_t tot = x.n_send_nodes + x.n_send_tets;
    if (tot)
        k_pack<<<nblk(tot), 256, 0, st>>>(u, state, x.d_send_nodes, x.n_send_nodes, x.d_send_ndst, x.d_send_tets,
                                          x.n_send_tets, x.d_send_tdst, x.d_sendbuf);
}

void exchange_unpack(const Exchange &x, double4 *u, uint8_t *state, const int32_t *eedge, int64_t E,
                     uint8_t *edge_dirty, cudaStream_t st, const uint8_t *recvbuf) {
    const int64_t tot = x.n_recv_nodes + x.n_recv_tets;
    if (tot)
        k_unpack<<<nblk(tot), 256, 0, st>>>(u, state, x.d_recv_nodes, x.n_recv_nodes, x.d_recv_nsrc, x.d_recv_tets,
                                            x.n_recv_tets, x.d_recv_tsrc, recvbuf ? recvbuf : x.d_recvbuf, eedge, E,
                                            edge_dirty);
}

void p2p_sync(const P2P &q, int npeers, int64_t target, bool wait, cudaStream_t st) {
    if (npeers) k_p2p_sync<<<1, 32, 0, st>>>(q.flags, q.d_peer_flag, q.d_peer_rank, npeers, target, wait ? 1 : 0, q.timeout);
}

void p2p_push_nodes(const P2P &q, const double4 *u, int64_t N, int par, int npeers, cudaStream_t st) {
    if (N) k_p2p_push<<<nblk(N), 256, 0, st>>>(u, N, q.d_noff, q.d_npeer, q.d_nbyte, q.d_peer_recv, npeers, par);
}

void count_mismatch(const uint8_t *a, const uint8_t *b, const int64_t *pos, int64_t n, int64_t width, int64_t *out,
                    cudaStream_t st) {
    if (n) k_mismatch<<<nblk(n), 256, 0, st>>>(a, b, pos, n, width, out);
}

bool nccl_allgather_bytes(const void *d_send, void *d_recv, size_t bytes, void *comm, cudaStream_t st, std::string &err) {
    Nccl &n = nccl();
    if (!n.h || !n.allgather) {
        err = "ncclAllGather not available";
        return false;
    }
    const int rc = n.allgather(d_send, d_recv, bytes, kNcclUint8, (ncclComm_t)comm, st);
    if (rc) err = std::string("ncclAllGather: ") + (n.err ? n.err(rc) : "error");
    return rc == 0;
}

bool nccl_allreduce_max_i64(const void *d_send, void *d_recv, size_t count, void *comm, cudaStream_t st, std::string &err) {
    Nccl &n = nccl();
    if (!n.h || !n.allreduce) {
        err = "ncclAllReduce not available";
        return false;
    }
    constexpr int kNcclInt64 = 4, kNcclMax = 2;
    const int rc = n.allreduce(d_send, d_recv, count, kNcclInt64, kNcclMax, (ncclComm_t)comm, st);
    if (rc) err = std::string("ncclAllReduce: ") + (n.err ? n.err(rc) : "error");
    return rc == 0;
}

bool exchange_nccl(const Exchange &x, void *comm, cudaStream_t st, std::string &err) {
    Nccl &n = nccl();
    if (!n.h) {
        err = "libnccl.so.2 not loadable";
        return false;
    }
    n.gstart();
    for (size_t j = 0; j < x.peers.size(); ++j) {
        const size_t sb = x.send_off[j + 1] - x.send_off[j], rb = x.recv_off[j + 1] - x.recv_off[j];
        if (sb) n.send(x.d_sendbuf + x.send_off[j], sb, kNcclUint8, x.peers[j], (ncclComm_t)comm, st);
        if (rb) n.recv(x.d_recvbuf + x.recv_off[j], rb, kNcclUint8, x.peers[j], (ncclComm_t)comm, st);
    }
    const int rc = n.gend();
    if (rc) {
        err = std::string("NCCL group: ") + (n.err ? n.err(rc) : "error");
        return false;
    }
    return true;
}

}  // namespace cem
