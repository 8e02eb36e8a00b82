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
        const int32_t e = tidx[i - nn];
        const uint8_t v = buf[tsrc[i - nn]];
        if (state[e] && !v)  // a ghost tet split on its owner: its edges' Vhat change
            for (int l = 0; l < 6; ++l) edge_dirty[eedge[(int64_t)l * E + e]] = 1;
        state[e] = v;
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
struct Nccl {
    void *h = nullptr;
    fn_getid getid;
    fn_init init;
    fn_destroy destroy;
    fn_sendrecv send, recv;
    fn_group gstart, gend;
    fn_err err;
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
                     uint8_t *edge_dirty, cudaStream_t st) {
    const int64_t tot = x.n_recv_nodes + x.n_recv_tets;
    if (tot)
        k_unpack<<<nblk(tot), 256, 0, st>>>(u, state, x.d_recv_nodes, x.n_recv_nodes, x.d_recv_nsrc, x.d_recv_tets,
                                            x.n_recv_tets, x.d_recv_tsrc, x.d_recvbuf, eedge, E, edge_dirty);
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
