// cem_dist.h -- halo exchange (cem_dist.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace cem {

// Byte layout of the send / receive buffers: per peer j a segment [off[j], off[j+1]) holding
// the peer's node displacements (3 doubles each, ascending global id) followed by the tet
// state bytes (ascending global id), padded to 8 bytes.
struct Exchange {
    std::vector<int> peers;
    std::vector<size_t> send_off, recv_off;       // [peers + 1] byte offsets
    int64_t n_send_nodes = 0, n_send_tets = 0, n_recv_nodes = 0, n_recv_tets = 0;
    int32_t *d_send_nodes = nullptr, *d_send_tets = nullptr, *d_recv_nodes = nullptr, *d_recv_tets = nullptr;
    int64_t *d_send_ndst = nullptr, *d_recv_nsrc = nullptr;  // byte positions of the node records
    int64_t *d_send_tdst = nullptr, *d_recv_tsrc = nullptr;  // byte positions of the state bytes
    uint8_t *d_sendbuf = nullptr, *d_recvbuf = nullptr;
};

// P2P halo: stage D stores the predicted displacement of every owned node a
// peer holds straight into that peer's receive buffer (double-buffered by step parity) over
// NVLink, the split pass stores the state byte of owned tets the peer holds as ghosts; one
// flag per (peer, step) then orders the peers' stores before the receiver's unpack.
struct P2P {
    bool on = false;
    uint8_t *recv[2] = {nullptr, nullptr};  // this rank's receive buffers (layout of Exchange::recv_off)
    int64_t *flags = nullptr;               // [nranks] last step each peer has completed its stores for
    int64_t *timeout = nullptr;             // = flags + nranks: set when a wait for a peer gave up
    std::vector<void *> opened;             // IPC-mapped peer allocations
    uint8_t **d_peer_recv = nullptr;        // [2][npeers] peer buffer + the offset of this rank's segment
    int64_t **d_peer_flag = nullptr;        // [npeers] &peer.flags[this rank]
    int32_t *d_peer_rank = nullptr;         // [npeers]
    int32_t *d_noff = nullptr, *d_npeer = nullptr, *d_nbyte = nullptr;  // storage node -> (peer, byte) CSR
    int32_t *d_toff = nullptr, *d_tpeer = nullptr, *d_tbyte = nullptr;  // storage tet -> (peer, byte) CSR
};

bool nccl_unique_id(void *id128, std::string &err);
bool nccl_comm_init(void **comm, int nranks, int rank, const void *id128, std::string &err);
void nccl_comm_destroy(void *comm);
// ncclCommGetAsyncError: true (and a message) if the communicator has failed asynchronously
bool nccl_async_error(void *comm, std::string &err);
void exchange_pack(const Exchange &x, const double4 *u, const uint8_t *state, cudaStream_t st);
void exchange_unpack(const Exchange &x, double4 *u, uint8_t *state, const int32_t *eedge, int64_t E,
                     uint8_t *edge_dirty, cudaStream_t st, const uint8_t *recvbuf = nullptr);
bool exchange_nccl(const Exchange &x, void *comm, cudaStream_t st, std::string &err);
bool nccl_allgather_bytes(const void *d_send, void *d_recv, size_t bytes, void *comm, cudaStream_t st, std::string &err);
bool nccl_allreduce_max_i64(const void *d_send, void *d_recv, size_t count, void *comm, cudaStream_t st, std::string &err);
// signal this rank's step `target` to the peers and (wait) until every peer has signalled it
void p2p_sync(const P2P &q, int npeers, int64_t target, bool wait, cudaStream_t st);
// push u of the send nodes into the peers' receive buffers[par] (the kernel stage D runs inline)
void p2p_push_nodes(const P2P &q, const double4 *u, int64_t N, int par, int npeers, cudaStream_t st);
// count of differing bytes between two device buffers (self-check)
void count_mismatch(const uint8_t *a, const uint8_t *b, const int64_t *pos, int64_t n, int64_t width, int64_t *out,
                    cudaStream_t st);

}  // namespace cem
