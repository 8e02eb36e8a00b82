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

bool nccl_unique_id(void *id128, std::string &err);
bool nccl_comm_init(void **comm, int nranks, int rank, const void *id128, std::string &err);
void nccl_comm_destroy(void *comm);
void exchange_pack(const Exchange &x, const double4 *u, const uint8_t *state, cudaStream_t st);
void exchange_unpack(const Exchange &x, double4 *u, uint8_t *state, const int32_t *eedge, int64_t E,
                     uint8_t *edge_dirty, cudaStream_t st);
bool exchange_nccl(const Exchange &x, void *comm, cudaStream_t st, std::string &err);

}  // namespace cem
