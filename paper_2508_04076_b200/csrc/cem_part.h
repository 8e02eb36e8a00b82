// cem_part.h -- domain decomposition plan for the multi-GPU step (cem_part.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace cem {

struct PartGlobal {
    int P = 1;
    std::vector<int32_t> tet_owner, node_owner;       // [E], [N]
    std::vector<int32_t> node_off, node_tets;         // node -> tets (ascending)
    std::vector<int32_t> edge_off, edge_tets, tet_edge;
    std::vector<std::vector<int32_t>> local_tets;     // per rank, ascending global id
    std::vector<std::vector<uint8_t>> layer1;         // per rank, aligned with local_tets
    std::vector<std::vector<int32_t>> local_nodes;    // per rank, ascending global id
};

struct PartLocal {
    int rank = 0, nranks = 1;
    std::vector<int32_t> tet_global, node_global;     // local -> global ids (ascending)
    std::vector<uint8_t> tet_flag;                    // bit0 layer 1 (criterion), bit1 owned (records)
    std::vector<uint8_t> node_owned;                  // 1 if this rank updates the node
    std::vector<int> peers;
    std::vector<std::vector<int32_t>> send_nodes, recv_nodes, send_tets, recv_tets;  // local ids per peer
};

void build_partition(int64_t N, const double *X, int64_t E, const int32_t *tet, int P, PartGlobal &g);
void build_exchange(const PartGlobal &g, int p, PartLocal &L);

}  // namespace cem
