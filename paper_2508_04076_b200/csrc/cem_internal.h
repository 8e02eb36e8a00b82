// cem_internal.h -- private structures of libcem.so (product path; shares nothing with oracle/).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/cem.h"

namespace cem {

// Host-side preprocessed mesh (cem_mesh.cpp).  All arrays are in the caller's numbering.
struct HostMesh {
    int64_t N = 0, E = 0, S = 0;
    std::vector<double> X;            // [N][3]
    std::vector<int32_t> tet;         // [E][4]
    std::vector<uint8_t> state;       // [E]
    std::vector<double> gc;           // [E]
    std::vector<double> geo;          // [E][16]: V, c6=V/6, pad, pad, grad[4][3]
    std::vector<int32_t> elem_edge;   // [E][6]
    std::vector<int32_t> edge_nodes;  // [S][2]
    std::vector<int32_t> edge_off;    // [S+1]
    std::vector<int32_t> edge_inc;    // [6E] ascending tet id per edge
    std::vector<int32_t> node_off;    // [N+1]
    std::vector<int32_t> node_ent;    // [4E] 4e+a, ascending e per node
    std::vector<double> mass;         // [N]
    std::vector<double> fext;         // [N][3]
    std::vector<uint8_t> nflag;       // [N] bit0-2 Dirichlet mask, bit3 has f_ext
    std::vector<double> dir_v0;       // [N][3] (only meaningful where mask bits set)
    double lam = 0, mu = 0, l2m = 0, rho = 0;
    double dt = 0, gamma = 0.5, t0 = 0;
    bool any_dirichlet = false;
};

// builds HostMesh; returns CEM_OK or an error with message
cem_status build_host_mesh(const cem_mesh_in *m, const cem_material *mat, const cem_load_in *ld,
                           const cem_opts *o, HostMesh &h, std::string &err);
cem_status count_edges(const cem_mesh_in *m, int64_t *S, std::string &err);

// ---------------------------------------------------------------- device views
struct DevMesh {
    int64_t N, E, S;
    const double4 *X;         // [N] (x,y,z,0)
    const int4 *tet;          // [E]
    uint8_t *state;           // [E]
    const double *gc;         // [E]
    const double *geo;        // [E][16]
    const int32_t *elem_edge; // [E][6]
    const int32_t *edge_off;  // [S+1]
    const int32_t *edge_inc;  // [6E]
    const int32_t *node_off;  // [N+1]
    const int32_t *node_ent;  // [4E]
    double *mass;             // [N]
    const double4 *fext;      // [N]
    const uint8_t *nflag;     // [N]
    const double4 *dir_v0;    // [N]
    double lam, mu, l2m, rho, dt, gamma, t0;
    uint32_t flags;
};

struct DevState {
    double4 *u[2];            // ping-pong: u[cur] = u_n, u[cur^1] = u_{n+1} (predicted)
    double4 *v, *a;           // [N]
    double *tau;              // [E][6]  V_e eps_e
    double *sig;              // [S][6]  edge stress
    double *fe;               // [E][12] element nodal forces
    // split bookkeeping
    int32_t *ctr;             // [8]: 0 n_flag, 1 nonfinite, 2 first bad node, 3 overflow
    int64_t *step;            // [1] completed steps n
    double *Ud;               // [1]
    int64_t *nrec;            // [1]
    int32_t *flag_list;       // [cap] unordered flagged tets
    int32_t *flag_cand;       // [cap]
    double *flag_G;           // [cap]
    double *flag_area;        // [cap]
    uint8_t *flag;            // [E] split flag (fallback path)
    int64_t *rec_step;        // [E]
    int32_t *rec_elem, *rec_cand;
    double *rec_G, *rec_area;
    int32_t flag_cap;
};

enum KernelId { K_STRAIN = 0, K_EDGE, K_FORCE, K_NODE, K_SPLIT, K_COUNT };
extern const char *kKernelNames[K_COUNT];

// kernels (cem_kernels.cu): enqueue one step on `stream` with u-buffer index `cur`
void launch_strain(const DevMesh &m, const DevState &s, int cur, cudaStream_t st);
void launch_edge(const DevMesh &m, const DevState &s, cudaStream_t st);
void launch_force(const DevMesh &m, const DevState &s, int cur, int crack_every, cudaStream_t st);
void launch_node(const DevMesh &m, const DevState &s, int cur, cudaStream_t st);
void launch_split(const DevMesh &m, const DevState &s, int cur, int crack_every, int advance, cudaStream_t st);

}  // namespace cem
