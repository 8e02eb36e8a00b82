// cem_internal.h -- private structures of libcem.so (product path; shares nothing with oracle/).
#pragma once
#include <cstddef>
#include <cstdint>
#include <memory>
#include <utility>
#include <string>
#include <vector>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

#include "../../include/cem.h"

namespace cem {

// force-slot layout: 3 (default) = the 4 slots of a tet packed (12 doubles, 96 B per tet, slot
// index 4e + a, written with three 256-bit stores); 4 = warp-tiled (x, y, z, 0) slots, one 32-B
// sector each, slot index ((e>>5)*4 + a)*32 + (e&31)
#ifndef CEM_FES
#define CEM_FES 3
#endif

// 1: stage C recomputes the element geometry from staged node coordinates instead of reading
// the 88-B geometry record (-75 MB/step DRAM, but +4 KB shared memory per block: slower)
// geometry layout: 0 (default) = warp-tiled planes (ten coalesced 8-B loads per tet), 1 = one
// 96-B record per tet (three 32-B loads; measured slower: 161 vs 158 us/step on config 3)
#ifndef CEM_GEO_AOS
#define CEM_GEO_AOS 0
#endif
#ifndef CEM_C_GEOX
#define CEM_C_GEOX 0
#endif

// stage AB: edges per thread (an AB block covers CEM_AB_EPT * blk consecutive edges).  2 cuts
// AB's own time (64 vs 68 us: fewer duplicated tets) but its larger blocks overlap less with the
// neighbouring stages under programmatic dependent launch: 164 vs 156 us per step -> 1
#ifndef CEM_AB_EPT
#define CEM_AB_EPT 1
#endif

// phase timer of the host preprocessing (CEM_TIMING=1 prints to stderr)
struct PhaseClock {
    bool on = getenv("CEM_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char *what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[cem timing] %-28s %8.3f s\n", what, std::chrono::duration<double>(n - t).count());
        t = n;
    }
};

// host vector whose resize() leaves new elements uninitialised (default-init): the large plan tables
// are written in full by parallel loops, so the serial zero-fill (and its page faults on one core)
// is skipped -- first touch happens in those loops
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = DefaultInitAlloc<U>;
    };
    DefaultInitAlloc() = default;
    template <class U>
    DefaultInitAlloc(const DefaultInitAlloc<U> &) noexcept {}
    template <class U>
    void construct(U *p) noexcept {
        ::new (static_cast<void *>(p)) U;
    }
    template <class U, class... A>
    void construct(U *p, A &&...a) {
        ::new (static_cast<void *>(p)) U(std::forward<A>(a)...);
    }
};
template <class T>
using hvec = std::vector<T, DefaultInitAlloc<T>>;

// ---------------------------------------------------------------- host preprocessing
// HostMesh holds the mesh in the caller's ("original") numbering (cem_mesh.cpp).
struct HostMesh {
    int64_t N = 0, E = 0, S = 0;
    std::vector<double> X;            // [N][3]
    std::vector<int32_t> tet;         // [E][4]
    std::vector<uint8_t> state;       // [E]
    std::vector<double> gc;           // [E]
    std::vector<double> V;            // [E]
    hvec<double> grad;                // [E][4][3]
    hvec<int32_t> elem_edge;          // [E][6]
    std::vector<int32_t> edge_nodes;  // [S][2]
    std::vector<int32_t> edge_off;    // [S+1]
    hvec<int32_t> edge_inc;           // [6E] ascending tet id per edge
    std::vector<int32_t> node_off;    // [N+1]
    std::vector<int32_t> node_ent;    // [4E] 4e+a, ascending e per node
    std::vector<double> mass;         // [N]
    std::vector<double> fext;         // [N][3]
    std::vector<uint8_t> nflag;       // [N] bit0-2 Dirichlet mask, bit3 has f_ext
    std::vector<double> dir_v0;       // [N][3]
    double lam = 0, mu = 0, l2m = 0, rho = 0;
    double dt = 0, gamma = 0.5, t0 = 0;
    bool any_dirichlet = false;
};

cem_status build_host_mesh(const cem_mesh_in *m, const cem_material *mat, const cem_load_in *ld,
                           const cem_opts *o, HostMesh &h, std::string &err);

// ---------------------------------------------------------------- hexahedra (ES-H-FEM, N3)
// local edges of a trilinear hex (p < q): bottom ring, top ring, verticals
constexpr int kHexEdgeP[12] = {0, 1, 2, 0, 4, 5, 6, 4, 0, 1, 2, 3};
constexpr int kHexEdgeQ[12] = {1, 2, 3, 3, 5, 6, 7, 7, 4, 5, 6, 7};
// local node pair (a, b) -> 0..27 (lexicographic over a < b), and the hex edge of a pair (-1: diagonal)
constexpr int kHexPairOf(int a, int b) {
    return a < b ? 7 * a - a * (a - 1) / 2 + (b - a - 1) : 7 * b - b * (b - 1) / 2 + (a - b - 1);
}
struct HexPairTab {
    int p[8][8];
    constexpr HexPairTab() : p() {
        for (int a = 0; a < 8; ++a)
            for (int b = 0; b < 8; ++b) p[a][b] = a == b ? -1 : kHexPairOf(a, b);
    }
    constexpr const int *operator[](int a) const { return p[a]; }
};
constexpr HexPairTab kHexPair{};
struct HexEdgeOfPairTab {
    int v[28];
    constexpr HexEdgeOfPairTab() : v() {
        for (int j = 0; j < 28; ++j) v[j] = -1;
        for (int l = 0; l < 12; ++l) v[kHexPairOf(kHexEdgeP[l], kHexEdgeQ[l])] = l;
    }
    constexpr int operator[](int j) const { return v[j]; }
};
constexpr HexEdgeOfPairTab kHexEdgeOfPair{};
struct HexHost {
    int64_t N = 0, E = 0, S = 0, S_h = 0;
    std::vector<int32_t> pair;        // [28][E] edge of the local node pair (R28)
    std::vector<double> gc;           // [4E] hexes, then remainder tets E + 3e + i
    std::vector<int32_t> hex;         // [E][8]
    std::vector<uint8_t> state;       // [E]
    std::vector<double> V, grad;      // [E], [E][8][3] mean gradients (R23)
    std::vector<int32_t> eedge;       // [12][E] edge of local edge l
    std::vector<int32_t> edge_off, edge_inc, node_off, node_ent;
    std::vector<double> vhat, mass, fext, dir_v0;
    std::vector<uint8_t> nflag;
    std::vector<int32_t> nodeE;       // [N][wn] hex slots 8e + a, then remainder slots 8E + 3 (8e + a) + i, padded with zslot
    int wn = 8;
    int wn0 = 8;                      // row prefix holding every sub-0 slot (multiple of 8): all stage D reads until a remainder exists
    int32_t zslot = 0;
    double lam = 0, mu = 0, l2m = 0, rho = 0, dt = 0, gamma = 0.5, t0 = 0;
    bool any_dirichlet = false;
};
bool hex_geometry(const double *X8, double &V, double *grad);
cem_status build_hex_host(const cem_mesh_in *m, const cem_material *mat, const cem_load_in *ld, const cem_opts *o,
                          HexHost &h, std::string &err);
cem_status count_edges(const cem_mesh_in *m, int64_t *S, std::string &err);
cem_status global_cfl_dt(const cem_mesh_in *m, const cem_material *mat, double cfl, double *dt, std::string &err);

// ---------------------------------------------------------------- storage plan
// Storage ("new") numbering: tets sorted by (sweep-axis slab of the centroid, original id),
// nodes and edges by first appearance in that tet order.  Summation lists keep the
// ORIGINAL tet order so every sum matches the oracle bit for bit.
// AB: strain of the block's tets + smoothed edge stress (fused), C: element force + crack
// criterion, D: node update.
enum Stage { ST_AB = 0, ST_C = 1, ST_D = 2, ST_COUNT = 3 };


struct Plan {
    std::vector<int32_t> tet_new2old, tet_old2new, node_new2old, node_old2new, edge_new2old;
    // storage-order arrays
    hvec<int32_t> conn;               // [E][4] new node ids (int4)
    std::vector<double> geoV, geoC;   // [E] V, V/6
    hvec<int32_t> eedge;              // [6][E] new edge ids
    std::vector<int32_t> edge_off, edge_inc;   // CSR over new edges, new tet ids, original order
    std::vector<int32_t> node_off, node_ent;   // CSR over new nodes, (new e << 2 | a), original order
    std::vector<uint8_t> state;
    std::vector<uint8_t> tflag;       // [E] bit0 evaluate the criterion, bit1 record splits (multi-GPU masks)
    std::vector<double> gc;
    // blocks and the wavefront schedule
    int blk = 256;                    // entities per work item (C: tets, D: nodes)
    int blk_ab = 256;                 // edges per stage-AB block (CEM_AB_EPT * blk)
    int nblk[ST_COUNT] = {0, 0, 0};
    int maxblk = 0;
    std::vector<int32_t> dep_off;     // [ST_COUNT * maxblk + 1] CSR of producer blocks per (stage, block)
    std::vector<int32_t> dep;         // producer block ids (of the producing stage)
    std::vector<int32_t> ncons;       // [ST_COUNT][maxblk] consumer blocks of each block (discard counts)
    std::vector<int32_t> sched;       // [P]: stage << 28 | block
    // block gather lists (deduplicated producer records staged in shared memory)
    std::vector<int32_t> nl_off, nl;  // tet block -> sorted unique node ids
    hvec<uint16_t> lconn;             // [E][4] index of each tet node in its block's node list
    std::vector<int32_t> el_off, el;  // tet block -> sorted unique edge ids
    hvec<uint16_t> ledge;             // [E][8] index of each tet edge in its block's edge list (6 used)
    std::vector<int32_t> tl_off, tl;  // edge block -> sorted unique incident tet ids
    std::vector<int32_t> nlb_off, nlb;  // edge block -> sorted unique nodes of its tet list
    hvec<uint16_t> tconn;             // [|tl|][4] staging row (in nlb) of each tet-list entry's nodes
    std::vector<uint16_t> trow;       // [|tl|] shared-memory row of each tet-list entry (bank-aware)
    std::vector<uint16_t> nrow;       // [|nlb|] shared-memory row of each node-list entry (bank-aware)
    hvec<uint16_t> inc_local;         // [6E] (CSR order of edge_inc) index into the edge block's tet list
    int max_nl = 0, max_el = 0, max_tl = 0, max_nlb = 0;
    // instruction-lean layouts
    hvec<double> geoT;                // geometry: [E][12] records or [E/32][11][32] tiles (CEM_GEO_AOS)
    int we = 8;                       // ELL width of edge incidences (multiple of 8)
    int we_max = 8;                   // largest incidence count (loop bound)
    hvec<uint16_t> incE;              // [S][we] index into the edge block's tet list, 0xFFFF = none
    int wn = 8;                       // ELL width of node incidences (multiple of 8)
    hvec<int32_t> nodeE;              // [N][wn] force slot of each incidence (original order), zslot = none
    int32_t zslot = 0;
    // exact partial sums of the nodal assembly (R27, DESIGN.md §6 "Partials"): stage C sums, for
    // each entry q of its block's node list, the contributions of the block's tets to that node
    // (partial q); stage D adds the partials of its node.  partials = false: force slots instead.
    bool partials = true;
    std::vector<int32_t> pinc_off;    // [|nl| + 1] entries of partial q in pinc
    hvec<uint16_t> pinc;              // [4E] a blk + t (t: tet within the block, a: corner), per partial
    std::vector<int32_t> pord;        // [|nl|] per block: node-list entries by descending incidence count
    std::vector<int32_t> poff;        // [N + 1] node-major partial records: node k's at [poff[k], poff[k+1])
    std::vector<int32_t> pdst;        // [|nl|] node-major record of partial q (ascending q per node)
};

void build_plan(const HostMesh &h, int blk, Plan &p, const uint8_t *tflag_orig = nullptr, bool with_deps = true);

// Dataflow ("wave") execution of the staged kernels (DESIGN.md §6 "Wavefront"): each stage's
// blocks are launched in chunks along the storage order, interleaved so that a consumer chunk is
// launched right after the producer chunks it reads; a block waits only for the producer blocks
// it reads (per-block completion counters), not for whole kernels, so consecutive stages and
// steps overlap and intermediates are consumed while they are still in L2.
struct WaveLaunch {
    int stage;      // ST_AB, ST_C or ST_D
    int b0, b1;     // block range [b0, b1) (D blocks are kDW nodes)
};
struct WavePlan {
    int nblk[ST_COUNT] = {0, 0, 0};   // AB: blk_ab edges, C: blk tets, D: kDW nodes per block
    int maxblk = 0;
    std::vector<int32_t> dep_off;     // [ST_COUNT * maxblk + 1] producer blocks of (stage, block)
    std::vector<int32_t> dep;         //   AB <- D (previous step), C <- AB, D <- C
    std::vector<int32_t> ncons;       // [2][maxblk]: consumer blocks of each AB (C-stage readers) / C block (D)
    std::vector<WaveLaunch> seq;      // launches of one step, in order
};
constexpr int kDW = 64;               // nodes per stage-D block (256 threads, four lanes per node)
void build_wave(const Plan &p, int64_t N, int chunks, int lookahead, WavePlan &w);
void build_schedule(Plan &p, int resident_ctas);

// ---------------------------------------------------------------- device view
struct Dev;
struct Dev {
    int64_t N, E, S;
    // read-only mesh tables (storage numbering)
    const int4 *conn;
    const int32_t *eedge;
    const double4 *X;
    const double4 *fext;
    const uint8_t *nflag;
    const double4 *dir_v0;
    const double *gc;
    const int32_t *tet_orig;   // storage -> original tet id
    const int32_t *node_orig;  // storage -> original node id
    // mutable state
    uint8_t *state;
    const uint8_t *tflag;      // [E] bit0 criterion here, bit1 record here (all 3 on one GPU)
    double *mass;
    int32_t *dirty;            // [N] step stamp of the last split touching the node
    double4 *ubuf[2];          // u_m lives in ubuf[m & 1]
    double4 *v, *a;
    double *rprev;             // [N][3] support force of prescribed dofs at the last step (NULL: none)
    double *wr_dof;            // [N][3] reaction work accumulated per prescribed dof (energy ledger)
    double *srec;              // [S][4]: sigma_s (11, 22, 33, 12), 32-B records
    double *srec2;             // [S][2]: sigma_s (23, 13), 16-B records
    double *fe;                // force slots f_{e,a}, CEM_FES doubles per slot (see CEM_FES)
    const double *geoT;        // geometry records (CEM_GEO_AOS) or warp-tiled planes
    const uint16_t *incE;      // [S][we]
    const int32_t *nodeE;      // [N][wn]
    int we, wn, we_max;        // ELL widths; we_max = largest edge incidence count
    int32_t zslot;             // index of the all-zero force slot (ELL padding)
    double *part;              // [|nl|][6] exact partials (s_x, s_y, s_z, c_x, c_y, c_z), node-major; null: force slots
    const int32_t *pinc_off;   // [|nl| + 1]
    const uint16_t *pinc;      // [4E] a blk + t per partial (stage C's force row)
    const int32_t *pord;       // [|nl|] per block: its node-list entries by descending incidence count
    const int32_t *poff;       // [N + 1] node k's partial records (node-major) at [poff[k], poff[k+1])
    const int32_t *pdst;       // [|nl|] node-major record of partial q
    const int32_t *nl_off, *nl, *el_off, *el, *tl_off, *tl, *nlb_off, *nlb;
    const uint16_t *tconn, *trow, *nrow;
    const uint16_t *lconn, *ledge;
    int smem_bytes, smem_ab, smem_c;  // dynamic shared memory: persistent kernel (max), per stage
    int cp_max_el, cp_max_nl;  // largest stage-C block edge / node lists (pipelined stage C, k_Cp)
    int cp_on, cp_grid;        // 1: stage C runs as k_Cp on cp_grid persistent CTAs
    const Dev *self;           // device-resident copy of this struct (for noinline helpers)
    int32_t *ctr;              // [0] records, [1] nonfinite, [2] first bad node (orig), [3] crit_list length,
                               // [8] survivors of the refined filter (crit_surv)
    int64_t *crit_list;        // [E] tets stage C flagged for the full criterion, entry (step + 1) << 32 | e
                               // (stamped: k_crit polls the entries of its own step while stage C runs)
    int32_t *crit_surv;        // [E] survivors of the refined filter (k_filter -> k_eval)
    int32_t *crit_seen;        // mapped host int: stage D writes the step's list length (kernel choice)
    double *vhat;              // [S] Vhat_s = sum V_e over the active incident tets (original order)
    uint8_t *edge_dirty;       // [S] 1: an incident tet split since stage AB last recomputed vhat[s]
    const int32_t *e_off, *e_inc;  // edge -> incident tets (storage ids, ascending original id)
    const uint8_t *edge_own;   // [S] 1 if this rank counts the edge in the energy ledger
    // P2P halo (multi-GPU); p2p_np = 0: the halo goes through NCCL / loopback copies
    uint8_t *const *p2p_recv;  // [2][p2p_np] peer receive buffer (+ this rank's segment) per step parity
    int p2p_np;
    const int32_t *p2p_noff, *p2p_npeer, *p2p_nbyte;  // storage node -> (peer, byte in segment) CSR
    const int32_t *p2p_toff, *p2p_tpeer, *p2p_tbyte;  // storage tet -> (peer, byte in segment) CSR
    int64_t *const *p2p_flag_out;  // [p2p_np] the peers' flag words for this rank (early signal)
    const int32_t *d_order;        // [nD] stage-D block order: blocks with peer-held nodes first
    int d_nbound;                  // how many of them
    unsigned long long *bdone;     // boundary D blocks finished (cumulative)
    int64_t *rec_step;
    int32_t *rec_elem, *rec_cand;
    double *rec_G, *rec_area;
    // parameters
    double lam, mu, l2m, rho, dt, hdt2, gamma, omg, t0;
    uint32_t flags;
    // persistent wavefront
    int32_t *cnt;              // [ST_COUNT][maxblk] completed-step counters
    const int32_t *dep_off, *dep;
    const int32_t *ncons;      // [ST_COUNT][maxblk] consumers of each AB/C block
    int32_t *cons_done;        // [ST_COUNT][maxblk] consumers finished with the block this step
    const int32_t *sched;      // [P]
    unsigned long long *head;  // work-queue head
    int blk, blk_ab, P, maxblk;
    int nblk[ST_COUNT];
    // dataflow ("wave") launches (WavePlan): per-block completion counters and producer lists
    int32_t *wcnt;             // [ST_COUNT][wmax]: the block has completed step value-1
    int64_t *wstep;            // base step of a graph replay (rel launches)
    // hexahedral contexts (npe = 8): [25][E] V + mean gradients, [8][E] connectivity, [12][E] edges,
    // [6][E] element strain planes
    int npe;
    const double *hgeo;
    const int32_t *hconn, *heedge;
    double *htau;
    // hex crack patterns III-VI (R28): [28][E] edge of each local node pair; per hex the remainder
    // (candidate k, -1 none), its tets' activity bits, local nodes [E][12], geometry [E][3][13]
    // (V, grad[4][3]) and strain [E][3][6]
    const int32_t *hpair;
    int64_t hS_h;              // edges [0, hS_h) are hex edges; the diagonals after them carry remainder tets only
    int8_t *hrem;
    uint8_t *htact, *htloc;
    double *htgeo, *httau;
    const int32_t *wncons;     // [2][wmax] consumers of each AB / C block (L2 discard of consumed intermediates)
    int32_t *wcons_done;       // [2][wmax] consumers finished with the block this step
    int wdiscard;              // 1: the last consumer discards a producer block's sigma / force-slot lines
    const int32_t *wdep_off, *wdep;
    int wmax;
    // (appended after every field the tet stage kernels read: their parameter offsets, and with them
    // the generated code and its measured time, stay those of the profiled build)
    int wn0;                   // hexahedra: the row prefix stage D reads for a node of no remainder prism (hnrem == 0); tets: wn
    uint8_t *hnrem;            // [N] node of some remainder prism (stage D then reads the node's remainder slots too)
    unsigned *hediag;          // bitmap over the diagonal edges [S_h, S): edge of some remainder prism, and ...
    int32_t *hdlist;           // ... the list of those edges (ctr[25] entries, appended by k_hexcrit): all stage B evaluates beyond the hex edges
    const int4 *heinc4;        // [S] the first four incidences of each edge (e << 5 | pair, -1 padding): one load instead of offsets + entries
    int32_t *hclist;           // hexes that failed the criterion's early-out this step (ctr[3] entries; k_hexcrit -> k_hexeval)
};

// cem_kernels.cu
// rel = 1: the step index is relative to the device word d.wstep (CUDA-graph replays)
int launch_wave_step(const Dev &d, const WavePlan &w, int64_t s, int crack_every, cudaStream_t st, int rel = 0);
void launch_wave_join(const Dev &d, int64_t nsteps_done, cudaStream_t st, int rel = 0);  // every block done
void launch_wave_base(const Dev &d, int64_t step0, cudaStream_t st);                    // d.wstep := step0
void launch_wave_fill(const Dev &d, int64_t step, cudaStream_t st);         // counters := step (after other modes)
void launch_persistent(const Dev &d, int64_t step0, int64_t nsteps, int crack_every, int grid, cudaStream_t st);
constexpr int kStagedEvents = 5;  // profiled staged step: AB | C | criterion | D
struct StagedSync {
    unsigned long long bdone = 0;  // cumulative boundary D blocks launched (early P2P signal)
};
// stage AB / C blocks of one chunk of a chunked staged step (CEM_STAGE_CHUNKS)
struct StageChunk {
    int ab0, ab1, c0, c1;
};
std::vector<StageChunk> build_stage_chunks(const Plan &p, int K);
// crit: how the criterion runs, from the recent list lengths -- CRIT_LIST: stage C lists the
// tets that fail the early-out, k_crit evaluates them after stage C (one warp each); CRIT_STREAM:
// k_crit takes the entries while stage C is still running; CRIT_IDLE: the same with a small grid
// (no recent list: fewer pollers); CRIT_HEAVY (long lists): k_filter + k_eval instead of k_crit.
// sy: the context's cumulative counts (multi-GPU early signal), may be null; chunks: AB/C in chunks
enum { CRIT_LIST = 0, CRIT_HEAVY = 1, CRIT_STREAM = 2, CRIT_IDLE = 3 };
int launch_staged_step(const Dev &d, int64_t s, int crack_every, cudaStream_t st, cudaEvent_t *ev /*5 or null*/,
                       int crit = CRIT_LIST, StagedSync *sy = nullptr,
                       const std::vector<StageChunk> *chunks = nullptr);  // kernels launched
void launch_energy(const Dev &d, int64_t n, double *part_edges, double *part_nodes, cudaStream_t st);
void launch_crack_only(const Dev &d, int64_t n, cudaStream_t st);
// cem_hex.cu: one explicit step of a hexahedral context (4 kernels, PDL-chained; stage D is the
// tet path's node update); returns the kernels launched
int launch_hex_step(const Dev &d, int64_t s, cudaStream_t st, bool crack, bool diagonals);
// hex criterion (patterns III-VI, remainder tets: the tet criterion) and split pass of step s
// (cem_kernels.cu), PDL-chained between stage C and stage D
void launch_hex_crit(const Dev &d, int64_t s, cudaStream_t st);
// energy ledger of a hexahedral context at step n: strain energy per edge block (U = sum_s
// psi(eps~_s) Vhat_s / 12, R26) into part_edges[ceil(S/256)], node terms as the tet ledger
void launch_hex_energy(const Dev &d, int64_t n, double *part_edges, double *part_nodes, cudaStream_t st);
void launch_energy_nodes(const Dev &d, int64_t n, double *part_nodes, cudaStream_t st);
// stage D alone (cem_kernels.cu), PDL-chained after the previous kernel
void launch_node_update(const Dev &d, int64_t s, cudaStream_t st);
int persistent_occupancy(int smem_bytes, int blk);  // resident CTAs per SM of the persistent kernel
void set_smem_limits(int smem_bytes);
void set_wave_carveout(int smem_ab, int smem_c, int pct = -1);  // same carveout for the three wave kernels
int cp_stage_c_smem(int max_el, int max_nl);  // dynamic shared memory of k_Cp (0: does not fit)
extern const int kThreads;

}  // namespace cem
