// cem_api.cu -- the C ABI of libcem.so (include/cem.h): context, device workspace layout,
// host<->device transfers, the persistent-kernel step loop and state readback.
#include <nvtx3/nvToolsExt.h>  // (header-only NVTX3: ranges cost nothing unless a tool attaches)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "cem_dist.h"
#include "cem_internal.h"
#include "cem_part.h"

using namespace cem;

struct cem_ctx {
    HostMesh h;
    Plan p;
    StagedSync sy;                // cumulative counts of the staged path (multi-GPU early signal)
    int cp_on = 0, cp_grid = 0;   // pipelined stage C (CEM_C_PIPE)
    std::vector<StageChunk> chunks;  // AB / C launched in chunks (CEM_STAGE_CHUNKS > 1)
    WavePlan w;                   // dataflow launches (opt-in, CEM_WAVE=1; w.seq empty = off)
    int64_t wcnt_valid = -1;      // the wave counters are valid for this step count
    struct WaveGraph {
        int crack_every, M;
        cudaGraphExec_t exec;
    };
    std::vector<WaveGraph> graphs;  // captured M-step wave sequences (replayed with a device base step)
    int graph_m = 16;             // steps per graph replay (env CEM_GRAPH_M; 0 = eager launches)
    Dev d{};
    cudaStream_t stream = nullptr;       // the library's private non-blocking stream (all its work)
    cudaStream_t user_stream = nullptr;  // opts.stream (NULL = the legacy default stream)
    cudaEvent_t fence_in = nullptr, fence_out = nullptr;  // ordering between the two
    bool own_stream = false;
    bool l2_limit_raised = false;        // this ctx raised the device's persisting-L2 set-aside
    size_t l2_limit_prev = 0;
    int device = 0;
    void *ws = nullptr;
    size_t ws_bytes = 0;
    bool own_ws = false;
    int64_t step = 0;             // steps enqueued so far (n)
    int64_t cnt_valid = 0;        // the wavefront counters are valid for this step count
    uint32_t flags = 0;
    int grid = 0;                 // persistent CTAs
    int64_t launches = 0;         // kernels this ctx has launched
    bool profiling = false;
    std::vector<cudaEvent_t> ev;  // staged profiling: 5 events per step
    int64_t prof_steps = 0;
    std::string err;
    // multi-GPU (nranks > 1)
    bool dist = false, loopback = false;
    bool hexa = false;            // trilinear hexahedra (ES-H-FEM, cem_hex.cpp / cem_hex.cu)
    bool hex_cracked = false;     // a crack step has run: remainder tets (and their diagonal edges) may exist
    int rank = 0, nranks = 1;
    PartLocal part;
    Exchange xch;
    void *comm = nullptr;
    bool init_exchange_pending = false;
    std::vector<void *> dist_allocs;
    P2P p2p;                      // P2P halo (multi-GPU), see cem_dist.h
    cem_allgather_fn host_allgather = nullptr;  // host-ordered CUDA-IPC halo (opts.host_allgather)
    void *host_user = nullptr;
    volatile int32_t *crit_seen = nullptr;  // mapped: criterion-list length of a recent step
    int critb_min = 1024;         // lists at least this long use k_filter + k_eval (env CEM_CRITB_MIN at init)
    bool crit_stream = true;      // k_crit takes its entries while stage C runs (env CEM_CRIT_STREAM=0: after it)
    double *epart = nullptr;      // energy-ledger partials (device)
    int64_t n_epart_edges = 0, n_epart_nodes = 0;
};

namespace {

thread_local std::string g_init_err;

// Every entry point that enqueues work orders the library's private stream after the caller's
// stream on entry and the caller's stream after the private one on exit (include/cem.h
// "Asynchrony"), so work the caller put on opts.stream -- or on the legacy default stream when
// opts.stream is NULL -- is ordered with the library's in both directions.
struct StreamFence {
    cem_ctx *c;
    explicit StreamFence(cem_ctx *ctx) : c(ctx) {
        if (c && c->fence_in) {
            cudaEventRecord(c->fence_in, c->user_stream);
            cudaStreamWaitEvent(c->stream, c->fence_in, 0);
        }
    }
    ~StreamFence() {
        if (c && c->fence_out) {
            cudaEventRecord(c->fence_out, c->stream);
            cudaStreamWaitEvent(c->user_stream, c->fence_out, 0);
        }
    }
};

#define CUDA_TRY(x)                                                                   \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            ctx->err = std::string(#x) + ": " + cudaGetErrorString(e_);               \
            return CEM_ECUDA;                                                         \
        }                                                                             \
    } while (0)

// entities per work item (= threads per CTA); CEM_BLK (128 or 256) is a tuning knob
int block_size() {
    const char *e = getenv("CEM_BLK");
    const int b = e ? atoi(e) : 256;
    return (b == 128 || b == 256) ? b : 256;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// NVTX range of one ABI call (SURVEY.md §5 "Tracing": nsys / ncu timelines show the calls)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
// force slots: 4 per tet in 32-tet tiles, + the all-zero slot
int64_t fe_slots(int64_t E) { return 4 * ((E + 31) / 32) * 32 + 1; }

struct Layout {
    size_t off = 0;
    template <class T>
    size_t take(int64_t n) {
        size_t o = off;
        off = align_up(off + sizeof(T) * (size_t)(n > 0 ? n : 1));
        return o;
    }
};

struct Offs {
    size_t conn, geoT, eedge, incE, nodeE, X, fext, nflag, dir_v0, gc;
    size_t tet_orig, node_orig, state, mass, dirty, u0, u1, v, a, srec, srec2, fe, ctr;
    size_t rec_step, rec_elem, rec_cand, rec_G, rec_area, cnt, dep_off, dep, sched, head;
    size_t nl_off, nl, lconn, el_off, el, ledge, tl_off, tl, self, ncons, cons_done;
    size_t nlb_off, nlb, tconn, trow, nrow, tflag;
    size_t rprev, wr_dof, epart, crit_list, crit_surv, vhat, edge_dirty, e_off, e_inc, edge_own;
    size_t wcnt, wdep_off, wdep, wstep, wncons, wcons_done;
    size_t part, pinc_off, pinc, poff, pdst, pord;
    size_t total;
};

Offs layout(const HostMesh &h, const Plan &p, const WavePlan &w) {
    const int64_t N = h.N, E = h.E, S = h.S;
    int64_t P = 0;
    for (int g = 0; g < ST_COUNT; ++g) P += p.nblk[g];
    Layout L;
    Offs o{};
    o.conn = L.take<int4>(E);
    o.geoT = L.take<double>((int64_t)p.geoT.size());
    o.eedge = L.take<int32_t>(6 * E);
    o.incE = L.take<uint16_t>((int64_t)p.incE.size());
    o.nodeE = L.take<int32_t>((int64_t)p.nodeE.size());
    o.X = L.take<double4>(N);
    o.fext = L.take<double4>(N);
    o.nflag = L.take<uint8_t>(N);
    o.dir_v0 = L.take<double4>(h.any_dirichlet ? N : 1);
    o.gc = L.take<double>(E);
    o.tet_orig = L.take<int32_t>(E);
    o.node_orig = L.take<int32_t>(N);
    o.state = L.take<uint8_t>(E);
    o.mass = L.take<double>(N);
    o.dirty = L.take<int32_t>(N);
    o.u0 = L.take<double4>(N);
    o.u1 = L.take<double4>(N);
    o.v = L.take<double4>(N);
    o.a = L.take<double4>(N);
    o.srec = L.take<double>(4 * S);
    o.srec2 = L.take<double>(2 * S);
    o.part = L.take<double>(6 * (int64_t)p.nl.size());  // (after the sigma planes: one L2 window can span both)
    o.fe = L.take<double>(CEM_FES * fe_slots(E));  // + the zero slot
    o.ctr = L.take<int32_t>(32);
    o.rec_step = L.take<int64_t>(E);
    o.rec_elem = L.take<int32_t>(E);
    o.rec_cand = L.take<int32_t>(E);
    o.rec_G = L.take<double>(E);
    o.rec_area = L.take<double>(E);
    o.cnt = L.take<int32_t>(ST_COUNT * (int64_t)p.maxblk);
    o.dep_off = L.take<int32_t>((int64_t)p.dep_off.size());
    o.dep = L.take<int32_t>((int64_t)p.dep.size());
    o.sched = L.take<int32_t>(P);
    o.head = L.take<unsigned long long>(1);
    o.nl_off = L.take<int32_t>((int64_t)p.nl_off.size());
    o.nl = L.take<int32_t>((int64_t)p.nl.size());
    o.lconn = L.take<uint16_t>((int64_t)p.lconn.size());
    o.el_off = L.take<int32_t>((int64_t)p.el_off.size());
    o.el = L.take<int32_t>((int64_t)p.el.size());
    o.ledge = L.take<uint16_t>((int64_t)p.ledge.size());
    o.tl_off = L.take<int32_t>((int64_t)p.tl_off.size());
    o.tl = L.take<int32_t>((int64_t)p.tl.size());
    o.self = L.take<Dev>(1);
    L.take<char>(256);  // tail padding: bulk-copy windows are rounded up to 16 B
    o.ncons = L.take<int32_t>(ST_COUNT * (int64_t)p.maxblk);
    o.cons_done = L.take<int32_t>(ST_COUNT * (int64_t)p.maxblk);
    o.nlb_off = L.take<int32_t>((int64_t)p.nlb_off.size());
    o.nlb = L.take<int32_t>((int64_t)p.nlb.size());
    o.tconn = L.take<uint16_t>((int64_t)p.tconn.size());
    o.trow = L.take<uint16_t>((int64_t)p.trow.size());
    o.nrow = L.take<uint16_t>((int64_t)p.nrow.size());
    o.tflag = L.take<uint8_t>(E);
    o.rprev = L.take<double>(h.any_dirichlet ? 3 * N : 1);
    o.wr_dof = L.take<double>(h.any_dirichlet ? 3 * N : 1);
    o.epart = L.take<double>(p.nblk[ST_AB] + 3 * ((N + 255) / 256));
    o.crit_list = L.take<int64_t>(E);  // the step's list (stamped entries)
    o.crit_surv = L.take<int32_t>(E);  // the refined filter's survivors
    o.vhat = L.take<double>(S);
    o.edge_dirty = L.take<uint8_t>(S);
    o.e_off = L.take<int32_t>(S + 1);
    o.e_inc = L.take<int32_t>((int64_t)p.edge_inc.size());
    o.edge_own = L.take<uint8_t>(S);
    o.wcnt = L.take<int32_t>(ST_COUNT * (int64_t)w.maxblk);
    o.wdep_off = L.take<int32_t>((int64_t)w.dep_off.size());
    o.wdep = L.take<int32_t>((int64_t)w.dep.size());
    o.wstep = L.take<int64_t>(1);
    o.wncons = L.take<int32_t>((int64_t)w.ncons.size());
    o.wcons_done = L.take<int32_t>((int64_t)w.ncons.size());
    o.pinc_off = L.take<int32_t>((int64_t)p.pinc_off.size());
    o.pinc = L.take<uint16_t>((int64_t)p.pinc.size());
    o.poff = L.take<int32_t>((int64_t)p.poff.size());
    o.pdst = L.take<int32_t>((int64_t)p.pdst.size());
    o.pord = L.take<int32_t>((int64_t)p.pord.size());
    o.total = L.off;
    return o;
}

int smem_ab_for(const Plan &p) { return 8 * (3 * (p.max_nlb | 1) + 7 * ((p.max_tl + 1) | 1)); }  // u: 3, tau + V: 7 planes
// stage C reuses its staging area for the warps' criterion scratch (<= 8 warps x ~840 B)
// (CEM_C_GEOX adds 3 planes of node coordinates; the default keeps stage C's shared memory small:
// its blocks then share the SM with a larger L1, which stage C measurably needs)
// (partials: + 12 planes of the block's element forces, f_{t,a,c} at [(3a + c) blk + t])
int smem_c_for(const Plan &p) {
    // (partials also stage the block's incidence entries, 4 x u16 per tet, and per-entry offsets)
    // the force planes (12 doubles per tet) overlay the sigma planes
    const int sig = p.partials ? std::max(6 * (p.max_el | 1), 12 * p.blk) : 6 * (p.max_el | 1);
    const int part = p.partials ? p.blk + (3 * p.max_nl + 2) / 2 + 1 : 0;  // pinc; offsets, order, destinations (int32)
    return std::max(8 * (sig + (CEM_C_GEOX ? 6 : 3) * (p.max_nl | 1) + part), 8 * 1024);
}
int smem_bytes_for(const Plan &p) { return std::max(smem_ab_for(p), smem_c_for(p)); }  // odd plane strides

template <class T>
T *at(void *base, size_t off) {
    return reinterpret_cast<T *>(static_cast<char *>(base) + off);
}

void bind_views(cem_ctx *ctx, const Offs &o) {
    void *b = ctx->ws;
    const HostMesh &h = ctx->h;
    const Plan &p = ctx->p;
    Dev &d = ctx->d;
    d.N = h.N;
    d.E = h.E;
    d.S = h.S;
    d.conn = at<int4>(b, o.conn);
    d.geoT = at<double>(b, o.geoT);
    d.eedge = at<int32_t>(b, o.eedge);
    d.incE = at<uint16_t>(b, o.incE);
    d.nodeE = at<int32_t>(b, o.nodeE);
    d.we = p.we;
    d.we_max = p.we_max;
    d.zslot = p.zslot;
    d.wn = p.wn;
    d.wn0 = p.wn;
    d.X = at<double4>(b, o.X);
    d.fext = at<double4>(b, o.fext);
    d.nflag = at<uint8_t>(b, o.nflag);
    d.dir_v0 = at<double4>(b, o.dir_v0);
    d.gc = at<double>(b, o.gc);
    d.tet_orig = at<int32_t>(b, o.tet_orig);
    d.node_orig = at<int32_t>(b, o.node_orig);
    d.state = at<uint8_t>(b, o.state);
    d.mass = at<double>(b, o.mass);
    d.dirty = at<int32_t>(b, o.dirty);
    d.ubuf[0] = at<double4>(b, o.u0);
    d.ubuf[1] = at<double4>(b, o.u1);
    d.v = at<double4>(b, o.v);
    d.a = at<double4>(b, o.a);
    d.srec = at<double>(b, o.srec);
    d.srec2 = at<double>(b, o.srec2);
    d.fe = at<double>(b, o.fe);
    d.part = p.partials ? at<double>(b, o.part) : nullptr;
    d.pinc_off = at<int32_t>(b, o.pinc_off);
    d.pinc = at<uint16_t>(b, o.pinc);
    d.poff = at<int32_t>(b, o.poff);
    d.pdst = at<int32_t>(b, o.pdst);
    d.pord = at<int32_t>(b, o.pord);
    d.nl_off = at<int32_t>(b, o.nl_off);
    d.nl = at<int32_t>(b, o.nl);
    d.lconn = at<uint16_t>(b, o.lconn);
    d.el_off = at<int32_t>(b, o.el_off);
    d.el = at<int32_t>(b, o.el);
    d.ledge = at<uint16_t>(b, o.ledge);
    d.tl_off = at<int32_t>(b, o.tl_off);
    d.tl = at<int32_t>(b, o.tl);
    d.smem_bytes = smem_bytes_for(p);
    d.smem_ab = smem_ab_for(p);
    d.smem_c = smem_c_for(p);
    d.cp_max_el = p.max_el;
    d.cp_max_nl = p.max_nl;
    d.cp_on = ctx->cp_on;
    d.cp_grid = ctx->cp_grid;
    d.self = at<Dev>(b, o.self);
    d.ncons = at<int32_t>(b, o.ncons);
    d.cons_done = at<int32_t>(b, o.cons_done);
    d.nlb_off = at<int32_t>(b, o.nlb_off);
    d.nlb = at<int32_t>(b, o.nlb);
    d.tconn = at<uint16_t>(b, o.tconn);
    d.trow = at<uint16_t>(b, o.trow);
    d.nrow = at<uint16_t>(b, o.nrow);
    d.tflag = at<uint8_t>(b, o.tflag);
    d.ctr = at<int32_t>(b, o.ctr);
    d.rec_step = at<int64_t>(b, o.rec_step);
    d.rec_elem = at<int32_t>(b, o.rec_elem);
    d.rec_cand = at<int32_t>(b, o.rec_cand);
    d.rec_G = at<double>(b, o.rec_G);
    d.rec_area = at<double>(b, o.rec_area);
    d.cnt = at<int32_t>(b, o.cnt);
    d.dep_off = at<int32_t>(b, o.dep_off);
    d.dep = at<int32_t>(b, o.dep);
    d.sched = at<int32_t>(b, o.sched);
    d.head = at<unsigned long long>(b, o.head);
    d.lam = h.lam;
    d.mu = h.mu;
    d.l2m = h.l2m;
    d.rho = h.rho;
    d.dt = h.dt;
    d.hdt2 = 0.5 * h.dt * h.dt;
    d.gamma = h.gamma;
    d.omg = 1.0 - h.gamma;
    d.t0 = h.t0;
    d.flags = ctx->flags;
    d.blk = p.blk;
    d.blk_ab = p.blk_ab;
    d.P = (int)p.sched.size();
    d.maxblk = p.maxblk;
    for (int g = 0; g < ST_COUNT; ++g) d.nblk[g] = p.nblk[g];
    d.rprev = h.any_dirichlet ? at<double>(b, o.rprev) : nullptr;
    d.wr_dof = at<double>(b, o.wr_dof);
    d.crit_list = at<int64_t>(b, o.crit_list);
    d.crit_surv = at<int32_t>(b, o.crit_surv);
    d.vhat = at<double>(b, o.vhat);
    d.edge_dirty = at<uint8_t>(b, o.edge_dirty);
    d.e_off = at<int32_t>(b, o.e_off);
    d.e_inc = at<int32_t>(b, o.e_inc);
    d.edge_own = at<uint8_t>(b, o.edge_own);
    d.wcnt = at<int32_t>(b, o.wcnt);
    d.wdep_off = at<int32_t>(b, o.wdep_off);
    d.wdep = at<int32_t>(b, o.wdep);
    d.wmax = ctx->w.maxblk;
    d.wstep = at<int64_t>(b, o.wstep);
    d.wncons = at<int32_t>(b, o.wncons);
    d.wcons_done = at<int32_t>(b, o.wcons_done);
    {
        const char *e = getenv("CEM_WAVE_DISCARD");
        d.wdiscard = (e ? atoi(e) : 0) != 0 && !ctx->w.ncons.empty();
    }
    ctx->epart = at<double>(b, o.epart);
    ctx->n_epart_edges = p.nblk[ST_AB];
    ctx->n_epart_nodes = (h.N + 255) / 256;
}

// Host -> device copies of the plan tables through two pinned staging halves (allocated once per
// process): the host copies chunk i+1 (OpenMP) while the DMA engine moves chunk i, instead of the
// driver's synchronous pageable staging.  Small copies go straight through.
struct Stager {
    static constexpr size_t kHalf = 16u << 20;
    std::mutex mu;
    char *buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int cur = 0;
    bool tried = false;
    bool ready() {
        if (!tried) {
            tried = true;
            for (int i = 0; i < 2; ++i)
                if (cudaHostAlloc(reinterpret_cast<void **>(&buf[i]), kHalf, cudaHostAllocPortable) != cudaSuccess ||
                    cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess) {
                    buf[0] = buf[1] = nullptr;
                    cudaGetLastError();
                    return false;
                }
        }
        return buf[0] && buf[1];
    }
    cudaError_t put(char *dst, const void *src, size_t bytes, cudaStream_t st) {
        if (bytes < (256u << 10) || !ready()) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
        const char *s = static_cast<const char *>(src);
        for (size_t done = 0; done < bytes;) {
            const size_t n = std::min(kHalf, bytes - done);
            cudaError_t e = cudaEventSynchronize(ev[cur]);  // the half's previous DMA has finished
            if (e != cudaSuccess) return e;
            char *d = buf[cur];
            const int64_t np = (int64_t)((n + (1u << 20) - 1) >> 20);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < np; ++i) {
                const size_t a = (size_t)i << 20, m = std::min<size_t>(1u << 20, n - a);
                std::memcpy(d + a, s + done + a, m);
            }
            e = cudaMemcpyAsync(dst + done, d, n, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) return e;
            e = cudaEventRecord(ev[cur], st);
            if (e != cudaSuccess) return e;
            cur ^= 1;
            done += n;
        }
        return cudaSuccess;
    }
};
// one Stager per device: its events are recorded on streams of that device only
Stager &stager(int device) {
    static std::mutex mu;
    static std::vector<Stager *> per_dev;  // process lifetime (pinned halves reused by the device's contexts)
    std::lock_guard<std::mutex> lock(mu);
    if (device < 0) device = 0;
    if ((size_t)device >= per_dev.size()) per_dev.resize(device + 1, nullptr);
    if (!per_dev[device]) per_dev[device] = new Stager();
    return *per_dev[device];
}

cem_status upload(cem_ctx *ctx, const Offs &o) {
    const HostMesh &h = ctx->h;
    const Plan &p = ctx->p;
    const int64_t N = h.N, E = h.E, S = h.S;
    void *b = ctx->ws;
    cudaStream_t st = ctx->stream;
    // node data in storage order; initial state (R17): u_0 = 0, v_0 = 0 / vbar(0),
    // a_0 = (f_ext - 0)/m / vbar'(0), frozen 0; u_1 = (u_0 + dt v_0) + (dt^2/2) a_0
    std::vector<double4> X4(N), f4(N), d4(h.any_dirichlet ? N : 1), z4(N, make_double4(0, 0, 0, 0)), v4(N), a4(N),
        u1(N);
    std::vector<uint8_t> nflag(N);
    std::vector<double> mass(N);
    const double dt = h.dt, hdt2 = 0.5 * h.dt * h.dt;
    for (int64_t kn = 0; kn < N; ++kn) {
        const int64_t n = p.node_new2old[kn];
        X4[kn] = make_double4(h.X[3 * n], h.X[3 * n + 1], h.X[3 * n + 2], 0.0);
        f4[kn] = make_double4(h.fext[3 * n], h.fext[3 * n + 1], h.fext[3 * n + 2], 0.0);
        if (h.any_dirichlet) d4[kn] = make_double4(h.dir_v0[3 * n], h.dir_v0[3 * n + 1], h.dir_v0[3 * n + 2], 0.0);
        nflag[kn] = h.nflag[n];
        mass[kn] = h.mass[n];
        double vv[3], aa[3], uu[3];
        for (int c = 0; c < 3; ++c) {
            const double mk = h.mass[n];
            if (mk == 0.0) {
                vv[c] = 0.0;
                aa[c] = 0.0;
            } else if (h.nflag[n] >> c & 1) {
                const double v0 = h.dir_v0[3 * n + c];
                if (h.t0 <= 0.0) {
                    vv[c] = v0;
                    aa[c] = 0.0;
                } else {
                    vv[c] = (0.0 / h.t0) * v0;
                    aa[c] = (0.0 < h.t0) ? v0 / h.t0 : 0.0;
                }
            } else {
                vv[c] = 0.0;
                aa[c] = (h.fext[3 * n + c] - 0.0) / mk;
            }
            uu[c] = (0.0 + dt * vv[c]) + hdt2 * aa[c];
        }
        v4[kn] = make_double4(vv[0], vv[1], vv[2], 0.0);
        a4[kn] = make_double4(aa[0], aa[1], aa[2], 0.0);
        u1[kn] = make_double4(uu[0], uu[1], uu[2], 0.0);
    }
    std::vector<int32_t> node_orig(p.node_new2old.begin(), p.node_new2old.end());
    Stager &sg = stager(ctx->device);
    std::lock_guard<std::mutex> lock(sg.mu);
    auto put = [&](size_t off, const void *src, size_t bytes) -> cudaError_t {
        return sg.put(at<char>(b, off), src, bytes, st);
    };
    CUDA_TRY(put(o.conn, p.conn.data(), sizeof(int32_t) * 4 * E));
    CUDA_TRY(put(o.geoT, p.geoT.data(), sizeof(double) * p.geoT.size()));
    CUDA_TRY(put(o.eedge, p.eedge.data(), sizeof(int32_t) * 6 * E));
    CUDA_TRY(put(o.incE, p.incE.data(), sizeof(uint16_t) * p.incE.size()));
    CUDA_TRY(put(o.nodeE, p.nodeE.data(), sizeof(int32_t) * p.nodeE.size()));
    CUDA_TRY(put(o.X, X4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.fext, f4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.nflag, nflag.data(), N));
    if (h.any_dirichlet) CUDA_TRY(put(o.dir_v0, d4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.gc, p.gc.data(), sizeof(double) * E));
    CUDA_TRY(put(o.tet_orig, p.tet_new2old.data(), sizeof(int32_t) * E));
    CUDA_TRY(put(o.node_orig, node_orig.data(), sizeof(int32_t) * N));
    CUDA_TRY(put(o.state, p.state.data(), E));
    CUDA_TRY(put(o.mass, mass.data(), sizeof(double) * N));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.dirty), 0, sizeof(int32_t) * N, st));
    CUDA_TRY(put(o.u0, z4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.u1, u1.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.v, v4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.a, a4.data(), sizeof(double4) * N));
    // energy ledger: support force at t = 0 of the prescribed dofs, R_0 = m a_0 - (f_ext - 0)
    // (f_int(u_0 = 0) = 0; oracle orc_create), reaction-work accumulators zeroed
    if (h.any_dirichlet) {
        std::vector<double> r0(3 * N, 0.0);
        for (int64_t kn = 0; kn < N; ++kn) {
            const int64_t n = p.node_new2old[kn];
            const double aa[3] = {a4[kn].x, a4[kn].y, a4[kn].z};
            for (int c = 0; c < 3; ++c)
                if (h.nflag[n] >> c & 1) r0[3 * kn + c] = h.mass[n] * aa[c] - (h.fext[3 * n + c] - 0.0);
        }
        CUDA_TRY(put(o.rprev, r0.data(), sizeof(double) * 3 * N));
    }
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.wr_dof), 0, sizeof(double) * (h.any_dirichlet ? 3 * N : 1), st));
    // Vhat_s = sum of V_e over the active incident tets in ascending original id (the oracle's
    // stage_edge order); kept in a table, recomputed by stage AB for edges marked dirty by a split
    {
        std::vector<double> vh(S, 0.0);
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < S; ++s) {
            double acc = 0.0;
            for (int32_t j = p.edge_off[s]; j < p.edge_off[s + 1]; ++j)
                if (p.state[p.edge_inc[j]]) acc = acc + p.geoV[p.edge_inc[j]];
            vh[s] = acc;
        }
        CUDA_TRY(put(o.vhat, vh.data(), sizeof(double) * S));
    }
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.edge_dirty), 0, S, st));
    CUDA_TRY(put(o.e_off, p.edge_off.data(), sizeof(int32_t) * (S + 1)));
    CUDA_TRY(put(o.e_inc, p.edge_inc.data(), sizeof(int32_t) * p.edge_inc.size()));
    // energy ledger ownership of an edge: the owner of its lowest-id incident tet (the first
    // entry of its incidence list; on one GPU every edge is owned).  Edges this rank owns are
    // edges of its layer-1 tets, whose incidences are complete locally.
    {
        std::vector<uint8_t> own(S, 1);
        for (int64_t s = 0; s < S; ++s)
            if (p.edge_off[s + 1] > p.edge_off[s]) own[s] = (p.tflag[p.edge_inc[p.edge_off[s]]] & 2) ? 1 : 0;
        CUDA_TRY(put(o.edge_own, own.data(), S));
    }
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.srec), 0, sizeof(double) * 4 * S, st));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.srec2), 0, sizeof(double) * 2 * S, st));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.fe), 0, sizeof(double) * CEM_FES * fe_slots(E), st));
    int32_t ctr[32] = {0, 0, INT32_MAX};
    CUDA_TRY(put(o.ctr, ctr, sizeof ctr));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.crit_list), 0, sizeof(int64_t) * E, st));  // stamp 0: no step's entry
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.cnt), 0, sizeof(int32_t) * ST_COUNT * p.maxblk, st));
    CUDA_TRY(put(o.dep_off, p.dep_off.data(), sizeof(int32_t) * p.dep_off.size()));
    CUDA_TRY(put(o.dep, p.dep.data(), sizeof(int32_t) * p.dep.size()));
    CUDA_TRY(put(o.nl_off, p.nl_off.data(), sizeof(int32_t) * p.nl_off.size()));
    CUDA_TRY(put(o.nl, p.nl.data(), sizeof(int32_t) * p.nl.size()));
    CUDA_TRY(put(o.lconn, p.lconn.data(), sizeof(uint16_t) * p.lconn.size()));
    CUDA_TRY(put(o.el_off, p.el_off.data(), sizeof(int32_t) * p.el_off.size()));
    CUDA_TRY(put(o.el, p.el.data(), sizeof(int32_t) * p.el.size()));
    CUDA_TRY(put(o.ledge, p.ledge.data(), sizeof(uint16_t) * p.ledge.size()));
    CUDA_TRY(put(o.tl_off, p.tl_off.data(), sizeof(int32_t) * p.tl_off.size()));
    CUDA_TRY(put(o.tl, p.tl.data(), sizeof(int32_t) * p.tl.size()));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.part), 0, sizeof(double) * 6 * p.nl.size(), st));
    CUDA_TRY(put(o.pinc_off, p.pinc_off.data(), sizeof(int32_t) * p.pinc_off.size()));
    CUDA_TRY(put(o.pinc, p.pinc.data(), sizeof(uint16_t) * p.pinc.size()));
    CUDA_TRY(put(o.poff, p.poff.data(), sizeof(int32_t) * p.poff.size()));
    CUDA_TRY(put(o.pdst, p.pdst.data(), sizeof(int32_t) * p.pdst.size()));
    CUDA_TRY(put(o.pord, p.pord.data(), sizeof(int32_t) * p.pord.size()));

    CUDA_TRY(put(o.sched, p.sched.data(), sizeof(int32_t) * p.sched.size()));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.head), 0, sizeof(unsigned long long), st));
    CUDA_TRY(put(o.ncons, p.ncons.data(), sizeof(int32_t) * p.ncons.size()));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.cons_done), 0, sizeof(int32_t) * ST_COUNT * p.maxblk, st));
    CUDA_TRY(put(o.nlb_off, p.nlb_off.data(), sizeof(int32_t) * p.nlb_off.size()));
    CUDA_TRY(put(o.nlb, p.nlb.data(), sizeof(int32_t) * p.nlb.size()));
    CUDA_TRY(put(o.tconn, p.tconn.data(), sizeof(uint16_t) * p.tconn.size()));
    CUDA_TRY(put(o.trow, p.trow.data(), sizeof(uint16_t) * p.trow.size()));
    CUDA_TRY(put(o.nrow, p.nrow.data(), sizeof(uint16_t) * p.nrow.size()));
    CUDA_TRY(put(o.tflag, p.tflag.data(), E));
    if (!ctx->w.dep.empty()) {
        CUDA_TRY(put(o.wdep_off, ctx->w.dep_off.data(), sizeof(int32_t) * ctx->w.dep_off.size()));
        CUDA_TRY(put(o.wdep, ctx->w.dep.data(), sizeof(int32_t) * ctx->w.dep.size()));
        CUDA_TRY(put(o.wncons, ctx->w.ncons.data(), sizeof(int32_t) * ctx->w.ncons.size()));
        CUDA_TRY(cudaMemsetAsync(at<char>(b, o.wcons_done), 0, sizeof(int32_t) * ctx->w.ncons.size(), st));
    }
    CUDA_TRY(put(o.self, &ctx->d, sizeof(Dev)));
    CUDA_TRY(cudaStreamSynchronize(st));
    return CEM_OK;
}

__global__ void k_fill(int32_t *p, int64_t n, int32_t v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// CEM_DEVICE readback (cem_get_state): storage-order device arrays -> the caller's device
// buffers in the caller's numbering ([n][3] for node vectors)
__global__ void k_export_vec(const double4 *__restrict__ src, const int32_t *__restrict__ node_orig, double *dst, int64_t N) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N) return;
    const double4 w = src[k];
    const int64_t o = 3 * (int64_t)node_orig[k];
    dst[o] = w.x;
    dst[o + 1] = w.y;
    dst[o + 2] = w.z;
}
__global__ void k_export_f64(const double *__restrict__ src, const int32_t *__restrict__ orig, double *dst, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[orig[i]] = src[i];
}
__global__ void k_export_u8(const uint8_t *__restrict__ src, const int32_t *__restrict__ orig, uint8_t *dst, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[orig[i]] = src[i];
}


// ---------------------------------------------------------------- multi-GPU helpers
struct LocalMesh {
    std::vector<double> X, tface_t, vbc_v0, f_nodal;
    std::vector<int32_t> tets, tface, vbc_node;
    std::vector<uint8_t> state, vbc_mask;
    std::vector<double> gc;
};

// the rank's sub-mesh in local numbering (ascending global id, so sums keep the global order)
void extract_local(const cem_mesh_in *m, const cem_material *mat, const cem_load_in *ld, const PartLocal &L,
                   LocalMesh &lm) {
    const int64_t El = L.tet_global.size(), Nl = L.node_global.size();
    std::vector<int32_t> g2l(m->n_nodes, -1);
    for (int64_t i = 0; i < Nl; ++i) g2l[L.node_global[i]] = (int32_t)i;
    lm.X.resize(3 * Nl);
    for (int64_t i = 0; i < Nl; ++i)
        for (int c = 0; c < 3; ++c) lm.X[3 * i + c] = m->X[3 * (int64_t)L.node_global[i] + c];
    lm.tets.resize(4 * El);
    lm.state.resize(El);
    lm.gc.resize(El);
    for (int64_t i = 0; i < El; ++i) {
        const int64_t e = L.tet_global[i];
        for (int a = 0; a < 4; ++a) lm.tets[4 * i + a] = g2l[m->tets[4 * e + a]];
        lm.state[i] = m->tet_state ? m->tet_state[e] : 1;
        lm.gc[i] = m->tet_gc ? m->tet_gc[e] : mat->Gc;
    }
    if (ld)
        for (int64_t f = 0; f < ld->n_tfaces; ++f) {
            const int32_t *t = ld->tface + 3 * f;
            if (g2l[t[0]] < 0 || g2l[t[1]] < 0 || g2l[t[2]] < 0) continue;
            for (int i = 0; i < 3; ++i) {
                lm.tface.push_back(g2l[t[i]]);
                lm.tface_t.push_back(ld->tface_t[3 * f + i]);
            }
        }
    if (ld && ld->f_nodal) {
        lm.f_nodal.resize(3 * Nl);
        for (int64_t i = 0; i < Nl; ++i)
            for (int c = 0; c < 3; ++c) lm.f_nodal[3 * i + c] = ld->f_nodal[3 * (int64_t)L.node_global[i] + c];
    }
    if (ld)
        for (int64_t b = 0; b < ld->n_vbc; ++b) {
            if (g2l[ld->vbc_node[b]] < 0) continue;
            lm.vbc_node.push_back(g2l[ld->vbc_node[b]]);
            lm.vbc_mask.push_back(ld->vbc_mask[b]);
            for (int c = 0; c < 3; ++c) lm.vbc_v0.push_back(ld->vbc_v0[3 * b + c]);
        }
}

cem_status setup_exchange(cem_ctx *ctx) {
    const PartLocal &L = ctx->part;
    const Plan &p = ctx->p;
    Exchange &x = ctx->xch;
    x.peers = L.peers;
    const size_t np = L.peers.size();
    x.send_off.assign(np + 1, 0);
    x.recv_off.assign(np + 1, 0);
    std::vector<int32_t> sn, st, rn, rt;
    std::vector<int64_t> sndst, stdst, rnsrc, rtsrc;
    auto pad8 = [](size_t v) { return (v + 7) & ~size_t(7); };
    for (size_t j = 0; j < np; ++j) {
        size_t off = x.send_off[j];
        for (int32_t k : L.send_nodes[j]) {
            sn.push_back(p.node_old2new[k]);
            sndst.push_back((int64_t)off);
            off += 24;
        }
        for (int32_t e : L.send_tets[j]) {
            st.push_back(p.tet_old2new[e]);
            stdst.push_back((int64_t)off);
            off += 1;
        }
        x.send_off[j + 1] = pad8(off);
        off = x.recv_off[j];
        for (int32_t k : L.recv_nodes[j]) {
            rn.push_back(p.node_old2new[k]);
            rnsrc.push_back((int64_t)off);
            off += 24;
        }
        for (int32_t e : L.recv_tets[j]) {
            rt.push_back(p.tet_old2new[e]);
            rtsrc.push_back((int64_t)off);
            off += 1;
        }
        x.recv_off[j + 1] = pad8(off);
    }
    x.n_send_nodes = sn.size();
    x.n_send_tets = st.size();
    x.n_recv_nodes = rn.size();
    x.n_recv_tets = rt.size();
    auto dev = [&](const void *src, size_t bytes, void **dst) -> cudaError_t {
        cudaError_t e = cudaMalloc(dst, bytes ? bytes : 8);
        if (e != cudaSuccess) return e;
        ctx->dist_allocs.push_back(*dst);
        if (bytes && src) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
        return e;
    };
    CUDA_TRY(dev(sn.data(), 4 * sn.size(), (void **)&x.d_send_nodes));
    CUDA_TRY(dev(st.data(), 4 * st.size(), (void **)&x.d_send_tets));
    CUDA_TRY(dev(rn.data(), 4 * rn.size(), (void **)&x.d_recv_nodes));
    CUDA_TRY(dev(rt.data(), 4 * rt.size(), (void **)&x.d_recv_tets));
    CUDA_TRY(dev(sndst.data(), 8 * sndst.size(), (void **)&x.d_send_ndst));
    CUDA_TRY(dev(stdst.data(), 8 * stdst.size(), (void **)&x.d_send_tdst));
    CUDA_TRY(dev(rnsrc.data(), 8 * rnsrc.size(), (void **)&x.d_recv_nsrc));
    CUDA_TRY(dev(rtsrc.data(), 8 * rtsrc.size(), (void **)&x.d_recv_tsrc));
    CUDA_TRY(dev(nullptr, x.send_off[np], (void **)&x.d_sendbuf));
    CUDA_TRY(dev(nullptr, x.recv_off[np], (void **)&x.d_recvbuf));
    return CEM_OK;
}

// exchange after a step whose predicted displacement sits in ubuf[parity]
cem_status exchange_nccl_step(cem_ctx *ctx, int parity) {
    exchange_pack(ctx->xch, ctx->d.ubuf[parity], ctx->d.state, ctx->stream);
    if (!exchange_nccl(ctx->xch, ctx->comm, ctx->stream, ctx->err)) return CEM_ENCCL;
    exchange_unpack(ctx->xch, ctx->d.ubuf[parity], ctx->d.state, ctx->d.eedge, ctx->h.E, ctx->d.edge_dirty, ctx->stream);
    ctx->launches += 2;
    return CEM_OK;
}

// ---------------------------------------------------------------- P2P halo
// Tables of this rank's stores into the peers' receive buffers: peer j's buffer for step parity
// par is peer_recv[par][j] (already offset to the segment the peer keeps for this rank); a node
// record sits at 24 i in the segment (i-th send node), a tet state byte after the node records.
cem_status p2p_tables(cem_ctx *ctx, const std::vector<uint8_t *> &r0, const std::vector<uint8_t *> &r1,
                      const std::vector<int64_t *> &flag_addr) {
    const PartLocal &L = ctx->part;
    const Plan &p = ctx->p;
    P2P &q = ctx->p2p;
    const int np = (int)L.peers.size();
    const int64_t N = ctx->h.N, E = ctx->h.E;
    std::vector<std::vector<std::pair<int32_t, int32_t>>> ne(N), te(E);
    for (int j = 0; j < np; ++j) {
        const auto &sn = L.send_nodes[j], &stt = L.send_tets[j];
        for (size_t i = 0; i < sn.size(); ++i) ne[p.node_old2new[sn[i]]].push_back({j, (int32_t)(24 * i)});
        for (size_t i = 0; i < stt.size(); ++i)
            te[p.tet_old2new[stt[i]]].push_back({j, (int32_t)(24 * sn.size() + i)});
    }
    auto csr = [](const std::vector<std::vector<std::pair<int32_t, int32_t>>> &v, std::vector<int32_t> &off,
                  std::vector<int32_t> &peer, std::vector<int32_t> &byte) {
        off.assign(v.size() + 1, 0);
        for (size_t k = 0; k < v.size(); ++k) {
            off[k + 1] = off[k] + (int32_t)v[k].size();
            for (auto &e : v[k]) {
                peer.push_back(e.first);
                byte.push_back(e.second);
            }
        }
    };
    std::vector<int32_t> noff, npeer, nbyte, toff, tpeer, tbyte;
    csr(ne, noff, npeer, nbyte);
    csr(te, toff, tpeer, tbyte);
    std::vector<uint8_t *> pr(2 * np);
    std::vector<int32_t> prank(np);
    for (int j = 0; j < np; ++j) {
        pr[j] = r0[j];
        pr[np + j] = r1[j];
        prank[j] = L.peers[j];
    }
    auto dev = [&](const void *src, size_t bytes, void **dst) -> cudaError_t {
        cudaError_t e = cudaMalloc(dst, bytes ? bytes : 8);
        if (e != cudaSuccess) return e;
        ctx->dist_allocs.push_back(*dst);
        if (bytes && src) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
        return e;
    };
    CUDA_TRY(dev(pr.data(), sizeof(uint8_t *) * pr.size(), (void **)&q.d_peer_recv));
    CUDA_TRY(dev(flag_addr.data(), sizeof(int64_t *) * flag_addr.size(), (void **)&q.d_peer_flag));
    CUDA_TRY(dev(prank.data(), 4 * prank.size(), (void **)&q.d_peer_rank));
    CUDA_TRY(dev(noff.data(), 4 * noff.size(), (void **)&q.d_noff));
    CUDA_TRY(dev(npeer.data(), 4 * npeer.size(), (void **)&q.d_npeer));
    CUDA_TRY(dev(nbyte.data(), 4 * nbyte.size(), (void **)&q.d_nbyte));
    CUDA_TRY(dev(toff.data(), 4 * toff.size(), (void **)&q.d_toff));
    CUDA_TRY(dev(tpeer.data(), 4 * tpeer.size(), (void **)&q.d_tpeer));
    CUDA_TRY(dev(tbyte.data(), 4 * tbyte.size(), (void **)&q.d_tbyte));
    return CEM_OK;
}

// this rank's receive buffers for the P2P halo, initialised from the exchanged state
cem_status p2p_alloc(cem_ctx *ctx) {
    P2P &q = ctx->p2p;
    const size_t bytes = std::max<size_t>(8, ctx->xch.recv_off.back());
    for (int par = 0; par < 2; ++par) {
        CUDA_TRY(cudaMalloc(&q.recv[par], bytes));
        ctx->dist_allocs.push_back(q.recv[par]);
        CUDA_TRY(cudaMemcpy(q.recv[par], ctx->xch.d_recvbuf, bytes, cudaMemcpyDeviceToDevice));
    }
    CUDA_TRY(cudaMalloc(&q.flags, sizeof(int64_t) * (std::max(1, ctx->nranks) + 1)));
    ctx->dist_allocs.push_back(q.flags);
    CUDA_TRY(cudaMemset(q.flags, 0, sizeof(int64_t) * (std::max(1, ctx->nranks) + 1)));
    q.timeout = q.flags + std::max(1, ctx->nranks);
    return CEM_OK;
}

void p2p_enable(cem_ctx *ctx) {
    P2P &q = ctx->p2p;
    Dev &d = ctx->d;
    d.p2p_recv = q.d_peer_recv;
    d.p2p_np = (int)ctx->part.peers.size();
    d.p2p_noff = q.d_noff;
    d.p2p_npeer = q.d_npeer;
    d.p2p_nbyte = q.d_nbyte;
    d.p2p_toff = q.d_toff;
    d.p2p_tpeer = q.d_tpeer;
    d.p2p_tbyte = q.d_tbyte;
    d.p2p_flag_out = q.d_peer_flag;
    // stage-D block order for the early signal: blocks holding a node some peer receives first
    // (CEM_P2P_EARLY=0 keeps the plain order and signals after the whole stage)
    const char *ee = getenv("CEM_P2P_EARLY");
    if (!(ee && atoi(ee) == 0) && d.p2p_np > 0) {
        const int64_t per = std::max(1, ctx->p.blk / 4), nD = (ctx->h.N + per - 1) / per;
        std::vector<uint8_t> hasp(nD, 0);
        for (const auto &sn : ctx->part.send_nodes)
            for (int32_t k : sn) hasp[ctx->p.node_old2new[k] / per] = 1;
        std::vector<int32_t> order;
        order.reserve(nD);
        for (int64_t b = 0; b < nD; ++b)
            if (hasp[b]) order.push_back((int32_t)b);
        const int nb = (int)order.size();
        for (int64_t b = 0; b < nD; ++b)
            if (!hasp[b]) order.push_back((int32_t)b);
        void *dord = nullptr, *dcnt = nullptr;
        if (cudaMalloc(&dord, 4 * order.size()) == cudaSuccess && cudaMalloc(&dcnt, 8) == cudaSuccess &&
            cudaMemcpy(dord, order.data(), 4 * order.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMemset(dcnt, 0, 8) == cudaSuccess) {
            ctx->dist_allocs.push_back(dord);
            ctx->dist_allocs.push_back(dcnt);
            d.d_order = static_cast<const int32_t *>(dord);
            d.d_nbound = nb;
            d.bdone = static_cast<unsigned long long *>(dcnt);
            ctx->sy.bdone = 0;
        } else {
            if (dord) cudaFree(dord);
            if (dcnt) cudaFree(dcnt);
            cudaGetLastError();
        }
    }
    q.on = true;
}

// Real multi-GPU: the receive buffers and flags are exported with CUDA IPC, the handles and the
// segment offsets all-gathered over NCCL, the peers' allocations mapped (peer access over
// NVLink).  Self-check before use: u_1 pushed through the P2P path must equal what the NCCL
// exchange delivered, on every rank; otherwise the halo stays on NCCL.
struct P2PBlob {
    cudaIpcMemHandle_t recv0, recv1, flags;
    int64_t seg_off_by_src[64];
};
cem_status p2p_setup_nccl(cem_ctx *ctx) {
    // every rank takes part in every collective below, whatever its own outcome (a rank that
    // returned early would leave the others waiting); the verdicts are all-reduced
    const int R = ctx->nranks, me = ctx->rank;
    const PartLocal &L = ctx->part;
    const int np = (int)L.peers.size();
    P2P &q = ctx->p2p;
    int64_t *dflag = nullptr;
    CUDA_TRY(cudaMalloc(&dflag, 2 * sizeof(int64_t)));
    ctx->dist_allocs.push_back(dflag);
    auto all_ok = [&](bool ok, bool &out) -> cem_status {  // logical AND over the ranks
        const int64_t notok = ok ? 0 : 1;
        CUDA_TRY(cudaMemcpy(dflag, &notok, sizeof(int64_t), cudaMemcpyHostToDevice));
        if (!nccl_allreduce_max_i64(dflag, dflag + 1, 1, ctx->comm, ctx->stream, ctx->err)) return CEM_ENCCL;
        int64_t any = 1;
        CUDA_TRY(cudaMemcpyAsync(&any, dflag + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        out = any == 0;
        return CEM_OK;
    };
    bool ok = R <= 64;
    if (ok && p2p_alloc(ctx) != CEM_OK) ok = false;
    P2PBlob mine{};
    for (int i = 0; i < 64; ++i) mine.seg_off_by_src[i] = -1;
    if (ok) {
        for (int j = 0; j < np; ++j) mine.seg_off_by_src[L.peers[j]] = (int64_t)ctx->xch.recv_off[j];
        if (cudaIpcGetMemHandle(&mine.recv0, q.recv[0]) != cudaSuccess ||
            cudaIpcGetMemHandle(&mine.recv1, q.recv[1]) != cudaSuccess ||
            cudaIpcGetMemHandle(&mine.flags, q.flags) != cudaSuccess)
            ok = false;
    }
    cudaGetLastError();
    bool every = false;
    cem_status st = all_ok(ok, every);
    if (st || !every) return st;
    void *dsend = nullptr, *drecv = nullptr;
    CUDA_TRY(cudaMalloc(&dsend, sizeof(P2PBlob)));
    CUDA_TRY(cudaMalloc(&drecv, sizeof(P2PBlob) * R));
    ctx->dist_allocs.push_back(dsend);
    ctx->dist_allocs.push_back(drecv);
    CUDA_TRY(cudaMemcpy(dsend, &mine, sizeof(P2PBlob), cudaMemcpyHostToDevice));
    if (!nccl_allgather_bytes(dsend, drecv, sizeof(P2PBlob), ctx->comm, ctx->stream, ctx->err)) return CEM_ENCCL;
    std::vector<P2PBlob> all(R);
    CUDA_TRY(cudaMemcpyAsync(all.data(), drecv, sizeof(P2PBlob) * R, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    std::vector<uint8_t *> r0(np), r1(np);
    std::vector<int64_t *> fl(np);
    for (int j = 0; j < np && ok; ++j) {
        const P2PBlob &b = all[L.peers[j]];
        void *a0 = nullptr, *a1 = nullptr, *af = nullptr;
        if (b.seg_off_by_src[me] < 0 ||
            cudaIpcOpenMemHandle(&a0, b.recv0, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
            cudaIpcOpenMemHandle(&a1, b.recv1, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
            cudaIpcOpenMemHandle(&af, b.flags, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            ok = false;
            break;
        }
        q.opened.push_back(a0);
        q.opened.push_back(a1);
        q.opened.push_back(af);
        r0[j] = static_cast<uint8_t *>(a0) + b.seg_off_by_src[me];
        r1[j] = static_cast<uint8_t *>(a1) + b.seg_off_by_src[me];
        fl[j] = static_cast<int64_t *>(af) + me;
    }
    cudaGetLastError();
    if (ok && p2p_tables(ctx, r0, r1, fl) != CEM_OK) ok = false;
    st = all_ok(ok, every);  // every rank can store into its peers: run the self-check together
    if (st || !every) return st;
    // self-check: poison buffer 1, push u_1 into the peers' buffers[1], sync, compare with the
    // NCCL delivery, then restore the buffer (its state bytes) from that delivery
    const size_t rbytes = std::max<size_t>(8, ctx->xch.recv_off.back());
    CUDA_TRY(cudaMemsetAsync(q.recv[1], 0xff, rbytes, ctx->stream));
    st = all_ok(true, every);  // every buffer poisoned before anybody pushes
    if (st) return st;
    p2p_push_nodes(q, ctx->d.ubuf[1], ctx->h.N, 1, np, ctx->stream);
    p2p_sync(q, np, 1, true, ctx->stream);
    CUDA_TRY(cudaMemsetAsync(dflag, 0, sizeof(int64_t), ctx->stream));
    count_mismatch(q.recv[1], ctx->xch.d_recvbuf, ctx->xch.d_recv_nsrc, ctx->xch.n_recv_nodes, 24, dflag, ctx->stream);
    int64_t bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, dflag, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(q.recv[1], ctx->xch.d_recvbuf, rbytes, cudaMemcpyDeviceToDevice, ctx->stream));
    st = all_ok(bad == 0, every);
    if (st || !every) return st;
    p2p_enable(ctx);
    CUDA_TRY(cudaMemcpy(const_cast<Dev *>(ctx->d.self), &ctx->d, sizeof(Dev), cudaMemcpyHostToDevice));
    return CEM_OK;
}

// Host-ordered CUDA-IPC halo (opts.host_allgather, no NCCL): the IPC handles and segment offsets
// are all-gathered through the caller's host callback, the peers' receive buffers mapped, and the
// initial halo (u_1 and the tet states) copied into them; every step the ranks then meet on the
// host after their stores completed (cem_step), so the device flag wait never spins.
cem_status host_barrier(cem_ctx *ctx) {
    std::vector<char> all(ctx->nranks);
    const char me = 1;
    if (ctx->host_allgather(&me, all.data(), 1, ctx->host_user) != 0) {
        ctx->err = "host_allgather callback failed";
        return CEM_ENCCL;
    }
    return CEM_OK;
}
cem_status p2p_setup_host(cem_ctx *ctx) {
    const int R = ctx->nranks, me = ctx->rank;
    const PartLocal &L = ctx->part;
    const int np = (int)L.peers.size();
    P2P &q = ctx->p2p;
    if (R > 64) {
        ctx->err = "host-ordered IPC halo: at most 64 ranks";
        return CEM_EINVAL;
    }
    cem_status st = p2p_alloc(ctx);
    if (st) return st;
    P2PBlob mine{};
    for (int i = 0; i < 64; ++i) mine.seg_off_by_src[i] = -1;
    for (int j = 0; j < np; ++j) mine.seg_off_by_src[L.peers[j]] = (int64_t)ctx->xch.recv_off[j];
    CUDA_TRY(cudaIpcGetMemHandle(&mine.recv0, q.recv[0]));
    CUDA_TRY(cudaIpcGetMemHandle(&mine.recv1, q.recv[1]));
    CUDA_TRY(cudaIpcGetMemHandle(&mine.flags, q.flags));
    std::vector<P2PBlob> all(R);
    if (ctx->host_allgather(&mine, all.data(), sizeof(P2PBlob), ctx->host_user) != 0) {
        ctx->err = "host_allgather callback failed";
        return CEM_ENCCL;
    }
    std::vector<uint8_t *> r0(np), r1(np);
    std::vector<int64_t *> fl(np);
    for (int j = 0; j < np; ++j) {
        const P2PBlob &b = all[L.peers[j]];
        if (b.seg_off_by_src[me] < 0) {
            ctx->err = "host-ordered IPC halo: a peer has no segment for this rank";
            return CEM_ESTATE;
        }
        void *a0 = nullptr, *a1 = nullptr, *af = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&a0, b.recv0, cudaIpcMemLazyEnablePeerAccess));
        q.opened.push_back(a0);
        CUDA_TRY(cudaIpcOpenMemHandle(&a1, b.recv1, cudaIpcMemLazyEnablePeerAccess));
        q.opened.push_back(a1);
        CUDA_TRY(cudaIpcOpenMemHandle(&af, b.flags, cudaIpcMemLazyEnablePeerAccess));
        q.opened.push_back(af);
        r0[j] = static_cast<uint8_t *>(a0) + b.seg_off_by_src[me];
        r1[j] = static_cast<uint8_t *>(a1) + b.seg_off_by_src[me];
        fl[j] = static_cast<int64_t *>(af) + me;
    }
    st = p2p_tables(ctx, r0, r1, fl);
    if (st) return st;
    // initial halo: the owners' u_1 and tet states into both parity buffers of every peer
    exchange_pack(ctx->xch, ctx->d.ubuf[1], ctx->d.state, ctx->stream);
    for (int j = 0; j < np; ++j) {
        const size_t bytes = ctx->xch.send_off[j + 1] - ctx->xch.send_off[j];
        if (!bytes) continue;
        CUDA_TRY(cudaMemcpyAsync(r0[j], ctx->xch.d_sendbuf + ctx->xch.send_off[j], bytes, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(r1[j], ctx->xch.d_sendbuf + ctx->xch.send_off[j], bytes, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    st = host_barrier(ctx);  // every rank's copies into this rank's buffers are complete
    if (st) return st;
    exchange_unpack(ctx->xch, ctx->d.ubuf[1], ctx->d.state, ctx->d.eedge, ctx->h.E, ctx->d.edge_dirty, ctx->stream,
                    q.recv[1]);
    ctx->launches += 2;
    p2p_enable(ctx);
    CUDA_TRY(cudaMemcpy(const_cast<Dev *>(ctx->d.self), &ctx->d, sizeof(Dev), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return CEM_OK;
}

// Loopback emulation (tests, one device): the peers' buffers are the other contexts' own.
cem_status p2p_setup_loopback(cem_ctx **c, int n) {
    for (int r = 0; r < n; ++r) {
        cem_ctx *ctx = c[r];
        cem_status st = p2p_alloc(ctx);
        if (st) return st;
    }
    for (int r = 0; r < n; ++r) {
        cem_ctx *ctx = c[r];
        const PartLocal &L = ctx->part;
        const int np = (int)L.peers.size();
        std::vector<uint8_t *> r0(np), r1(np);
        std::vector<int64_t *> fl(np);
        for (int j = 0; j < np; ++j) {
            cem_ctx *pc = c[L.peers[j]];
            size_t off = 0;
            for (size_t i = 0; i < pc->part.peers.size(); ++i)
                if (pc->part.peers[i] == r) off = pc->xch.recv_off[i];
            r0[j] = pc->p2p.recv[0] + off;
            r1[j] = pc->p2p.recv[1] + off;
            fl[j] = pc->p2p.flags + r;
        }
        cem_status st = p2p_tables(ctx, r0, r1, fl);
        if (st) return st;
        p2p_enable(ctx);
        CUDA_TRY(cudaMemcpy(const_cast<Dev *>(ctx->d.self), &ctx->d, sizeof(Dev), cudaMemcpyHostToDevice));
    }
    return CEM_OK;
}

// loopback: all ranks in this process, transport = device copies on ctxs[0]'s stream
cem_status exchange_loopback(cem_ctx **c, int n, int parity) {
    cudaStream_t st = c[0]->stream;
    for (int r = 0; r < n; ++r) exchange_pack(c[r]->xch, c[r]->d.ubuf[parity], c[r]->d.state, st);
    for (int r = 0; r < n; ++r) {
        const Exchange &xs = c[r]->xch;
        for (size_t j = 0; j < xs.peers.size(); ++j) {
            const int q = xs.peers[j];
            const Exchange &xq = c[q]->xch;
            size_t jq = 0;
            while (jq < xq.peers.size() && xq.peers[jq] != r) ++jq;
            const size_t bytes = xs.send_off[j + 1] - xs.send_off[j];
            if (jq == xq.peers.size() || bytes != xq.recv_off[jq + 1] - xq.recv_off[jq]) {
                c[r]->err = "loopback exchange lists do not match";
                return CEM_ESTATE;
            }
            if (bytes &&
                cudaMemcpyAsync(xq.d_recvbuf + xq.recv_off[jq], xs.d_sendbuf + xs.send_off[j], bytes,
                                cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
                c[r]->err = "loopback copy failed";
                return CEM_ECUDA;
            }
        }
    }
    for (int r = 0; r < n; ++r)
        exchange_unpack(c[r]->xch, c[r]->d.ubuf[parity], c[r]->d.state, c[r]->d.eedge, c[r]->h.E, c[r]->d.edge_dirty, st);
    for (int r = 0; r < n; ++r) c[r]->launches += 2;
    return CEM_OK;
}

void fill_part_out(const PartGlobal &g, const PartLocal &L, cem_part_out *o) {
    auto dup32 = [](const std::vector<int32_t> &v) {
        int32_t *p = (int32_t *)malloc(sizeof(int32_t) * (v.size() ? v.size() : 1));
        if (!v.empty()) std::memcpy(p, v.data(), sizeof(int32_t) * v.size());
        return p;
    };
    auto dup8 = [](const std::vector<uint8_t> &v) {
        uint8_t *p = (uint8_t *)malloc(v.size() ? v.size() : 1);
        if (!v.empty()) std::memcpy(p, v.data(), v.size());
        return p;
    };
    auto csr = [&](const std::vector<std::vector<int32_t>> &lists, int64_t **off, int32_t **flat) {
        std::vector<int32_t> f;
        *off = (int64_t *)malloc(sizeof(int64_t) * (lists.size() + 1));
        (*off)[0] = 0;
        for (size_t j = 0; j < lists.size(); ++j) {
            f.insert(f.end(), lists[j].begin(), lists[j].end());
            (*off)[j + 1] = (int64_t)f.size();
        }
        *flat = dup32(f);
    };
    o->n_tets = L.tet_global.size();
    o->n_nodes = L.node_global.size();
    o->tet_global = dup32(L.tet_global);
    o->tet_flag = dup8(L.tet_flag);
    o->node_global = dup32(L.node_global);
    o->node_owned = dup8(L.node_owned);
    o->n_peers = (int32_t)L.peers.size();
    o->peers = dup32(std::vector<int32_t>(L.peers.begin(), L.peers.end()));
    csr(L.send_nodes, &o->send_node_off, &o->send_nodes);
    csr(L.recv_nodes, &o->recv_node_off, &o->recv_nodes);
    csr(L.send_tets, &o->send_tet_off, &o->send_tets);
    csr(L.recv_tets, &o->recv_tet_off, &o->recv_tets);
    o->tet_owner = dup32(g.tet_owner);
    o->node_owner = dup32(g.node_owner);
}

// ---------------------------------------------------------------- hexahedral contexts (N3)
struct HexOffs {
    size_t hgeo, hconn, heedge, htau, e_off, e_inc, hpair, hrem, htact, htloc, hnrem, hediag, hdlist, hclist, heinc4, htgeo, httau, gc, X, rec_step, rec_elem,
        rec_cand, rec_G, rec_area, nodeE, fext, nflag, dir_v0, state, mass, dirty, u0, u1, v, a,
        srec, srec2, fe, ctr, rprev, wr_dof, node_orig, tet_orig, self, epart, total;
};
HexOffs hex_layout(const HexHost &h) {
    Layout L;
    HexOffs o{};
    const int64_t N = h.N, E = h.E, S = h.S;
    o.hgeo = L.take<double>(25 * E);
    o.hconn = L.take<int32_t>(8 * E);
    o.heedge = L.take<int32_t>(12 * E);
    o.htau = L.take<double>(6 * E);
    o.e_off = L.take<int32_t>(S + 1);
    o.e_inc = L.take<int32_t>((int64_t)h.edge_inc.size());
    o.hpair = L.take<int32_t>(28 * E);
    o.hrem = L.take<int8_t>(E);
    o.htact = L.take<uint8_t>(E);
    o.hnrem = L.take<uint8_t>(N);
    o.hediag = L.take<uint32_t>((S - h.S_h + 31) / 32 + 1);
    o.hdlist = L.take<int32_t>(S - h.S_h);
    o.hclist = L.take<int32_t>(E);
    o.heinc4 = L.take<int4>(S);
    o.htloc = L.take<uint8_t>(12 * E);
    o.htgeo = L.take<double>(39 * E);
    o.httau = L.take<double>(18 * E);
    o.gc = L.take<double>(E);
    o.X = L.take<double4>(N);
    o.rec_step = L.take<int64_t>(4 * E);
    o.rec_elem = L.take<int32_t>(4 * E);
    o.rec_cand = L.take<int32_t>(4 * E);
    o.rec_G = L.take<double>(4 * E);
    o.rec_area = L.take<double>(4 * E);
    o.nodeE = L.take<int32_t>((int64_t)h.nodeE.size());
    o.fext = L.take<double4>(N);
    o.nflag = L.take<uint8_t>(N);
    o.dir_v0 = L.take<double4>(h.any_dirichlet ? N : 1);
    o.state = L.take<uint8_t>(E);
    o.mass = L.take<double>(N);
    o.dirty = L.take<int32_t>(N);
    o.u0 = L.take<double4>(N);
    o.u1 = L.take<double4>(N);
    o.v = L.take<double4>(N);
    o.a = L.take<double4>(N);
    o.srec = L.take<double>(4 * S);
    o.srec2 = L.take<double>(2 * S);
    o.fe = L.take<double>(3 * (32 * E + 1));
    o.ctr = L.take<int32_t>(32);
    o.rprev = L.take<double>(h.any_dirichlet ? 3 * N : 1);
    o.wr_dof = L.take<double>(h.any_dirichlet ? 3 * N : 1);
    o.node_orig = L.take<int32_t>(N);
    o.tet_orig = L.take<int32_t>(E);
    o.self = L.take<Dev>(1);
    o.epart = L.take<double>((S + 255) / 256 + 3 * ((N + 255) / 256));
    o.total = L.off;
    return o;
}

// allocate the device workspace as cem_init_mesh does (caller buffer, allocation callback or cudaMalloc)
cem_status alloc_workspace(cem_ctx *ctx, const cem_opts *opts, size_t total) {
    if (opts && opts->workspace) {
        if (opts->workspace_bytes < total) {
            ctx->err = "workspace too small: need " + std::to_string(total) + " bytes";
            return CEM_ENOMEM;
        }
        ctx->ws = opts->workspace;
        ctx->ws_bytes = opts->workspace_bytes;
    } else if (opts && opts->dev_alloc) {
        if (opts->dev_alloc(total, opts->alloc_user, &ctx->ws) != 0 || !ctx->ws) {
            ctx->err = "dev_alloc callback failed for " + std::to_string(total) + " bytes";
            return CEM_ENOMEM;
        }
        ctx->ws_bytes = total;
    } else {
        cudaError_t e = cudaMalloc(&ctx->ws, total);
        if (e != cudaSuccess) {
            ctx->err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
            ctx->ws = nullptr;
            return CEM_ENOMEM;
        }
        ctx->own_ws = true;
        ctx->ws_bytes = total;
    }
    return CEM_OK;
}

cem_status hex_init(const cem_mesh_in *mesh, const cem_material *mat, const cem_load_in *load, const cem_opts *opts,
                    cem_ctx **out) {
    cem_ctx *ctx = new cem_ctx();
    auto fail = [&](cem_status s) {
        g_init_err = ctx->err;
        if (ctx->own_ws && ctx->ws) cudaFree(ctx->ws);
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        if (ctx->fence_in) cudaEventDestroy(ctx->fence_in);
        if (ctx->fence_out) cudaEventDestroy(ctx->fence_out);
        delete ctx;
        return s;
    };
    if (opts && opts->nranks > 1) {
        ctx->err = "hexahedral meshes run on one GPU (nranks = 1)";
        return fail(CEM_EINVAL);
    }
    HexHost h;
    cem_status st = build_hex_host(mesh, mat, load, opts, h, ctx->err);
    if (st) return fail(st);
    ctx->hexa = true;
    ctx->device = opts ? opts->device : 0;
    ctx->flags = opts ? opts->flags : 0;
    ctx->user_stream = opts ? (cudaStream_t)opts->stream : nullptr;
    if (cudaSetDevice(ctx->device) != cudaSuccess) {
        ctx->err = "cudaSetDevice failed (no CUDA device?)";
        return fail(CEM_ECUDA);
    }
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->fence_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->fence_out, cudaEventDisableTiming) != cudaSuccess) {
        ctx->err = "cudaStreamCreate / cudaEventCreate failed";
        return fail(CEM_ECUDA);
    }
    ctx->own_stream = true;
    cudaEventRecord(ctx->fence_in, ctx->user_stream);
    cudaStreamWaitEvent(ctx->stream, ctx->fence_in, 0);
    const int64_t N = h.N, E = h.E, S = h.S;
    // the host views cem_get_state uses (identity numbering: no storage reordering for hexes)
    ctx->h.N = N;
    ctx->h.E = E;
    ctx->h.S = S;
    ctx->h.dt = h.dt;
    ctx->h.gc = h.gc;  // [4E]: records of remainder tets E + 3e + i carry their parent's Gc
    ctx->p.node_new2old.resize(N);
    std::iota(ctx->p.node_new2old.begin(), ctx->p.node_new2old.end(), 0);
    ctx->p.tet_new2old.resize(E);
    std::iota(ctx->p.tet_new2old.begin(), ctx->p.tet_new2old.end(), 0);
    const HexOffs o = hex_layout(h);
    st = alloc_workspace(ctx, opts, o.total);
    if (st) return fail(st);
    void *b = ctx->ws;
    Dev &d = ctx->d;
    d = Dev{};
    d.N = N;
    d.E = E;
    d.S = S;
    d.npe = 8;
    d.hgeo = at<double>(b, o.hgeo);
    d.hconn = at<int32_t>(b, o.hconn);
    d.heedge = at<int32_t>(b, o.heedge);
    d.htau = at<double>(b, o.htau);
    d.e_off = at<int32_t>(b, o.e_off);
    d.e_inc = at<int32_t>(b, o.e_inc);
    d.vhat = nullptr;  // Vhat summed per step by stage B (splits change it)
    d.hpair = at<int32_t>(b, o.hpair);
    d.hS_h = h.S_h;
    d.hrem = at<int8_t>(b, o.hrem);
    d.htact = at<uint8_t>(b, o.htact);
    d.hnrem = at<uint8_t>(b, o.hnrem);
    d.hediag = at<unsigned>(b, o.hediag);
    d.hdlist = at<int32_t>(b, o.hdlist);
    d.hclist = at<int32_t>(b, o.hclist);
    d.heinc4 = at<int4>(b, o.heinc4);
    d.htloc = at<uint8_t>(b, o.htloc);
    d.htgeo = at<double>(b, o.htgeo);
    d.httau = at<double>(b, o.httau);
    d.gc = at<double>(b, o.gc);
    d.X = at<double4>(b, o.X);
    d.rec_step = at<int64_t>(b, o.rec_step);
    d.rec_elem = at<int32_t>(b, o.rec_elem);
    d.rec_cand = at<int32_t>(b, o.rec_cand);
    d.rec_G = at<double>(b, o.rec_G);
    d.rec_area = at<double>(b, o.rec_area);
    d.nodeE = at<int32_t>(b, o.nodeE);
    d.wn = h.wn;
    d.wn0 = h.wn0;
    d.zslot = h.zslot;
    d.fext = at<double4>(b, o.fext);
    d.nflag = at<uint8_t>(b, o.nflag);
    d.dir_v0 = at<double4>(b, o.dir_v0);
    d.state = at<uint8_t>(b, o.state);
    d.mass = at<double>(b, o.mass);
    d.dirty = at<int32_t>(b, o.dirty);
    d.ubuf[0] = at<double4>(b, o.u0);
    d.ubuf[1] = at<double4>(b, o.u1);
    d.v = at<double4>(b, o.v);
    d.a = at<double4>(b, o.a);
    d.srec = at<double>(b, o.srec);
    d.srec2 = at<double>(b, o.srec2);
    d.fe = at<double>(b, o.fe);
    d.part = nullptr;  // hexahedra: force slots (4 per hex incidence: the hex, its 3 remainder tets)
    d.ctr = at<int32_t>(b, o.ctr);
    d.rprev = h.any_dirichlet ? at<double>(b, o.rprev) : nullptr;
    d.wr_dof = at<double>(b, o.wr_dof);
    d.node_orig = at<int32_t>(b, o.node_orig);
    d.tet_orig = at<int32_t>(b, o.tet_orig);
    d.self = at<Dev>(b, o.self);
    ctx->epart = at<double>(b, o.epart);
    ctx->n_epart_edges = (S + 255) / 256;
    ctx->n_epart_nodes = (N + 255) / 256;
    d.lam = h.lam;
    d.mu = h.mu;
    d.l2m = h.l2m;
    d.rho = h.rho;
    d.dt = h.dt;
    d.hdt2 = 0.5 * h.dt * h.dt;
    d.gamma = h.gamma;
    d.omg = 1.0 - h.gamma;
    d.t0 = h.t0;
    d.flags = ctx->flags;
    d.blk = 256;
    d.blk_ab = 256;
    // device tables: planes [25][E] (V, then dN_a/dx_c at 1 + 3a + c), [8][E], [12][E]
    cudaStream_t s = ctx->stream;
    std::vector<double> geo(25 * E);
    std::vector<int32_t> conn(8 * E);
    for (int64_t e = 0; e < E; ++e) {
        geo[e] = h.V[e];
        for (int i = 0; i < 24; ++i) geo[(1 + i) * E + e] = h.grad[24 * e + i];
        for (int a = 0; a < 8; ++a) conn[a * E + e] = h.hex[8 * e + a];
    }
    // initial state as the tet path (R17): u_0 = 0, a_0 = M^-1 f_ext (prescribed: v(0), v'(0)), u_1 predicted
    std::vector<double4> f4(N), d4(h.any_dirichlet ? N : 1), z4(N, make_double4(0, 0, 0, 0)), v4(N), a4(N), u1(N);
    std::vector<double> r0(h.any_dirichlet ? 3 * N : 1, 0.0);
    const double dt = h.dt, hdt2 = 0.5 * h.dt * h.dt;
    for (int64_t n = 0; n < N; ++n) {
        f4[n] = make_double4(h.fext[3 * n], h.fext[3 * n + 1], h.fext[3 * n + 2], 0.0);
        if (h.any_dirichlet) d4[n] = make_double4(h.dir_v0[3 * n], h.dir_v0[3 * n + 1], h.dir_v0[3 * n + 2], 0.0);
        double vv[3], aa[3], uu[3];
        for (int c = 0; c < 3; ++c) {
            const double mk = h.mass[n];
            if (mk == 0.0) {
                vv[c] = 0.0;
                aa[c] = 0.0;
            } else if (h.nflag[n] >> c & 1) {
                const double v0 = h.dir_v0[3 * n + c];
                if (h.t0 <= 0.0) {
                    vv[c] = v0;
                    aa[c] = 0.0;
                } else {
                    vv[c] = (0.0 / h.t0) * v0;
                    aa[c] = (0.0 < h.t0) ? v0 / h.t0 : 0.0;
                }
            } else {
                vv[c] = 0.0;
                aa[c] = (h.fext[3 * n + c] - 0.0) / mk;
            }
            uu[c] = (0.0 + dt * vv[c]) + hdt2 * aa[c];
            if (h.any_dirichlet && (h.nflag[n] >> c & 1)) r0[3 * n + c] = mk * aa[c] - (h.fext[3 * n + c] - 0.0);
        }
        v4[n] = make_double4(vv[0], vv[1], vv[2], 0.0);
        a4[n] = make_double4(aa[0], aa[1], aa[2], 0.0);
        u1[n] = make_double4(uu[0], uu[1], uu[2], 0.0);
    }
    std::vector<int32_t> ident(std::max(N, E));
    std::iota(ident.begin(), ident.end(), 0);
    int32_t ctr[32] = {0, 0, INT32_MAX};
    auto put = [&](size_t off, const void *src, size_t bytes) { return cudaMemcpyAsync(at<char>(b, off), src, bytes, cudaMemcpyHostToDevice, s); };
    CUDA_TRY(put(o.hgeo, geo.data(), 8 * geo.size()));
    CUDA_TRY(put(o.hconn, conn.data(), 4 * conn.size()));
    CUDA_TRY(put(o.heedge, h.eedge.data(), 4 * h.eedge.size()));
    CUDA_TRY(put(o.e_off, h.edge_off.data(), 4 * h.edge_off.size()));
    CUDA_TRY(put(o.e_inc, h.edge_inc.data(), 4 * h.edge_inc.size()));
    {
        std::vector<int4> q4((size_t)S, make_int4(-1, -1, -1, -1));
        for (int64_t k = 0; k < S; ++k) {
            int32_t *q = &q4[k].x;
            for (int32_t j = h.edge_off[k]; j < std::min(h.edge_off[k + 1], h.edge_off[k] + 4); ++j) q[j - h.edge_off[k]] = h.edge_inc[j];
        }
        CUDA_TRY(put(o.heinc4, q4.data(), sizeof(int4) * q4.size()));
        CUDA_TRY(cudaStreamSynchronize(s));  // q4 leaves scope
    }
    CUDA_TRY(put(o.hpair, h.pair.data(), 4 * h.pair.size()));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.hrem), 0xff, E, s));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.htact), 0, E, s));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.hnrem), 0, N, s));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.hediag), 0, 4 * ((S - h.S_h + 31) / 32 + 1), s));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.htloc), 0, 12 * E, s));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.htgeo), 0, 8 * 39 * E, s));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.httau), 0, 8 * 18 * E, s));
    CUDA_TRY(put(o.gc, h.gc.data(), 8 * E));
    {
        std::vector<double4> x4(N);
        for (int64_t n = 0; n < N; ++n) x4[n] = make_double4(mesh->X[3 * n], mesh->X[3 * n + 1], mesh->X[3 * n + 2], 0.0);
        CUDA_TRY(put(o.X, x4.data(), sizeof(double4) * N));
        CUDA_TRY(cudaStreamSynchronize(s));  // x4 leaves scope
    }
    CUDA_TRY(put(o.nodeE, h.nodeE.data(), 4 * h.nodeE.size()));
    CUDA_TRY(put(o.fext, f4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.nflag, h.nflag.data(), N));
    if (h.any_dirichlet) {
        CUDA_TRY(put(o.dir_v0, d4.data(), sizeof(double4) * N));
        CUDA_TRY(put(o.rprev, r0.data(), 8 * r0.size()));
    }
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.wr_dof), 0, 8 * (h.any_dirichlet ? 3 * N : 1), s));
    CUDA_TRY(put(o.state, h.state.data(), E));
    CUDA_TRY(put(o.mass, h.mass.data(), 8 * N));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.dirty), 0, 4 * N, s));
    CUDA_TRY(put(o.u0, z4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.u1, u1.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.v, v4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.a, a4.data(), sizeof(double4) * N));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.srec), 0, 8 * 4 * S, s));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.srec2), 0, 8 * 2 * S, s));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.fe), 0, 8 * 3 * (32 * E + 1), s));
    CUDA_TRY(put(o.ctr, ctr, sizeof ctr));
    CUDA_TRY(put(o.node_orig, ident.data(), 4 * N));
    CUDA_TRY(put(o.tet_orig, ident.data(), 4 * E));
    CUDA_TRY(put(o.self, &ctx->d, sizeof(Dev)));
    CUDA_TRY(cudaStreamSynchronize(s));
    *out = ctx;
    return CEM_OK;
}

// undo this context's L2 persistence: clear the window on its stream and, if it raised the
// device's persisting set-aside, restore the previous limit and demote the lines it pinned
void release_l2(cem_ctx *ctx) {
    if (ctx->stream) {
        cudaStreamAttrValue a = {};
        a.accessPolicyWindow.num_bytes = 0;
        cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &a);
    }
    if (ctx->l2_limit_raised) {
        if (ctx->stream) cudaStreamSynchronize(ctx->stream);
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, ctx->l2_limit_prev);
        ctx->l2_limit_raised = false;
    }
    cudaGetLastError();
}

}  // namespace

extern "C" {

int32_t cem_abi_version(void) { return CEM_ABI_VERSION; }

const char *cem_last_error(const cem_ctx *ctx) { return ctx ? ctx->err.c_str() : g_init_err.c_str(); }

cem_status cem_workspace_size(const cem_mesh_in *mesh, const cem_opts *opts, size_t *bytes) {
    if (!mesh || !bytes) return CEM_EINVAL;
    // the exact size depends on the storage plan: build it (no device work)
    const cem_material mat = {1.0, 0.0, 1.0, 0.0};
    cem_opts o{};
    if (opts) o = *opts;
    o.dt = 1.0;
    if (mesh->nodes_per_elem == 8) {
        HexHost hh;
        cem_load_in ld{};
        ld.n_vbc = 0;
        cem_status st = build_hex_host(mesh, &mat, &ld, &o, hh, g_init_err);
        if (st) return st;
        hh.any_dirichlet = true;
        *bytes = hex_layout(hh).total;
        return CEM_OK;
    }
    HostMesh h;
    Plan p;
    cem_status st = build_host_mesh(mesh, &mat, nullptr, &o, h, g_init_err);
    if (st) return st;
    h.any_dirichlet = true;
    build_plan(h, block_size(), p);
    WavePlan w;
    if (!(opts && opts->nranks > 1)) build_wave(p, h.N, 8, 1, w);  // (sizes only)
    *bytes = layout(h, p, w).total;
    return CEM_OK;
}

cem_status cem_init_mesh(const cem_mesh_in *mesh, const cem_material *mat, const cem_load_in *load,
                         const cem_opts *opts, cem_ctx **out) {
    if (!out) return CEM_EINVAL;
    *out = nullptr;
    NvtxRange nv("cem_init_mesh");
    g_init_err.clear();
    if (mesh && mesh->nodes_per_elem != 0 && mesh->nodes_per_elem != 4 && mesh->nodes_per_elem != 8) {
        g_init_err = "cem_init_mesh: nodes_per_elem must be 0, 4 (tets) or 8 (hexahedra)";
        return CEM_EINVAL;
    }
    if (mesh && mesh->nodes_per_elem == 8) return hex_init(mesh, mat, load, opts, out);
    cem_ctx *ctx = new cem_ctx();
    auto fail = [&](cem_status s) {
        g_init_err = ctx->err;
        release_l2(ctx);
        if (ctx->own_ws && ctx->ws) cudaFree(ctx->ws);
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        if (ctx->fence_in) cudaEventDestroy(ctx->fence_in);
        if (ctx->fence_out) cudaEventDestroy(ctx->fence_out);
        delete ctx;
        return s;
    };
    cem_status st;
    std::vector<uint8_t> tflag_local;
    if (opts && opts->nranks > 1) {
        // multi-GPU: this rank's sub-mesh with a 2-ring ghost layer
        if (!mesh || !mesh->X || !mesh->tets || !mat || opts->rank < 0 || opts->rank >= opts->nranks) {
            ctx->err = "cem_init_mesh: bad multi-rank arguments";
            return fail(CEM_EINVAL);
        }
        ctx->dist = true;
        ctx->loopback = (opts->flags & CEM_F_LOOPBACK) != 0;
        ctx->rank = opts->rank;
        ctx->nranks = opts->nranks;
        cem_opts lo = *opts;
        if (!(lo.dt > 0)) {  // the global time step, identical on every rank
            st = global_cfl_dt(mesh, mat, lo.cfl > 0 ? lo.cfl : 0.5, &lo.dt, ctx->err);
            if (st) return fail(st);
        }
        lo.nranks = 1;
        PartGlobal g;
        build_partition(mesh->n_nodes, mesh->X, mesh->n_tets, mesh->tets, opts->nranks, g);
        build_exchange(g, opts->rank, ctx->part);
        LocalMesh lm;
        extract_local(mesh, mat, load, ctx->part, lm);
        cem_mesh_in m2 = {(int64_t)ctx->part.node_global.size(), lm.X.data(), (int64_t)ctx->part.tet_global.size(),
                          lm.tets.data(), lm.state.data(), lm.gc.data()};
        cem_load_in l2 = {(int64_t)lm.tface.size() / 3, lm.tface.data(), lm.tface_t.data(), (int64_t)lm.vbc_node.size(),
                          lm.vbc_node.data(), lm.vbc_mask.data(), lm.vbc_v0.data(), load ? load->vbc_t0 : 0.0,
                          lm.f_nodal.empty() ? nullptr : lm.f_nodal.data(),
                          {load ? load->body[0] : 0.0, load ? load->body[1] : 0.0, load ? load->body[2] : 0.0}};
        st = build_host_mesh(&m2, mat, &l2, &lo, ctx->h, ctx->err);
        if (st) return fail(st);
        for (size_t i = 0; i < ctx->part.node_owned.size(); ++i)
            if (!ctx->part.node_owned[i]) ctx->h.nflag[i] |= 16;  // not updated here
        tflag_local = ctx->part.tet_flag;
    } else {
        st = build_host_mesh(mesh, mat, load, opts, ctx->h, ctx->err);
        if (st) return fail(st);
    }
    ctx->device = opts ? opts->device : 0;
    ctx->flags = opts ? opts->flags : 0;
    ctx->user_stream = opts ? (cudaStream_t)opts->stream : nullptr;
    if (cudaSetDevice(ctx->device) != cudaSuccess) {
        ctx->err = "cudaSetDevice failed (no CUDA device?)";
        return fail(CEM_ECUDA);
    }
    const bool persistent = opts && (opts->flags & CEM_F_PERSISTENT);
    build_plan(ctx->h, block_size(), ctx->p, tflag_local.empty() ? nullptr : tflag_local.data(), persistent);
    PhaseClock clk;
    const int smem = smem_bytes_for(ctx->p);
    if (smem > 227 * 1024) {
        ctx->err = "a block's gather list exceeds shared memory (" + std::to_string(smem) + " bytes)";
        return fail(CEM_EINVAL);
    }
    set_smem_limits(smem);
    if (const char *ek = getenv("CEM_STAGE_CHUNKS"))
        if (atoi(ek) > 1) ctx->chunks = build_stage_chunks(ctx->p, atoi(ek));
    {  // software-pipelined stage C (k_Cp): CEM_C_PIPE=1 (measured in DESIGN.md §6)
        const char *e = getenv("CEM_C_PIPE");
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        // (k_Cp writes force slots: only with CEM_PARTIALS=0)
        if (e && atoi(e) > 0 && ctx->p.blk == 256 && !ctx->p.partials &&
            cp_stage_c_smem(ctx->p.max_el, ctx->p.max_nl) > 0) {
            ctx->cp_on = 1;
            ctx->cp_grid = std::max(1, sms) * std::max(1, atoi(e));
        }
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    const int occ = std::max(1, persistent_occupancy(smem, ctx->p.blk));
    ctx->grid = sms * occ;
    if (persistent) {
        const char *ev = getenv("CEM_SCHED_SLACK");  // tuning knob: slack in units of resident CTAs
        const double slack = ev ? atof(ev) : 3.0;
        build_schedule(ctx->p, (int)(slack * ctx->grid));
    }
    if (!ctx->dist && !persistent && getenv("CEM_WAVE") && atoi(getenv("CEM_WAVE")) != 0) {
        // (opt-in: measured slower than the staged path on B200, DESIGN.md §6 "Wavefront")
        // dataflow launches: K chunks per stage, lookahead in chunks (DESIGN.md §6 "Wavefront")
        const char *ek = getenv("CEM_WAVE_K"), *el = getenv("CEM_WAVE_LA");
        build_wave(ctx->p, ctx->h.N, ek ? atoi(ek) : 8, el ? atoi(el) : 1, ctx->w);
        if (const char *gm = getenv("CEM_GRAPH_M")) ctx->graph_m = std::max(0, atoi(gm));
        const char *cv = getenv("CEM_WAVE_CARVE");
        if (!(cv && atoi(cv) == -2)) set_wave_carveout(smem_ab_for(ctx->p), smem_c_for(ctx->p), cv ? atoi(cv) : -1);
    }
    clk.mark("init: schedule");
    {  // the library's own stream (graphs, access-policy window); fenced against opts.stream
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->fence_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->fence_out, cudaEventDisableTiming) != cudaSuccess) {
            ctx->err = "cudaStreamCreate / cudaEventCreate failed";
            return fail(CEM_ECUDA);
        }
        ctx->own_stream = true;
        cudaEventRecord(ctx->fence_in, ctx->user_stream);  // a caller-allocated workspace is ready
        cudaStreamWaitEvent(ctx->stream, ctx->fence_in, 0);
    }
    Offs o = layout(ctx->h, ctx->p, ctx->w);
    if (opts && opts->workspace) {
        if (opts->workspace_bytes < o.total) {
            ctx->err = "workspace too small: need " + std::to_string(o.total) + " bytes";
            return fail(CEM_ENOMEM);
        }
        ctx->ws = opts->workspace;
        ctx->ws_bytes = opts->workspace_bytes;
    } else if (opts && opts->dev_alloc) {
        if (opts->dev_alloc(o.total, opts->alloc_user, &ctx->ws) != 0 || !ctx->ws) {
            ctx->err = "dev_alloc callback failed for " + std::to_string(o.total) + " bytes";
            return fail(CEM_ENOMEM);
        }
        ctx->ws_bytes = o.total;
    } else {
        cudaError_t e = cudaMalloc(&ctx->ws, o.total);
        if (e != cudaSuccess) {
            ctx->err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
            ctx->ws = nullptr;
            return fail(CEM_ENOMEM);
        }
        ctx->own_ws = true;
        ctx->ws_bytes = o.total;
    }
    clk.mark("init: workspace");
    bind_views(ctx, o);
    {
        // the criterion kernel is chosen per step on the host from the list length of a recent
        // step, which stage D stores here (a heuristic: results do not depend on the choice)
        void *hp = nullptr, *dp = nullptr;
        cudaError_t e = cudaHostAlloc(&hp, sizeof(int32_t), cudaHostAllocMapped);
        if (e == cudaSuccess) e = cudaHostGetDevicePointer(&dp, hp, 0);
        if (e != cudaSuccess) {
            ctx->err = std::string("cudaHostAlloc (mapped): ") + cudaGetErrorString(e);
            return fail(CEM_ECUDA);
        }
        *static_cast<int32_t *>(hp) = 0;
        if (const char *m = getenv("CEM_CRITB_MIN")) ctx->critb_min = atoi(m);
        if (const char *m = getenv("CEM_CRIT_STREAM")) ctx->crit_stream = atoi(m) != 0;
        ctx->crit_seen = static_cast<volatile int32_t *>(hp);
        ctx->d.crit_seen = static_cast<int32_t *>(dp);
    }
    st = upload(ctx, o);
    if (st) return fail(st);
    clk.mark("init: upload");
    {
        // L2 persistence for the sigma records between their writer (stage AB) and their reader
        // (stage C): a stream access-policy window over the two sigma planes, persisting up to the
        // device's set-aside limit (CEM_L2_PERSIST=0 disables it, =r < 1 sets the hit ratio).
        // Measured: config 3 153.9 -> 147.8 us/step, config 2 167.7 -> 162.1; windows reaching into
        // the force slots were slower.
        const char *lp = getenv("CEM_L2_PERSIST");
        const double want = lp ? atof(lp) : 1.0;
        int maxwin = 0, maxpers = 0;
        cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
        cudaDeviceGetAttribute(&maxpers, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
        // CEM_L2_WIN (measurement knob): 1 sigma planes (default), 2 the partials, 3 both
        const int wsel = getenv("CEM_L2_WIN") ? atoi(getenv("CEM_L2_WIN")) : 1;
        char *wbase = (char *)ctx->d.srec, *wend = (char *)(ctx->d.srec2 + 2 * ctx->h.S);
        if (ctx->d.part && wsel >= 2) {
            if (wsel == 2) wbase = (char *)ctx->d.part;
            wend = (char *)(ctx->d.part + 6 * ctx->p.nl.size());
        }
        const size_t bytes = (size_t)(wend - wbase);
        const size_t win = std::min(bytes, (size_t)std::max(0, maxwin));
        // only when the planes fit the set-aside whole: a partial window (hit ratio < 1 over a larger
        // mesh's planes) thrashed -- config 4 on one GPU 1087 -> 1614 us/step
        // (single-GPU contexts only: loopback ranks share rank 0's stream; the window lives on the
        // library's private stream, and cem_destroy restores the set-aside it raised)
        const bool fits = bytes <= (size_t)std::max(0, maxpers) || wsel == 3;
        if (!ctx->dist && want > 0.0 && win > 0 && win == bytes && fits) {
            const double hit = std::min(want, std::min(1.0, (double)std::max(0, maxpers) / (double)bytes));
            size_t cur = 0;
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            const size_t aside = std::min((size_t)maxpers, (size_t)(win * hit));
            if (aside > cur && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, aside) == cudaSuccess) {
                ctx->l2_limit_raised = true;  // (device-wide: restored by cem_destroy)
                ctx->l2_limit_prev = cur;
            }
            cudaStreamAttrValue a = {};
            a.accessPolicyWindow.base_ptr = wbase;
            a.accessPolicyWindow.num_bytes = win;
            a.accessPolicyWindow.hitRatio = (float)hit;
            a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &a);
            cudaGetLastError();  // best effort: a refused window only costs the speed-up
        }
    }
    if (ctx->dist) {
        st = setup_exchange(ctx);
        if (st) return fail(st);
        if (ctx->loopback) {
            ctx->init_exchange_pending = true;  // done by the first cem_step_group
        } else {
            if (!opts->nccl_id && opts->host_allgather) {  // host-ordered CUDA-IPC halo, no NCCL
                ctx->host_allgather = opts->host_allgather;
                ctx->host_user = opts->host_user;
                st = p2p_setup_host(ctx);
                if (st) return fail(st);
                *out = ctx;
                return CEM_OK;
            }
            if (!opts->nccl_id) {
                ctx->err = "cem_init_mesh: nranks > 1 needs opts.nccl_id, opts.host_allgather or CEM_F_LOOPBACK";
                return fail(CEM_EINVAL);
            }
            if (!nccl_comm_init(&ctx->comm, ctx->nranks, ctx->rank, opts->nccl_id, ctx->err)) return fail(CEM_ENCCL);
            st = exchange_nccl_step(ctx, 1);  // owners' u_1 to the ranks holding their nodes
            if (st) return fail(st);
            CUDA_TRY(cudaStreamSynchronize(ctx->stream));
            if (!getenv("CEM_NO_P2P")) {  // NVLink P2P halo when every rank can map its peers
                st = p2p_setup_nccl(ctx);
                if (st) return fail(st);
            }
        }
    }
    *out = ctx;
    return CEM_OK;
}

void cem_destroy(cem_ctx *ctx) {
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto &g : ctx->graphs) cudaGraphExecDestroy(g.exec);
    release_l2(ctx);
    for (auto e : ctx->ev) cudaEventDestroy(e);
    for (void *p : ctx->p2p.opened) cudaIpcCloseMemHandle(p);
    if (ctx->comm) nccl_comm_destroy(ctx->comm);
    for (void *p : ctx->dist_allocs) cudaFree(p);
    if (ctx->own_ws && ctx->ws) cudaFree(ctx->ws);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->fence_in) cudaEventDestroy(ctx->fence_in);
    if (ctx->fence_out) cudaEventDestroy(ctx->fence_out);
    if (ctx->crit_seen) cudaFreeHost(const_cast<int32_t *>(ctx->crit_seen));
    delete ctx;
}

cem_status cem_sizes(const cem_ctx *ctx, int64_t *n_nodes, int64_t *n_tets, int64_t *n_edges) {
    if (!ctx) return CEM_EINVAL;
    if (n_nodes) *n_nodes = ctx->h.N;
    if (n_tets) *n_tets = ctx->h.E;
    if (n_edges) *n_edges = ctx->h.S;
    return CEM_OK;
}

int64_t cem_launch_count(const cem_ctx *ctx) { return ctx ? ctx->launches : 0; }

cem_status cem_set_profiling(cem_ctx *ctx, int on) {
    if (!ctx) return CEM_EINVAL;
    ctx->profiling = on != 0;
    ctx->prof_steps = 0;
    return CEM_OK;
}

// long criterion lists (cracking phases) go to k_filter + k_eval; CEM_CRITB_MIN overrides the threshold
bool crit_heavy(const cem_ctx *ctx) { return ctx->crit_seen && *ctx->crit_seen >= ctx->critb_min; }
// the staged path's criterion mode from the recent list length (racy by design: results never depend on it)
int crit_mode(const cem_ctx *ctx) {
    static const int forced = getenv("CEM_CRIT_MODE") ? atoi(getenv("CEM_CRIT_MODE")) : -1;  // (measurement knob)
    if (forced >= 0 && forced <= CRIT_IDLE) return forced;
    if (!ctx->crit_seen) return CRIT_LIST;
    const int n = *ctx->crit_seen;
    if (n >= ctx->critb_min) return CRIT_HEAVY;
    if (!ctx->crit_stream) return CRIT_LIST;
    return n == 0 ? CRIT_IDLE : CRIT_STREAM;
}

cem_status cem_step(cem_ctx *ctx, int64_t nsteps, int32_t crack_every) {
    if (!ctx || nsteps < 0) return CEM_EINVAL;
    NvtxRange nv("cem_step");
    if (ctx->dist && ctx->comm) {  // a failed communicator (ncclCommGetAsyncError) stops the run
        std::string e;
        if (nccl_async_error(ctx->comm, e)) {
            ctx->err = e;
            return CEM_ENCCL;
        }
    }
    if (nsteps == 0) return CEM_OK;
    if (crack_every < 0) crack_every = 0;
    StreamFence fence(ctx);
    if (ctx->hexa) {  // crack steps (R16): the criterion of patterns III-VI between stages C and D
        for (int64_t i = 0; i < nsteps; ++i) {
            const int64_t s1 = ctx->step + i + 1;
            const bool crack = crack_every > 0 && s1 % crack_every == 0;
            ctx->launches += launch_hex_step(ctx->d, ctx->step + i, ctx->stream, crack, ctx->hex_cracked);
            ctx->hex_cracked |= crack;
        }
        CUDA_TRY(cudaGetLastError());
        ctx->step += nsteps;
        return CEM_OK;
    }
    // default: one kernel per stage (measured faster than the persistent wavefront kernel on
    // B200 for the current stage bodies; CEM_F_PERSISTENT selects the latter)
    if (ctx->dist) {
        if (ctx->loopback) {
            ctx->err = "loopback contexts are stepped with cem_step_group";
            return CEM_ESTATE;
        }
        for (int64_t i = 0; i < nsteps; ++i) {
            const int64_t sstep = ctx->step + i;
            ctx->launches += launch_staged_step(ctx->d, sstep, crack_every, ctx->stream, nullptr, crit_mode(ctx), &ctx->sy,
                                                &ctx->chunks);
            if (ctx->p2p.on && ctx->host_allgather) {
                // host-ordered: signal, wait for this rank's stores, meet the peers on the host, then
                // the flag wait (already satisfied: it never spins) and the unpack
                p2p_sync(ctx->p2p, (int)ctx->part.peers.size(), sstep + 2, false, ctx->stream);
                CUDA_TRY(cudaStreamSynchronize(ctx->stream));
                cem_status hs = host_barrier(ctx);
                if (hs) return hs;
            }
            if (ctx->p2p.on) {  // stage D / the split pass already stored into the peers' buffers
                p2p_sync(ctx->p2p, (int)ctx->part.peers.size(), sstep + 2, true, ctx->stream);
                exchange_unpack(ctx->xch, ctx->d.ubuf[sstep & 1], ctx->d.state, ctx->d.eedge, ctx->h.E,
                                ctx->d.edge_dirty, ctx->stream, ctx->p2p.recv[sstep & 1]);
                ctx->launches += 2;
                continue;
            }
            cem_status st = exchange_nccl_step(ctx, (int)(sstep & 1));
            if (st) return st;
        }
        CUDA_TRY(cudaGetLastError());
        ctx->step += nsteps;
        return CEM_OK;
    }
    if (!ctx->profiling && !(ctx->flags & CEM_F_PERSISTENT) && !ctx->w.seq.empty()) {
        // dataflow launches (DESIGN.md §6 "Wavefront"); steps whose recent criterion lists are long
        // go to the staged k_filter + k_eval path instead (joined / refilled at the switch)
        bool in_wave = false;
        for (int64_t i = 0; i < nsteps;) {
            const int64_t sstep = ctx->step + i;
            const bool heavy = crack_every > 0 && crit_heavy(ctx);
            const int M = ctx->graph_m;
            if (!heavy && M > 0 && nsteps - i >= M) {
                // M steps as one CUDA-graph replay (captured once per crack_every): the kernels read
                // the base step from d.wstep, set by a plain launch that follows all earlier work
                cudaGraphExec_t ex = nullptr;
                for (auto &g : ctx->graphs)
                    if (g.crack_every == crack_every && g.M == M) ex = g.exec;
                if (!ex) {
                    cudaGraph_t gr = nullptr;
                    CUDA_TRY(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
                    for (int j = 0; j < M; ++j) launch_wave_step(ctx->d, ctx->w, j, crack_every, ctx->stream, 1);
                    launch_wave_join(ctx->d, M, ctx->stream, 1);
                    CUDA_TRY(cudaStreamEndCapture(ctx->stream, &gr));
                    const cudaError_t e = cudaGraphInstantiate(&ex, gr, 0);
                    cudaGraphDestroy(gr);
                    CUDA_TRY(e);
                    ctx->graphs.push_back({crack_every, M, ex});
                }
                if (in_wave) {
                    launch_wave_join(ctx->d, sstep, ctx->stream);
                    ctx->launches += 1;
                    in_wave = false;
                }
                if (ctx->wcnt_valid != sstep) {
                    launch_wave_fill(ctx->d, sstep, ctx->stream);
                    ctx->launches += 1;
                }
                launch_wave_base(ctx->d, sstep, ctx->stream);
                CUDA_TRY(cudaGraphLaunch(ex, ctx->stream));
                ctx->launches += 2 + (int64_t)M * (int64_t)ctx->w.seq.size();
                ctx->wcnt_valid = sstep + M;
                i += M;
                continue;
            }
            ++i;
            if (!heavy) {
                if (ctx->wcnt_valid != sstep) {
                    launch_wave_fill(ctx->d, sstep, ctx->stream);
                    ctx->launches += 1;
                }
                ctx->launches += launch_wave_step(ctx->d, ctx->w, sstep, crack_every, ctx->stream);
                ctx->wcnt_valid = sstep + 1;
                in_wave = true;
            } else {
                if (in_wave) {
                    launch_wave_join(ctx->d, sstep, ctx->stream);
                    ctx->launches += 1;
                    in_wave = false;
                }
                ctx->launches += launch_staged_step(ctx->d, sstep, crack_every, ctx->stream, nullptr, CRIT_HEAVY);
            }
        }
        if (in_wave) {
            launch_wave_join(ctx->d, ctx->step + nsteps, ctx->stream);
            ctx->launches += 1;
        }
        CUDA_TRY(cudaGetLastError());
        ctx->step += nsteps;
        return CEM_OK;
    }
    const bool staged = ctx->profiling || !(ctx->flags & CEM_F_PERSISTENT);
    if (staged) {
        // one kernel per stage; with profiling, CUDA events bracket every stage
        if (ctx->profiling) {
            const size_t need = (size_t)(ctx->prof_steps + nsteps) * kStagedEvents;
            while (ctx->ev.size() < need) {
                cudaEvent_t e;
                CUDA_TRY(cudaEventCreate(&e));
                ctx->ev.push_back(e);
            }
        }
        for (int64_t i = 0; i < nsteps; ++i) {
            cudaEvent_t *E = ctx->profiling ? ctx->ev.data() + (ctx->prof_steps + i) * kStagedEvents : nullptr;
            ctx->launches += launch_staged_step(ctx->d, ctx->step + i, crack_every, ctx->stream, E, crit_mode(ctx), &ctx->sy,
                                                &ctx->chunks);
        }
        CUDA_TRY(cudaGetLastError());
        if (ctx->profiling) ctx->prof_steps += nsteps;
        ctx->step += nsteps;
        return CEM_OK;
    }
    if (ctx->cnt_valid != ctx->step) {
        // steps ran outside the wavefront: every block is complete through ctx->step
        const int64_t n = ST_COUNT * (int64_t)ctx->p.maxblk;
        k_fill<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->d.cnt, n, (int32_t)ctx->step);
        ctx->launches += 1;
    }
    launch_persistent(ctx->d, ctx->step, nsteps, crack_every, ctx->grid, ctx->stream);
    CUDA_TRY(cudaGetLastError());
    ctx->launches += 1;
    ctx->step += nsteps;
    ctx->cnt_valid = ctx->step;
    return CEM_OK;
}

cem_status cem_kernel_times(const cem_ctx *ctx, int32_t *n, const char **names, double *ms, int32_t cap) {
    constexpr int K = kStagedEvents - 1;
    static const char *kNames[K] = {"stage_AB_strain_edge_stress", "stage_C_force_earlyout", "criterion_split",
                                    "stage_D_node_update"};  // (profiled: plain launches, no PDL overlap)
    if (!ctx || !n) return CEM_EINVAL;
    *n = K;
    if (cap < K) return CEM_OK;
    for (int k = 0; k < K; ++k) {
        if (names) names[k] = kNames[k];
        double tot = 0.0;
        for (int64_t i = 0; i < ctx->prof_steps; ++i) {
            float t = 0.f;
            cudaEvent_t *E = const_cast<cudaEvent_t *>(ctx->ev.data()) + i * kStagedEvents;
            if (cudaEventSynchronize(E[k + 1]) != cudaSuccess) return CEM_ECUDA;
            if (cudaEventElapsedTime(&t, E[k], E[k + 1]) != cudaSuccess) return CEM_ECUDA;
            tot += t;
        }
        ms[k] = tot;
    }
    return CEM_OK;
}

cem_status cem_crack_update(cem_ctx *ctx, int64_t *n_split_out) {
    if (!ctx) return CEM_EINVAL;
    if (ctx->dist) {
        ctx->err = "cem_crack_update: single-GPU contexts only";
        return CEM_ESTATE;
    }
    if (ctx->hexa) {
        ctx->err = "cem_crack_update: not available for hexahedral contexts (their criterion runs inside cem_step)";
        return CEM_ESTATE;
    }
    StreamFence fence(ctx);
    int32_t before = 0, after = 0;
    CUDA_TRY(cudaMemcpyAsync(&before, ctx->d.ctr, sizeof before, cudaMemcpyDeviceToHost, ctx->stream));
    launch_crack_only(ctx->d, ctx->step, ctx->stream);
    ctx->launches += 3;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(&after, ctx->d.ctr, sizeof after, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (n_split_out) *n_split_out = after - before;
    return CEM_OK;
}

cem_status cem_set_state(cem_ctx *ctx, const cem_state_out *in) {
    if (!ctx || !in) return CEM_EINVAL;
    NvtxRange nv("cem_set_state");
    if (ctx->dist || ctx->hexa) {
        ctx->err = "cem_set_state: single-GPU tetrahedral contexts only";
        return CEM_ESTATE;
    }
    const HostMesh &h = ctx->h;
    const Plan &p = ctx->p;
    const int64_t N = h.N, E = h.E, S = h.S, nr = in->n_records;
    if (!in->u || !in->v || !in->a || !in->tet_state || !in->mass || in->step < 0 || nr < 0 || nr > E ||
        (nr > 0 && (!in->rec_step || !in->rec_elem || !in->rec_cand || !in->rec_G || !in->rec_area))) {
        ctx->err = "cem_set_state: a required array is NULL or a count is out of range";
        return CEM_EINVAL;
    }
    StreamFence fence(ctx);
    cudaStream_t st = ctx->stream;
    CUDA_TRY(cudaStreamSynchronize(st));  // earlier steps done before their buffers are overwritten
    const int64_t n = in->step;
    const double dt = ctx->d.dt, hdt2 = ctx->d.hdt2;
    std::vector<double4> u0(N), u1(N), v4(N), a4(N);
    std::vector<double> m(N);
    for (int64_t kn = 0; kn < N; ++kn) {
        const int64_t k = p.node_new2old[kn];
        double uu[3], vv[3], aa[3], up[3];
        for (int c = 0; c < 3; ++c) {
            uu[c] = in->u[3 * k + c];
            vv[c] = in->v[3 * k + c];
            aa[c] = in->a[3 * k + c];
            up[c] = (uu[c] + dt * vv[c]) + hdt2 * aa[c];  // predictor (stage D's expression)
        }
        u0[kn] = make_double4(uu[0], uu[1], uu[2], 0.0);
        u1[kn] = make_double4(up[0], up[1], up[2], 0.0);
        v4[kn] = make_double4(vv[0], vv[1], vv[2], 0.0);
        a4[kn] = make_double4(aa[0], aa[1], aa[2], 0.0);
        m[kn] = in->mass[k];
    }
    std::vector<uint8_t> stt(E);
    for (int64_t en = 0; en < E; ++en) stt[en] = in->tet_state[p.tet_new2old[en]] ? 1 : 0;
    std::vector<double> vh(S, 0.0);  // Vhat_s over the active incident tets, ascending original id
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < S; ++s) {
        double acc = 0.0;
        for (int32_t j = p.edge_off[s]; j < p.edge_off[s + 1]; ++j)
            if (stt[p.edge_inc[j]]) acc = acc + p.geoV[p.edge_inc[j]];
        vh[s] = acc;
    }
    std::vector<double> nanv(3 * N, std::nan(""));
    CUDA_TRY(cudaMemcpyAsync(ctx->d.ubuf[n & 1], u0.data(), sizeof(double4) * N, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ctx->d.ubuf[(n + 1) & 1], u1.data(), sizeof(double4) * N, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ctx->d.v, v4.data(), sizeof(double4) * N, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ctx->d.a, a4.data(), sizeof(double4) * N, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ctx->d.mass, m.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ctx->d.state, stt.data(), E, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ctx->d.vhat, vh.data(), sizeof(double) * S, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(ctx->d.edge_dirty, 0, S, st));
    CUDA_TRY(cudaMemsetAsync(ctx->d.dirty, 0, sizeof(int32_t) * N, st));
    if (ctx->d.rprev) {  // (the reaction-work ledger is not part of the checkpoint)
        CUDA_TRY(cudaMemcpyAsync(ctx->d.rprev, nanv.data(), sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(ctx->d.wr_dof, nanv.data(), sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    }
    if (nr > 0) {
        CUDA_TRY(cudaMemcpyAsync(ctx->d.rec_step, in->rec_step, 8 * nr, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(ctx->d.rec_elem, in->rec_elem, 4 * nr, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(ctx->d.rec_cand, in->rec_cand, 4 * nr, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(ctx->d.rec_G, in->rec_G, 8 * nr, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(ctx->d.rec_area, in->rec_area, 8 * nr, cudaMemcpyHostToDevice, st));
    }
    int32_t ctr[32] = {(int32_t)nr, 0, INT32_MAX};  // records, no non-finite value, empty lists
    CUDA_TRY(cudaMemcpyAsync(ctx->d.ctr, ctr, sizeof ctr, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(ctx->d.crit_list, 0, sizeof(int64_t) * E, st));  // (stamps of the old steps)
    CUDA_TRY(cudaStreamSynchronize(st));  // (the host vectors above go out of scope)
    ctx->step = n;
    ctx->cnt_valid = -1;   // persistent / wave counters refilled for the new step
    ctx->wcnt_valid = -1;
    return CEM_OK;
}

cem_status cem_energy(cem_ctx *ctx, cem_energy_out *out) {
    if (!ctx || !out) return CEM_EINVAL;
    NvtxRange nv("cem_energy");
    StreamFence fence(ctx);
    cudaStream_t st = ctx->stream;
    cem_state_out so{};
    const cem_status rc = cem_get_state(ctx, &so, CEM_HOST);  // synchronises; U_d, nonfinite
    if (rc != CEM_OK) return rc;
    if (ctx->hexa) {
        launch_hex_energy(ctx->d, ctx->step, ctx->epart, ctx->epart + ctx->n_epart_edges, st);
        ctx->launches += 1;
    } else {
        launch_energy(ctx->d, ctx->step, ctx->epart, ctx->epart + ctx->n_epart_edges, st);
    }
    ctx->launches += 2;
    std::vector<double> pe(ctx->n_epart_edges + 3 * ctx->n_epart_nodes);
    CUDA_TRY(cudaMemcpyAsync(pe.data(), ctx->epart, sizeof(double) * pe.size(), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaGetLastError());
    double U = 0.0, T = 0.0, W = 0.0, Wr = 0.0;  // partials summed in block order
    for (int64_t i = 0; i < ctx->n_epart_edges; ++i) U = U + pe[i];
    for (int64_t i = 0; i < ctx->n_epart_nodes; ++i) {
        T = T + pe[ctx->n_epart_edges + 3 * i];
        W = W + pe[ctx->n_epart_edges + 3 * i + 1];
        Wr = Wr + pe[ctx->n_epart_edges + 3 * i + 2];
    }
    out->step = ctx->step;
    out->time = (double)ctx->step * ctx->h.dt;
    out->kinetic = 0.5 * T;
    out->strain = U;
    out->external_work = W;
    out->reaction_work = Wr;
    out->dissipated = so.dissipated;
    return CEM_OK;
}

cem_status cem_get_state(cem_ctx *ctx, cem_state_out *out, int where) {
    if (!ctx || !out) return CEM_EINVAL;
    NvtxRange nv("cem_get_state");
    if (ctx->dist && ctx->comm) {
        std::string e;
        if (nccl_async_error(ctx->comm, e)) {
            ctx->err = e;
            return CEM_ENCCL;
        }
    }
    StreamFence fence(ctx);
    cudaStream_t st = ctx->stream;
    const HostMesh &h = ctx->h;
    const Plan &p = ctx->p;
    const int64_t N = h.N, E = h.E;
    int32_t ctr[16];
    CUDA_TRY(cudaMemcpyAsync(ctr, ctx->d.ctr, sizeof ctr, cudaMemcpyDeviceToHost, st));
    int64_t p2p_timeout = 0;
    if (ctx->p2p.on && ctx->p2p.timeout)
        CUDA_TRY(cudaMemcpyAsync(&p2p_timeout, ctx->p2p.timeout, sizeof p2p_timeout, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (p2p_timeout) {
        ctx->err = "P2P halo: a peer stopped signalling (waited 60 s); the state is invalid";
        return CEM_ENCCL;
    }
    const int64_t nrec = ctr[0];
#ifdef CEM_DEBUG_BOUNDS
    {
        int32_t bline = 0;
        CUDA_TRY(cudaMemcpy(&bline, ctx->d.ctr + 20, sizeof bline, cudaMemcpyDeviceToHost));
        if (bline) {
            ctx->err = "debug build: a device bounds check failed at cem_kernels.cu line " + std::to_string(bline);
            return CEM_ESTATE;
        }
    }
#endif
#ifdef CEM_WAVE_STATS
    fprintf(stderr, "[cem wave stats] blocks that waited: AB %d C %d D %d; polls %u\n", ctr[12], ctr[13], ctr[14],
            (unsigned)ctr[7]);
#endif
#ifdef CEM_POLL_STATS
    fprintf(stderr, "[cem poll stats] polls AB %d C %d D %d, items that waited %d\n", ctr[4], ctr[5], ctr[6], ctr[7]);
#endif
    // records: unordered on the device; ordered here by (step, element) and U_d summed in
    // that order (the oracle's split-pass order)
    std::vector<int64_t> rs(nrec);
    std::vector<int32_t> re(nrec), rk(nrec);
    std::vector<double> rg(nrec), ra(nrec);
    if (nrec > 0) {
        CUDA_TRY(cudaMemcpyAsync(rs.data(), ctx->d.rec_step, 8 * nrec, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(re.data(), ctx->d.rec_elem, 4 * nrec, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(rk.data(), ctx->d.rec_cand, 4 * nrec, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(rg.data(), ctx->d.rec_G, 8 * nrec, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(ra.data(), ctx->d.rec_area, 8 * nrec, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    std::vector<int64_t> ord(nrec);
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) {
        return rs[x] < rs[y] || (rs[x] == rs[y] && re[x] < re[y]);
    });
    double Ud = 0.0;
    for (int64_t i = 0; i < nrec; ++i) Ud = Ud + h.gc[re[ord[i]]] * ra[ord[i]];
    if (ctx->dist)  // records carry GLOBAL element ids (local ids ascend with global ids: order kept)
        for (int64_t i = 0; i < nrec; ++i) re[i] = ctx->part.tet_global[re[i]];
    std::vector<uint8_t> stt(E);
    CUDA_TRY(cudaMemcpyAsync(stt.data(), ctx->d.state, E, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    int64_t na = 0;
    for (int64_t e = 0; e < E; ++e) na += stt[e] != 0;
    double4 *ucur = ctx->d.ubuf[ctx->step & 1];
    if (where == CEM_DEVICE) {
        // the caller's DEVICE buffers, filled in the caller's numbering on the ctx stream (same
        // layout as CEM_HOST); records sorted here and copied up
        const unsigned gn = (unsigned)((N + 255) / 256), ge = (unsigned)((E + 255) / 256);
        if (N > 0) {
            if (out->u) k_export_vec<<<gn, 256, 0, st>>>(ucur, ctx->d.node_orig, out->u, N);
            if (out->v) k_export_vec<<<gn, 256, 0, st>>>(ctx->d.v, ctx->d.node_orig, out->v, N);
            if (out->a) k_export_vec<<<gn, 256, 0, st>>>(ctx->d.a, ctx->d.node_orig, out->a, N);
            if (out->mass) k_export_f64<<<gn, 256, 0, st>>>(ctx->d.mass, ctx->d.node_orig, out->mass, N);
        }
        if (out->tet_state && E > 0) k_export_u8<<<ge, 256, 0, st>>>(ctx->d.state, ctx->d.tet_orig, out->tet_state, E);
        const int64_t nr = std::min<int64_t>(nrec, out->rec_capacity);
        if (nr > 0) {
            std::vector<int64_t> s2(nr);
            std::vector<int32_t> e2(nr), k2(nr);
            std::vector<double> g2(nr), a2(nr);
            for (int64_t i = 0; i < nr; ++i) {
                const int64_t j = ord[i];
                s2[i] = rs[j]; e2[i] = re[j]; k2[i] = rk[j]; g2[i] = rg[j]; a2[i] = ra[j];
            }
            auto up = [&](void *dst, const void *src, size_t bytes) -> cudaError_t {
                return dst ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st) : cudaSuccess;
            };
            CUDA_TRY(up(out->rec_step, s2.data(), 8 * nr));
            CUDA_TRY(up(out->rec_elem, e2.data(), 4 * nr));
            CUDA_TRY(up(out->rec_cand, k2.data(), 4 * nr));
            CUDA_TRY(up(out->rec_G, g2.data(), 8 * nr));
            CUDA_TRY(up(out->rec_area, a2.data(), 8 * nr));
        }
        ctx->launches += (N > 0 ? (out->u != nullptr) + (out->v != nullptr) + (out->a != nullptr) + (out->mass != nullptr) : 0) +
                         (out->tet_state && E > 0 ? 1 : 0);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(st));  // the host record vectors above go out of scope
    } else {
        std::vector<double4> tmp;
        auto get3 = [&](double *dst, const double4 *src) -> cudaError_t {
            if (!dst) return cudaSuccess;
            tmp.resize(N);
            cudaError_t e = cudaMemcpyAsync(tmp.data(), src, sizeof(double4) * N, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return e;
            for (int64_t kn = 0; kn < N; ++kn) {
                const int64_t k = p.node_new2old[kn];
                dst[3 * k] = tmp[kn].x;
                dst[3 * k + 1] = tmp[kn].y;
                dst[3 * k + 2] = tmp[kn].z;
            }
            return cudaSuccess;
        };
        CUDA_TRY(get3(out->u, ucur));
        CUDA_TRY(get3(out->v, ctx->d.v));
        CUDA_TRY(get3(out->a, ctx->d.a));
        if (out->tet_state)
            for (int64_t en = 0; en < E; ++en) out->tet_state[p.tet_new2old[en]] = stt[en];
        if (out->mass) {
            std::vector<double> m(N);
            CUDA_TRY(cudaMemcpyAsync(m.data(), ctx->d.mass, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaStreamSynchronize(st));
            for (int64_t kn = 0; kn < N; ++kn) out->mass[p.node_new2old[kn]] = m[kn];
        }
        const int64_t nr = std::min<int64_t>(nrec, out->rec_capacity);
        for (int64_t i = 0; i < nr; ++i) {
            const int64_t j = ord[i];
            if (out->rec_step) out->rec_step[i] = rs[j];
            if (out->rec_elem) out->rec_elem[i] = re[j];
            if (out->rec_cand) out->rec_cand[i] = rk[j];
            if (out->rec_G) out->rec_G[i] = rg[j];
            if (out->rec_area) out->rec_area[i] = ra[j];
        }
    }
    out->step = ctx->step;
    out->dt = h.dt;
    out->time = (double)ctx->step * h.dt;
    out->n_records = nrec;
    out->dissipated = Ud;
    out->n_active = na;
    out->nonfinite = ctr[1];
    out->nonfinite_node = ctr[1] ? ctr[2] : -1;
    return ctr[1] ? CEM_ENONFINITE : CEM_OK;
}

cem_status cem_partition(const cem_mesh_in *mesh, int nranks, int rank, cem_part_out *out) {
    if (!mesh || !mesh->X || !mesh->tets || !out || nranks < 1 || rank < 0 || rank >= nranks) return CEM_EINVAL;
    for (int64_t i = 0; i < 4 * mesh->n_tets; ++i)
        if (mesh->tets[i] < 0 || mesh->tets[i] >= mesh->n_nodes) {
            g_init_err = "cem_partition: node index out of range";
            return CEM_ETOPOLOGY;
        }
    PartGlobal g;
    PartLocal L;
    build_partition(mesh->n_nodes, mesh->X, mesh->n_tets, mesh->tets, nranks, g);
    build_exchange(g, rank, L);
    fill_part_out(g, L, out);
    return CEM_OK;
}

void cem_partition_free(cem_part_out *o) {
    if (!o) return;
    free(o->tet_global); free(o->tet_flag); free(o->node_global); free(o->node_owned); free(o->peers);
    free(o->send_node_off); free(o->recv_node_off); free(o->send_tet_off); free(o->recv_tet_off);
    free(o->send_nodes); free(o->recv_nodes); free(o->send_tets); free(o->recv_tets);
    free(o->tet_owner); free(o->node_owner);
    std::memset(o, 0, sizeof *o);
}

cem_status cem_nccl_unique_id(void *id128) {
    if (!id128) return CEM_EINVAL;
    return nccl_unique_id(id128, g_init_err) ? CEM_OK : CEM_ENCCL;
}

cem_status cem_step_group(cem_ctx **c, int32_t n, int64_t nsteps, int32_t crack_every) {
    if (!c || n < 1 || nsteps < 0) return CEM_EINVAL;
    for (int r = 0; r < n; ++r)
        if (!c[r] || !c[r]->dist || !c[r]->loopback || c[r]->nranks != n || c[r]->rank != r || c[r]->step != c[0]->step)
            return CEM_EINVAL;
    cem_ctx *ctx = c[0];
    if (crack_every < 0) crack_every = 0;
    for (int r = 1; r < n; ++r) {  // every rank's work goes on rank 0's stream, in rank order
        CUDA_TRY(cudaStreamSynchronize(c[r]->stream));
    }
    for (int r = 0; r < n; ++r) {  // ... after the work the callers put on their streams
        CUDA_TRY(cudaEventRecord(c[r]->fence_in, c[r]->user_stream));
        CUDA_TRY(cudaStreamWaitEvent(ctx->stream, c[r]->fence_in, 0));
    }
    if (c[0]->init_exchange_pending) {
        cem_status st = exchange_loopback(c, n, 1);
        if (st) return st;
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        for (int r = 0; r < n; ++r) c[r]->init_exchange_pending = false;
        if (c[0]->flags & CEM_F_P2P) {
            st = p2p_setup_loopback(c, n);
            if (st) return st;
        }
    }
    for (int64_t i = 0; i < nsteps; ++i) {
        const int64_t sstep = c[0]->step + i;
        for (int r = 0; r < n; ++r) {
            c[r]->launches += launch_staged_step(c[r]->d, sstep, crack_every, ctx->stream, nullptr,
                                                    crit_heavy(c[r]) ? CRIT_HEAVY : CRIT_LIST, &c[r]->sy);
        }
        if (c[0]->p2p.on) {  // the stores went straight into the peers' buffers; stream order syncs
            for (int r = 0; r < n; ++r) {
                exchange_unpack(c[r]->xch, c[r]->d.ubuf[sstep & 1], c[r]->d.state, c[r]->d.eedge, c[r]->h.E,
                                c[r]->d.edge_dirty, ctx->stream, c[r]->p2p.recv[sstep & 1]);
                c[r]->launches += 1;
            }
            continue;
        }
        cem_status st = exchange_loopback(c, n, (int)(sstep & 1));
        if (st) return st;
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < n; ++r) c[r]->step += nsteps;
    return CEM_OK;
}

cem_status cem_merge_records(int64_t n, const int64_t *step, const int32_t *elem, const double *area,
                             const double *gc, int64_t *order_out, double *dissipated_out) {
    if (n < 0 || (n > 0 && (!step || !elem || !area || !gc))) return CEM_EINVAL;
    std::vector<int64_t> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) {
        return step[x] < step[y] || (step[x] == step[y] && elem[x] < elem[y]);
    });
    double Ud = 0.0;
    for (int64_t i = 0; i < n; ++i) Ud = Ud + gc[elem[ord[i]]] * area[ord[i]];
    if (order_out) std::memcpy(order_out, ord.data(), sizeof(int64_t) * n);
    if (dissipated_out) *dissipated_out = Ud;
    return CEM_OK;
}

}  // extern "C"
