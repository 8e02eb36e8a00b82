// cem_api.cu -- the C ABI of libcem.so (include/cem.h): context, device workspace layout,
// host<->device transfers, CUDA-graph step loop, state readback.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "cem_internal.h"

namespace cem {
void launch_crack_only(const DevMesh &m, const DevState &s, int cur, cudaStream_t st);
}

using namespace cem;

struct cem_ctx {
    HostMesh h;
    DevMesh m{};
    DevState s{};
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int device = 0;
    void *ws = nullptr;
    size_t ws_bytes = 0;
    bool own_ws = false;
    int cur = 0;                  // u[cur] = u_n
    int64_t host_step = 0;        // steps enqueued
    uint32_t flags = 0;
    // graphs: [parity] for a given crack_every
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    int graph_crack = -1;
    bool profiling = false;
    std::vector<cudaEvent_t> ev;  // profiling events, (K_COUNT + 1) per step
    int64_t prof_steps = 0;
    std::string err;
};

namespace {

thread_local std::string g_init_err;

#define CUDA_TRY(x)                                                                   \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            ctx->err = std::string(#x) + ": " + cudaGetErrorString(e_);               \
            return CEM_ECUDA;                                                         \
        }                                                                             \
    } while (0)

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
    size_t off = 0;
    template <class T>
    size_t take(int64_t n) {
        size_t o = off;
        off = align_up(off + sizeof(T) * (size_t)(n > 0 ? n : 1));
        return o;
    }
};

// device layout, in one workspace
struct Offs {
    size_t X, tet, state, gc, geo, elem_edge, edge_off, edge_inc, node_off, node_ent, mass, fext, nflag, dir_v0;
    size_t u0, u1, v, a, tau, sig, fe, ctr, step, Ud, nrec, flag_list, flag_cand, flag_G, flag_area, flag;
    size_t rec_step, rec_elem, rec_cand, rec_G, rec_area;
    size_t total;
};

Offs layout(int64_t N, int64_t E, int64_t S, bool dir) {
    Layout L;
    Offs o{};
    o.X = L.take<double4>(N);
    o.tet = L.take<int4>(E);
    o.state = L.take<uint8_t>(E);
    o.gc = L.take<double>(E);
    o.geo = L.take<double>(16 * E);
    o.elem_edge = L.take<int32_t>(6 * E);
    o.edge_off = L.take<int32_t>(S + 1);
    o.edge_inc = L.take<int32_t>(6 * E);
    o.node_off = L.take<int32_t>(N + 1);
    o.node_ent = L.take<int32_t>(4 * E);
    o.mass = L.take<double>(N);
    o.fext = L.take<double4>(N);
    o.nflag = L.take<uint8_t>(N);
    o.dir_v0 = L.take<double4>(dir ? N : 1);
    o.u0 = L.take<double4>(N);
    o.u1 = L.take<double4>(N);
    o.v = L.take<double4>(N);
    o.a = L.take<double4>(N);
    o.tau = L.take<double>(6 * E);
    o.sig = L.take<double>(6 * S);
    o.fe = L.take<double>(12 * E);
    o.ctr = L.take<int32_t>(8);
    o.step = L.take<int64_t>(1);
    o.Ud = L.take<double>(1);
    o.nrec = L.take<int64_t>(1);
    o.flag_list = L.take<int32_t>(E);
    o.flag_cand = L.take<int32_t>(E);
    o.flag_G = L.take<double>(E);
    o.flag_area = L.take<double>(E);
    o.flag = L.take<uint8_t>(E);
    o.rec_step = L.take<int64_t>(E);
    o.rec_elem = L.take<int32_t>(E);
    o.rec_cand = L.take<int32_t>(E);
    o.rec_G = L.take<double>(E);
    o.rec_area = L.take<double>(E);
    o.total = L.off;
    return o;
}

template <class T>
T *at(void *base, size_t off) {
    return reinterpret_cast<T *>(static_cast<char *>(base) + off);
}

cem_status upload(cem_ctx *ctx, const Offs &o) {
    const HostMesh &h = ctx->h;
    const int64_t N = h.N, E = h.E, S = h.S;
    void *b = ctx->ws;
    cudaStream_t st = ctx->stream;
    std::vector<double4> X4(N), f4(N), d4(ctx->h.any_dirichlet ? N : 1), z4(N, make_double4(0, 0, 0, 0));
    for (int64_t n = 0; n < N; ++n) {
        X4[n] = make_double4(h.X[3 * n], h.X[3 * n + 1], h.X[3 * n + 2], 0.0);
        f4[n] = make_double4(h.fext[3 * n], h.fext[3 * n + 1], h.fext[3 * n + 2], 0.0);
        if (h.any_dirichlet) d4[n] = make_double4(h.dir_v0[3 * n], h.dir_v0[3 * n + 1], h.dir_v0[3 * n + 2], 0.0);
    }
    // initial state (R17): u_0 = 0, v_0 = 0 / vbar(0), a_0 = f_ext/m / vbar'(0), frozen 0;
    // u_1 = (u_0 + dt v_0) + (dt^2/2) a_0
    std::vector<double4> v4(N), a4(N), u1(N);
    const double dt = h.dt, hdt2 = 0.5 * h.dt * h.dt;
    for (int64_t n = 0; n < N; ++n) {
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
        v4[n] = make_double4(vv[0], vv[1], vv[2], 0.0);
        a4[n] = make_double4(aa[0], aa[1], aa[2], 0.0);
        u1[n] = make_double4(uu[0], uu[1], uu[2], 0.0);
    }
    std::vector<int4> t4(E);
    for (int64_t e = 0; e < E; ++e) t4[e] = make_int4(h.tet[4 * e], h.tet[4 * e + 1], h.tet[4 * e + 2], h.tet[4 * e + 3]);
    auto put = [&](size_t off, const void *src, size_t bytes) -> cudaError_t {
        return cudaMemcpyAsync(at<char>(b, off), src, bytes, cudaMemcpyHostToDevice, st);
    };
    CUDA_TRY(put(o.X, X4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.tet, t4.data(), sizeof(int4) * E));
    CUDA_TRY(put(o.state, h.state.data(), E));
    CUDA_TRY(put(o.gc, h.gc.data(), sizeof(double) * E));
    CUDA_TRY(put(o.geo, h.geo.data(), sizeof(double) * 16 * E));
    CUDA_TRY(put(o.elem_edge, h.elem_edge.data(), sizeof(int32_t) * 6 * E));
    CUDA_TRY(put(o.edge_off, h.edge_off.data(), sizeof(int32_t) * (S + 1)));
    CUDA_TRY(put(o.edge_inc, h.edge_inc.data(), sizeof(int32_t) * 6 * E));
    CUDA_TRY(put(o.node_off, h.node_off.data(), sizeof(int32_t) * (N + 1)));
    CUDA_TRY(put(o.node_ent, h.node_ent.data(), sizeof(int32_t) * 4 * E));
    CUDA_TRY(put(o.mass, h.mass.data(), sizeof(double) * N));
    CUDA_TRY(put(o.fext, f4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.nflag, h.nflag.data(), N));
    if (h.any_dirichlet) CUDA_TRY(put(o.dir_v0, d4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.u0, z4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.u1, u1.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.v, v4.data(), sizeof(double4) * N));
    CUDA_TRY(put(o.a, a4.data(), sizeof(double4) * N));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.tau), 0, sizeof(double) * 6 * E, st));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.sig), 0, sizeof(double) * 6 * S, st));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.fe), 0, sizeof(double) * 12 * E, st));
    int32_t ctr[8] = {0, 0, INT32_MAX, 0, 0, 0, 0, 0};
    CUDA_TRY(put(o.ctr, ctr, sizeof ctr));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.step), 0, sizeof(int64_t), st));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.Ud), 0, sizeof(double), st));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.nrec), 0, sizeof(int64_t), st));
    CUDA_TRY(cudaMemsetAsync(at<char>(b, o.flag), 0, E, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return CEM_OK;
}

void bind_views(cem_ctx *ctx, const Offs &o) {
    void *b = ctx->ws;
    const HostMesh &h = ctx->h;
    DevMesh &m = ctx->m;
    m.N = h.N;
    m.E = h.E;
    m.S = h.S;
    m.X = at<double4>(b, o.X);
    m.tet = at<int4>(b, o.tet);
    m.state = at<uint8_t>(b, o.state);
    m.gc = at<double>(b, o.gc);
    m.geo = at<double>(b, o.geo);
    m.elem_edge = at<int32_t>(b, o.elem_edge);
    m.edge_off = at<int32_t>(b, o.edge_off);
    m.edge_inc = at<int32_t>(b, o.edge_inc);
    m.node_off = at<int32_t>(b, o.node_off);
    m.node_ent = at<int32_t>(b, o.node_ent);
    m.mass = at<double>(b, o.mass);
    m.fext = at<double4>(b, o.fext);
    m.nflag = at<uint8_t>(b, o.nflag);
    m.dir_v0 = at<double4>(b, o.dir_v0);
    m.lam = h.lam;
    m.mu = h.mu;
    m.l2m = h.l2m;
    m.rho = h.rho;
    m.dt = h.dt;
    m.gamma = h.gamma;
    m.t0 = h.t0;
    m.flags = ctx->flags;
    DevState &s = ctx->s;
    s.u[0] = at<double4>(b, o.u0);
    s.u[1] = at<double4>(b, o.u1);
    s.v = at<double4>(b, o.v);
    s.a = at<double4>(b, o.a);
    s.tau = at<double>(b, o.tau);
    s.sig = at<double>(b, o.sig);
    s.fe = at<double>(b, o.fe);
    s.ctr = at<int32_t>(b, o.ctr);
    s.step = at<int64_t>(b, o.step);
    s.Ud = at<double>(b, o.Ud);
    s.nrec = at<int64_t>(b, o.nrec);
    s.flag_list = at<int32_t>(b, o.flag_list);
    s.flag_cand = at<int32_t>(b, o.flag_cand);
    s.flag_G = at<double>(b, o.flag_G);
    s.flag_area = at<double>(b, o.flag_area);
    s.flag = at<uint8_t>(b, o.flag);
    s.rec_step = at<int64_t>(b, o.rec_step);
    s.rec_elem = at<int32_t>(b, o.rec_elem);
    s.rec_cand = at<int32_t>(b, o.rec_cand);
    s.rec_G = at<double>(b, o.rec_G);
    s.rec_area = at<double>(b, o.rec_area);
    s.flag_cap = (int32_t)h.E;
}

void enqueue_step(cem_ctx *ctx, int cur, int crack_every, cudaStream_t st) {
    launch_strain(ctx->m, ctx->s, cur, st);
    launch_edge(ctx->m, ctx->s, st);
    launch_force(ctx->m, ctx->s, cur, crack_every, st);
    launch_node(ctx->m, ctx->s, cur, st);
    launch_split(ctx->m, ctx->s, cur, crack_every, 1, st);
}

void destroy_graphs(cem_ctx *ctx) {
    for (auto &g : ctx->graph)
        if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
        }
    ctx->graph_crack = -1;
}

cem_status build_graphs(cem_ctx *ctx, int crack_every) {
    destroy_graphs(ctx);
    for (int par = 0; par < 2; ++par) {
        cudaGraph_t g;
        CUDA_TRY(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        enqueue_step(ctx, par, crack_every, ctx->stream);
        CUDA_TRY(cudaStreamEndCapture(ctx->stream, &g));
        CUDA_TRY(cudaGraphInstantiate(&ctx->graph[par], g, 0));
        cudaGraphDestroy(g);
    }
    ctx->graph_crack = crack_every;
    return CEM_OK;
}

}  // namespace

extern "C" {

int32_t cem_abi_version(void) { return CEM_ABI_VERSION; }

const char *cem_last_error(const cem_ctx *ctx) { return ctx ? ctx->err.c_str() : g_init_err.c_str(); }

cem_status cem_workspace_size(const cem_mesh_in *mesh, const cem_opts *opts, size_t *bytes) {
    if (!mesh || !bytes) return CEM_EINVAL;
    int64_t S = 0;
    cem_status st = count_edges(mesh, &S, g_init_err);
    if (st) return st;
    (void)opts;
    *bytes = layout(mesh->n_nodes, mesh->n_tets, S, true).total;
    return CEM_OK;
}

cem_status cem_init_mesh(const cem_mesh_in *mesh, const cem_material *mat, const cem_load_in *load,
                         const cem_opts *opts, cem_ctx **out) {
    if (!out) return CEM_EINVAL;
    *out = nullptr;
    g_init_err.clear();
    cem_ctx *ctx = new cem_ctx();
    cem_status st = build_host_mesh(mesh, mat, load, opts, ctx->h, ctx->err);
    auto fail = [&](cem_status s) {
        g_init_err = ctx->err;
        if (ctx->own_ws && ctx->ws) cudaFree(ctx->ws);
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        delete ctx;
        return s;
    };
    if (st) return fail(st);
    if (opts && opts->nranks > 1) {
        ctx->err = "multi-GPU context not supported by this entry point (use the partitioned driver)";
        return fail(CEM_EINVAL);
    }
    ctx->device = opts ? opts->device : 0;
    ctx->flags = opts ? opts->flags : 0;
    ctx->stream = opts ? (cudaStream_t)opts->stream : nullptr;
    if (cudaSetDevice(ctx->device) != cudaSuccess) {
        ctx->err = "cudaSetDevice failed";
        return fail(CEM_ECUDA);
    }
    if (!ctx->stream) {  // graphs cannot be captured on the legacy default stream
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
            ctx->err = "cudaStreamCreate failed";
            return fail(CEM_ECUDA);
        }
        ctx->own_stream = true;
    }
    Offs o = layout(ctx->h.N, ctx->h.E, ctx->h.S, ctx->h.any_dirichlet);
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
    bind_views(ctx, o);
    st = upload(ctx, o);
    if (st) return fail(st);
    *out = ctx;
    return CEM_OK;
}

void cem_destroy(cem_ctx *ctx) {
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    else cudaDeviceSynchronize();
    destroy_graphs(ctx);
    for (auto e : ctx->ev) cudaEventDestroy(e);
    if (ctx->own_ws && ctx->ws) cudaFree(ctx->ws);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

cem_status cem_sizes(const cem_ctx *ctx, int64_t *n_nodes, int64_t *n_tets, int64_t *n_edges) {
    if (!ctx) return CEM_EINVAL;
    if (n_nodes) *n_nodes = ctx->h.N;
    if (n_tets) *n_tets = ctx->h.E;
    if (n_edges) *n_edges = ctx->h.S;
    return CEM_OK;
}

int32_t cem_launches_per_step(const cem_ctx *ctx) { return ctx ? (int32_t)K_COUNT : 0; }

cem_status cem_set_profiling(cem_ctx *ctx, int on) {
    if (!ctx) return CEM_EINVAL;
    ctx->profiling = on != 0;
    ctx->prof_steps = 0;
    return CEM_OK;
}

cem_status cem_step(cem_ctx *ctx, int64_t nsteps, int32_t crack_every) {
    if (!ctx || nsteps < 0) return CEM_EINVAL;
    if (crack_every < 0) crack_every = 0;
    if (ctx->profiling) {
        // eager launches bracketed by events (per-kernel durations on the launching stream)
        const size_t need = (size_t)(ctx->prof_steps + nsteps) * (K_COUNT + 1);
        while (ctx->ev.size() < need) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreate(&e));
            ctx->ev.push_back(e);
        }
        for (int64_t i = 0; i < nsteps; ++i) {
            cudaEvent_t *E = ctx->ev.data() + (ctx->prof_steps + i) * (K_COUNT + 1);
            CUDA_TRY(cudaEventRecord(E[0], ctx->stream));
            launch_strain(ctx->m, ctx->s, ctx->cur, ctx->stream);
            CUDA_TRY(cudaEventRecord(E[1], ctx->stream));
            launch_edge(ctx->m, ctx->s, ctx->stream);
            CUDA_TRY(cudaEventRecord(E[2], ctx->stream));
            launch_force(ctx->m, ctx->s, ctx->cur, crack_every, ctx->stream);
            CUDA_TRY(cudaEventRecord(E[3], ctx->stream));
            launch_node(ctx->m, ctx->s, ctx->cur, ctx->stream);
            CUDA_TRY(cudaEventRecord(E[4], ctx->stream));
            launch_split(ctx->m, ctx->s, ctx->cur, crack_every, 1, ctx->stream);
            CUDA_TRY(cudaEventRecord(E[5], ctx->stream));
            ctx->cur ^= 1;
        }
        CUDA_TRY(cudaGetLastError());
        ctx->prof_steps += nsteps;
        ctx->host_step += nsteps;
        return CEM_OK;
    }
    if (ctx->graph_crack != crack_every) {
        cem_status st = build_graphs(ctx, crack_every);
        if (st) return st;
    }
    for (int64_t i = 0; i < nsteps; ++i) {
        CUDA_TRY(cudaGraphLaunch(ctx->graph[ctx->cur], ctx->stream));
        ctx->cur ^= 1;
    }
    ctx->host_step += nsteps;
    return CEM_OK;
}

cem_status cem_kernel_times(const cem_ctx *ctx, int32_t *n, const char **names, double *ms, int32_t cap) {
    if (!ctx || !n) return CEM_EINVAL;
    *n = K_COUNT;
    if (cap < K_COUNT) return CEM_OK;
    for (int k = 0; k < K_COUNT; ++k) {
        if (names) names[k] = kKernelNames[k];
        double tot = 0.0;
        for (int64_t i = 0; i < ctx->prof_steps; ++i) {
            float t = 0.f;
            cudaEvent_t *E = const_cast<cudaEvent_t *>(ctx->ev.data()) + i * (K_COUNT + 1);
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
    int64_t before = 0, after = 0;
    CUDA_TRY(cudaMemcpyAsync(&before, ctx->s.nrec, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    launch_crack_only(ctx->m, ctx->s, ctx->cur, ctx->stream);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(&after, ctx->s.nrec, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (n_split_out) *n_split_out = after - before;
    return CEM_OK;
}

cem_status cem_get_state(cem_ctx *ctx, cem_state_out *out, int where) {
    if (!ctx || !out) return CEM_EINVAL;
    cudaStream_t st = ctx->stream;
    const int64_t N = ctx->h.N, E = ctx->h.E;
    int64_t step = 0, nrec = 0;
    double Ud = 0.0;
    int32_t ctr[8];
    CUDA_TRY(cudaMemcpyAsync(&step, ctx->s.step, sizeof step, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&nrec, ctx->s.nrec, sizeof nrec, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&Ud, ctx->s.Ud, sizeof Ud, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(ctr, ctx->s.ctr, sizeof ctr, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    double4 *ucur = ctx->s.u[ctx->cur];
    if (where == CEM_DEVICE) {
        out->u = reinterpret_cast<double *>(ucur);  // NB: device views are double4-strided
        out->v = reinterpret_cast<double *>(ctx->s.v);
        out->a = reinterpret_cast<double *>(ctx->s.a);
        out->tet_state = ctx->m.state;
        out->mass = ctx->m.mass;
        out->rec_step = ctx->s.rec_step;
        out->rec_elem = ctx->s.rec_elem;
        out->rec_cand = ctx->s.rec_cand;
        out->rec_G = ctx->s.rec_G;
        out->rec_area = ctx->s.rec_area;
    } else {
        std::vector<double4> tmp;
        auto get3 = [&](double *dst, const double4 *src) -> cudaError_t {
            if (!dst) return cudaSuccess;
            tmp.resize(N);
            cudaError_t e = cudaMemcpyAsync(tmp.data(), src, sizeof(double4) * N, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) return e;
            e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return e;
            for (int64_t n = 0; n < N; ++n) {
                dst[3 * n] = tmp[n].x;
                dst[3 * n + 1] = tmp[n].y;
                dst[3 * n + 2] = tmp[n].z;
            }
            return cudaSuccess;
        };
        CUDA_TRY(get3(out->u, ucur));
        CUDA_TRY(get3(out->v, ctx->s.v));
        CUDA_TRY(get3(out->a, ctx->s.a));
        if (out->tet_state) CUDA_TRY(cudaMemcpyAsync(out->tet_state, ctx->m.state, E, cudaMemcpyDeviceToHost, st));
        if (out->mass) CUDA_TRY(cudaMemcpyAsync(out->mass, ctx->m.mass, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        const int64_t nr = std::min<int64_t>(nrec, out->rec_capacity);
        if (nr > 0) {
            if (out->rec_step) CUDA_TRY(cudaMemcpyAsync(out->rec_step, ctx->s.rec_step, 8 * nr, cudaMemcpyDeviceToHost, st));
            if (out->rec_elem) CUDA_TRY(cudaMemcpyAsync(out->rec_elem, ctx->s.rec_elem, 4 * nr, cudaMemcpyDeviceToHost, st));
            if (out->rec_cand) CUDA_TRY(cudaMemcpyAsync(out->rec_cand, ctx->s.rec_cand, 4 * nr, cudaMemcpyDeviceToHost, st));
            if (out->rec_G) CUDA_TRY(cudaMemcpyAsync(out->rec_G, ctx->s.rec_G, 8 * nr, cudaMemcpyDeviceToHost, st));
            if (out->rec_area) CUDA_TRY(cudaMemcpyAsync(out->rec_area, ctx->s.rec_area, 8 * nr, cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    out->step = step;
    out->dt = ctx->h.dt;
    out->time = (double)step * ctx->h.dt;
    out->n_records = nrec;
    out->dissipated = Ud;
    out->n_active = 0;
    {
        // active count from the state bytes (host copy when available)
        std::vector<uint8_t> stt(E);
        CUDA_TRY(cudaMemcpyAsync(stt.data(), ctx->m.state, E, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        int64_t na = 0;
        for (int64_t e = 0; e < E; ++e) na += stt[e] != 0;
        out->n_active = na;
    }
    out->nonfinite = ctr[1];
    out->nonfinite_node = ctr[1] ? ctr[2] : -1;
    return ctr[1] ? CEM_ENONFINITE : CEM_OK;
}

}  // extern "C"
