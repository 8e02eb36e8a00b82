// cem_kernels.cu -- sm_100a kernels of the CEM explicit step.
//
// Compiled with --fmad=false: every product and sum rounds exactly as written, in the
// association order fixed by the oracle, so results are
// bitwise reproducible and equal to the CPU oracle's.  No floating-point atomics: every
// output is produced by one thread that sums its inputs sequentially in ascending
// ORIGINAL element id (deterministic CSR gathers).
//
// Stages of one explicit step s -> s+1 (u_{s+1} already predicted, stored in ubuf[(s+1)&1]):
//   A  tau_e = V_e eps_e(u_{s+1}) per tet
//   B  Vhat_s, eps~_s = (sum tau_e)/Vhat_s, sigma_s per edge
//   C  f_e = (V_e/6) B^T sum_l sigma_{s(e,l)} per tet; crack
//      criterion's conservative early-out; the tets that fail it
//      are listed for k_crit (24 candidates, one warp per tet),
//      which splits
//   D  f_int gather, Newmark + BC, mass/freeze of split nodes,
//      predictor u_{s+2} -> ubuf[s&1] (+ reaction work, N1)
// Vhat_s is kept per edge (table, recomputed only where a split changed it).
//
// k_persistent runs K steps in ONE launch: CTAs pull (stage, block) work items from a
// global queue in a precomputed wavefront order (cem_plan.cpp) and wait only on the
// completed-step counters of the producer blocks they read.  Consecutive steps overlap;
// intermediates stay L2-resident between producer and consumer.
#include <algorithm>
#include <cstdint>
#include <mutex>

#include "cem_internal.h"

namespace cem {

const int kThreads = 256;

namespace {

// Bounds checks of the debug build (-DCEM_DEBUG_BOUNDS, libcem_dbg.so; compute-sanitizer is not
// available on the GPU pool): the first violated check stores its source line in ctr[20], which
// cem_get_state reports as CEM_ESTATE.  Compiled out of the product build.
#ifdef CEM_DEBUG_BOUNDS
#define CEM_BOUND(dev, cond)                                        \
    do {                                                            \
        if (!(cond)) atomicCAS(&(dev).ctr[20], 0, (int)__LINE__);   \
    } while (0)
#else
#define CEM_BOUND(dev, cond) \
    do {                     \
    } while (0)
#endif

// read-only tables: non-coherent path
__device__ __forceinline__ double ldro(const double *p) { return __ldg(p); }
__device__ __forceinline__ int ldro(const int32_t *p) { return __ldg(p); }
// criterion-list entry of step s's crack check (rec_step = s + 1): the stamp tells k_crit's
// pollers an entry of their own step from one left by an earlier step
__device__ __forceinline__ int64_t crit_entry(int64_t rec_step, int64_t e) { return (rec_step << 32) | e; }
__device__ __forceinline__ double4 ldro4(const double4 *p) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
    const double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}
// data written inside the kernel (coherent path; L1 invalidated after every acquire)
__device__ __forceinline__ double4 ld4(const double4 *p) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
    const double2 a = q[0], b = q[1];
    return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st4(double4 *p, double x, double y, double z, double w) {
    double2 *q = reinterpret_cast<double2 *>(p);
    q[0] = make_double2(x, y);
    q[1] = make_double2(z, w);
}

[[maybe_unused]] __device__ __forceinline__ void st256(double4 *p, double x, double y, double z, double w) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(x), "d"(y), "d"(z), "d"(w) : "memory");
}
#if CEM_FES == 4
__device__ __forceinline__ void store_slot(double *p, double x, double y, double z) {  // (x, y, z, 0)
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(x), "d"(y), "d"(z), "d"(0.0) : "memory");
}
#endif
__device__ __forceinline__ void st128(double *p, double x, double y) {
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ double2 ldcg128(const double *p) {
    double2 r;
    asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
// Data produced inside the same (persistent) kernel by other CTAs is read at L2 (.cg,
// LDG.STRONG.GPU): no stale L1 lines, so no SM-wide L1 invalidation is needed per work item.
__device__ __forceinline__ double4 ldcg256(const double4 *p) {
    double4 r;
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ double4 ldro256(const double *p) {  // read-only 32-B load (LDG.E.256.CONSTANT)
    double4 r;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
#if CEM_GEO_AOS
// geometry record per tet (96 B): V, V/6, gradN1..3 (x, y, z), 0 -- three 32-B loads
__device__ __forceinline__ double geo_V(const Dev &d, uint32_t e) { return __ldg(d.geoT + 12u * e); }
__device__ __forceinline__ void geo_record(const Dev &d, uint32_t e, double (&g)[4][3], double &V, double &V6) {
    const double *p = d.geoT + 12u * e;
    const double4 a = ldro256(p), b = ldro256(p + 4), c = ldro256(p + 8);
    V = a.x;
    V6 = a.y;
    g[1][0] = a.z; g[1][1] = a.w; g[1][2] = b.x;
    g[2][0] = b.y; g[2][1] = b.z; g[2][2] = b.w;
    g[3][0] = c.x; g[3][1] = c.y; g[3][2] = c.z;
}
#else
// warp-tiled geometry: tet e -> tile e>>5, lane e&31, component c at [tile][c][lane]
__device__ __forceinline__ const double *geo_ptr(const Dev &d, uint32_t e) { return d.geoT + ((e >> 5) * 352u + (e & 31u)); }
__device__ __forceinline__ double geo_V(const Dev &d, uint32_t e) { return __ldg(geo_ptr(d, e)); }
__device__ __forceinline__ void geo_record(const Dev &d, uint32_t e, double (&g)[4][3], double &V, double &V6) {
    const double *gp = geo_ptr(d, e);
#pragma unroll
    for (int a = 1; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) g[a][c] = __ldg(gp + 32 * (2 + 3 * (a - 1) + c));
    V = __ldg(gp);
    V6 = __ldg(gp + 32);
}
#endif
#if CEM_FES == 3
__device__ __forceinline__ int64_t slot_tet(int32_t slot) { return slot >> 2; }  // slot = 4e + a
#else
__device__ __forceinline__ int64_t slot_tet(int32_t slot) { return ((int64_t)(slot >> 7) << 5) + (slot & 31); }
#endif

// lumped mass of node k from its active incidences in original order
#ifndef CEM_MASS_BATCH
#define CEM_MASS_BATCH 4  // (8 costs stage D a spill: +2.6 us per step on config 3)
#endif
// (CEM_MASS_BATCH incidences at a time: their slot, state and volume loads are issued together,
// three round trips per batch instead of three per incidence; the sum stays sequential in
// ascending order)
__device__ __forceinline__ double node_mass(const Dev &d, int64_t k) {
    constexpr int B = CEM_MASS_BATCH;
    double acc = 0.0;
    const int32_t *row = d.nodeE + k * d.wn;  // wn is a multiple of 8
    for (int j = 0; j < d.wn; j += B) {
        int32_t sl[B];
        uint8_t st[B];
        double V[B];
#pragma unroll
        for (int t = 0; t < B; ++t) sl[t] = __ldg(row + j + t);
#pragma unroll
        for (int t = 0; t < B; ++t) {
            const bool ok = sl[t] != d.zslot;
            const int64_t e = ok ? slot_tet(sl[t]) : 0;
            st[t] = ok ? __ldcg(d.state + e) : (uint8_t)0;
            V[t] = ok ? geo_V(d, (uint32_t)e) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < B; ++t)
            if (st[t]) acc = acc + (d.rho * V[t]) / 4.0;
        if (sl[B - 1] == d.zslot) break;  // padding only at the row's end
    }
    return acc;
}

// The same mass, computed by the node's four stage-D lanes together (called by all four, lane c
// = threadIdx.x & 3): each round, lane c loads incidences j+4c .. j+4c+3 (one 16-B row load, then
// their state and volume), so 16 incidences cost one round trip instead of four; every lane then
// forms the identical sequential sum in ascending order from the shuffled terms.  An inactive
// incidence contributes -0.0, which leaves any partial sum bit-for-bit unchanged (acc + -0 = acc),
// so the sum equals node_mass()'s conditional one.
__device__ __forceinline__ double node_mass4(const Dev &d, int64_t k, int c) {
    const unsigned gm = 0xFu << (threadIdx.x & 28u);
    const int g0 = (int)(threadIdx.x & 28u);
    const int4 *row = reinterpret_cast<const int4 *>(d.nodeE + k * d.wn);  // wn is a multiple of 8
    double acc = 0.0;
    for (int j = 0; j < d.wn; j += 16) {
        const int4 q = j + 4 * c < d.wn ? __ldg(row + (j >> 2) + c) : make_int4(d.zslot, d.zslot, d.zslot, d.zslot);
        const int32_t sl[4] = {q.x, q.y, q.z, q.w};
        double x[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const bool ok = sl[t] != d.zslot;
            const int64_t e = ok ? slot_tet(sl[t]) : 0;
            const uint8_t st = ok ? __ldcg(d.state + e) : (uint8_t)0;
            const double V = ok ? geo_V(d, (uint32_t)e) : 0.0;
            x[t] = st ? (d.rho * V) / 4.0 : -0.0;
        }
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
#pragma unroll
            for (int t = 0; t < 4; ++t) acc = acc + __shfl_sync(gm, x[t], g0 + cc);
        if (__shfl_sync(gm, q.w, g0 + 3) == d.zslot) break;  // padding only at the row's end
    }
    return acc;
}

// lumped mass of node k of a hexahedral context (R24, R29; the hex oracle's node_mass): incidences
// (e, a) ascending, the hex's rho V / 8 or its active remainder tets' rho V_t / 4
__device__ __noinline__ double hex_node_mass(const Dev *__restrict__ dp, int64_t k) {
    const Dev &d = *dp;
    const int32_t *row = d.nodeE + k * d.wn;
    double acc = 0.0;
    for (int j = 0; j < d.wn; ++j) {  // the row's sub-0 prefix: one entry per incident hex, ascending e
        const int32_t sl = __ldg(row + j);
        if (sl >= 8 * (int32_t)d.E) break;  // (a remainder slot or the padding)
        const int64_t e = sl >> 3;
        const int a = sl & 7;
        if (__ldcg(d.state + e)) {
            acc = acc + (d.rho * __ldg(d.hgeo + e)) / 8.0;
            continue;
        }
        if (__ldcg(d.hrem + e) < 0) continue;
        const uint8_t ta = __ldcg(d.htact + e);
        for (int i = 0; i < 3; ++i) {
            if (!(ta >> i & 1)) continue;
            const uint8_t *tl = d.htloc + 12 * e + 4 * i;
            if (tl[0] == a || tl[1] == a || tl[2] == a || tl[3] == a)
                acc = acc + (d.rho * __ldcg(d.htgeo + 39 * e + 13 * i)) / 4.0;
        }
    }
    return acc;
}

// Shared-memory staging: a block's deduplicated producer records (u of its nodes, sigma of its
// edges) are loaded once into component planes plane[c][row], so that every later per-thread
// gather hits shared memory; rows are assigned bank-aware by the plan (cem_plan.cpp bank_rows).

// programmatic dependent launch (PDL): let the next stage kernel launch early, and wait for
// the previous one only where its outputs are read
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- dataflow ("wave") launches (cem_plan.cpp build_wave): a block waits only for the producer
// blocks it reads.  Producer: all threads' writes, barrier, thread 0 stores the block's
// completed-step value (wcnt) with st.release.gpu (MEMBAR.ALL.GPU + strong store).  Consumer:
// warp 0 polls its producers' counters with ld.relaxed.gpu (strong L2 loads), then a barrier
// releases the block.  Every load of produced data in the stage bodies is a strong GPU-scope
// load served by L2 (__ldcg / ld.global.cg -> LDG.E.STRONG.GPU), issued after the poll that
// observed the flag returned, so it sees the producer's writes.  Deliberately NO acquire
// loads or __threadfence(): on sm_100a those compile to CCTL.IVALL, an invalidation of the
// SM's whole L1, and one per block start/finish cost the stage kernels 15-50 us per step
// (ncu, measured).  Launch order is a topological order of the dependencies and every kernel
// triggers its dependents at entry, so all producers of a resident block are resident or done.
__device__ __forceinline__ int ld_acquire_gpu(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int32_t *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int32_t *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wave_wait(const Dev &d, int g, int b, int need) {
    const int pg = g == ST_AB ? ST_D : g - 1;
    {  // every warp polls the block's producers itself (no barrier: warps start independently)
        const int lane = (int)(threadIdx.x & 31);
        const int64_t q = (int64_t)g * d.wmax + b;
        const int lo = __ldg(d.wdep_off + q), hi = __ldg(d.wdep_off + q + 1);
        const int32_t *c = d.wcnt + (int64_t)pg * d.wmax;
#ifdef CEM_WAVE_STATS
        int polls = 0;
#endif
        for (int i = lo + lane; i < hi; i += 32) {
            const int32_t *cp = c + __ldg(d.wdep + i);
            while (ld_relaxed_gpu(cp) < need) {
                __nanosleep(32);
#ifdef CEM_WAVE_STATS
                ++polls;
#endif
            }
        }
        __syncwarp();
#ifdef CEM_WAVE_STATS
        polls = __reduce_add_sync(0xffffffffu, polls);
        if (threadIdx.x == 0) {
            atomicAdd(&d.ctr[12 + (g == ST_D ? 2 : 0) + (g == ST_C ? 1 : 0)], polls ? 1 : 0);  // blocks that waited
            atomicAdd(reinterpret_cast<unsigned int *>(&d.ctr[7]), (unsigned)polls);
        }
#endif
    }
}
__device__ __forceinline__ void discard_lines(const void *base, int64_t off, int64_t bytes) {
    const char *p = static_cast<const char *>(base) + off;
    for (int64_t l = threadIdx.x; l < bytes / 128; l += blockDim.x)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(p + 128 * l) : "memory");
}
// Consumer block (stage g = C or D) done with its inputs: count it against each producer block; the
// last consumer of a producer block invalidates that block's intermediate lines in L2 without
// write-back (sigma records of an AB block, force slots of a C block), BEFORE it publishes its
// own completion -- the producer's next write happens-after that publication.
__device__ __forceinline__ void wave_discard(const Dev &d, int g, int b) {
    __shared__ int sh_n;
    __shared__ int sh_pb[32];
    __syncthreads();
    if (threadIdx.x == 0) sh_n = 0;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int64_t q = (int64_t)g * d.wmax + b;
        const int lo = __ldg(d.wdep_off + q), hi = __ldg(d.wdep_off + q + 1);
        int32_t *cd = d.wcons_done + (int64_t)(g - 1) * d.wmax;
        const int32_t *nc = d.wncons + (int64_t)(g - 1) * d.wmax;
        for (int i = lo + (int)threadIdx.x; i < hi; i += 32) {
            const int pb = __ldg(d.wdep + i);
            if (atomicAdd(cd + pb, 1) == __ldg(nc + pb) - 1) {
                cd[pb] = 0;
                const int k = atomicAdd(&sh_n, 1);
                if (k < 32) sh_pb[k] = pb;
            }
        }
    }
    __syncthreads();
    const int n = min(sh_n, 32);  // (a producer beyond 32 is left to normal eviction)
    for (int j = 0; j < n; ++j) {
        const int pb = sh_pb[j];
        if (g == ST_C) {  // sigma records of AB block pb: 32-B and 16-B planes
            const int64_t e0 = (int64_t)pb * d.blk_ab, ne = min((int64_t)d.blk_ab, d.S - e0);
            discard_lines(d.srec, e0 * 32, ne * 32);
            discard_lines(d.srec2, e0 * 16, ne * 16);
        } else {          // force slots of C block pb (12 doubles per tet)
#if CEM_FES == 3
            const int64_t t0 = (int64_t)pb * d.blk, nt = min((int64_t)d.blk, d.E - t0);
            discard_lines(d.fe, t0 * 96, nt * 96);
#endif
        }
    }
}
__device__ __forceinline__ void wave_done(const Dev &d, int g, int b, int val) {
    if (d.wdiscard && g != ST_AB) wave_discard(d, g, b);
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(d.wcnt + (int64_t)g * d.wmax + b, val);
}
// the stage bodies wait for their inputs here: wave launches on their producers' counters
// (wneed >= 0), staged launches on the previous kernel (PDL)
__device__ __forceinline__ void stage_wait(const Dev &d, int g, int b, int wneed) {
    if (wneed >= 0) wave_wait(d, g, b, wneed);
    else pdl_wait();
}

// plane strides are odd so the 8-byte planes of a record fall into different bank pairs
__host__ __device__ __forceinline__ int pstride(int n) { return n | 1; }

// exact-sum accumulation of the nodal assembly (reading R27): s is the running rounded sum, c
// collects the TwoSum rounding errors; RN(s + c) is the exact sum rounded once whenever c's
// additions are exact (the node's partial sums within 2^49 of its smallest nonzero term).
// Compiled with --fmad=false: no contraction may fuse these operations.
__device__ __forceinline__ void xacc(double &s, double &c, double x) {
    const double t = s + x;
    const double z = t - s;
    c = c + ((s - (t - z)) + (x - z));
    s = t;
}

// deterministic block sum (fixed shuffle tree, then the warps in order); valid in thread 0.
// Every thread of the block must call it.
__device__ __forceinline__ double block_sum(double x, double *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = x + __shfl_down_sync(0xffffffffu, x, o);
    __syncthreads();  // red may still be read by a previous call
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = t + red[i];
    return t;
}

// ------------------------------------------------------------------ stage AB: strain + edge stress
// For the edge block's deduplicated tet list: eps = sum_a B_a u_a (a = 0..3 in order), Voigt
// (11,22,33,12,23,13) with engineering shears, gradN0 = -((gradN1 + gradN2) + gradN3),
// tau = V eps -> shared-memory planes (V = 0 marks an inactive tet).
// Then per edge: Vhat = sum V_e, T = sum tau_e over the active incident tets in original-id
// order, eps~ = T * (1/Vhat), sigma_ii = (lam+2mu) eps_ii + lam (eps_jj +
// eps_kk), sigma_ij = mu gamma_ij, stored as a packed 48-B record.
// tau = V eps of one tet from its staged nodes (a = 0..3 in order) into row i of the planes
__device__ __forceinline__ void tau_row(double *T, int tn, int i, const double *U, int un, const double (&g)[4][3],
                                        double V, ushort4 lc) {
    const int li[4] = {lc.x, lc.y, lc.z, lc.w};
    double ex = 0.0, ey = 0.0, ez = 0.0, gxy = 0.0, gyz = 0.0, gxz = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const double ux = U[li[a]], uy = U[un + li[a]], uz = U[2 * un + li[a]];
        const double gx = g[a][0], gy = g[a][1], gz = g[a][2];
        ex = ex + gx * ux;
        ey = ey + gy * uy;
        ez = ez + gz * uz;
        gxy = gxy + (gy * ux + gx * uy);
        gyz = gyz + (gz * uy + gy * uz);
        gxz = gxz + (gz * ux + gx * uz);
    }
    T[i] = V * ex;
    T[tn + i] = V * ey;
    T[2 * tn + i] = V * ez;
    T[3 * tn + i] = V * gxy;
    T[4 * tn + i] = V * gyz;
    T[5 * tn + i] = V * gxz;
    T[6 * tn + i] = V;  // (plane 6: the volume of an active tet, for a dirty edge's Vhat)
}
__device__ __forceinline__ void zero_row(double *T, int tn, int i) {
#pragma unroll
    for (int c = 0; c < 6; ++c) T[c * tn + i] = 0.0;
    T[6 * tn + i] = -0.0;  // inactive tet / sentinel: adding -0.0 leaves any sum bit-for-bit unchanged
}
// the 9 stored gradients (nodes 1..3) and V of tet e; gradN0 = -((gradN1 + gradN2) + gradN3)
__device__ __forceinline__ void load_geo(const Dev &d, uint32_t e, double (&g)[4][3], double &V) {
    double V6;
    geo_record(d, e, g, V, V6);
}

__device__ __forceinline__ void grad0(double (&g)[4][3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) g[0][c] = -((g[1][c] + g[2][c]) + g[3][c]);
}

// Vhat_s of an edge with a tet split since the last step (splits mark their 6 edges; ghost splits
// arrive marked by the halo unpack), recomputed inside stage AB from the block's staged rows:
// plane 6 holds V of each active tet of the block's list (-0.0 for an inactive tet and for the
// sentinel row), and the edge's ELL row lists its incident tets in ascending original id -- the
// same terms in the same order as the oracle's stage_edge sum (V_e of the active incident tets,
// ascending original id; an inactive one adds -0.0), without a walk of the global incidence lists.  `update` writes the value back and clears the flag.
__device__ __forceinline__ double vhat_rows(const Dev &d, int64_t s, const double *T, int tn, int nt, uint4 q,
                                            bool update) {
    const double *Vr = T + 6 * tn;
    const uint4 *row = reinterpret_cast<const uint4 *>(d.incE + (uint32_t)s * (uint32_t)d.we);
    double acc = 0.0;
    for (int w = 0;;) {
        const uint32_t qq[4] = {q.x, q.y, q.z, q.w};
        const int lim = d.we_max - w;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (t >= lim) break;
            const int raw = (int)((qq[t >> 1] >> (16 * (t & 1))) & 0xffff);
            acc = acc + Vr[min(raw, nt)];
        }
        w += 8;
        if (w >= d.we_max) break;
        q = __ldg(row + (w >> 3));
    }
    if (update) {
        d.vhat[s] = acc;
        d.edge_dirty[s] = 0;
    }
    return acc;
}

// edge s: T = sum of tau over its incidences (ELL row, 8 per 16-B load, ascending original id;
// padding -> the all-zero sentinel row nt), eps~ = T / Vhat, sigma = D eps~ -> the two sigma
// planes; energy mode (epart): psi(eps~_s) Vhat_s / 6 added to U instead (oracle
// orc_strain_energy, same association)
__device__ __forceinline__ void edge_sigma(const Dev &d, int64_t s, const double *T, int tn, int nt, uint4 q,
                                           double Vh, const double *epart, double &U) {
    double T0 = 0.0, T1 = 0.0, T2 = 0.0, T3 = 0.0, T4 = 0.0, T5 = 0.0;
    const uint4 *row = reinterpret_cast<const uint4 *>(d.incE + (uint32_t)s * (uint32_t)d.we);
    for (int w = 0;;) {
        const uint32_t qq[4] = {q.x, q.y, q.z, q.w};
        const int lim = d.we_max - w;  // warp-uniform: slots past the mesh's max incidence are skipped
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (t >= lim) break;
            const int raw = (int)((qq[t >> 1] >> (16 * (t & 1))) & 0xffff);
            CEM_BOUND(d, raw == 0xffff || raw <= nt);
            const int r = min(raw, nt);
            T0 = T0 + T[r];
            T1 = T1 + T[tn + r];
            T2 = T2 + T[2 * tn + r];
            T3 = T3 + T[3 * tn + r];
            T4 = T4 + T[4 * tn + r];
            T5 = T5 + T[5 * tn + r];
        }
        w += 8;
        if (w >= d.we_max) break;  // (we_max <= we)
        q = __ldg(row + (w >> 3));
    }
    if (epart) {
        if (Vh != 0.0 && __ldg(d.edge_own + s)) {
            const double inv = 1.0 / Vh;
            const double e11 = T0 * inv, e22 = T1 * inv, e33 = T2 * inv, g12 = T3 * inv, g23 = T4 * inv, g13 = T5 * inv;
            const double tr = e11 + e22 + e33;
            const double ee = e11 * e11 + e22 * e22 + e33 * e33 + 0.5 * (g12 * g12 + g23 * g23 + g13 * g13);
            U = U + (0.5 * d.lam * tr * tr + d.mu * ee) * (Vh / 6.0);
        }
        return;
    }
    // sigma_s in two planes: (11, 22, 33, 12) as one 32-B record, (23, 13) as one 16-B record
    double4 *o4 = reinterpret_cast<double4 *>(d.srec) + s;
    double *o2 = d.srec2 + 2 * s;
    if (Vh == 0.0) {
        st256(o4, 0.0, 0.0, 0.0, 0.0);
        st128(o2, 0.0, 0.0);
        return;
    }
    const double inv = 1.0 / Vh;
    const double e11 = T0 * inv, e22 = T1 * inv, e33 = T2 * inv, g12 = T3 * inv, g23 = T4 * inv, g13 = T5 * inv;
    st256(o4, d.l2m * e11 + d.lam * (e22 + e33), d.l2m * e22 + d.lam * (e11 + e33), d.l2m * e33 + d.lam * (e11 + e22),
          d.mu * g12);
    st128(o2, d.mu * g23, d.mu * g13);
}

__device__ __forceinline__ void block_AB(const Dev &d, int b, const double4 *u, double *sm, double *epart = nullptr,
                                         int wneed = -1) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int32_t t0 = __ldg(d.tl_off + b);
    const int nt = __ldg(d.tl_off + b + 1) - t0;
    const int32_t n0 = __ldg(d.nlb_off + b);
    const int nn = __ldg(d.nlb_off + b + 1) - n0;
    const int un = pstride(nn), tn = pstride(nt + 1);  // row nt: all-zero sentinel
    double *U = sm, *T = sm + 3 * un;
    // static tables of this thread's first tet and node before the dependency wait (they
    // overlap the previous stage's tail and the u gather)
    const bool has0 = tid < nt;
    const uint32_t e0 = has0 ? (uint32_t)__ldg(d.tl + t0 + tid) : 0u;
    double g0[4][3], V0 = 0.0;
    ushort4 lc0 = make_ushort4(0, 0, 0, 0);
    int r0 = tid;  // shared-memory row of this thread's tet (bank-aware order, trow)
    if (has0) {
        load_geo(d, e0, g0, V0);
        lc0 = __ldg(reinterpret_cast<const ushort4 *>(d.tconn) + t0 + tid);
        r0 = __ldg(d.trow + t0 + tid);
    }
    const int32_t k0 = tid < nn ? __ldg(d.nlb + n0 + tid) : 0;
    const int q0 = tid < nn ? __ldg(d.nrow + n0 + tid) : 0;
    CEM_BOUND(d, k0 >= 0 && k0 < d.N && q0 >= 0 && q0 < un);
    CEM_BOUND(d, !has0 || (e0 < (uint32_t)d.E && r0 >= 0 && r0 < tn && lc0.x < un && lc0.y < un && lc0.z < un && lc0.w < un));
    // the second tet's list entry (most blocks hold 1.5 tets per thread): index, row, nodes
    const int i1 = tid + nthr;
    const bool has1 = i1 < nt;
    const uint32_t e1 = has1 ? (uint32_t)__ldg(d.tl + t0 + i1) : 0u;
    const int r1 = has1 ? (int)__ldg(d.trow + t0 + i1) : nt;
    const ushort4 lc1 = has1 ? __ldg(reinterpret_cast<const ushort4 *>(d.tconn) + t0 + i1) : make_ushort4(0, 0, 0, 0);
    stage_wait(d, ST_AB, b, wneed);  // u and the tet states come from the previous step's D (and splits)
    const uint8_t act0 = has0 ? __ldcg(d.state + e0) : (uint8_t)0;
    if (tid < nn) {  // one node per thread (list in ascending order, rows bank-aware)
        const double4 w = ldcg256(u + k0);
        U[q0] = w.x;
        U[un + q0] = w.y;
        U[2 * un + q0] = w.z;
    }
    for (int i = tid + nthr; i < nn; i += nthr) {
        const double4 w = ldcg256(u + __ldg(d.nlb + n0 + i));
        const int q = __ldg(d.nrow + n0 + i);
        U[q] = w.x;
        U[un + q] = w.y;
        U[2 * un + q] = w.z;
    }
    __syncthreads();
    // inactive tet / sentinel: exact zeros. Running sums here never hold -0.0, so adding
    // +0.0 is bit-identical to skipping the entry.
    if (act0) {
        grad0(g0);
        tau_row(T, tn, r0, U, un, g0, V0, lc0);
    } else if (tid <= nt) {
        zero_row(T, tn, r0);  // (tid == nt: the sentinel row)
    }
    if (has1) {  // second tet: indices prefetched, geometry and state issued together
        double g[4][3], V;
        load_geo(d, e1, g, V);
        if (__ldcg(d.state + e1)) {
            grad0(g);
            tau_row(T, tn, r1, U, un, g, V, lc1);
        } else {
            zero_row(T, tn, r1);
        }
    } else if (i1 == nt) {
        zero_row(T, tn, nt);  // sentinel
    }
    for (int i = tid + 2 * nthr; i <= nt; i += nthr) {
        const uint32_t e = i < nt ? (uint32_t)__ldg(d.tl + t0 + i) : 0u;
        double g[4][3], V;
        load_geo(d, e, g, V);
        const ushort4 lc = __ldg(reinterpret_cast<const ushort4 *>(d.tconn) + t0 + min(i, nt - 1));
        const int r = i < nt ? (int)__ldg(d.trow + t0 + i) : nt;
        if (i == nt || !__ldcg(d.state + e)) {
            zero_row(T, tn, r);
            continue;
        }
        grad0(g);
        tau_row(T, tn, r, U, un, g, V, lc);
    }
    // the block's edges: blk_ab = CEM_AB_EPT * nthr consecutive edges, thread tid takes edges
    // sbase + j nthr + tid (j < CEM_AB_EPT); the first one's row and Vhat before the barrier
    const int64_t sbase = (int64_t)b * d.blk_ab;
    const int64_t send = min(d.S, sbase + d.blk_ab);
    const int64_t s0 = sbase + tid;
    const bool hs0 = s0 < send;
    const uint4 qe0 = hs0 ? __ldg(reinterpret_cast<const uint4 *>(d.incE + (uint32_t)s0 * (uint32_t)d.we))
                          : make_uint4(0, 0, 0, 0);
    // Vhat from the table, issued with its dirty flag (one round trip) before the barrier
    const uint8_t dty0 = hs0 ? __ldcg(d.edge_dirty + s0) : (uint8_t)0;
    double Vh0 = hs0 ? __ldcg(d.vhat + s0) : 0.0;
    __syncthreads();
    double Ue = 0.0;  // energy mode: this thread's strain energy
    if (hs0) {
        if (dty0) Vh0 = vhat_rows(d, s0, T, tn, nt, qe0, epart == nullptr);
        edge_sigma(d, s0, T, tn, nt, qe0, Vh0, epart, Ue);
    }
    for (int64_t s = s0 + nthr; s < send; s += nthr) {  // (CEM_AB_EPT > 1: more edges per thread)
        const uint4 q = __ldg(reinterpret_cast<const uint4 *>(d.incE + (uint32_t)s * (uint32_t)d.we));
        double Vh = __ldcg(d.vhat + s);
        if (__ldcg(d.edge_dirty + s)) Vh = vhat_rows(d, s, T, tn, nt, q, epart == nullptr);
        edge_sigma(d, s, T, tn, nt, q, Vh, epart, Ue);
    }
    if (epart) {
        const double t = block_sum(Ue, sm);  // the planes are no longer read
        if (tid == 0) epart[b] = t;
    }
}

// ------------------------------------------------------------------ crack criterion (rare path)
__constant__ int c_ep[6] = {0, 0, 0, 1, 1, 2};
__constant__ int c_eq[6] = {1, 2, 3, 2, 3, 3};
__device__ __forceinline__ int ledge(int a, int b) {
    const int p = a < b ? a : b, q = a < b ? b : a;
    return p == 0 ? q - 1 : (p == 1 ? q + 1 : 5);
}
struct Vec3 {
    double x, y, z;
};
__device__ __forceinline__ Vec3 vsub(Vec3 a, Vec3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double vdot(Vec3 a, Vec3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ Vec3 vcross(Vec3 a, Vec3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// Principal decomposition by cyclic Jacobi (R8): pivots (0,1),(0,2),(1,2),
// <= 8 sweeps, stop when all off-diagonals are 0, a pivot with |a_pq| <= 2^-60(|a_pp|+|a_qq|)
// is zeroed without rotation; theta = (a_qq-a_pp)/(2a_pq), t = sgn(theta)/(|theta|+sqrt(theta^2+1)),
// c = 1/sqrt(t^2+1), s = t c.
struct Eig {
    double l[3];
    double ev[3][3];
    int k1, deg;
};

__device__ void principal(const double *s6, Eig &E) {
    double A[3][3] = {{s6[0], s6[3], s6[5]}, {s6[3], s6[1], s6[4]}, {s6[5], s6[4], s6[2]}};
    double Vm[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
    for (int sweep = 0; sweep < 8; ++sweep) {
        if (A[0][1] == 0.0 && A[0][2] == 0.0 && A[1][2] == 0.0) break;
#pragma unroll
        for (int r3 = 0; r3 < 3; ++r3) {
            const int p = r3 == 2 ? 1 : 0;
            const int q = r3 == 0 ? 1 : 2;
            const int r = 2 - r3;
            const double apq = A[p][q], app = A[p][p], aqq = A[q][q];
            if (fabs(apq) <= 0x1p-60 * (fabs(app) + fabs(aqq))) {
                A[p][q] = 0.0;
                A[q][p] = 0.0;
                continue;
            }
            const double theta = (aqq - app) / (2.0 * apq);
            double t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
            if (theta < 0.0) t = -t;
            const double c = 1.0 / sqrt(t * t + 1.0);
            const double s = t * c;
            A[p][p] = app - t * apq;
            A[q][q] = aqq + t * apq;
            A[p][q] = 0.0;
            A[q][p] = 0.0;
            const double arp = A[r][p], arq = A[r][q];
            A[r][p] = c * arp - s * arq;
            A[p][r] = A[r][p];
            A[r][q] = s * arp + c * arq;
            A[q][r] = A[r][q];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const double vip = Vm[i][p], viq = Vm[i][q];
                Vm[i][p] = c * vip - s * viq;
                Vm[i][q] = s * vip + c * viq;
            }
        }
    }
    E.l[0] = A[0][0];
    E.l[1] = A[1][1];
    E.l[2] = A[2][2];
    int k1 = 0;
    if (E.l[1] > E.l[k1]) k1 = 1;
    if (E.l[2] > E.l[k1]) k1 = 2;
    int deg = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (E.l[k1] - E.l[k] <= 1e-10 * fabs(E.l[k1])) deg |= 1 << k;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) E.ev[i][k] = Vm[i][k];
    E.k1 = k1;
    E.deg = deg;
}

// sigma_G . m unnormalised (R8): sigma1 |e1.m|, degenerate top eigenspace -> projector norm
__device__ double sig_proj(const Eig &E, Vec3 m) {
    const int cnt = (E.deg & 1) + ((E.deg >> 1) & 1) + ((E.deg >> 2) & 1);
    if (cnt == 1) {
        const Vec3 e = {E.ev[0][E.k1], E.ev[1][E.k1], E.ev[2][E.k1]};
        return E.l[E.k1] * fabs(vdot(e, m));
    }
    double acc = 0.0;
    for (int k = 0; k < 3; ++k) {
        if (!(E.deg >> k & 1)) continue;
        const Vec3 e = {E.ev[0][k], E.ev[1][k], E.ev[2][k]};
        const double dd = vdot(e, m);
        acc = acc + dd * dd;
    }
    return E.l[E.k1] * sqrt(acc);
}

__device__ __forceinline__ double dsgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

// Full criterion of one tet, evaluated by a whole warp (the tets that fail the early-out;
// called with all 32 lanes, uniform arguments).  Lanes 0-3 gather the nodes, lanes 0-5 the
// Heaviside flags and the principal pair of their edge's sigma (R6, R8), lanes
// 0-23 one candidate each, k = 6c + 2f + t (R7): corner c, front {p,q} among the other nodes
// o0<o1<o2 as (o0,o1),(o0,o2),(o1,o2), r the remaining node; t=0 pattern I (eq:G-I) with
// m = (X_q-X_p)x(X_r-X_c), t=1 pattern II (eq:G-II) with m = (X_q-X_p)x(X_r-X_p).  The
// selection (max G, ties -> larger area, then lower k; R14) is a butterfly argmax over
// (G, area, -k), which equals the oracle's sequential scan.  Split: deactivate
// now (this step's readers of the state are done), append a record (unordered; sorted by
// (step, element) on readback), stamp the 4 nodes so stage D recomputes their mass.
#ifndef CEM_D_PIPE
#define CEM_D_PIPE 1  // stage D: double-buffered slot gathers (batch i+1 in flight while batch i is summed)
#endif
#ifndef CEM_D_BATCH
#define CEM_D_BATCH 8  // stage D: force slots gathered per batch (multiple of 4)
#endif
// sigma_s of edge s from its two planes (rare path)
__device__ __forceinline__ void load_sigma(const Dev &d, int64_t s, double *s6) {
    const double4 a = ldcg256(reinterpret_cast<const double4 *>(d.srec) + s);
    const double2 b = ldcg128(d.srec2 + 2 * s);
    s6[0] = a.x;
    s6[1] = a.y;
    s6[2] = a.z;
    s6[3] = a.w;
    s6[4] = b.x;
    s6[5] = b.y;
}

#ifndef CEM_CRIT_GRID
#define CEM_CRIT_GRID (148 * 2)  // k_crit blocks (8 warps each, grid-stride over the list)
#endif
#ifndef CEM_CRIT_BATCH
#define CEM_CRIT_BATCH 5  // k_eval: survivors evaluated together by one warp (6 x 5 = 30 eigen lanes)
#endif
#ifndef CEM_CRIT_THREADS
#define CEM_CRIT_THREADS 128  // k_eval block size
#endif
#ifndef CEM_CRITB_GRID
#define CEM_CRITB_GRID (148 * 4)  // k_eval blocks
#endif
#ifndef CEM_FILTER_MINB
#define CEM_FILTER_MINB 2  // 128 registers: fewer warps but no large spills (measured best)
#endif
#ifndef CEM_FILTER_GRID
#define CEM_FILTER_GRID (148 * 2)  // k_filter blocks (256 threads, grid-stride over the list)
#endif
#ifndef CEM_CRITB_MINB
#define CEM_CRITB_MINB 4
#endif
#ifndef CEM_CRIT_COOP_MAX
#define CEM_CRIT_COOP_MAX 1
#endif
struct CritScratch {
    double X[4][3], U[4][3];
    int H[6];
    Eig eg[6];
};

static_assert(sizeof(CritScratch) <= 1024, "stage C's staging area holds 8 warp scratches of <= 1 KB");

// Candidate k of a tet (R7): both patterns through one instruction stream (no divergent branch
// per pattern or per Heaviside flag: selects instead), so a warp evaluating 24 candidates side by
// side runs one division and one square root per lane.  Every value is the same expression as
// the oracle's (orc candidate): pattern I  A1 = S(s_pr,m) Dd_p, A2 = S(s_qr,m) Dd_q,
// G = (1/2 (A1 + A2)) / |m|^2, area |m| / 4; pattern II  G = (1/2 (S(s_cr,m) (Dd_p + Dd_q))) / |m|^2,
// area |m| / 8 (x / 4 and x * 0.25 are the same correctly rounded value); Dd = 0 where H = 0.
__device__ void candidate(const CritScratch &w, int k, bool both, double &G, double &area) {
    const int c = k / 6, f = (k % 6) / 2, tt = k & 1;
    // the other three nodes in ascending order, o0 < o1 < o2
    const int o0 = c == 0 ? 1 : 0, o1 = c <= 1 ? 2 : 1, o2 = c <= 2 ? 3 : 2;
    const int p = f == 2 ? o1 : o0, q = f == 0 ? o1 : o2, r = f == 0 ? o2 : (f == 1 ? o1 : o0);
    auto X = [&](int a) { return Vec3{w.X[a][0], w.X[a][1], w.X[a][2]}; };
    auto U = [&](int a) { return Vec3{w.U[a][0], w.U[a][1], w.U[a][2]}; };
    const Vec3 Xc = X(c), Xp = X(p), Xq = X(q), Xr = X(r);
    const Vec3 d1 = vsub(Xq, Xp);
    const Vec3 d2 = vsub(Xr, tt == 0 ? Xc : Xp);
    const Vec3 mv = vcross(d1, d2);
    const double mm = vdot(mv, mv);
    const Vec3 Uc = U(c);
    const bool hp = w.H[ledge(c, p)], hq = w.H[ledge(c, q)];
    const double vp = vdot(vsub(U(p), Uc), mv) * dsgn(vdot(vsub(Xp, Xc), mv));
    const double vq = vdot(vsub(U(q), Uc), mv) * dsgn(vdot(vsub(Xq, Xc), mv));
    const double Dp = hp ? vp : 0.0, Dq = hq ? vq : 0.0;
    const double S1 = sig_proj(w.eg[tt == 0 ? ledge(p, r) : ledge(c, r)], mv);
    const double S2 = sig_proj(w.eg[ledge(q, r)], mv);  // (pattern I only)
    const double num = tt == 0 ? S1 * Dp + S2 * Dq : S1 * (Dp + Dq);
    G = (0.5 * num) / mm;
    area = sqrt(mm) * (tt == 0 ? 0.25 : 0.125);
    // R11 variant (CEM_F_FRONT_BOTH_STRETCHED): the front must be stretched at both edges
    if (both && !(hp && hq)) G = 0.0;
}

__device__ __forceinline__ void split_tet(const Dev &d, int64_t e, int4 t, double G, int k, double A, int64_t rec_step,
                                          int32_t stamp, bool record) {
    d.state[e] = 0;
#pragma unroll
    for (int l = 0; l < 6; ++l) d.edge_dirty[ldro(d.eedge + (int64_t)l * d.E + e)] = 1;  // their Vhat changes
    if (d.p2p_np && record) {
        // P2P halo: the owner stores the new state byte into the buffers of the peers holding the
        // tet as a ghost (parity of the step whose sync consumes it: s for step s -> s+1,
        // n for cem_crack_update at step n, which uses negative stamps)
        const int par = (int)((stamp > 0 ? rec_step - 1 : rec_step) & 1);
        for (int32_t i = __ldg(d.p2p_toff + e); i < __ldg(d.p2p_toff + e + 1); ++i)
            d.p2p_recv[par * d.p2p_np + __ldg(d.p2p_tpeer + i)][__ldg(d.p2p_tbyte + i)] = 0;
    }
    if (record) {  // multi-GPU: only the owning rank records (every holder deactivates)
        const int slot = atomicAdd(&d.ctr[0], 1);
        CEM_BOUND(d, slot < d.E);
        d.rec_step[slot] = rec_step;
        d.rec_elem[slot] = ldro(d.tet_orig + e);
        d.rec_cand[slot] = k;
        d.rec_G[slot] = G;
        d.rec_area[slot] = A;
    }
    d.dirty[t.x] = stamp;
    d.dirty[t.y] = stamp;
    d.dirty[t.z] = stamp;
    d.dirty[t.w] = stamp;
}

// The same criterion evaluated by one lane (used when many lanes of a warp need it: they
// then run it side by side): the oracle's sequential scan over k = 0..23.
__device__ __noinline__ void criterion_lane(const Dev *__restrict__ dp, int64_t e, const double4 *u, double gc,
                                            int64_t rec_step, int32_t stamp, bool record) {
    const Dev &d = *dp;
    CritScratch w;
    const int4 t = __ldg(&d.conn[e]);
    const int nid[4] = {t.x, t.y, t.z, t.w};
    for (int a = 0; a < 4; ++a) {
        const double4 x = ldro4(&d.X[nid[a]]);
        const double4 uu = ldcg256(&u[nid[a]]);
        w.X[a][0] = x.x;
        w.X[a][1] = x.y;
        w.X[a][2] = x.z;
        w.U[a][0] = uu.x;
        w.U[a][1] = uu.y;
        w.U[a][2] = uu.z;
    }
    for (int l = 0; l < 6; ++l) {
        const Vec3 du = {w.U[c_eq[l]][0] - w.U[c_ep[l]][0], w.U[c_eq[l]][1] - w.U[c_ep[l]][1],
                         w.U[c_eq[l]][2] - w.U[c_ep[l]][2]};
        const Vec3 dX = {w.X[c_eq[l]][0] - w.X[c_ep[l]][0], w.X[c_eq[l]][1] - w.X[c_ep[l]][1],
                         w.X[c_eq[l]][2] - w.X[c_ep[l]][2]};
        const Vec3 ww = {2.0 * dX.x + du.x, 2.0 * dX.y + du.y, 2.0 * dX.z + du.z};
        w.H[l] = vdot(du, ww) > 0.0;
        double s6[6];
        load_sigma(d, ldro(d.eedge + (int64_t)l * d.E + e), s6);
        principal(s6, w.eg[l]);
    }
    double Gb = 0.0, Ab = 0.0;
    int kb = -1;
    for (int k = 0; k < 24; ++k) {
        double G, A;
        candidate(w, k, (d.flags & CEM_F_FRONT_BOTH_STRETCHED) != 0, G, A);
        if (kb < 0 || G > Gb || (G == Gb && A > Ab)) {
            Gb = G;
            kb = k;
            Ab = A;
        }
    }
    if (Gb > gc) split_tet(d, e, t, Gb, kb, Ab, rec_step, stamp, record);
}

#ifdef CEM_CRIT_TRACE
// (measurement build only) SM clock after the value v has arrived: the setp consumes v
__device__ __forceinline__ long long clk_after(double v) {
    long long t;
    asm volatile("{ .reg .pred p; setp.eq.f64 p, %1, 0d7FF0DEADBEEF0001; mov.u64 %0, %%clock64; @p mov.u64 %0, 0; }"
                 : "=l"(t) : "d"(v) : "memory");
    return t;
}
#define CT(i, v) tr[i] = clk_after((double)(v))
#else
#define CT(i, v) ((void)0)
#endif
__device__ __forceinline__ void criterion_warp_body(const Dev &d, int64_t e, const double4 *u, double gc,
                                                    int64_t rec_step, int32_t stamp, bool record, CritScratch &w) {
    const int lane = threadIdx.x & 31;
#ifdef CEM_CRIT_TRACE
    long long tr[10] = {0};
    CT(0, e);
#endif
    // every load that depends only on e is issued first: the edge ids (lanes 0-5), then the nodes'
    // X and u (lanes 0-3) and the edges' sigma, so that the eigen-solves start as soon as sigma
    // arrives and the node loads land while they run
    const int4 t = __ldg(&d.conn[e]);
    const int64_t es = lane < 6 ? ldro(d.eedge + (int64_t)lane * d.E + e) : 0;
    const int n = lane == 0 ? t.x : (lane == 1 ? t.y : (lane == 2 ? t.z : t.w));
    const int32_t orig = lane == 0 && record ? ldro(d.tet_orig + e) : 0;  // (the record, if it splits)
    double4 x = make_double4(0.0, 0.0, 0.0, 0.0), uu = x;
    if (lane < 4) {
        x = ldro4(&d.X[n]);
        uu = ldcg256(&u[n]);
    }
    Eig eg;
    if (lane < 6) {
        double s6[6];
        CT(1, t.x + es);
        load_sigma(d, es, s6);
        CT(2, s6[0] + s6[5]);
        principal(s6, eg);
        CT(3, eg.l[0] + eg.ev[2][2]);
    }
    if (lane < 4) {
        w.X[lane][0] = x.x;
        w.X[lane][1] = x.y;
        w.X[lane][2] = x.z;
        w.U[lane][0] = uu.x;
        w.U[lane][1] = uu.y;
        w.U[lane][2] = uu.z;
    }
    __syncwarp();
    if (lane < 6) {
        const int l = lane;
        // local edge l = (ep, eq): (0,1) (0,2) (0,3) (1,2) (1,3) (2,3) -- c_ep / c_eq without
        // lane-divergent constant-bank reads
        const int ep = l < 3 ? 0 : (l < 5 ? 1 : 2), eq = l < 3 ? l + 1 : (l == 3 ? 2 : 3);
        const Vec3 du = {w.U[eq][0] - w.U[ep][0], w.U[eq][1] - w.U[ep][1], w.U[eq][2] - w.U[ep][2]};
        const Vec3 dX = {w.X[eq][0] - w.X[ep][0], w.X[eq][1] - w.X[ep][1], w.X[eq][2] - w.X[ep][2]};
        const Vec3 ww = {2.0 * dX.x + du.x, 2.0 * dX.y + du.y, 2.0 * dX.z + du.z};
        w.H[l] = vdot(du, ww) > 0.0;  // eq:stretch-delta Heaviside, R6
        w.eg[l] = eg;
    }
    __syncwarp();
    double G = -INFINITY, A = -INFINITY;
    int k = 1 << 20;
    CT(5, w.H[0]);
    if (lane < 24) {
        candidate(w, lane, (d.flags & CEM_F_FRONT_BOTH_STRETCHED) != 0, G, A);
        k = lane;
    }
    CT(6, G + A);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double G2 = __shfl_xor_sync(0xffffffffu, G, o), A2 = __shfl_xor_sync(0xffffffffu, A, o);
        const int k2 = __shfl_xor_sync(0xffffffffu, k, o);
        if (G2 > G || (G2 == G && (A2 > A || (A2 == A && k2 < k)))) {
            G = G2;
            A = A2;
            k = k2;
        }
    }
    // lane 0's selection decides for the whole warp (with a NaN G the butterfly need not agree)
    CT(4, G);
    G = __shfl_sync(0xffffffffu, G, 0);
#ifdef CEM_CRIT_TRACE
    if (lane == 0 && blockIdx.x < 3 && threadIdx.x == 0)
        printf("[crit] blk %d: eedge+conn %lld  sigma %lld  jacobi %lld  heaviside %lld  cand %lld  argmax %lld\n", blockIdx.x,
               tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], tr[5] - tr[3], tr[6] - tr[5], tr[4] - tr[6]);
#endif
    if (G > gc) {  // split_tet's stores, spread over the lanes that hold their indices
        A = __shfl_sync(0xffffffffu, A, 0);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (lane < 6) d.edge_dirty[es] = 1;  // their Vhat changes
        if (lane < 4) d.dirty[n] = stamp;
        if (lane == 0) {
            d.state[e] = 0;
            if (d.p2p_np && record) {
                const int par = (int)((stamp > 0 ? rec_step - 1 : rec_step) & 1);
                for (int32_t i = __ldg(d.p2p_toff + e); i < __ldg(d.p2p_toff + e + 1); ++i)
                    d.p2p_recv[par * d.p2p_np + __ldg(d.p2p_tpeer + i)][__ldg(d.p2p_tbyte + i)] = 0;
            }
            if (record) {
                const int slot = atomicAdd(&d.ctr[0], 1);
                CEM_BOUND(d, slot < d.E);
                d.rec_step[slot] = rec_step;
                d.rec_elem[slot] = orig;
                d.rec_cand[slot] = k;
                d.rec_G[slot] = G;
                d.rec_area[slot] = A;
            }
        }
    }
    __syncwarp();  // the scratch is reused by the warp's next call
}

// (out of line for the stage-C callers, whose register budget it must not raise; k_crit inlines the
// body and reads the Dev fields from its parameter bank instead of through d.self)
__device__ __noinline__ void criterion_warp(const Dev *__restrict__ dp, int64_t e, const double4 *u, double gc,
                                            int64_t rec_step, int32_t stamp, bool record, CritScratch &w) {
    criterion_warp_body(*dp, e, u, gc, rec_step, stamp, record, w);
}

// Refined early-out of one listed tet, evaluated by one thread (k_filter).  Candidate k
// has G_k = 1/2 (S(s1,m) Dd1 + S(s2,m) Dd2) / |m|^2 with |S(s,m)| <= |sigma_1(s)| |m| <= g_s |m|
// (g_s: Gershgorin bound of sigma_s) and |Dd(a,b,m)| = H_ab |du_ab . m|, so
//   |G_k| <= N_k / |m|,  N_k = 1/2 (g_pr H_cp |du_cp.m| + g_qr H_cq |du_cq.m|)   (pattern I)
//                        N_k = 1/2 g_cr (H_cp |du_cp.m| + H_cq |du_cq.m|)      (pattern II),
// with m, du and H computed by the same expressions as the full evaluation (candidate()).  The
// tet needs the full evaluation unless every candidate has (N_k (1 + 1e-6))^2 <= Gc_e^2 |m|^2
// (the margin dwarfs the rounding; Gc_e = 0 keeps exactly the tets with some N_k > 0, for which
// G_k could be positive).  Costs no eigen-solve, square root or division.
__device__ __forceinline__ bool crit_refined_need(const Dev *__restrict__ dp, int64_t e, const double4 *u, double gc) {
    const Dev &d = *dp;
    const int4 t = __ldg(&d.conn[e]);
    const int nid[4] = {t.x, t.y, t.z, t.w};
    Vec3 X[4], U[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const double4 x = ldro4(&d.X[nid[a]]);
        const double4 uu = ldcg256(&u[nid[a]]);
        X[a] = Vec3{x.x, x.y, x.z};
        U[a] = Vec3{uu.x, uu.y, uu.z};
    }
    double g[6];
    bool H[6];
#pragma unroll
    for (int l = 0; l < 6; ++l) {
        const int pp = c_ep[l], qq = c_eq[l];
        const Vec3 du = vsub(U[qq], U[pp]), dX = vsub(X[qq], X[pp]);
        const Vec3 ww = {2.0 * dX.x + du.x, 2.0 * dX.y + du.y, 2.0 * dX.z + du.z};
        H[l] = vdot(du, ww) > 0.0;
        double s6[6];
        load_sigma(d, ldro(d.eedge + (int64_t)l * d.E + e), s6);
        const double r0 = fabs(s6[0]) + fabs(s6[3]) + fabs(s6[5]);
        const double r1 = fabs(s6[1]) + fabs(s6[3]) + fabs(s6[4]);
        const double r2 = fabs(s6[2]) + fabs(s6[4]) + fabs(s6[5]);
        g[l] = fmax(r0, fmax(r1, r2));
    }
    const double thr2 = gc * gc;
#pragma unroll
    for (int k = 0; k < 24; ++k) {
        const int c = k / 6, f = (k % 6) / 2, tt = k & 1;
        const int o0 = c == 0 ? 1 : 0, o1 = c <= 1 ? 2 : 1, o2 = c == 3 ? 2 : 3;
        const int p = f == 2 ? o1 : o0, q = f == 0 ? o1 : o2, r = f == 0 ? o2 : (f == 1 ? o1 : o0);
        const Vec3 d1 = vsub(X[q], X[p]);
        const Vec3 d2 = tt == 0 ? vsub(X[r], X[c]) : vsub(X[r], X[p]);
        const Vec3 mv = vcross(d1, d2);
        const double mm = vdot(mv, mv);
        const int lp = ledge(c, p), lq = ledge(c, q);
        const double ap = H[lp] ? fabs(vdot(vsub(U[p], U[c]), mv)) : 0.0;
        const double aq = H[lq] ? fabs(vdot(vsub(U[q], U[c]), mv)) : 0.0;
        const double N = tt == 0 ? 0.5 * (g[ledge(p, r)] * ap + g[ledge(q, r)] * aq) : 0.5 * (g[ledge(c, r)] * (ap + aq));
        const double Nm = N * (1.0 + 1e-6);
        if (!(Nm * Nm <= thr2 * mm)) return true;
    }
    return false;
}

// ------------------------------------------------------------------ stage C: force + criterion
// S = sum_{l=0..5} sigma_{s(e,l)}; f_{e,a} = c((gx S11 + gy S12) + gz S13), ... with c = V/6
// (PAPER.md:L340-L367), written to the warp-tiled force slots.  Early-out (DESIGN.md
// "Early-out"): every candidate satisfies |G| <= max_l g_{s(e,l)} * max_l |u_q - u_p|; tets
// below Gc_e (1 - 1e-6) skip the 24-candidate evaluation.
#ifndef CEM_C_KME
#define CEM_C_KME 3
#endif

__device__ __forceinline__ void stage_sigma(double *sm, int np, int i, double4 x, double2 z) {
    sm[i] = x.x;
    sm[np + i] = x.y;
    sm[2 * np + i] = x.z;
    sm[3 * np + i] = x.w;
    sm[4 * np + i] = z.x;
    sm[5 * np + i] = z.y;
}
// asynchronous global -> shared copies (cp.async: no registers held while in flight)
__device__ __forceinline__ void cpa16(void *sdst, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(g)
                 : "memory");
}
__device__ __forceinline__ void cpa8(void *sdst, const void *g) {  // static tables only (.ca)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(g)
                 : "memory");
}
__device__ __forceinline__ void cpa4(void *sdst, const void *g) {  // static tables only (.ca)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(g)
                 : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// stage C, partial mode (R27): entry i of the block's node list sums the contributions of the
// block's tets to that node (any order: the sum is exact), stored as (s, c) per component.  One
// thread per entry, entries in descending incidence count (nearly equal trip counts per warp);
// the forces are row a nthr + t of an (x, y) plane and a z plane.  Every thread calls it (barrier).
__device__ __forceinline__ void c_partials(const Dev &d, int b, const double *sm) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    // (block geometry reloaded here rather than kept live through stage C's body: registers)
    const int32_t n0 = __ldg(d.nl_off + b);
    const int nn = __ldg(d.nl_off + b + 1) - n0;
    const int ne = __ldg(d.el_off + b + 1) - __ldg(d.el_off + b);
    // (x, y) plane of 16-B rows and z plane of 8-B rows (overlay the sigma planes): random rows of
    // a warp then spread over 8 / 16 bank positions (32-B rows would give 4: 3x the wavefronts)
    const double2 *fxy = reinterpret_cast<const double2 *>(sm);
    const double *fz = sm + 8 * nthr;
    const uint16_t *spinc = reinterpret_cast<const uint16_t *>(sm + max(6 * pstride(ne), 12 * nthr) +
                                                               (CEM_C_GEOX ? 6 : 3) * pstride(nn));  // staged at block start
    const int32_t *spoff = reinterpret_cast<const int32_t *>(spinc + 4 * nthr);  // global offsets [nn + 1]
    const int32_t *spord = spoff + nn + 1;                                       // entry order [nn]
    const int32_t *spdst = spord + nn;                                           // node-major record [nn]
    const int32_t base = 4 * b * d.blk;
    cpa_wait_all();
    __syncthreads();
    for (int k = tid; k < nn; k += nthr) {
        const int i = spord[k];
        const int32_t j1 = spoff[i + 1] - base;
        double sx = 0.0, sy = 0.0, sz = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
        // eight entries per pass (their shared-memory loads all in flight); padding adds +0.0
        for (int32_t j = spoff[i] - base; j < j1; j += 8) {
            int ri[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) ri[u] = j + u < j1 ? (int)spinc[j + u] : -1;
            double2 xy[8];
            double z[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int r = ri[u] < 0 ? 0 : ri[u];
                xy[u] = ri[u] < 0 ? make_double2(0.0, 0.0) : fxy[r];
                z[u] = ri[u] < 0 ? 0.0 : fz[r];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                xacc(sx, cx, xy[u].x);
                xacc(sy, cy, xy[u].y);
                xacc(sz, cz, z[u]);
            }
        }
        double2 *o = reinterpret_cast<double2 *>(d.part + 6 * (int64_t)spdst[i]);
        o[0] = make_double2(sx, sy);
        o[1] = make_double2(sz, cx);
        o[2] = make_double2(cy, cz);
    }
}

// PM: exact partials (d.part != null, R27) instead of force slots (a compile-time choice: one
// register allocation per mode)
template <bool PM>
__device__ __forceinline__ void block_C(const Dev &d, int b, const double4 *u, bool crack, int64_t rec_step,
                                        int32_t stamp, double *sm, bool defer = false, int wneed = -1) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int32_t s0i = __ldg(d.el_off + b);
    const int ne = __ldg(d.el_off + b + 1) - s0i;
    const int32_t n0 = __ldg(d.nl_off + b);
    const int nn = __ldg(d.nl_off + b + 1) - n0;
    const bool early = crack && !(d.flags & CEM_F_NO_EARLY_OUT);
    const int np = pstride(ne), nq = pstride(nn);
    // partials: the block's element forces, row a nthr + t in a (f_x, f_y) 16-B plane and an f_z plane, overlay the sigma
    // planes once every thread has formed its S (barrier); the u (/ X) planes and the staged
    // partial tables follow
    double *smu = sm + (PM ? max(6 * np, 12 * nthr) : 6 * np);
    double *smf = sm;
    uint16_t *spinc_w = reinterpret_cast<uint16_t *>(smu + (CEM_C_GEOX ? 6 : 3) * nq);
    // ---- wave 1: list indices
    constexpr int kME = CEM_C_KME;  // sigma records per thread in flight (more -> tail loop)
    uint32_t sid[kME];
#pragma unroll
    for (int m = 0; m < kME; ++m) sid[m] = tid + m * nthr < ne ? (uint32_t)__ldg(d.el + s0i + tid + m * nthr) : 0u;
#ifdef CEM_DEBUG_BOUNDS
#pragma unroll
    for (int m = 0; m < kME; ++m) CEM_BOUND(d, sid[m] < (uint32_t)d.S);
#endif
#if CEM_C_GEOX
    // geometry from the block's node coordinates (static: staged before the dependency wait)
    double *smx = smu + 3 * nq;
    const int32_t nid = tid < nn ? __ldg(d.nl + n0 + tid) : 0;
    for (int i = tid; i < nn; i += nthr) {
        const double4 x = ldro4(&d.X[i == tid ? nid : __ldg(d.nl + n0 + i)]);
        smx[i] = x.x;
        smx[nq + i] = x.y;
        smx[2 * nq + i] = x.z;
    }
#else
    const int32_t nid = (early && tid < nn) ? __ldg(d.nl + n0 + tid) : 0;
#endif
    if (PM) {
        // partial tables of this block (static; staged before the dependency wait): its tets'
        // incidence entries (4 per tet, grouped by node-list entry) and the per-entry offsets
        // (cp.async: in flight without registers until c_partials waits for them)
        uint16_t *spinc = spinc_w;
        int32_t *spoff = reinterpret_cast<int32_t *>(spinc + 4 * nthr);
        const int64_t e0 = (int64_t)b * d.blk;
        if (e0 + tid < d.E) cpa8(reinterpret_cast<uint2 *>(spinc) + tid, reinterpret_cast<const uint2 *>(d.pinc) + e0 + tid);
        for (int i = tid; i <= nn; i += nthr) cpa4(spoff + i, d.pinc_off + n0 + i);
        for (int i = tid; i < nn; i += nthr) cpa4(spoff + nn + 1 + i, d.pord + n0 + i);
        for (int i = tid; i < nn; i += nthr) cpa4(spoff + 2 * nn + 1 + i, d.pdst + n0 + i);
        cpa_commit();
    }
    stage_wait(d, ST_C, b, wneed);  // sigma records come from stage AB
    // ---- wave 2: gathered records (one 32-B and one 16-B load each) -> planes 0..5
    double4 rx[kME];
    double2 rz[kME];
#pragma unroll
    for (int m = 0; m < kME; ++m)
        if (tid + m * nthr < ne) {
            rx[m] = ldcg256(reinterpret_cast<const double4 *>(d.srec) + sid[m]);
            rz[m] = ldcg128(d.srec2 + 2u * sid[m]);
        }
    const double4 uw = (early && tid < nn) ? ldcg256(u + nid) : make_double4(0, 0, 0, 0);
#pragma unroll
    for (int m = 0; m < kME; ++m) {
        const int i = tid + m * nthr;
        if (i < ne) stage_sigma(sm, np, i, rx[m], rz[m]);
    }
    for (int i = tid + kME * nthr; i < ne; i += nthr) {  // tail
        const uint32_t r = (uint32_t)__ldg(d.el + s0i + i);
        stage_sigma(sm, np, i, ldcg256(reinterpret_cast<const double4 *>(d.srec) + r), ldcg128(d.srec2 + 2u * r));
    }
    if (early) {
        if (tid < nn) {
            smu[tid] = uw.x;
            smu[nq + tid] = uw.y;
            smu[2 * nq + tid] = uw.z;
        }
        for (int i = tid + nthr; i < nn; i += nthr) {
            const double4 w = ldcg256(u + __ldg(d.nl + n0 + i));
            smu[i] = w.x;
            smu[nq + i] = w.y;
            smu[2 * nq + i] = w.z;
        }
    }
    // this thread's tet: state and static tables issued before the barrier, so their latency
    // overlaps the other warps' staging
    const int64_t e = (int64_t)b * d.blk + threadIdx.x;
    const bool he = e < d.E;
    const uint8_t act = he ? __ldcg(d.state + e) : (uint8_t)0;
    uint4 lq = make_uint4(0, 0, 0, 0);
    double g[4][3], cc = 0.0, gc = 0.0;
    uint8_t tf = 0;
    ushort4 lc = make_ushort4(0, 0, 0, 0);
    if (he) {
        if (crack) {  // criterion inputs (static): issued with the rest, not after the force
            tf = __ldg(d.tflag + e);
            gc = ldro(d.gc + e);
#if !CEM_C_GEOX
            if (early) lc = __ldg(reinterpret_cast<const ushort4 *>(d.lconn) + e);
#endif
        }
        lq = __ldg(reinterpret_cast<const uint4 *>(d.ledge) + e);
#if CEM_C_GEOX
        lc = __ldg(reinterpret_cast<const ushort4 *>(d.lconn) + e);
#else
        double Vd;
        geo_record(d, (uint32_t)e, g, Vd, cc);
#endif
    }
    __syncthreads();
#if CEM_C_GEOX
    if (he) {
        // the host preprocessing's formula (cem_mesh.cpp, = the oracle's): d_a = X_a - X_0,
        // det = d1.(d2 x d3), gradN1..3 = (d2xd3, d3xd1, d1xd2) / det, c = (det / 6) / 6
        const int li[4] = {lc.x, lc.y, lc.z, lc.w};
        Vec3 xa[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) xa[a] = Vec3{smx[li[a]], smx[nq + li[a]], smx[2 * nq + li[a]]};
        const Vec3 d1 = vsub(xa[1], xa[0]), d2 = vsub(xa[2], xa[0]), d3 = vsub(xa[3], xa[0]);
        const Vec3 c23 = vcross(d2, d3), c31 = vcross(d3, d1), c12 = vcross(d1, d2);
        const double det = vdot(d1, c23);
        const double inv = 1.0 / det;
        cc = (det / 6.0) / 6.0;
        g[1][0] = c23.x * inv; g[1][1] = c23.y * inv; g[1][2] = c23.z * inv;
        g[2][0] = c31.x * inv; g[2][1] = c31.y * inv; g[2][2] = c31.z * inv;
        g[3][0] = c12.x * inv; g[3][1] = c12.y * inv; g[3][2] = c12.z * inv;
    }
#endif
    bool need = false;  // this tet needs the full criterion (failed the early-out)
    double fr[PM ? 12 : 1];  // partials: the tet's forces, stored after the barrier (zeros if inactive)
#pragma unroll
    for (int q = 0; q < (PM ? 12 : 1); ++q) fr[q] = 0.0;
    if (he) {
#if CEM_FES == 3
        // the tet's 4 slots packed (f0, f1, f2, f3: 12 doubles, 96 B) -> three 256-bit stores
        double *fo = d.fe + 12 * (uint32_t)e;
#else
        // slot (e,a) = slot0 + 32 a, CEM_FES doubles per slot
        double *fo = d.fe + CEM_FES * (((uint32_t)e >> 5) * 128u + ((uint32_t)e & 31u));
#endif
        if (!act) {
#if CEM_FES == 3
            if (!PM)
                for (int q = 0; q < 3; ++q) st256(reinterpret_cast<double4 *>(fo) + q, 0.0, 0.0, 0.0, 0.0);
#else
#pragma unroll
            for (int a = 0; a < 4; ++a) store_slot(fo + 32 * CEM_FES * a, 0.0, 0.0, 0.0);
#endif
        } else {
            const int le[6] = {(int)(lq.x & 0xffff), (int)(lq.x >> 16), (int)(lq.y & 0xffff),
                               (int)(lq.y >> 16), (int)(lq.z & 0xffff), (int)(lq.z >> 16)};
#ifdef CEM_DEBUG_BOUNDS
#pragma unroll
            for (int l = 0; l < 6; ++l) CEM_BOUND(d, le[l] < ne);
#endif
            double S0 = 0.0, S1 = 0.0, S2 = 0.0, S3 = 0.0, S4 = 0.0, S5 = 0.0, gmax = 0.0;
#pragma unroll
            for (int l = 0; l < 6; ++l) {
                const int r = le[l];
                const double a0 = sm[r], a1 = sm[np + r], a2 = sm[2 * np + r];
                const double a3 = sm[3 * np + r], a4 = sm[4 * np + r], a5 = sm[5 * np + r];
                S0 = S0 + a0;
                S1 = S1 + a1;
                S2 = S2 + a2;
                S3 = S3 + a3;
                S4 = S4 + a4;
                S5 = S5 + a5;
                if (early) {  // Gershgorin bound g_s = max_i sum_j |sigma_ij| of the edge
                    const double r0 = fabs(a0) + fabs(a3) + fabs(a5);
                    const double r1 = fabs(a1) + fabs(a3) + fabs(a4);
                    const double r2 = fabs(a2) + fabs(a4) + fabs(a5);
                    gmax = fmax(gmax, fmax(r0, fmax(r1, r2)));
                }
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) g[0][c] = -((g[1][c] + g[2][c]) + g[3][c]);
#if CEM_FES == 3
            double f[12];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                f[3 * a] = cc * ((g[a][0] * S0 + g[a][1] * S3) + g[a][2] * S5);
                f[3 * a + 1] = cc * ((g[a][1] * S1 + g[a][0] * S3) + g[a][2] * S4);
                f[3 * a + 2] = cc * ((g[a][2] * S2 + g[a][1] * S4) + g[a][0] * S5);
            }
            if (PM) {
#pragma unroll
                for (int q = 0; q < 12; ++q) fr[q] = f[q];
            } else {
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    st256(reinterpret_cast<double4 *>(fo) + q, f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
            }
#else
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const double fx = cc * ((g[a][0] * S0 + g[a][1] * S3) + g[a][2] * S5);
                const double fy = cc * ((g[a][1] * S1 + g[a][0] * S3) + g[a][2] * S4);
                const double fz = cc * ((g[a][2] * S2 + g[a][1] * S4) + g[a][0] * S5);
                store_slot(fo + 32 * CEM_FES * a, fx, fy, fz);
            }
#endif
            // ghost tets (tflag bit 0 clear): the owner decides, the state arrives by exchange
            need = crack && (tf & 1);
            if (need && early) {
                const int li[4] = {lc.x, lc.y, lc.z, lc.w};
                double ux[4], uy[4], uz[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    ux[a] = smu[li[a]];
                    uy[a] = smu[nq + li[a]];
                    uz[a] = smu[2 * nq + li[a]];
                }
                double d2 = 0.0;
#pragma unroll
                for (int l = 0; l < 6; ++l) {
                    const int p = l < 3 ? 0 : (l < 5 ? 1 : 2), q = l < 3 ? l + 1 : (l < 5 ? l - 1 : 3);
                    const double dx = ux[q] - ux[p], dy = uy[q] - uy[p], dz = uz[q] - uz[p];
                    d2 = fmax(d2, (dx * dx + dy * dy) + dz * dz);
                }
                need = !(gmax * sqrt(d2) * (1.0 + 1e-6) <= gc);
            }
        }
    }
    if (PM) {
        __syncthreads();  // every S is formed: the sigma planes are free
        if (he) {  // row a nthr + t of corner a: (f_x, f_y) in the 16-B plane, f_z in the 8-B plane
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                reinterpret_cast<double2 *>(smf)[a * nthr + tid] = make_double2(fr[3 * a], fr[3 * a + 1]);
                smf[8 * nthr + a * nthr + tid] = fr[3 * a + 2];
            }
        }
    }
    if (!crack) {  // block-uniform
        if (PM) c_partials(d, b, sm);
        return;
    }
    if (defer) {
        // staged path: append the flagged tets to the step's list (warp-aggregated); k_crit
        // evaluates them all concurrently, one warp per tet, as they appear (it polls the
        // entries while stage C runs); ctr[9] counts the stage-C blocks that got here, a hint
        // only (k_crit stops polling at the block count, then waits for stage C's completion)
        if (threadIdx.x == 0) atomicAdd(&d.ctr[9], 1);
        const unsigned mm = __ballot_sync(0xffffffffu, need);
        if (mm) {
            const int lane = threadIdx.x & 31, lead = __ffs(mm) - 1;
            int base = 0;
            if (lane == lead) base = atomicAdd(&d.ctr[3], __popc(mm));
            base = __shfl_sync(0xffffffffu, base, lead);
            if (need) d.crit_list[base + __popc(mm & ((1u << lane) - 1))] = crit_entry(rec_step, e);
        }
        if (PM) c_partials(d, b, sm);
        return;
    }
    if (PM) c_partials(d, b, sm);
    // few flagged tets in the warp: the warp evaluates them one after another, 24 candidates
    // in parallel (scratch in the staging area, free after the barrier); many: each lane
    // evaluates its own (side by side)
    unsigned m = __ballot_sync(0xffffffffu, need);
    if (wneed >= 0 && m && (threadIdx.x & 31) == 0) atomicAdd(&d.ctr[10], __popc(m));  // (kernel-choice heuristic)
    __syncthreads();
    if (__popc(m) > CEM_CRIT_COOP_MAX) {
        if (need) criterion_lane(d.self, e, u, gc, rec_step, stamp, (tf & 2) != 0);
        return;
    }
    CritScratch &cs = reinterpret_cast<CritScratch *>(sm)[threadIdx.x >> 5];
    while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int64_t te = __shfl_sync(0xffffffffu, e, src);
        const double tgc = __shfl_sync(0xffffffffu, gc, src);
        const int trec = __shfl_sync(0xffffffffu, (int)(tf & 2), src);
        criterion_warp(d.self, te, u, tgc, rec_step, stamp, trec != 0, cs);
    }
}

__host__ __device__ __forceinline__ bool crack_on(int crack_every, int64_t s) {
    return crack_every > 0 && ((s + 1) % crack_every) == 0;
}

// ------------------------------------------------------------------ stage C, software-pipelined
// k_Cp: one persistent CTA per SM walks the stage-C blocks b = blockIdx.x + j gridDim.x.  While it
// computes block j, the asynchronous copies (cp.async, no registers held) of block j+1's inputs are
// in flight: the sigma records and node displacements it gathers (the index lists came one block
// earlier) and its contiguous per-tet tables (geometry tile, local edge / node indices, Gc, state,
// flags).  The per-tet arithmetic and every store are those of block_C (same bits); only the data
// movement differs: sigma rows (48 B) and u rows (32 B) are AoS in shared memory.
struct CpSlot {  // byte offsets inside one data slot
    int sig, u, geo, ledge, lconn, gc, st, tf, bytes;
};
__host__ __device__ inline CpSlot cp_slot(int max_el, int max_nl) {
    CpSlot c;
    c.sig = 0;
    c.u = (48 * max_el + 15) & ~15;
    c.geo = c.u + 32 * max_nl;
    c.ledge = c.geo + 8 * 352 * 8;
    c.lconn = c.ledge + 256 * 16;
    c.gc = c.lconn + 256 * 8;
    c.st = c.gc + 256 * 8;
    c.tf = c.st + 256;
    c.bytes = (c.tf + 256 + 127) & ~127;
    return c;
}
__host__ __device__ inline int cp_idx_ints(int max_el, int max_nl) { return (max_el + max_nl + 3) & ~3; }
#ifndef CEM_CP_DEPTH
#define CEM_CP_DEPTH 3  // data slots in flight (block j computed while j+1 .. j+DEPTH-1 load)
#endif
__host__ __device__ inline int cp_smem_bytes(int max_el, int max_nl) {
    return CEM_CP_DEPTH * cp_slot(max_el, max_nl).bytes + (CEM_CP_DEPTH + 2) * 4 * cp_idx_ints(max_el, max_nl);
}

// the index lists (edge list, node list) of block b -> an index slot
__device__ __forceinline__ void cp_issue_idx(const Dev &d, int b, int32_t *idx, bool early) {
    const int32_t s0i = __ldg(d.el_off + b), ne = __ldg(d.el_off + b + 1) - s0i;
    for (int i = threadIdx.x; i < ne; i += blockDim.x) cpa4(idx + i, d.el + s0i + i);
    if (early) {
        const int32_t n0 = __ldg(d.nl_off + b), nn = __ldg(d.nl_off + b + 1) - n0;
        for (int i = threadIdx.x; i < nn; i += blockDim.x) cpa4(idx + d.cp_max_el + i, d.nl + n0 + i);
    }
}
// the gathered records and the contiguous per-tet tables of block b -> a data slot
__device__ __forceinline__ void cp_issue_data(const Dev &d, int b, char *slot, const CpSlot &L, const int32_t *idx,
                                              const double4 *u, bool early) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int ne = __ldg(d.el_off + b + 1) - __ldg(d.el_off + b);
    for (int i = tid; i < ne; i += nthr) {  // sigma: 32-B record (11,22,33,12) + 16-B record (23,13) -> 48-B row
        const int64_t e = idx[i];
        char *row = slot + L.sig + 48 * i;
        cpa16(row, d.srec + 4 * e);
        cpa16(row + 16, d.srec + 4 * e + 2);
        cpa16(row + 32, d.srec2 + 2 * e);
    }
    if (early) {
        const int nn = __ldg(d.nl_off + b + 1) - __ldg(d.nl_off + b);
        for (int i = tid; i < nn; i += nthr) {
            const double *w = reinterpret_cast<const double *>(u + idx[d.cp_max_el + i]);
            char *row = slot + L.u + 32 * i;
            cpa16(row, w);
            cpa16(row + 16, w + 2);
        }
    }
    const int64_t t0 = (int64_t)b * d.blk;
    const int nt = (int)min((int64_t)d.blk, d.E - t0);
    const int ntile = (nt + 31) >> 5;
    const double *gsrc = d.geoT + (t0 >> 5) * 352;  // (blk is a multiple of 32)
    for (int i = tid; i < ntile * 176; i += nthr) cpa16(slot + L.geo + 16 * i, gsrc + 2 * i);
    for (int i = tid; i < nt; i += nthr) {
        cpa16(slot + L.ledge + 16 * i, d.ledge + 8 * (t0 + i));
        cpa8(slot + L.lconn + 8 * i, d.lconn + 4 * (t0 + i));
        cpa8(slot + L.gc + 8 * i, d.gc + t0 + i);
    }
    for (int i = tid; i < (nt + 3) / 4; i += nthr) {  // (the byte arrays are padded past E)
        cpa4(slot + L.st + 4 * i, d.state + t0 + 4 * i);
        cpa4(slot + L.tf + 4 * i, d.tflag + t0 + 4 * i);
    }
}

__global__ void __launch_bounds__(256, 1) k_Cp(Dev d, int64_t s, int crack_every) {
    extern __shared__ __align__(128) char cpsm[];
    pdl_trigger();
    const bool crack = crack_on(crack_every, s);
    const bool early = crack && !(d.flags & CEM_F_NO_EARLY_OUT);
    // ring: data slot of block j = j % D, index slot of block j = j % (D + 2); cp.async groups:
    // group g (one per iteration) = {data of block g + D - 1, indices of block g + D + 1}, so the
    // indices a data issue needs are two groups old (complete after wait_group D - 2)
    constexpr int D = CEM_CP_DEPTH;
    const CpSlot L = cp_slot(d.cp_max_el, d.cp_max_nl);
    const int nidx = cp_idx_ints(d.cp_max_el, d.cp_max_nl);
    int32_t *idx = reinterpret_cast<int32_t *>(cpsm + D * L.bytes);
    const double4 *u = d.ubuf[(s + 1) & 1];
    const int nC = d.nblk[ST_C], G = (int)gridDim.x;
    const int64_t rec_step = s + 1;
    const int32_t stamp = (int32_t)(s + 1);
    const int b0 = (int)blockIdx.x;
    for (int q = 0; q <= D; ++q)
        if (b0 + q * G < nC) cp_issue_idx(d, b0 + q * G, idx + (q % (D + 2)) * nidx, early);
    cpa_commit();
    pdl_wait();  // sigma (stage AB) and u (previous stage D) are complete from here on
    cpa_wait_all();
    __syncthreads();
    for (int q = 0; q < D - 1; ++q) {  // data of blocks 0 .. D-2, one group each
        if (b0 + q * G < nC)
            cp_issue_data(d, b0 + q * G, cpsm + (q % D) * L.bytes, L, idx + (q % (D + 2)) * nidx, u, early);
        cpa_commit();
    }
    const int tid = threadIdx.x;
    for (int j = 0;; ++j) {
        const int b = b0 + j * G;
        if (b >= nC) break;
        // block j's data (committed D - 1 groups ago) has arrived; later groups may still fly
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 2) : "memory");
        __syncthreads();
        {
            const int jn = j + D - 1, bn = b0 + jn * G;  // its indices arrived earlier
            if (bn < nC) cp_issue_data(d, bn, cpsm + (jn % D) * L.bytes, L, idx + (jn % (D + 2)) * nidx, u, early);
            const int ji = j + D + 1, bi = b0 + ji * G;
            if (bi < nC) cp_issue_idx(d, bi, idx + (ji % (D + 2)) * nidx, early);
            cpa_commit();
        }
        // ---- compute block b from its data slot (block_C's per-tet arithmetic)
        const char *sl = cpsm + (j % D) * L.bytes;
        const int64_t e = (int64_t)b * d.blk + tid;
        const bool he = e < d.E;
        bool need = false;
        if (he) {
            const uint8_t act = reinterpret_cast<const uint8_t *>(sl + L.st)[tid];
            double *fo = d.fe + 12 * (uint32_t)e;
            if (!act) {
                for (int q = 0; q < 3; ++q) st256(reinterpret_cast<double4 *>(fo) + q, 0.0, 0.0, 0.0, 0.0);
            } else {
                const uint4 lq = reinterpret_cast<const uint4 *>(sl + L.ledge)[tid];
                const int le[6] = {(int)(lq.x & 0xffff), (int)(lq.x >> 16), (int)(lq.y & 0xffff),
                                   (int)(lq.y >> 16), (int)(lq.z & 0xffff), (int)(lq.z >> 16)};
                double S0 = 0.0, S1 = 0.0, S2 = 0.0, S3 = 0.0, S4 = 0.0, S5 = 0.0, gmax = 0.0;
#pragma unroll
                for (int l = 0; l < 6; ++l) {
                    const double2 *row = reinterpret_cast<const double2 *>(sl + L.sig + 48 * le[l]);
                    const double2 p0 = row[0], p1 = row[1], p2 = row[2];
                    const double a0 = p0.x, a1 = p0.y, a2 = p1.x, a3 = p1.y, a4 = p2.x, a5 = p2.y;
                    S0 = S0 + a0;
                    S1 = S1 + a1;
                    S2 = S2 + a2;
                    S3 = S3 + a3;
                    S4 = S4 + a4;
                    S5 = S5 + a5;
                    if (early) {
                        const double r0 = fabs(a0) + fabs(a3) + fabs(a5);
                        const double r1 = fabs(a1) + fabs(a3) + fabs(a4);
                        const double r2 = fabs(a2) + fabs(a4) + fabs(a5);
                        gmax = fmax(gmax, fmax(r0, fmax(r1, r2)));
                    }
                }
                const double *gt = reinterpret_cast<const double *>(sl + L.geo) + (tid >> 5) * 352 + (tid & 31);
                double g[4][3];
#pragma unroll
                for (int a = 1; a < 4; ++a)
#pragma unroll
                    for (int c = 0; c < 3; ++c) g[a][c] = gt[32 * (2 + 3 * (a - 1) + c)];
                const double cc = gt[32];
#pragma unroll
                for (int c = 0; c < 3; ++c) g[0][c] = -((g[1][c] + g[2][c]) + g[3][c]);
                double f[12];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    f[3 * a] = cc * ((g[a][0] * S0 + g[a][1] * S3) + g[a][2] * S5);
                    f[3 * a + 1] = cc * ((g[a][1] * S1 + g[a][0] * S3) + g[a][2] * S4);
                    f[3 * a + 2] = cc * ((g[a][2] * S2 + g[a][1] * S4) + g[a][0] * S5);
                }
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    st256(reinterpret_cast<double4 *>(fo) + q, f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
                const uint8_t tf = reinterpret_cast<const uint8_t *>(sl + L.tf)[tid];
                need = crack && (tf & 1);
                if (need && early) {
                    const ushort4 lc = reinterpret_cast<const ushort4 *>(sl + L.lconn)[tid];
                    const int li[4] = {lc.x, lc.y, lc.z, lc.w};
                    double ux[4], uy[4], uz[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        const double2 *row = reinterpret_cast<const double2 *>(sl + L.u + 32 * li[a]);
                        const double2 q0 = row[0], q1 = row[1];
                        ux[a] = q0.x;
                        uy[a] = q0.y;
                        uz[a] = q1.x;
                    }
                    double d2 = 0.0;
#pragma unroll
                    for (int l = 0; l < 6; ++l) {
                        const int p = l < 3 ? 0 : (l < 5 ? 1 : 2), q = l < 3 ? l + 1 : (l < 5 ? l - 1 : 3);
                        const double dx = ux[q] - ux[p], dy = uy[q] - uy[p], dz = uz[q] - uz[p];
                        d2 = fmax(d2, (dx * dx + dy * dy) + dz * dz);
                    }
                    const double gcv = reinterpret_cast<const double *>(sl + L.gc)[tid];
                    need = !(gmax * sqrt(d2) * (1.0 + 1e-6) <= gcv);
                }
            }
        }
        if (crack) {  // the tets that fail the early-out: the step's criterion list (k_crit / k_filter)
            const unsigned mm = __ballot_sync(0xffffffffu, need);
            if (mm) {
                const int lane = threadIdx.x & 31, lead = __ffs(mm) - 1;
                int base = 0;
                if (lane == lead) base = atomicAdd(&d.ctr[3], __popc(mm));
                base = __shfl_sync(0xffffffffu, base, lead);
                if (need) d.crit_list[base + __popc(mm & ((1u << lane) - 1))] = crit_entry(rec_step, e);
            }
            if (threadIdx.x == 0) atomicAdd(&d.ctr[9], 1);  // (k_crit's polling hint, as in block_C)
        }
        __syncthreads();  // this data slot is refilled by the copies issued in iteration j + 1
    }
    (void)stamp;
}

// ------------------------------------------------------------------ stage D: node update
// Four lanes per node, lane c = component c (lane 3 carries the zero w component): the three
// component sums f_int,k,c = sum over the node's ELL row of force-slot components (ascending
// original tet id) are independent, so splitting them across lanes keeps every sum sequential
// in the oracle's order while a warp reads whole 32-B slot sectors with 8-B loads and holds
// 4x fewer registers per slot in flight.  Newmark + BC are per component as well.
// nodes per D block: four lanes per node (lane 3 carries the zero w component)
__host__ __device__ __forceinline__ int d_nodes_per_block(int threads) { return threads >> 2; }

// mode: ND_INLINE (staged and persistent kernels) -- PDL wait, resets the criterion list;
// ND_WAVE -- inputs already awaited at kernel entry, kernel-choice heuristic from stage C's count
enum { ND_INLINE = 0, ND_WAVE = 1 };
template <bool PM>
__device__ __forceinline__ void node_update(const Dev &d, int64_t kbase, int64_t kend, const double4 *u1p, double4 *u2p,
                                            int64_t s, int mode = ND_INLINE) {
    const bool wave = mode == ND_WAVE;
    const int c = threadIdx.x & 3;
    const int64_t k = kbase + (threadIdx.x >> 2);
    if (wave) {
        if (kbase == 0 && threadIdx.x == 0 && d.crit_seen && (s & 15) == 0) {
            // kernel-choice heuristic: tets that failed the early-out per step, averaged over the
            // last 16 steps (racy by design: results never depend on it)
            const int cur = *(volatile int32_t *)&d.ctr[10];
            *(volatile int32_t *)d.crit_seen = (cur - d.ctr[11]) / 16;
            d.ctr[11] = cur;
        }
    } else if (kbase == 0 && threadIdx.x == 0) {  // k_crit (if any) has consumed the step's list
        pdl_wait();
        if (d.crit_seen && (s & 15) == 0) *(volatile int32_t *)d.crit_seen = d.ctr[3];  // (host-side kernel choice)
#ifdef CEM_DEBUG_LIST
        if (s % 100 == 0) printf("[list] step %lld: %d listed of %lld tets\n", (long long)s, d.ctr[3], (long long)d.E);
#endif
        d.ctr[3] = 0;
        d.ctr[8] = 0;
        d.ctr[9] = 0;
    }
    if (k >= kend) return;
    const uint8_t fl = __ldg(&d.nflag[k]);
    if (fl & 16) return;  // multi-GPU: another rank owns (and updates) this node
    // static tables before the dependency wait (overlaps the previous stage's tail)
    const int4 *row = reinterpret_cast<const int4 *>(d.nodeE + (uint32_t)k * (uint32_t)d.wn);
    constexpr int kB = CEM_D_BATCH, kQ = kB / 4;  // slots per batch, int4 index loads per batch
    int4 q[kQ];
    // partial mode (R27): the node's exact partials from stage C, consecutive records [p0, p1)
    constexpr bool pm = PM;
    int32_t p0 = 0, p1 = 0;
    if (pm) {
        p0 = __ldg(d.poff + k);
        p1 = __ldg(d.poff + k + 1);
    } else {
#pragma unroll
        for (int j = 0; j < kQ; ++j) q[j] = j * 4 < d.wn ? __ldg(row + j) : make_int4(d.zslot, d.zslot, d.zslot, d.zslot);
    }
    const double fxc = (fl & 8) ? __ldg(reinterpret_cast<const double *>(d.fext + k) + c) : 0.0;
    const double vb0 = (fl & 7) ? __ldg(reinterpret_cast<const double *>(d.dir_v0 + k) + c) : 0.0;
    if (!wave) pdl_wait();  // force slots come from stage C (wave launches waited at kernel entry)
    // node state issued before the slot gathers (consumed after them)
    double mk = __ldcg(d.mass + k);
    const double u1 = __ldcg(reinterpret_cast<const double *>(u1p + k) + c);
    double vv = __ldcg(reinterpret_cast<const double *>(d.v + k) + c);
    double aa = __ldcg(reinterpret_cast<const double *>(d.a + k) + c);
    const int32_t dirty = __ldcg(d.dirty + k);
    const double *fec = d.fe + (c < 3 ? c : 0);  // lane c: component c of each slot (lane 3: unused sum)
    // hexahedra: the remainder-tet slots follow the row's hex-slot prefix and hold zeros unless the
    // node belongs to a remainder prism (hnrem, set by k_hexcrit; read after the wait: every
    // earlier kernel has completed)
    const int wl = (!pm && d.npe == 8 && !__ldcg(d.hnrem + k)) ? d.wn0 : d.wn;
    double f = 0.0, fc = 0.0;  // exact-sum accumulator (R27)
    if (pm) {
        // lane c: component c of each partial, s and c terms, four records per pass
        const double *pc = d.part + (c < 3 ? c : 0);
        for (int32_t p = p0; p < p1; p += 4) {
            double xs[4], xe[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const bool live = p + t < p1;
                xs[t] = live ? __ldcg(pc + 6 * (int64_t)(p + t)) : 0.0;  // (+0.0: an exact no-op)
                xe[t] = live ? __ldcg(pc + 6 * (int64_t)(p + t) + 3) : 0.0;
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                xacc(f, fc, xs[t]);
                xacc(f, fc, xe[t]);
            }
        }
    } else {
#if CEM_D_PIPE
    // software pipeline: batch i+1's slot loads are issued before batch i is summed
    {
        auto unpack = [&](const int4 (&qq)[kQ], int32_t (&sl)[kB]) {
#pragma unroll
            for (int j = 0; j < kQ; ++j) {
                sl[4 * j] = qq[j].x;
                sl[4 * j + 1] = qq[j].y;
                sl[4 * j + 2] = qq[j].z;
                sl[4 * j + 3] = qq[j].w;
            }
        };
        int32_t sl[kB];
        unpack(q, sl);
        double x[kB];
#pragma unroll
        for (int t = 0; t < kB; ++t) {
            CEM_BOUND(d, sl[t] >= 0 && sl[t] <= d.zslot);
            x[t] = __ldcg(fec + (uint32_t)CEM_FES * (uint32_t)sl[t]);
        }
        int w = kB;
        bool more = sl[kB - 1] != d.zslot && w < wl;
        if (more) {
#pragma unroll
            for (int j = 0; j < kQ; ++j)
                q[j] = w + 4 * j < wl ? __ldg(row + (w >> 2) + j) : make_int4(d.zslot, d.zslot, d.zslot, d.zslot);
        }
        for (;;) {
            double y[kB];
            bool more2 = false;
            if (more) {
                unpack(q, sl);
#pragma unroll
                for (int t = 0; t < kB; ++t) {
                    CEM_BOUND(d, sl[t] >= 0 && sl[t] <= d.zslot);
                    y[t] = __ldcg(fec + (uint32_t)CEM_FES * (uint32_t)sl[t]);
                }
                w += kB;
                more2 = sl[kB - 1] != d.zslot && w < wl;
                if (more2) {
#pragma unroll
                    for (int j = 0; j < kQ; ++j)
                        q[j] = w + 4 * j < wl ? __ldg(row + (w >> 2) + j)
                                                : make_int4(d.zslot, d.zslot, d.zslot, d.zslot);
                }
            }
#pragma unroll
            for (int t = 0; t < kB; ++t) xacc(f, fc, x[t]);
            if (!more) break;
#pragma unroll
            for (int t = 0; t < kB; ++t) x[t] = y[t];
            more = more2;
        }
    }
#else
    for (int w = 0;;) {
        // padding entries point at an all-zero slot: adding +0.0 is an exact no-op here
        int32_t sl[kB];
#pragma unroll
        for (int j = 0; j < kQ; ++j) {
            sl[4 * j] = q[j].x;
            sl[4 * j + 1] = q[j].y;
            sl[4 * j + 2] = q[j].z;
            sl[4 * j + 3] = q[j].w;
        }
        double x[kB];
#pragma unroll
        for (int t = 0; t < kB; ++t) {
            CEM_BOUND(d, sl[t] >= 0 && sl[t] <= d.zslot);
            x[t] = __ldcg(fec + (uint32_t)CEM_FES * (uint32_t)sl[t]);
        }
        w += kB;
        const bool more = sl[kB - 1] != d.zslot && w < wl;
        if (more) {
#pragma unroll
            for (int j = 0; j < kQ; ++j)
                q[j] = w + 4 * j < wl ? __ldg(row + (w >> 2) + j) : make_int4(d.zslot, d.zslot, d.zslot, d.zslot);
        }
#pragma unroll
        for (int t = 0; t < kB; ++t) xacc(f, fc, x[t]);
        if (!more) break;
    }
#endif
    }
    f = f + fc;  // RN(s + c) (R27)
    const double dt = d.dt;
    const double t1 = (double)(s + 1) * dt;
    if (c == 3) {
        vv = aa = 0.0;
    } else if (mk == 0.0) {  // frozen node (R15)
        vv = 0.0;
        aa = 0.0;
    } else if (fl >> c & 1) {  // prescribed velocity ramp (R17)
        const double t0 = d.t0;
        if (t0 <= 0.0) {
            vv = vb0;
            aa = 0.0;
        } else {
            vv = (t1 <= t0) ? (t1 / t0) * vb0 : vb0;
            aa = (t1 < t0) ? vb0 / t0 : 0.0;
        }
    } else {  // a = (f_ext - f_int)/m ; v += dt ((1-gamma) a_old + gamma a_new)
        const double an = (fxc - f) / mk;
        vv = vv + dt * (d.omg * aa + d.gamma * an);
        aa = an;
    }
    if (d.rprev && c < 3 && (fl >> c & 1)) {
        // energy ledger: support force R = m a - (f_ext - f_int) of the prescribed dof and its
        // trapezoidal work 1/2 (R_s + R_{s+1}) (u_{s+1} - u_s) (oracle reaction_work, R22),
        // accumulated per dof (one writer: independent of how nodes are blocked)
        const double R = mk * aa - (fxc - f);
        const double us = __ldcg(reinterpret_cast<const double *>(u2p + k) + c);  // u_s, overwritten below
        double *rp = d.rprev + 3 * k + c;
        d.wr_dof[3 * k + c] += 0.5 * (*rp + R) * (u1 - us);
        *rp = R;
    }
    if (dirty == (int32_t)(s + 1)) {
        // an incident tet split in this step: lumped mass from the active incidences;
        // m = 0 -> frozen, v = a = 0 (R15)
        mk = d.npe == 8 ? hex_node_mass(d.self, k) : node_mass4(d, k, c);
        if (c == 0) d.mass[k] = mk;
        if (mk == 0.0) vv = aa = 0.0;
    }
    // predictor u_{s+2} = u_{s+1} + dt v + dt^2/2 a
    const double u2 = c == 3 ? 0.0 : (u1 + dt * vv) + d.hdt2 * aa;
    reinterpret_cast<double *>(d.v + k)[c] = vv;
    reinterpret_cast<double *>(d.a + k)[c] = aa;
    reinterpret_cast<double *>(u2p + k)[c] = u2;
    if (d.p2p_np && c < 3)  // P2P halo: the peers holding this owned node receive u_{s+2} now
        for (int32_t i = __ldg(d.p2p_noff + k); i < __ldg(d.p2p_noff + k + 1); ++i)
            reinterpret_cast<double *>(d.p2p_recv[(s & 1) * d.p2p_np + __ldg(d.p2p_npeer + i)] + __ldg(d.p2p_nbyte + i))[c] = u2;
    if (c < 3 && (!isfinite(u1) || !isfinite(vv) || !isfinite(aa))) {
        d.ctr[1] = 1;
        atomicMin(&d.ctr[2], ldro(d.node_orig + k));
    }
}



template <bool PM>
__device__ __forceinline__ void block_D(const Dev &d, int64_t kbase, int64_t kend, const double4 *u1p, double4 *u2p,
                                        int64_t s) {
    node_update<PM>(d, kbase, min(kend, d.N), u1p, u2p, s);
}


// ------------------------------------------------------------------ persistent wavefront kernel
__device__ __forceinline__ int ld_relaxed(const int32_t *p) {  // poll without invalidating L1
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void discard_l2(const void *p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// Invalidate, without write-back, the L2 lines holding producer block pb's intermediate
// records (tau / sigma / f_e).  Called by the LAST consumer block of pb in a step, before it
// publishes its own completion (the next writer of those lines transitively waits for it).
__device__ __forceinline__ void discard_block(const Dev &d, int pg, int pb) {
    const char *base;
    int64_t bytes, off;
    if (pg == ST_AB) {  // the 16-B plane is left to the normal eviction
        base = reinterpret_cast<const char *>(d.srec);
        off = (int64_t)pb * d.blk_ab * 32;
        bytes = min((int64_t)d.blk_ab, d.S - (int64_t)pb * d.blk_ab) * 32;
    } else {
        base = reinterpret_cast<const char *>(d.fe);
        off = (int64_t)pb * d.blk * 32 * CEM_FES;
        bytes = min((int64_t)d.blk, d.E - (int64_t)pb * d.blk) * 32 * CEM_FES;
    }
    for (int64_t l = threadIdx.x; l < bytes / 128; l += blockDim.x) discard_l2(base + off + 128 * l);
}

#ifndef CEM_PERSIST_MINB
#define CEM_PERSIST_MINB 4
#endif
__global__ void __launch_bounds__(256, CEM_PERSIST_MINB) k_persistent(Dev d, int64_t step0, int64_t nsteps, int crack_every) {
    extern __shared__ __align__(16) double sm[];
    __shared__ unsigned long long sh_q;
    __shared__ int sh_ndisc;
    __shared__ int sh_disc[64];
    const unsigned long long total = (unsigned long long)nsteps * (unsigned long long)d.P;
    const int tid = threadIdx.x;
    unsigned long long qn = 0;
    if (tid == 0) qn = atomicAdd(d.head, 1ull);
    for (;;) {
        if (tid == 0) {
            sh_q = qn;
            qn = atomicAdd(d.head, 1ull);  // next item, in flight while this one runs
            sh_ndisc = 0;
        }
        __syncthreads();
        const unsigned long long q = sh_q;
        if (q >= total) return;
        const int64_t s = step0 + (int64_t)(q / (unsigned long long)d.P);
        const int code = __ldg(d.sched + (q % (unsigned long long)d.P));
        const int g = code >> 28, b = code & 0x0FFFFFFF;
        const int64_t qd = (int64_t)g * d.maxblk + b;
        const int dlo = __ldg(d.dep_off + qd), dhi = __ldg(d.dep_off + qd + 1);
        const int pg = g == ST_AB ? ST_D : g - 1;
        // wait for the producer blocks (warp 0; lanes poll counters in parallel)
        if (tid < 32) {
            const int need = g == ST_AB ? (int)s : (int)(s + 1);
            const int32_t *c = d.cnt + (int64_t)pg * d.maxblk;
            int polls = 0;
            for (int i = dlo + tid; i < dhi; i += 32) {
                const int pb = __ldg(d.dep + i);
                while (ld_relaxed(c + pb) < need) {
                    ++polls;
                    __nanosleep(64);
                }
            }
            __syncwarp();
            if (tid == 0) __threadfence();  // one acquire-side fence per item (produced data is read via .cg)
#ifdef CEM_POLL_STATS
            polls = __reduce_add_sync(0xffffffffu, polls);
            if (tid == 0) {
                atomicAdd(&d.ctr[4 + g], polls);
                if (polls) atomicAdd(&d.ctr[7], 1);
            }
#endif
        }
        __syncthreads();
        const double4 *u1 = d.ubuf[(s + 1) & 1];
        switch (g) {
            case ST_AB: block_AB(d, b, u1, sm); break;
            case ST_C:
                if (d.part) block_C<true>(d, b, u1, crack_on(crack_every, s), s + 1, (int32_t)(s + 1), sm);
                else block_C<false>(d, b, u1, crack_on(crack_every, s), s + 1, (int32_t)(s + 1), sm);
                break;
            default:
                for (int64_t k0 = (int64_t)b * d.blk; k0 < (int64_t)(b + 1) * d.blk; k0 += d_nodes_per_block(blockDim.x))
                    if (d.part) block_D<true>(d, k0, (int64_t)(b + 1) * d.blk, u1, d.ubuf[s & 1], s);  // a D item covers blk nodes
                    else block_D<false>(d, k0, (int64_t)(b + 1) * d.blk, u1, d.ubuf[s & 1], s);
                break;
        }
        __syncthreads();
        if (g != ST_AB && !(d.flags & CEM_F_NO_DISCARD)) {
            // consumers of intermediates: the last one of each producer block discards it
            if (tid < 32) {
                int32_t *cd = d.cons_done + (int64_t)(g - 1) * d.maxblk;
                const int32_t *nc = d.ncons + (int64_t)(g - 1) * d.maxblk;
                for (int i = dlo + tid; i < dhi; i += 32) {
                    const int pb = __ldg(d.dep + i);
                    const int old = atomicAdd(cd + pb, 1);
                    if (old == __ldg(nc + pb) - 1) {
                        cd[pb] = 0;
                        const int slot = atomicAdd(&sh_ndisc, 1);
                        if (slot < 64) sh_disc[slot] = pb;
                        else discard_block(d, g - 1, pb);  // (rare) overflow: this lane alone
                    }
                }
            }
            __syncthreads();
            const int nd = min(sh_ndisc, 64);
            for (int i = 0; i < nd; ++i) discard_block(d, g - 1, sh_disc[i]);
            __syncthreads();
        }
        if (tid == 0) {
            __threadfence();
            atomicExch(d.cnt + qd, (int)(s + 1));
        }
    }
}

// ------------------------------------------------------------------ staged kernels (one per stage)
#ifndef CEM_AB_MINB
#define CEM_AB_MINB 4
#endif
#ifndef CEM_C_MINB
#define CEM_C_MINB 4
#endif
#ifndef CEM_D_MINB
#define CEM_D_MINB 5
#endif

__global__ void __launch_bounds__(256, CEM_AB_MINB) k_AB(Dev d, int64_t s, int boff) {
    extern __shared__ __align__(16) double sm[];
    pdl_trigger();
    block_AB(d, (int)blockIdx.x + boff, d.ubuf[(s + 1) & 1], sm);
}
// crack: crack_on(crack_every, s), decided on the host (a 64-bit modulo per thread otherwise).
// k_C: exact partials (R27, the default); k_Cs: force slots (CEM_PARTIALS=0, hexahedral D path)
#define CEM_K_C_BODY(PM)                                                                                      \
    extern __shared__ double sm[];                                                                            \
    pdl_trigger();                                                                                            \
    block_C<PM>(d, (int)blockIdx.x + boff, d.ubuf[(s + 1) & 1], crack != 0, s + 1, (int32_t)(s + 1), sm, true);
__global__ void __launch_bounds__(256, CEM_C_MINB) k_C(Dev d, int64_t s, int crack, int boff) { CEM_K_C_BODY(true) }
__global__ void __launch_bounds__(256, CEM_C_MINB) k_Cs(Dev d, int64_t s, int crack, int boff) { CEM_K_C_BODY(false) }
// full criterion of the tets stage C flagged (ctr[3] of them in crit_list), one warp per tet.
// Its inputs other than the list (sigma from stage AB, u, X, the tables) are final before stage C
// writes any entry, and its outputs (the split tets' state, Vhat flags, node stamps, records) are
// read only by stage D and the next step -- never by stage C, which is done with a tet when it
// lists it.  So the warps take their entries while stage C is still running (PDL launches k_crit
// once every stage-C block has started): the warp owning list index i polls it (relaxed, no L1
// invalidation, with a back-off) until it holds an entry stamped with this step -- visible only
// after stage C passed its wait, hence after every earlier kernel completed -- or stage C's blocks
// have all reached their list append (ctr[9], a hint) or a poll budget runs out; then it waits for
// stage C's completion (griddepcontrol.wait: the list and its length ctr[3] are final) and takes
// its remaining indices.  Every listed tet is evaluated exactly once, by the warp owning its
// index, with the same inputs whatever the timing.
__device__ __forceinline__ long long ld_relaxed64(const int64_t *p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
#ifndef CEM_CRIT_POLLS
#define CEM_CRIT_POLLS 256  // poll budget per warp before the completion wait (a safety bound)
#endif
#ifndef CEM_CRIT_IGRID
#define CEM_CRIT_IGRID 37  // k_crit blocks when no recent step had a list (fewer pollers beside stage C's tail)
#endif
__global__ void __launch_bounds__(256) k_crit(Dev d, int64_t s, int poll_budget) {
    __shared__ CritScratch scratch[8];
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const int nw = (int)(gridDim.x * (blockDim.x >> 5));
    const double4 *u = d.ubuf[(s + 1) & 1];
    const int64_t rec = s + 1;
    int i = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
    // phase 1: entries as stage C writes them
    for (int polls = 0; i < d.E && polls < poll_budget;) {
        long long v = 0;
        int done = 0;
        if (lane == 0) {
            v = ld_relaxed64(d.crit_list + i);
            if ((v >> 32) != rec) done = ld_relaxed(&d.ctr[9]) >= d.nblk[ST_C];
        }
        v = __shfl_sync(0xffffffffu, v, 0);
        if ((v >> 32) == rec) {
            const int64_t e = (int32_t)(v & 0xffffffff);
            CEM_BOUND(d, e >= 0 && e < d.E);
            criterion_warp_body(d, e, u, ldro(d.gc + e), rec, (int32_t)rec, (__ldg(d.tflag + e) & 2) != 0,
                                scratch[threadIdx.x >> 5]);
            i += nw;
            continue;
        }
        if (__shfl_sync(0xffffffffu, done, 0)) break;
        ++polls;
        __nanosleep(256);
    }
    // phase 2: stage C complete, the list final
    pdl_wait();
    const int n = *(volatile int32_t *)&d.ctr[3];
    for (; i < n; i += nw) {
        const int64_t e = (int32_t)(d.crit_list[i] & 0xffffffff);
        CEM_BOUND(d, n <= d.E && e >= 0 && e < d.E && (d.crit_list[i] >> 32) == rec);
        criterion_warp_body(d, e, u, ldro(d.gc + e), rec, (int32_t)rec, (__ldg(d.tflag + e) & 2) != 0,
                            scratch[threadIdx.x >> 5]);
    }
}

// The same decisions for long lists (cracking phases), in two kernels.  k_filter: one thread per
// listed tet applies the refined early-out (crit_refined_need) and appends the survivors (order
// irrelevant: every decision is independent) -- a latency-bound pass that runs at full
// occupancy.  k_eval: each warp evaluates kCB survivors at a time so that every warp instruction
// carries several tets: lanes (j, a) gather the nodes, lanes (j, l) the Heaviside flags and
// principal pairs of the kCB x 6 edges, all lanes the kCB x 24 candidates, then lane j scans tet
// j's candidates in the oracle's order (k = 0..23; max G, ties -> larger area, then lower k: R14)
// and splits.
constexpr int kCB = CEM_CRIT_BATCH;
struct CritBatch {
    CritScratch t[kCB];
    double G[kCB][24], A[kCB][24];
};
__host__ __device__ constexpr int crit_batch_warps() { return CEM_CRIT_THREADS / 32; }
__global__ void __launch_bounds__(256, CEM_FILTER_MINB) k_filter(Dev d, int64_t s) {
    pdl_trigger();
    pdl_wait();  // the list and the sigma records come from stage C / AB
    const int n = *(volatile int32_t *)&d.ctr[3];
    const double4 *u = d.ubuf[(s + 1) & 1];
    const int lane = threadIdx.x & 31;
    const int stride = (int)(gridDim.x * blockDim.x);
    for (int i0 = (int)(blockIdx.x * blockDim.x + (threadIdx.x & ~31u)); i0 < n; i0 += stride) {  // warp-uniform
        const int i = i0 + lane;
        int32_t e = 0;
        bool need = false;
        if (i < n) {
            e = (int32_t)(d.crit_list[i] & 0xffffffff);
            CEM_BOUND(d, n <= d.E && e >= 0 && e < d.E);
            // CEM_F_NO_EARLY_OUT: every listed tet gets the full 24-candidate evaluation
            need = (d.flags & CEM_F_NO_EARLY_OUT) || crit_refined_need(d.self, e, u, ldro(d.gc + e));
        }
        const unsigned mm = __ballot_sync(0xffffffffu, need);
        if (mm) {
            const int lead = __ffs(mm) - 1;
            int base = 0;
            if (lane == lead) base = atomicAdd(&d.ctr[8], __popc(mm));
            base = __shfl_sync(0xffffffffu, base, lead);
            if (need) d.crit_surv[base + __popc(mm & ((1u << lane) - 1u))] = e;
        }
    }
}
__global__ void __launch_bounds__(CEM_CRIT_THREADS, CEM_CRITB_MINB) k_eval(Dev d, int64_t s) {
    extern __shared__ __align__(16) unsigned char crit_smem[];
    CritBatch &wb = reinterpret_cast<CritBatch *>(crit_smem)[threadIdx.x >> 5];
    pdl_trigger();
    pdl_wait();  // the survivors come from k_filter
    const int ns = *(volatile int32_t *)&d.ctr[8];
    const int nw = (int)(gridDim.x * (blockDim.x >> 5));
    const double4 *u = d.ubuf[(s + 1) & 1];
    const int lane = threadIdx.x & 31;
    const int32_t *ids = d.crit_surv;
    for (int b0 = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kCB; b0 < ns; b0 += nw * kCB) {
        const int cnt = min(kCB, ns - b0);
        if (lane < 4 * cnt) {  // (j, a): node a of tet j
            const int j = lane >> 2, a = lane & 3;
            const int4 t = __ldg(&d.conn[ids[b0 + j]]);
            const int nd = a == 0 ? t.x : (a == 1 ? t.y : (a == 2 ? t.z : t.w));
            const double4 x = ldro4(&d.X[nd]);
            const double4 uu = ldcg256(&u[nd]);
            CritScratch &w = wb.t[j];
            w.X[a][0] = x.x;
            w.X[a][1] = x.y;
            w.X[a][2] = x.z;
            w.U[a][0] = uu.x;
            w.U[a][1] = uu.y;
            w.U[a][2] = uu.z;
        }
        __syncwarp();
        if (lane < 6 * cnt) {  // (j, l): edge l of tet j
            const int j = lane / 6, l = lane - 6 * j;
            CritScratch &w = wb.t[j];
            const Vec3 du = {w.U[c_eq[l]][0] - w.U[c_ep[l]][0], w.U[c_eq[l]][1] - w.U[c_ep[l]][1],
                             w.U[c_eq[l]][2] - w.U[c_ep[l]][2]};
            const Vec3 dX = {w.X[c_eq[l]][0] - w.X[c_ep[l]][0], w.X[c_eq[l]][1] - w.X[c_ep[l]][1],
                             w.X[c_eq[l]][2] - w.X[c_ep[l]][2]};
            const Vec3 ww = {2.0 * dX.x + du.x, 2.0 * dX.y + du.y, 2.0 * dX.z + du.z};
            w.H[l] = vdot(du, ww) > 0.0;  // eq:stretch-delta Heaviside, R6
            double s6[6];
            load_sigma(d, ldro(d.eedge + (int64_t)l * d.E + ids[b0 + j]), s6);
            Eig eg;
            principal(s6, eg);
            w.eg[l] = eg;
        }
        __syncwarp();
        for (int q = lane; q < 24 * cnt; q += 32) {  // (j, k): candidate k of tet j
            const int j = q / 24, k = q - 24 * j;
            double G, A;
            candidate(wb.t[j], k, (d.flags & CEM_F_FRONT_BOTH_STRETCHED) != 0, G, A);
            wb.G[j][k] = G;
            wb.A[j][k] = A;
        }
        __syncwarp();
        if (lane < cnt) {
            const int j = lane;
            const int64_t te = ids[b0 + j];
            double Gb = 0.0, Ab = 0.0;
            int kb = -1;
            for (int k = 0; k < 24; ++k) {
                const double G = wb.G[j][k], A = wb.A[j][k];
                if (kb < 0 || G > Gb || (G == Gb && A > Ab)) {
                    Gb = G;
                    kb = k;
                    Ab = A;
                }
            }
            if (Gb > ldro(d.gc + te))
                split_tet(d, te, __ldg(&d.conn[te]), Gb, kb, Ab, s + 1, (int32_t)(s + 1), (__ldg(d.tflag + te) & 2) != 0);
        }
        __syncwarp();  // the scratch is reused by the next batch
    }
}
// bd_target > 0 (multi-GPU P2P halo): the blocks are taken in d.d_order, the blocks holding nodes
// that peers need first; the last of those to finish signals the peers (st.release.sys of step
// s + 2, the value the per-step sync kernel waits for) while the interior blocks still run, so a
// peer's unpack and next step overlap this rank's interior update (SURVEY.md §8(e) "update the
// boundary nodes first").  bd_target = the cumulative count of boundary blocks after this step.
// k_D: exact partials (default); k_Ds: force slots
__global__ void __launch_bounds__(256, CEM_D_MINB) k_D(Dev d, int64_t s) {
    pdl_trigger();
    const int64_t k0 = (int64_t)blockIdx.x * d_nodes_per_block(blockDim.x);
    block_D<true>(d, k0, k0 + d_nodes_per_block(blockDim.x), d.ubuf[(s + 1) & 1], d.ubuf[s & 1], s);
}
__global__ void __launch_bounds__(256, CEM_D_MINB) k_Ds(Dev d, int64_t s) {
    pdl_trigger();
    const int64_t k0 = (int64_t)blockIdx.x * d_nodes_per_block(blockDim.x);
    block_D<false>(d, k0, k0 + d_nodes_per_block(blockDim.x), d.ubuf[(s + 1) & 1], d.ubuf[s & 1], s);
}
// hexahedral contexts: the slot-mode body under a looser register bound (k_Ds spills 56 B at the 48
// registers that fit 5 CTAs per SM)
#ifndef CEM_DH_MINB
#define CEM_DH_MINB 4  // (61 registers, no spill; 3 / 4 CTAs per SM: 385 / 368 us per step on 100^3 hexes, k_Ds at 5: 387)
#endif
__global__ void __launch_bounds__(256, CEM_DH_MINB) k_Dh(Dev d, int64_t s) {
    pdl_trigger();
    const int64_t k0 = (int64_t)blockIdx.x * d_nodes_per_block(blockDim.x);
    block_D<false>(d, k0, k0 + d_nodes_per_block(blockDim.x), d.ubuf[(s + 1) & 1], d.ubuf[s & 1], s);
}
// (a separate kernel, so that the single-GPU stage D keeps its register allocation)
template <bool PM>
__device__ __forceinline__ void k_Db_body(const Dev &d, int64_t s, unsigned long long bd_target) {
    pdl_trigger();
    const int bi = (int)blockIdx.x;
    const int b = __ldg(d.d_order + bi);
    const int64_t k0 = (int64_t)b * d_nodes_per_block(blockDim.x);
    block_D<PM>(d, k0, k0 + d_nodes_per_block(blockDim.x), d.ubuf[(s + 1) & 1], d.ubuf[s & 1], s);
    if (bi < d.d_nbound) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();  // this block's stores into the peers' buffers
            if (atomicAdd(d.bdone, 1ull) + 1ull == bd_target)
                for (int j = 0; j < d.p2p_np; ++j)
                    asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(d.p2p_flag_out[j]), "l"(s + 2) : "memory");
        }
    }
}
__global__ void __launch_bounds__(256, CEM_D_MINB) k_Db(Dev d, int64_t s, unsigned long long bd_target) { k_Db_body<true>(d, s, bd_target); }
__global__ void __launch_bounds__(256, CEM_D_MINB) k_Dbs(Dev d, int64_t s, unsigned long long bd_target) { k_Db_body<false>(d, s, bd_target); }

__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// ---- dataflow ("wave") kernels: block b = blockIdx.x + boff of the stage; the crack criterion
// is evaluated inside stage C's block (warp-cooperative), as in the persistent kernel
// (rel: the step is s + *d.wstep -- graph replays read the base step from device memory)
__device__ __forceinline__ int64_t wave_step(const Dev &d, int64_t s, int rel) {
    return rel ? s + *(volatile const int64_t *)d.wstep : s;
}
__global__ void __launch_bounds__(256, CEM_AB_MINB) k_AB_w(Dev d, int64_t s, int boff, int rel) {
    extern __shared__ __align__(16) double sm[];
    pdl_trigger();
    s = wave_step(d, s, rel);
    const int b = (int)blockIdx.x + boff;
    block_AB(d, b, d.ubuf[(s + 1) & 1], sm, nullptr, (int)s);
    wave_done(d, ST_AB, b, (int)(s + 1));
}
__global__ void __launch_bounds__(256, CEM_C_MINB) k_C_w(Dev d, int64_t s, int crack_every, int boff, int rel) {
    extern __shared__ double sm[];
    pdl_trigger();
    s = wave_step(d, s, rel);
    const int b = (int)blockIdx.x + boff;
    if (d.part) block_C<true>(d, b, d.ubuf[(s + 1) & 1], crack_on(crack_every, s), s + 1, (int32_t)(s + 1), sm, false, (int)(s + 1));
    else block_C<false>(d, b, d.ubuf[(s + 1) & 1], crack_on(crack_every, s), s + 1, (int32_t)(s + 1), sm, false, (int)(s + 1));
    wave_done(d, ST_C, b, (int)(s + 1));
}
__global__ void __launch_bounds__(256, CEM_D_MINB) k_D_w(Dev d, int64_t s, int boff, int rel) {
    pdl_trigger();
    s = wave_step(d, s, rel);
    const int b = (int)blockIdx.x + boff;
    wave_wait(d, ST_D, b, (int)(s + 1));
    if (d.part) node_update<true>(d, (int64_t)b * kDW, min((int64_t)(b + 1) * kDW, d.N), d.ubuf[(s + 1) & 1], d.ubuf[s & 1], s, ND_WAVE);
    else node_update<false>(d, (int64_t)b * kDW, min((int64_t)(b + 1) * kDW, d.N), d.ubuf[(s + 1) & 1], d.ubuf[s & 1], s, ND_WAVE);
    wave_done(d, ST_D, b, (int)(s + 1));
}

// end of a run of wave launches: returns once every block of every stage has published step
// value `need` (launched without the PDL attribute; what follows on the stream sees all the work)
__global__ void __launch_bounds__(1024) k_wave_join(Dev d, int64_t need64, int rel) {
    const int need = (int)wave_step(d, need64, rel);
    for (int g = 0; g < ST_COUNT; ++g) {
        const int n = g == ST_D ? (int)((d.N + kDW - 1) / kDW) : d.nblk[g];
        const int32_t *c = d.wcnt + (int64_t)g * d.wmax;
        for (int i = (int)threadIdx.x; i < n; i += (int)blockDim.x)
            while (ld_acquire_gpu(c + i) < need) __nanosleep(64);
    }
    __syncthreads();
    if (threadIdx.x == 0) __threadfence();
}

// energy ledger on the current state u_n, v_n (cem_energy): per-block partials, fixed order
__global__ void __launch_bounds__(256) k_energy_edges(Dev d, int64_t n, double *part) {
    extern __shared__ __align__(16) double sm[];
    block_AB(d, blockIdx.x, d.ubuf[n & 1], sm, part);
}
__global__ void __launch_bounds__(256) k_energy_nodes(Dev d, int64_t n, double *part) {
    __shared__ double red[32];
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double t = 0.0, w = 0.0, r = 0.0;
    if (k < d.N && !(__ldg(&d.nflag[k]) & 16)) {
        const double4 v = ld4(&d.v[k]), u = ld4(&d.ubuf[n & 1][k]);
        t = d.mass[k] * ((v.x * v.x + v.y * v.y) + v.z * v.z);  // oracle orc_energy
        if (__ldg(&d.nflag[k]) & 8) {
            const double4 f = ldro4(&d.fext[k]);
            w = (f.x * u.x + f.y * u.y) + f.z * u.z;
        }
        if (d.rprev) r = (d.wr_dof[3 * k] + d.wr_dof[3 * k + 1]) + d.wr_dof[3 * k + 2];
    }
    const double ts = block_sum(t, red);
    const double ws = block_sum(w, red);
    const double rs = block_sum(r, red);
    if (threadIdx.x == 0) {
        part[3 * blockIdx.x] = ts;
        part[3 * blockIdx.x + 1] = ws;
        part[3 * blockIdx.x + 2] = rs;
    }
}

// criterion on the current state u_n (cem_crack_update)
__global__ void __launch_bounds__(256) k_AB_cur(Dev d, int64_t n) {
    extern __shared__ __align__(16) double sm[];
    block_AB(d, blockIdx.x, d.ubuf[n & 1], sm);
}
__global__ void __launch_bounds__(256, 4) k_C_cur(Dev d, int64_t n, int32_t stamp) {
    extern __shared__ double sm[];
    if (d.part) block_C<true>(d, blockIdx.x, d.ubuf[n & 1], true, n, stamp, sm);
    else block_C<false>(d, blockIdx.x, d.ubuf[n & 1], true, n, stamp, sm);
}
// nodes of tets split by cem_crack_update: new mass; frozen -> v = a = 0 and the pending
// prediction u_{n+1} restarts from u_n
__global__ void __launch_bounds__(256) k_fix_cur(Dev d, int64_t n, int32_t stamp) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= d.N || d.dirty[k] != stamp) return;
    const double acc = node_mass(d, k);
    d.mass[k] = acc;
    if (acc == 0.0) {
        st4(&d.v[k], 0.0, 0.0, 0.0, 0.0);
        st4(&d.a[k], 0.0, 0.0, 0.0, 0.0);
        const double4 un = ld4(&d.ubuf[n & 1][k]);
        st4(&d.ubuf[(n + 1) & 1][k], (un.x + d.dt * 0.0) + d.hdt2 * 0.0, (un.y + d.dt * 0.0) + d.hdt2 * 0.0,
            (un.z + d.dt * 0.0) + d.hdt2 * 0.0, 0.0);
    }
}

// ------------------------------------------------------------------ hexahedral crack patterns III-VI
// (R28; the hex oracle's hex_candidate / hex_crack, same expressions).  One thread
// per hex on crack steps, between stage C and stage D: an active hex evaluates its 84 candidates
// (III k = 2f + j, IV 12 + 4f + 2j + t, V 36 + 4f + i, VI 60 + 4f + i), a split hex with a remainder
// evaluates its active tets with the tet criterion (candidate(), R7).  Decisions use the pre-split
// state (R18): this thread's own hex and tets only.  A split deactivates, records (hex e or tet
// E + 3e + i) and stamps the element's nodes for stage D's mass recomputation; IV-VI activate the
// three tets of the half-hex prism (A,B,C,A'), (B,C,A',B'), (C,A',B',C').
__constant__ int8_t c_hf[6][4] = {{0, 1, 2, 3}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};
__constant__ int8_t c_hpartner[6][8] = {{4, 5, 6, 7, -1, -1, -1, -1}, {-1, -1, -1, -1, 0, 1, 2, 3},
                                        {3, 2, -1, -1, 7, 6, -1, -1},   {-1, 0, 3, -1, -1, 4, 7, -1},
                                        {-1, -1, 1, 0, -1, -1, 5, 4},   {1, -1, -1, 2, 5, -1, -1, 6}};
__constant__ int8_t c_hep[12] = {0, 1, 2, 0, 4, 5, 6, 4, 0, 1, 2, 3};
__constant__ int8_t c_heq[12] = {1, 2, 3, 3, 5, 6, 7, 7, 4, 5, 6, 7};
__constant__ int8_t c_hpair2[8][8] = {{-1, 0, 1, 2, 3, 4, 5, 6},     {0, -1, 7, 8, 9, 10, 11, 12},
                                      {1, 7, -1, 13, 14, 15, 16, 17}, {2, 8, 13, -1, 18, 19, 20, 21},
                                      {3, 9, 14, 18, -1, 22, 23, 24}, {4, 10, 15, 19, 22, -1, 25, 26},
                                      {5, 11, 16, 20, 23, 25, -1, 27}, {6, 12, 17, 21, 24, 26, 27, -1}};
__device__ __forceinline__ int hedge(int a, int b) {  // local hex edge of (a, b), -1 for a diagonal
    const int p = a < b ? a : b, q = a < b ? b : a;
    for (int l = 0; l < 12; ++l)
        if (c_hep[l] == p && c_heq[l] == q) return l;
    return -1;
}
struct HexScratch {
    double X[8][3], U[8][3], G[12][3];
    int H[12];
    Eig eg[12];
};
__device__ double hex_Dd(const HexScratch &w, int l, Vec3 m) {
    if (!w.H[l]) return 0.0;
    const int p = c_hep[l], q = c_heq[l];
    const Vec3 du = {w.U[q][0] - w.U[p][0], w.U[q][1] - w.U[p][1], w.U[q][2] - w.U[p][2]};
    const Vec3 dX = {w.X[q][0] - w.X[p][0], w.X[q][1] - w.X[p][1], w.X[q][2] - w.X[p][2]};
    return vdot(du, m) * dsgn(vdot(dX, m));
}
// m = (Gq - Gp) x (R - M), M = (Gp + Gq)/2, R = Rm or (Rm + Rn)/2
__device__ Vec3 hex_m(const double *Gp, const double *Gq, const double *Rm, const double *Rn) {
    double d1[3], d2[3];
    for (int c = 0; c < 3; ++c) {
        const double M = 0.5 * (Gp[c] + Gq[c]), R = Rn ? 0.5 * (Rm[c] + Rn[c]) : Rm[c];
        d1[c] = Gq[c] - Gp[c];
        d2[c] = R - M;
    }
    return vcross(Vec3{d1[0], d1[1], d1[2]}, Vec3{d2[0], d2[1], d2[2]});
}
__device__ __noinline__ bool hex_candidate(const HexScratch &w, int k, bool both, double &G, double &area, int *P) {
    int lp, lq;
    bool rem = true;
    if (k < 36) {
        int f, j, t = 0;
        if (k < 12) {
            f = k / 2;
            j = k % 2;
        } else {
            f = (k - 12) / 4;
            j = ((k - 12) / 2) % 2;
            t = (k - 12) % 2;
        }
        const int a = c_hf[f][j], b = c_hf[f][j + 1], c = c_hf[f][(j + 2) % 4], dd = c_hf[f][(j + 3) % 4];
        const int a1 = c_hpartner[f][a], b1 = c_hpartner[f][b], c1 = c_hpartner[f][c], d1 = c_hpartner[f][dd];
        lp = hedge(a, b);
        lq = hedge(dd, c);
        if (k < 12) {
            const int lp1 = hedge(a1, b1), lq1 = hedge(d1, c1);
            const Vec3 m = hex_m(w.G[lp], w.G[lq], w.G[lp1], w.G[lq1]);
            const double mm = vdot(m, m);
            const double A1 = sig_proj(w.eg[lp1], m) * hex_Dd(w, lp, m);
            const double A2 = sig_proj(w.eg[lq1], m) * hex_Dd(w, lq, m);
            G = (0.5 * (A1 + A2)) / mm;
            area = sqrt(mm);
            rem = false;
        } else {
            const int g = t == 0 ? hedge(a1, d1) : hedge(b1, c1);
            const Vec3 m = hex_m(w.G[lp], w.G[lq], w.G[g], nullptr);
            const double mm = vdot(m, m);
            const double A1 = sig_proj(w.eg[g], m) * hex_Dd(w, lp, m);
            const double A2 = sig_proj(w.eg[g], m) * hex_Dd(w, lq, m);
            G = (0.5 * (A1 + A2)) / mm;
            area = sqrt(mm);
            if (t == 0) {
                P[0] = b; P[1] = b1; P[2] = a1; P[3] = c; P[4] = c1; P[5] = d1;
            } else {
                P[0] = a; P[1] = a1; P[2] = b1; P[3] = dd; P[4] = d1; P[5] = c1;
            }
        }
    } else {
        const int vi = k < 60 ? k - 36 : k - 60, f = vi / 4, i = vi % 4;
        const int c = c_hf[f][i], x = c_hf[f][(i + 1) % 4], z = c_hf[f][(i + 2) % 4], y = c_hf[f][(i + 3) % 4];
        const int c1 = c_hpartner[f][c], x1 = c_hpartner[f][x], z1 = c_hpartner[f][z], y1 = c_hpartner[f][y];
        lp = hedge(c, x);
        lq = hedge(c, y);
        const int lr = hedge(c, c1);
        if (k < 60) {
            const int lp1 = hedge(c1, x1), lq1 = hedge(c1, y1);
            const Vec3 m = hex_m(w.G[lp], w.G[lq], w.G[lp1], w.G[lq1]);
            const double mm = vdot(m, m);
            const double A1 = sig_proj(w.eg[lp1], m) * hex_Dd(w, lp, m);
            const double A2 = sig_proj(w.eg[lq1], m) * hex_Dd(w, lq, m);
            G = (0.5 * (A1 + A2)) / mm;
            area = sqrt(mm);
        } else {
            const Vec3 m = hex_m(w.G[lp], w.G[lq], w.G[lr], nullptr);
            const double mm = vdot(m, m);
            const double Sg = sig_proj(w.eg[lr], m);
            G = (0.5 * (Sg * (hex_Dd(w, lp, m) + hex_Dd(w, lq, m)))) / mm;
            area = sqrt(mm) / 2.0;
        }
        P[0] = x; P[1] = z; P[2] = y; P[3] = x1; P[4] = z1; P[5] = y1;
    }
    if (both && !(w.H[lp] && w.H[lq])) G = 0.0;
    return rem;
}
// tet volume and gradients (eq:CSTet_strain_discretization; the oracle's orc_tet_geometry)
__device__ void tet_geo(const double X[4][3], double *g13) {
    double d1[3], d2[3], d3[3];
    for (int c = 0; c < 3; ++c) {
        d1[c] = X[1][c] - X[0][c];
        d2[c] = X[2][c] - X[0][c];
        d3[c] = X[3][c] - X[0][c];
    }
    const Vec3 a1 = {d1[0], d1[1], d1[2]}, a2 = {d2[0], d2[1], d2[2]}, a3 = {d3[0], d3[1], d3[2]};
    const Vec3 c23 = vcross(a2, a3), c31 = vcross(a3, a1), c12 = vcross(a1, a2);
    const double det = vdot(a1, c23);
    g13[0] = det / 6.0;
    const double inv = 1.0 / det;
    const double r1[3] = {c23.x, c23.y, c23.z}, r2[3] = {c31.x, c31.y, c31.z}, r3[3] = {c12.x, c12.y, c12.z};
    for (int c = 0; c < 3; ++c) {
        g13[4 + c] = r1[c] * inv;
        g13[7 + c] = r2[c] * inv;
        g13[10 + c] = r3[c] * inv;
        g13[1 + c] = -((g13[4 + c] + g13[7 + c]) + g13[10 + c]);
    }
}
__device__ __forceinline__ void hex_record(const Dev &d, int64_t step, int32_t elem, int k, double G, double A) {
    const int slot = atomicAdd(&d.ctr[0], 1);
    CEM_BOUND(d, slot < 4 * d.E);
    d.rec_step[slot] = step;
    d.rec_elem[slot] = elem;
    d.rec_cand[slot] = k;
    d.rec_G[slot] = G;
    d.rec_area[slot] = A;
}

__global__ void __launch_bounds__(128) k_hexcrit(Dev d, int64_t s) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t E = d.E;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int32_t n[8];
    for (int a = 0; a < 8; ++a) n[a] = __ldg(d.hconn + a * E + e);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // sigma (stage B) and u_{s+1}, stage C done
    const double4 *u = d.ubuf[(s + 1) & 1];
    const int32_t stamp = (int32_t)(s + 1);
    const bool both = (d.flags & CEM_F_FRONT_BOTH_STRETCHED) != 0;
    const double gc = ldro(d.gc + e);
    if (__ldcg(d.state + e)) {
        if (!(d.flags & CEM_F_NO_EARLY_OUT)) {
            // conservative early-out (as for tets): every candidate is
            // 1/2 (S_1 Dd_1 + S_2 Dd_2) / |m|^2 with |S_i| <= |sigma_1| |m| <= g |m| (g the Gershgorin
            // bound of the stress of one of the hex's 12 edges) and |Dd_i| <= |du| |m| (du along one
            // of them), so |G_k| <= max_l g_l max_l |du_l| for all 84; skipped when that bound
            // (1 + 1e-6) <= Gc_e -- the decision "no split" either way
            // (tests/test_early_out_bounds.py pins the bound against the hex oracle's candidates)
            double U8[8][3];
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const double4 uu = ldcg256(&u[n[a]]);
                U8[a][0] = uu.x; U8[a][1] = uu.y; U8[a][2] = uu.z;
            }
            double d2 = 0.0, gmax = 0.0;
            constexpr int kp[12] = {0, 1, 2, 0, 4, 5, 6, 4, 0, 1, 2, 3}, kq[12] = {1, 2, 3, 3, 5, 6, 7, 7, 4, 5, 6, 7};  // (= c_hep, c_heq)
#pragma unroll
            for (int l = 0; l < 12; ++l) {
                const int p = kp[l], q = kq[l];
                const double dx = U8[q][0] - U8[p][0], dy = U8[q][1] - U8[p][1], dz = U8[q][2] - U8[p][2];
                d2 = fmax(d2, (dx * dx + dy * dy) + dz * dz);
                double s6[6];
                load_sigma(d, __ldg(d.heedge + (int64_t)l * E + e), s6);
                const double r0 = fabs(s6[0]) + fabs(s6[3]) + fabs(s6[5]);
                const double r1 = fabs(s6[1]) + fabs(s6[3]) + fabs(s6[4]);
                const double r2 = fabs(s6[2]) + fabs(s6[4]) + fabs(s6[5]);
                gmax = fmax(gmax, fmax(r0, fmax(r1, r2)));
            }
            if (gmax * sqrt(d2) * (1.0 + 1e-6) <= gc) return;
        }
        // failed the early-out: listed for k_hexeval (one warp per listed hex)
        d.hclist[atomicAdd(&d.ctr[3], 1)] = (int32_t)e;
        return;
    }
    if (__ldcg(d.hrem + e) < 0) return;
    const uint8_t ta = __ldcg(d.htact + e);
    uint8_t keep = ta;
    for (int i = 0; i < 3; ++i) {
        if (!(ta >> i & 1)) continue;
        const uint8_t *tl = d.htloc + 12 * e + 4 * i;
        CritScratch w;
        for (int a = 0; a < 4; ++a) {
            const double4 x = ldro4(&d.X[n[tl[a]]]);
            const double4 uu = ldcg256(&u[n[tl[a]]]);
            w.X[a][0] = x.x; w.X[a][1] = x.y; w.X[a][2] = x.z;
            w.U[a][0] = uu.x; w.U[a][1] = uu.y; w.U[a][2] = uu.z;
        }
        for (int l = 0; l < 6; ++l) {
            const Vec3 du = {w.U[c_eq[l]][0] - w.U[c_ep[l]][0], w.U[c_eq[l]][1] - w.U[c_ep[l]][1],
                             w.U[c_eq[l]][2] - w.U[c_ep[l]][2]};
            const Vec3 dX = {w.X[c_eq[l]][0] - w.X[c_ep[l]][0], w.X[c_eq[l]][1] - w.X[c_ep[l]][1],
                             w.X[c_eq[l]][2] - w.X[c_ep[l]][2]};
            const Vec3 ww = {2.0 * dX.x + du.x, 2.0 * dX.y + du.y, 2.0 * dX.z + du.z};
            w.H[l] = vdot(du, ww) > 0.0;
            double s6[6];
            load_sigma(d, __ldg(d.hpair + (int64_t)c_hpair2[tl[c_ep[l]]][tl[c_eq[l]]] * E + e), s6);
            principal(s6, w.eg[l]);
        }
        double Gb = 0.0, Ab = 0.0;
        int kb = -1;
        for (int k = 0; k < 24; ++k) {
            double G, A;
            candidate(w, k, both, G, A);
            if (kb < 0 || G > Gb || (G == Gb && A > Ab)) {
                Gb = G;
                kb = k;
                Ab = A;
            }
        }
        if (!(Gb > gc)) continue;
        keep &= (uint8_t)~(1u << i);
        hex_record(d, s + 1, (int32_t)(E + 3 * e + i), kb, Gb, Ab);
        for (int a = 0; a < 4; ++a) d.dirty[n[tl[a]]] = stamp;
    }
    if (keep != ta) d.htact[e] = keep;
}

// The listed hexes (those the early-out could not rule out), one warp each: lanes 0-7 gather the
// nodes, lanes 0-11 the edge midpoints, Heaviside flags and principal pairs (one cyclic-Jacobi solve
// per lane instead of twelve in sequence), every lane the candidates k = lane, lane + 32, lane + 64
// in ascending k; a butterfly argmax over (G, area, -k) equals the oracle's sequential scan (first
// of the largest (G, area)).  Lane 0 splits: the serial code of the first version, same expressions.
constexpr int kHexEvalWarps = 4;
__global__ void __launch_bounds__(32 * kHexEvalWarps) k_hexeval(Dev d, int64_t s) {
    __shared__ HexScratch ws[kHexEvalWarps];
    __shared__ int32_t wn[kHexEvalWarps][8];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // k_hexcrit's list is complete
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    HexScratch &w = ws[wib];
    int32_t *n = wn[wib];
    const int64_t E = d.E;
    const int nl = __ldcg(d.ctr + 3);
    const double4 *u = d.ubuf[(s + 1) & 1];
    const int32_t stamp = (int32_t)(s + 1);
    const bool both = (d.flags & CEM_F_FRONT_BOTH_STRETCHED) != 0;
    for (int it = (int)blockIdx.x * kHexEvalWarps + wib; it < nl; it += (int)gridDim.x * kHexEvalWarps) {
        const int64_t e = __ldcg(d.hclist + it);
        __syncwarp();
        if (lane < 8) {
            const int32_t na = __ldg(d.hconn + lane * E + e);
            n[lane] = na;
            const double4 x = ldro4(&d.X[na]);
            const double4 uu = ldcg256(&u[na]);
            w.X[lane][0] = x.x; w.X[lane][1] = x.y; w.X[lane][2] = x.z;
            w.U[lane][0] = uu.x; w.U[lane][1] = uu.y; w.U[lane][2] = uu.z;
        }
        __syncwarp();
        if (lane < 12) {
            const int l = lane;
            const int p = c_hep[l], q = c_heq[l];
            double du[3], dX[3], ww[3];
            for (int c = 0; c < 3; ++c) {
                w.G[l][c] = 0.5 * (w.X[p][c] + w.X[q][c]);
                du[c] = w.U[q][c] - w.U[p][c];
                dX[c] = w.X[q][c] - w.X[p][c];
                ww[c] = 2.0 * dX[c] + du[c];
            }
            w.H[l] = vdot(Vec3{du[0], du[1], du[2]}, Vec3{ww[0], ww[1], ww[2]}) > 0.0;
            double s6[6];
            load_sigma(d, __ldg(d.heedge + (int64_t)l * E + e), s6);
            principal(s6, w.eg[l]);
        }
        __syncwarp();
        double Gb = 0.0, Ab = 0.0;
        int kb = -1, P[6];
        for (int k = lane; k < 84; k += 32) {
            double G, A;
            hex_candidate(w, k, both, G, A, P);
            if (kb < 0 || G > Gb || (G == Gb && A > Ab)) {
                Gb = G;
                Ab = A;
                kb = k;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double G2 = __shfl_xor_sync(0xffffffffu, Gb, o), A2 = __shfl_xor_sync(0xffffffffu, Ab, o);
            const int k2 = __shfl_xor_sync(0xffffffffu, kb, o);
            if (G2 > Gb || (G2 == Gb && (A2 > Ab || (A2 == Ab && k2 < kb)))) {
                Gb = G2;
                Ab = A2;
                kb = k2;
            }
        }
        if (lane != 0 || !(Gb > ldro(d.gc + e))) continue;
        d.state[e] = 0;
        hex_record(d, s + 1, (int32_t)e, kb, Gb, Ab);
        double G, A;
        if (hex_candidate(w, kb, both, G, A, P)) {  // the half-hex prism remainder
            const int TT[3][4] = {{0, 1, 2, 3}, {1, 2, 3, 4}, {2, 3, 4, 5}};
            for (int i = 0; i < 3; ++i) {
                int t[4];
                for (int a = 0; a < 4; ++a) t[a] = P[TT[i][a]];
                double g13[13];
                for (int pass = 0; pass < 2; ++pass) {
                    double X4[4][3];
                    for (int a = 0; a < 4; ++a)
                        for (int c = 0; c < 3; ++c) X4[a][c] = w.X[t[a]][c];
                    tet_geo(X4, g13);
                    if (g13[0] >= 0.0 || pass) break;
                    const int sw = t[0];
                    t[0] = t[1];
                    t[1] = sw;
                }
                for (int a = 0; a < 4; ++a) d.htloc[12 * e + 4 * i + a] = (uint8_t)t[a];
                for (int j = 0; j < 13; ++j) d.htgeo[39 * e + 13 * i + j] = g13[j];
            }
            d.htact[e] = 7;
            d.hrem[e] = (int8_t)kb;
            atomicAdd(&d.ctr[24], 1);  // (count of remainders)
            // from the next step on stage D reads the remainder slots of this hex's nodes and stage B
            // evaluates its 16 diagonal edges (the three tets lie among them)
            for (int a = 0; a < 8; ++a) d.hnrem[n[a]] = 1;
            for (int a = 0; a < 8; ++a)
                for (int b = a + 1; b < 8; ++b)
                    if (hedge(a, b) < 0) {  // (a face diagonal is shared with a neighbour: listed once)
                        const int32_t kd = __ldg(d.hpair + (int64_t)c_hpair2[a][b] * E + e);
                        const unsigned i = (unsigned)(kd - d.hS_h), bit = 1u << (i & 31);
                        if (!(atomicOr(d.hediag + (i >> 5), bit) & bit)) d.hdlist[atomicAdd(&d.ctr[25], 1)] = kd;
                    }
        }
        for (int a = 0; a < 8; ++a) d.dirty[n[a]] = stamp;
    }
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }
inline size_t crit_smem_bytes() { return sizeof(CritBatch) * crit_batch_warps(); }
inline unsigned nblk_d(const Dev &d) {  // staged D: 10 nodes per warp
    const int64_t per = d_nodes_per_block(d.blk);
    return (unsigned)((d.N + per - 1) / per);
}

}  // namespace

int persistent_occupancy(int smem_bytes, int blk) {
    int n = 0;
    cudaFuncSetAttribute(k_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_persistent, blk, smem_bytes);
    return n;
}

// Wave launches put blocks of the three stage kernels on the same SM at the same time; an SM can
// only change its shared-memory / L1 split when it is idle, so the three kernels get the same
// preferred carveout (enough shared memory for the stage-AB / C occupancy), else every switch
// between a D block (no shared memory) and an AB / C block drains the SM.  pct < 0: leave unset.
void set_wave_carveout(int smem_ab, int smem_c, int pct) {
    if (pct < 0) {
        const int need = std::max(4 * (smem_ab + 1024), 4 * (smem_c + 1024));
        int maxsm = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        if (maxsm <= 0) return;
        pct = std::min(100, (int)((100LL * need + maxsm - 1) / maxsm));
    }
    cudaFuncSetAttribute(k_AB_w, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(k_C_w, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(k_D_w, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaGetLastError();
}

int cp_stage_c_smem(int max_el, int max_nl) {
    const int b = cp_smem_bytes(max_el, max_nl);
    if (b > 227 * 1024) return 0;
    if (cudaFuncSetAttribute(k_Cp, cudaFuncAttributeMaxDynamicSharedMemorySize, b) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return b;
}

void set_smem_limits(int smem_bytes) {
    // the attribute is per function AND per device: keep the largest any context of the current
    // device needs (called after cudaSetDevice)
    static std::mutex mu;
    static int cur[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 0 || dev >= 64) dev = 0;
    if (smem_bytes <= cur[dev]) return;
    cur[dev] = smem_bytes;
    cudaFuncSetAttribute(k_AB, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_Cs, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_C, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_AB_w, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_C_w, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_AB_cur, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_energy_edges, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_C_cur, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaFuncSetAttribute(k_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)crit_smem_bytes());
}

void launch_persistent(const Dev &d, int64_t step0, int64_t nsteps, int crack_every, int grid, cudaStream_t st) {
    cudaMemsetAsync(d.head, 0, sizeof(unsigned long long), st);
    k_persistent<<<grid, d.blk, d.smem_bytes, st>>>(d, step0, nsteps, crack_every);
}

template <class K, class... Args>
void launch_pdl(K kern, unsigned grid, unsigned blk, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(blk);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

// One staged step: k_AB, k_C, [k_crit | k_filter + k_eval], k_D chained with programmatic dependent
// launch.  With ev (5 events), plain launches bracketed per stage: AB | C | criterion | D.
// (Measured and rejected: stage D waiting on stage C's block-completion count so that the criterion
// kernels run concurrently with it, plus a fix-up kernel for the split nodes' masses -- config 3
// 152.3 / 168.9 us per step steady / cracking vs 148.3 / 166.7.)
int launch_staged_step(const Dev &d, int64_t s, int crack_every, cudaStream_t st, cudaEvent_t *ev, int cmode,
                       StagedSync *sy, const std::vector<StageChunk> *chunks) {
    const bool heavy = cmode == CRIT_HEAVY;
    unsigned long long bd = 0;  // early peer signal from stage D (P2P halo, boundary blocks first)
    if (sy && d.p2p_np && d.d_order && d.d_nbound > 0) bd = sy->bdone += (unsigned long long)d.d_nbound;
    const bool crit = crack_on(crack_every, s);
    // one warp per flagged tet, grid-stride; streaming (short recent lists): fewer blocks, polling
    const bool stream = (cmode == CRIT_STREAM || cmode == CRIT_IDLE) && !ev;
    const unsigned gcrit = stream && cmode == CRIT_IDLE ? CEM_CRIT_IGRID : CEM_CRIT_GRID;
    if (!ev && chunks && chunks->size() > 1) {
        // AB and C in chunks along the storage order, AB(c) C(c) AB(c+1) ...: each C chunk reads
        // only the AB chunks before it (chunk bounds from the plan), every kernel waits for its
        // predecessor, so the chain is transitive; C(c) runs while AB(c)'s outputs are in L2
        int n = 0;
        for (const StageChunk &c : *chunks) {
            if (c.ab1 > c.ab0) {
                launch_pdl(k_AB, (unsigned)(c.ab1 - c.ab0), (unsigned)d.blk, (size_t)d.smem_ab, st, d, s, c.ab0);
                ++n;
            }
            if (c.c1 > c.c0) {
                launch_pdl(d.part ? k_C : k_Cs, (unsigned)(c.c1 - c.c0), (unsigned)d.blk, (size_t)d.smem_c, st, d, s, (int)crack_on(crack_every, s), c.c0);
                ++n;
            }
        }
        if (crit) {
            if (heavy) {
                launch_pdl(k_filter, (unsigned)CEM_FILTER_GRID, 256u, (size_t)0, st, d, s);
                launch_pdl(k_eval, (unsigned)CEM_CRITB_GRID, (unsigned)CEM_CRIT_THREADS, crit_smem_bytes(), st, d, s);
                n += 2;
            } else {
                launch_pdl(k_crit, (unsigned)CEM_CRIT_GRID, 256u, (size_t)0, st, d, s, 0);
                ++n;
            }
        }
        if (bd) launch_pdl(d.part ? k_Db : k_Dbs, nblk_d(d), (unsigned)d.blk, (size_t)0, st, d, s, bd);
        else launch_pdl(d.part ? k_D : k_Ds, nblk_d(d), (unsigned)d.blk, (size_t)0, st, d, s);
        return n + 1;
    }
    if (!ev) {  // programmatic dependent launches: stages overlap each other's launch and tail
        launch_pdl(k_AB, (unsigned)d.nblk[ST_AB], (unsigned)d.blk, (size_t)d.smem_ab, st, d, s, 0);
        if (d.cp_on)
            launch_pdl(k_Cp, (unsigned)d.cp_grid, 256u, (size_t)cp_smem_bytes(d.cp_max_el, d.cp_max_nl), st, d, s,
                       crack_every);
        else
            launch_pdl(d.part ? k_C : k_Cs, (unsigned)d.nblk[ST_C], (unsigned)d.blk, (size_t)d.smem_c, st, d, s, (int)crack_on(crack_every, s), 0);
        if (crit) {
            if (heavy) {
                launch_pdl(k_filter, (unsigned)CEM_FILTER_GRID, 256u, (size_t)0, st, d, s);
                launch_pdl(k_eval, (unsigned)CEM_CRITB_GRID, (unsigned)CEM_CRIT_THREADS, crit_smem_bytes(), st, d, s);
            } else {
                launch_pdl(k_crit, gcrit, 256u, (size_t)0, st, d, s, stream ? CEM_CRIT_POLLS : 0);
            }
        }
        if (bd) launch_pdl(d.part ? k_Db : k_Dbs, nblk_d(d), (unsigned)d.blk, (size_t)0, st, d, s, bd);
        else launch_pdl(d.part ? k_D : k_Ds, nblk_d(d), (unsigned)d.blk, (size_t)0, st, d, s);
        return crit ? (heavy ? 5 : 4) : 3;
    }
    cudaEventRecord(ev[0], st);
    k_AB<<<d.nblk[ST_AB], d.blk, d.smem_ab, st>>>(d, s, 0);
    cudaEventRecord(ev[1], st);
    if (d.cp_on)
        k_Cp<<<d.cp_grid, 256, cp_smem_bytes(d.cp_max_el, d.cp_max_nl), st>>>(d, s, crack_every);
    else
        (d.part ? k_C : k_Cs)<<<d.nblk[ST_C], d.blk, d.smem_c, st>>>(d, s, (int)crack_on(crack_every, s), 0);
    cudaEventRecord(ev[2], st);
    if (crit) {
        if (heavy) {
            k_filter<<<CEM_FILTER_GRID, 256, 0, st>>>(d, s);
            k_eval<<<CEM_CRITB_GRID, CEM_CRIT_THREADS, crit_smem_bytes(), st>>>(d, s);
        } else {
            k_crit<<<gcrit, 256, 0, st>>>(d, s, 0);
        }
    }
    cudaEventRecord(ev[3], st);
    if (bd) (d.part ? k_Db : k_Dbs)<<<nblk_d(d), d.blk, 0, st>>>(d, s, bd);
    else (d.part ? k_D : k_Ds)<<<nblk_d(d), d.blk, 0, st>>>(d, s);
    cudaEventRecord(ev[4], st);
    return crit ? (heavy ? 5 : 4) : 3;
}

void launch_wave_join(const Dev &d, int64_t nsteps_done, cudaStream_t st, int rel) {
    k_wave_join<<<1, 1024, 0, st>>>(d, nsteps_done, rel);
}
__global__ void k_set_i64(int64_t *p, int64_t v) { *p = v; }
void launch_wave_base(const Dev &d, int64_t step0, cudaStream_t st) { k_set_i64<<<1, 1, 0, st>>>(d.wstep, step0); }
void launch_wave_fill(const Dev &d, int64_t step, cudaStream_t st) {
    const int64_t n = ST_COUNT * (int64_t)d.wmax;
    k_fill_i32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d.wcnt, n, (int32_t)step);
}

void launch_hex_crit(const Dev &d, int64_t s, cudaStream_t st) {
    launch_pdl(k_hexcrit, (unsigned)((d.E + 127) / 128), 128u, (size_t)0, st, d, s);
    launch_pdl(k_hexeval, 148u * 4u, (unsigned)(32 * kHexEvalWarps), (size_t)0, st, d, s);
}

void launch_node_update(const Dev &d, int64_t s, cudaStream_t st) {
    launch_pdl(d.part ? k_D : (d.npe == 8 ? k_Dh : k_Ds), nblk_d(d), (unsigned)d.blk, (size_t)0, st, d, s);
}

int launch_wave_step(const Dev &d, const WavePlan &w, int64_t s, int crack_every, cudaStream_t st, int rel) {
    for (const WaveLaunch &L : w.seq) {
        const unsigned nb = (unsigned)(L.b1 - L.b0);
        if (L.stage == ST_AB) launch_pdl(k_AB_w, nb, (unsigned)d.blk, (size_t)d.smem_ab, st, d, s, L.b0, rel);
        else if (L.stage == ST_C) launch_pdl(k_C_w, nb, (unsigned)d.blk, (size_t)d.smem_c, st, d, s, crack_every, L.b0, rel);
        else launch_pdl(k_D_w, nb, 256u, (size_t)0, st, d, s, L.b0, rel);
    }
    return (int)w.seq.size();
}

void launch_energy_nodes(const Dev &d, int64_t n, double *part_nodes, cudaStream_t st) {
    k_energy_nodes<<<nblk(d.N), 256, 0, st>>>(d, n, part_nodes);
}

void launch_energy(const Dev &d, int64_t n, double *part_edges, double *part_nodes, cudaStream_t st) {
    k_energy_edges<<<d.nblk[ST_AB], d.blk, d.smem_ab, st>>>(d, n, part_edges);
    k_energy_nodes<<<nblk(d.N), 256, 0, st>>>(d, n, part_nodes);
}

void launch_crack_only(const Dev &d, int64_t n, cudaStream_t st) {
    const int32_t stamp = -(int32_t)(n + 1);
    k_AB_cur<<<d.nblk[ST_AB], d.blk, d.smem_ab, st>>>(d, n);
    k_C_cur<<<d.nblk[ST_C], d.blk, d.smem_c, st>>>(d, n, stamp);
    k_fix_cur<<<nblk(d.N), 256, 0, st>>>(d, n, stamp);
}

}  // namespace cem
