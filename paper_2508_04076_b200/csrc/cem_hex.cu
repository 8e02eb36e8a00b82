// cem_hex.cu -- sm_100a kernels of the ES-H-FEM step on trilinear hexahedra (
// PAPER.md:L311-L338 eq:hex_strain_discretization, L368-L390 eq:hex_fint_discretization).
// Same bitwise contract as the tet path (--fmad=false, sequential sums in the order of
// DESIGN.md §5 for hexes); no criterion (crack patterns III-VI are not built).
//   A  tau_e = V_e eps_e, eps from the mean gradients (R23), a = 0..7      -> [6][E] planes
//   B  sigma_s = D (sum tau_e) / Vhat_s over the active incident hexes (ascending id)
//   C  S_e = sum_{l=0..11} sigma_{s(e,l)}; f_{e,a} = (V_e/12) B_a^T S_e (R26)  -> slots 8e + a
//   D  the tet path's node update (force-slot gather, Newmark, BC, predictor)
#include <cstdint>

#include "cem_internal.h"

namespace cem {

namespace {

__device__ __forceinline__ void pdl_trigger_h() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_h() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(256) k_hexA(Dev d, int64_t s) {
    pdl_trigger_h();
    const int64_t E = d.E;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int32_t n[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) n[a] = __ldg(d.hconn + a * E + e);
    const double V = __ldg(d.hgeo + e);
    double g[8][3];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) g[a][c] = __ldg(d.hgeo + (1 + 3 * a + c) * E + e);
    pdl_wait_h();  // u_{s+1} comes from the previous step's stage D
    const uint8_t act = __ldcg(d.state + e);
    const double4 *u = d.ubuf[(s + 1) & 1];
    double ex = 0.0, ey = 0.0, ez = 0.0, gxy = 0.0, gyz = 0.0, gxz = 0.0;
    if (act) {
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double *ua = reinterpret_cast<const double *>(u + n[a]);
            const double ux = __ldcg(ua), uy = __ldcg(ua + 1), uz = __ldcg(ua + 2);
            ex = ex + g[a][0] * ux;
            ey = ey + g[a][1] * uy;
            ez = ez + g[a][2] * uz;
            gxy = gxy + (g[a][1] * ux + g[a][0] * uy);
            gyz = gyz + (g[a][2] * uy + g[a][1] * uz);
            gxz = gxz + (g[a][2] * ux + g[a][0] * uz);
        }
    }
    double *t = d.htau;
    t[e] = act ? V * ex : 0.0;
    t[E + e] = act ? V * ey : 0.0;
    t[2 * E + e] = act ? V * ez : 0.0;
    t[3 * E + e] = act ? V * gxy : 0.0;
    t[4 * E + e] = act ? V * gyz : 0.0;
    t[5 * E + e] = act ? V * gxz : 0.0;
}

__global__ void __launch_bounds__(256) k_hexB(Dev d, int64_t s) {
    pdl_trigger_h();
    const int64_t S = d.S, E = d.E;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= S) return;
    const int32_t j0 = __ldg(d.e_off + k), j1 = __ldg(d.e_off + k + 1);
    const double Vh = __ldg(d.vhat + k);
    pdl_wait_h();  // tau from stage A
    double T0 = 0.0, T1 = 0.0, T2 = 0.0, T3 = 0.0, T4 = 0.0, T5 = 0.0;
    for (int32_t j = j0; j < j1; ++j) {  // ascending hex id; inactive hexes hold exact zeros
        const int64_t e = __ldg(d.e_inc + j);
        if (!__ldcg(d.state + e)) continue;
        T0 = T0 + __ldcg(d.htau + e);
        T1 = T1 + __ldcg(d.htau + E + e);
        T2 = T2 + __ldcg(d.htau + 2 * E + e);
        T3 = T3 + __ldcg(d.htau + 3 * E + e);
        T4 = T4 + __ldcg(d.htau + 4 * E + e);
        T5 = T5 + __ldcg(d.htau + 5 * E + e);
    }
    double4 *o4 = reinterpret_cast<double4 *>(d.srec) + k;
    double2 *o2 = reinterpret_cast<double2 *>(d.srec2) + k;
    if (Vh == 0.0) {
        *o4 = make_double4(0.0, 0.0, 0.0, 0.0);
        *o2 = make_double2(0.0, 0.0);
        return;
    }
    const double inv = 1.0 / Vh;
    const double e11 = T0 * inv, e22 = T1 * inv, e33 = T2 * inv, g12 = T3 * inv, g23 = T4 * inv, g13 = T5 * inv;
    *o4 = make_double4(d.l2m * e11 + d.lam * (e22 + e33), d.l2m * e22 + d.lam * (e11 + e33),
                       d.l2m * e33 + d.lam * (e11 + e22), d.mu * g12);
    *o2 = make_double2(d.mu * g23, d.mu * g13);
}

__global__ void __launch_bounds__(256) k_hexC(Dev d, int64_t s) {
    pdl_trigger_h();
    const int64_t E = d.E;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int32_t sid[12];
#pragma unroll
    for (int l = 0; l < 12; ++l) sid[l] = __ldg(d.heedge + l * E + e);
    const double V = __ldg(d.hgeo + e);
    pdl_wait_h();  // sigma from stage B
    double *fo = d.fe + 24 * e;  // slots 8e + a, 3 doubles each
    if (!__ldcg(d.state + e)) {
#pragma unroll
        for (int i = 0; i < 24; ++i) fo[i] = 0.0;
        return;
    }
    double S0 = 0.0, S1 = 0.0, S2 = 0.0, S3 = 0.0, S4 = 0.0, S5 = 0.0;
#pragma unroll
    for (int l = 0; l < 12; ++l) {
        const double2 a0 = __ldcg(reinterpret_cast<const double2 *>(d.srec) + 2 * (int64_t)sid[l]);
        const double2 a1 = __ldcg(reinterpret_cast<const double2 *>(d.srec) + 2 * (int64_t)sid[l] + 1);
        const double4 a = make_double4(a0.x, a0.y, a1.x, a1.y);
        const double2 b = __ldcg(reinterpret_cast<const double2 *>(d.srec2) + sid[l]);
        S0 = S0 + a.x;
        S1 = S1 + a.y;
        S2 = S2 + a.z;
        S3 = S3 + a.w;
        S4 = S4 + b.x;
        S5 = S5 + b.y;
    }
    const double c = V / 12.0;  // R26: the smoothing-domain share of each of the 12 edges
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const double gx = __ldg(d.hgeo + (1 + 3 * a) * E + e), gy = __ldg(d.hgeo + (2 + 3 * a) * E + e),
                     gz = __ldg(d.hgeo + (3 + 3 * a) * E + e);
        fo[3 * a] = c * ((gx * S0 + gy * S3) + gz * S5);
        fo[3 * a + 1] = c * ((gy * S1 + gx * S3) + gz * S4);
        fo[3 * a + 2] = c * ((gz * S2 + gy * S4) + gx * S5);
    }
}

// strain energy of the edges of one 256-edge block on u_n (tau from k_hexA(n - 1)): psi(eps~_s)
// Vhat_s / 12 with psi = 1/2 lam tr^2 + mu eps:eps (the hex oracle's hx_strain_energy), summed by a
// fixed shuffle tree and the warps in order
__global__ void __launch_bounds__(256) k_hex_energy_edges(Dev d, double *part) {
    __shared__ double red[8];
    const int64_t S = d.S, E = d.E;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double U = 0.0;
    if (k < S) {
        const double Vh = __ldg(d.vhat + k);
        if (Vh != 0.0) {
            double T[6] = {0, 0, 0, 0, 0, 0};
            for (int32_t j = __ldg(d.e_off + k); j < __ldg(d.e_off + k + 1); ++j) {
                const int64_t e = __ldg(d.e_inc + j);
                if (!__ldcg(d.state + e)) continue;
#pragma unroll
                for (int c = 0; c < 6; ++c) T[c] = T[c] + __ldcg(d.htau + c * E + e);
            }
            const double inv = 1.0 / Vh;
            const double e11 = T[0] * inv, e22 = T[1] * inv, e33 = T[2] * inv, g12 = T[3] * inv, g23 = T[4] * inv,
                         g13 = T[5] * inv;
            const double tr = e11 + e22 + e33;
            const double ee = e11 * e11 + e22 * e22 + e33 * e33 + 0.5 * (g12 * g12 + g23 * g23 + g13 * g13);
            U = (0.5 * d.lam * tr * tr + d.mu * ee) * (Vh / 12.0);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) U = U + __shfl_down_sync(0xffffffffu, U, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = U;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = t + red[i];
        part[blockIdx.x] = t;
    }
}

template <class K, class... Args>
void launch_pdl_h(K kern, unsigned grid, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace

void launch_hex_energy(const Dev &d, int64_t n, double *part_edges, double *part_nodes, cudaStream_t st) {
    const unsigned ge = (unsigned)((d.E + 255) / 256), gs = (unsigned)((d.S + 255) / 256);
    k_hexA<<<ge, 256, 0, st>>>(d, n - 1);  // tau of u_n = ubuf[n & 1]
    k_hex_energy_edges<<<gs, 256, 0, st>>>(d, part_edges);
    launch_energy_nodes(d, n, part_nodes, st);
}

int launch_hex_step(const Dev &d, int64_t s, cudaStream_t st) {
    const unsigned ge = (unsigned)((d.E + 255) / 256), gs = (unsigned)((d.S + 255) / 256);
    launch_pdl_h(k_hexA, ge, st, d, s);
    launch_pdl_h(k_hexB, gs, st, d, s);
    launch_pdl_h(k_hexC, ge, st, d, s);
    launch_node_update(d, s, st);
    return 4;
}

}  // namespace cem
