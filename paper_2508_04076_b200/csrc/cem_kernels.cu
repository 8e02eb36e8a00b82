// cem_kernels.cu -- sm_100a kernels of the CEM explicit step.
//
// Compiled with --fmad=false: every product and sum rounds exactly as written, in the
// association order fixed in DESIGN.md ("Association order"), so results are bitwise
// reproducible and equal to the CPU oracle's.  No floating-point atomics anywhere: each
// output is produced by one thread that sums its inputs sequentially in ascending
// element id (deterministic CSR gathers).
//
// Stages (one explicit step n -> n+1, u_{n+1} already predicted):
//   k_strain  (a1) tau_e = V_e eps_e(u_{n+1})
//   k_edge    (a2) Vhat_s, eps~_s = (sum tau_e)/Vhat_s, sigma_s
//   k_force   (a3) f_e = (V_e/6) B^T sum_l sigma_{s(e,l)}; criterion PAPER.md:L340-L367, L426-L476
//   k_node    (a4) f_int gather, Newmark, BC, predictor u_{n+2}
//   k_split   (a5) ordered split pass (deactivate, records, mass)
#include <cstdint>

#include "cem_internal.h"

namespace cem {

const char *kKernelNames[K_COUNT] = {"k_strain", "k_edge", "k_force", "k_node", "k_split"};

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ double ld_nc(const double *p) { return __ldg(p); }
__device__ __forceinline__ double4 ldg4(const double4 *p) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
    const double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// ------------------------------------------------------------------ a1: element strain
__global__ void __launch_bounds__(kBlock) k_strain(DevMesh m, const double4 *__restrict__ u, double *__restrict__ tau) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m.E) return;
    if (!m.state[e]) return;  // inactive: tau is never read (k_edge skips it)
    const int4 t = __ldg(&m.tet[e]);
    const double *g = m.geo + 16 * e;
    const double V = ld_nc(g);
    const int nid[4] = {t.x, t.y, t.z, t.w};
    double ex = 0.0, ey = 0.0, ez = 0.0, gxy = 0.0, gyz = 0.0, gxz = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const double4 ua = ldg4(&u[nid[a]]);
        const double gx = ld_nc(g + 4 + 3 * a), gy = ld_nc(g + 5 + 3 * a), gz = ld_nc(g + 6 + 3 * a);
        ex = ex + gx * ua.x;
        ey = ey + gy * ua.y;
        ez = ez + gz * ua.z;
        gxy = gxy + (gy * ua.x + gx * ua.y);
        gyz = gyz + (gz * ua.y + gy * ua.z);
        gxz = gxz + (gz * ua.x + gx * ua.z);
    }
    double2 *o = reinterpret_cast<double2 *>(tau + 6 * e);
    o[0] = make_double2(V * ex, V * ey);
    o[1] = make_double2(V * ez, V * gxy);
    o[2] = make_double2(V * gyz, V * gxz);
}

// ------------------------------------------------------------------ a2: edge smoothed strain -> stress
__global__ void __launch_bounds__(kBlock) k_edge(DevMesh m, const double *__restrict__ tau, double *__restrict__ sig) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m.S) return;
    const int32_t j0 = __ldg(&m.edge_off[s]), j1 = __ldg(&m.edge_off[s + 1]);
    double Vh = 0.0, T0 = 0.0, T1 = 0.0, T2 = 0.0, T3 = 0.0, T4 = 0.0, T5 = 0.0;
    for (int32_t j = j0; j < j1; ++j) {
        const int32_t e = __ldg(&m.edge_inc[j]);
        if (!m.state[e]) continue;
        Vh = Vh + ld_nc(m.geo + 16 * (int64_t)e);
        const double2 *tp = reinterpret_cast<const double2 *>(tau + 6 * (int64_t)e);
        const double2 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
        T0 = T0 + a.x; T1 = T1 + a.y; T2 = T2 + b.x;
        T3 = T3 + b.y; T4 = T4 + c.x; T5 = T5 + c.y;
    }
    double2 *o = reinterpret_cast<double2 *>(sig + 6 * s);
    if (Vh == 0.0) {
        o[0] = o[1] = o[2] = make_double2(0.0, 0.0);
        return;
    }
    const double inv = 1.0 / Vh;
    const double e11 = T0 * inv, e22 = T1 * inv, e33 = T2 * inv, g12 = T3 * inv, g23 = T4 * inv, g13 = T5 * inv;
    const double lam = m.lam, mu = m.mu, l2m = m.l2m;
    o[0] = make_double2(l2m * e11 + lam * (e22 + e33), l2m * e22 + lam * (e11 + e33));
    o[1] = make_double2(l2m * e33 + lam * (e11 + e22), mu * g12);
    o[2] = make_double2(mu * g23, mu * g13);
}

// ------------------------------------------------------------------ crack criterion (device)
// Local edge l -> (p,q), p < q, and the inverse map.
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

// Principal decomposition of a symmetric 3x3 (Voigt 11,22,33,12,23,13) by cyclic Jacobi
// with pivots (0,1),(0,2),(1,2), <= 8 sweeps, early stop when all off-diagonals are 0,
// a pivot with |a_pq| <= 2^-60 (|a_pp|+|a_qq|) zeroed without rotation; rotation
// theta = (a_qq-a_pp)/(2a_pq), t = sgn(theta)/(|theta|+sqrt(theta^2+1)), c = 1/sqrt(t^2+1),
// s = t c (R8).  Output: eigenvalues l[3], eigenvector columns ev[i][k].
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

// sigma_G . m, unnormalised (R8): sigma1 |e1.m|, or sigma1 sqrt(sum_{k in deg}(e_k.m)^2)
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
        const double d = vdot(e, m);
        acc = acc + d * d;
    }
    return E.l[E.k1] * sqrt(acc);
}

__device__ __forceinline__ double dsgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

// Full evaluation of the 24 candidates (R7): returns best G, candidate, area.
__device__ void evaluate_candidates(const Vec3 Xn[4], const Vec3 un[4], const int H[6], const double *sig6[6],
                                    double &Gbest, int &kbest, double &Abest) {
    Eig eg[6];
    for (int l = 0; l < 6; ++l) principal(sig6[l], eg[l]);
    Gbest = 0.0;
    kbest = -1;
    Abest = 0.0;
    for (int c = 0; c < 4; ++c) {
        int o[3], no = 0;
        for (int b = 0; b < 4; ++b)
            if (b != c) o[no++] = b;
        for (int f = 0; f < 3; ++f) {
            const int p = o[f == 2 ? 1 : 0], q = o[f == 0 ? 1 : 2], r = o[2 - f];
            for (int t = 0; t < 2; ++t) {
                const Vec3 d1 = vsub(Xn[q], Xn[p]);
                const Vec3 d2 = t == 0 ? vsub(Xn[r], Xn[c]) : vsub(Xn[r], Xn[p]);
                const Vec3 mv = vcross(d1, d2);
                const double mm = vdot(mv, mv);
                double Dd[2];
                const int ends[2] = {p, q};
                for (int z = 0; z < 2; ++z) {
                    const int b = ends[z];
                    if (!H[ledge(c, b)]) {
                        Dd[z] = 0.0;
                        continue;
                    }
                    const Vec3 du = vsub(un[b], un[c]), dX = vsub(Xn[b], Xn[c]);
                    Dd[z] = vdot(du, mv) * dsgn(vdot(dX, mv));
                }
                double G, area;
                if (t == 0) {
                    const double A1 = sig_proj(eg[ledge(p, r)], mv) * Dd[0];
                    const double A2 = sig_proj(eg[ledge(q, r)], mv) * Dd[1];
                    G = (0.5 * (A1 + A2)) / mm;
                    area = sqrt(mm) / 4.0;
                } else {
                    const double Sg = sig_proj(eg[ledge(c, r)], mv);
                    G = (0.5 * (Sg * (Dd[0] + Dd[1]))) / mm;
                    area = sqrt(mm) / 8.0;
                }
                const int k = 6 * c + 2 * f + t;
                if (kbest < 0 || G > Gbest || (G == Gbest && area > Abest)) {
                    Gbest = G;
                    kbest = k;
                    Abest = area;
                }
            }
        }
    }
}

// ------------------------------------------------------------------ a3: element force + criterion
__global__ void __launch_bounds__(kBlock) k_force(DevMesh m, DevState s, const double4 *__restrict__ u, int crack_every,
                                                  int force_crack) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m.E) return;
    double2 *fo = reinterpret_cast<double2 *>(s.fe + 12 * e);
    if (!m.state[e]) {
#pragma unroll
        for (int i = 0; i < 6; ++i) fo[i] = make_double2(0.0, 0.0);
        return;
    }
    const int32_t *ee = m.elem_edge + 6 * e;
    double S0 = 0.0, S1 = 0.0, S2 = 0.0, S3 = 0.0, S4 = 0.0, S5 = 0.0;
    double gmax = 0.0;
    const double *sp[6];
#pragma unroll
    for (int l = 0; l < 6; ++l) {
        const double *sg = s.sig + 6 * (int64_t)__ldg(&ee[l]);
        sp[l] = sg;
        const double2 *q = reinterpret_cast<const double2 *>(sg);
        const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
        S0 = S0 + a.x; S1 = S1 + a.y; S2 = S2 + b.x;
        S3 = S3 + b.y; S4 = S4 + c.x; S5 = S5 + c.y;
        // Gershgorin bound on the spectral radius of sigma_s (early-out)
        const double r0 = fabs(a.x) + fabs(b.y) + fabs(c.y);
        const double r1 = fabs(a.y) + fabs(b.y) + fabs(c.x);
        const double r2 = fabs(b.x) + fabs(c.x) + fabs(c.y);
        gmax = fmax(gmax, fmax(r0, fmax(r1, r2)));
    }
    const double *g = m.geo + 16 * e;
    const double cc = ld_nc(g + 1);  // V_e / 6
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const double gx = ld_nc(g + 4 + 3 * a), gy = ld_nc(g + 5 + 3 * a), gz = ld_nc(g + 6 + 3 * a);
        const double fx = cc * ((gx * S0 + gy * S3) + gz * S5);
        const double fy = cc * ((gy * S1 + gx * S3) + gz * S4);
        const double fz = cc * ((gz * S2 + gy * S4) + gx * S5);
        s.fe[12 * e + 3 * a + 0] = fx;
        s.fe[12 * e + 3 * a + 1] = fy;
        s.fe[12 * e + 3 * a + 2] = fz;
    }
    // ---------------- crack criterion on (u_{n+1}, sigma(u_{n+1}))
    if (!force_crack) {
        if (crack_every <= 0) return;
        const int64_t n1 = *s.step + 1;
        if (n1 % crack_every != 0) return;
    }
    const int4 t = __ldg(&m.tet[e]);
    const int nid[4] = {t.x, t.y, t.z, t.w};
    Vec3 Xn[4], un[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const double4 x = ldg4(&m.X[nid[a]]);
        const double4 uu = ldg4(&u[nid[a]]);
        Xn[a] = {x.x, x.y, x.z};
        un[a] = {uu.x, uu.y, uu.z};
    }
    int H[6];
    double d2max = 0.0;
#pragma unroll
    for (int l = 0; l < 6; ++l) {
        const Vec3 du = vsub(un[c_eq[l]], un[c_ep[l]]);
        const Vec3 dX = vsub(Xn[c_eq[l]], Xn[c_ep[l]]);
        const Vec3 w = {2.0 * dX.x + du.x, 2.0 * dX.y + du.y, 2.0 * dX.z + du.z};
        H[l] = vdot(du, w) > 0.0;
        if (H[l]) d2max = fmax(d2max, vdot(du, du));
    }
    const double gc = __ldg(&m.gc[e]);
    // every candidate satisfies |G| <= gmax * max_l H_l |du_l|
    if (!(m.flags & CEM_F_NO_EARLY_OUT) && gmax * sqrt(d2max) * (1.0 + 1e-6) <= gc) return;
    double G, A;
    int k;
    evaluate_candidates(Xn, un, H, sp, G, k, A);
    if (G > gc) {
        const int slot = atomicAdd(&s.ctr[0], 1);
        if (slot < s.flag_cap) s.flag_list[slot] = (int32_t)e;
        s.flag[e] = 1;
        s.flag_cand[e] = k;
        s.flag_G[e] = G;
        s.flag_area[e] = A;
    }
}

// ------------------------------------------------------------------ a4: node update
__global__ void __launch_bounds__(kBlock) k_node(DevMesh m, DevState s, const double4 *__restrict__ ucur,
                                                 double4 *__restrict__ unext, double hdt2) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m.N) return;
    const int32_t j0 = __ldg(&m.node_off[k]), j1 = __ldg(&m.node_off[k + 1]);
    double f0 = 0.0, f1 = 0.0, f2 = 0.0;
    for (int32_t j = j0; j < j1; ++j) {
        const int32_t ent = __ldg(&m.node_ent[j]);
        const double *f = s.fe + 12 * (int64_t)(ent >> 2) + 3 * (ent & 3);
        f0 = f0 + __ldg(f);
        f1 = f1 + __ldg(f + 1);
        f2 = f2 + __ldg(f + 2);
    }
    const double mk = m.mass[k];
    const uint8_t fl = __ldg(&m.nflag[k]);
    const double4 u1 = ucur[k];
    double4 v = s.v[k], a = s.a[k];
    const double dt = m.dt, gamma = m.gamma, omg = 1.0 - m.gamma;
    double4 fx = make_double4(0.0, 0.0, 0.0, 0.0);
    if (fl & 8) fx = ldg4(&m.fext[k]);
    const double fi[3] = {f0, f1, f2};
    const double fe3[3] = {fx.x, fx.y, fx.z};
    double vv[3] = {v.x, v.y, v.z}, aa[3] = {a.x, a.y, a.z};
    double vb0[3] = {0.0, 0.0, 0.0};
    if (fl & 7) {
        const double4 w = ldg4(&m.dir_v0[k]);
        vb0[0] = w.x; vb0[1] = w.y; vb0[2] = w.z;
    }
    const double t1 = (double)(*s.step + 1) * dt;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if (mk == 0.0) {
            vv[c] = 0.0;
            aa[c] = 0.0;
        } else if (fl >> c & 1) {  // prescribed velocity ramp (R17)
            const double t0 = m.t0, v0 = vb0[c];
            if (t0 <= 0.0) {
                vv[c] = v0;
                aa[c] = 0.0;
            } else {
                vv[c] = (t1 <= t0) ? (t1 / t0) * v0 : v0;
                aa[c] = (t1 < t0) ? v0 / t0 : 0.0;
            }
        } else {
            const double an = (fe3[c] - fi[c]) / mk;
            vv[c] = vv[c] + dt * (omg * aa[c] + gamma * an);
            aa[c] = an;
        }
    }
    s.v[k] = make_double4(vv[0], vv[1], vv[2], 0.0);
    s.a[k] = make_double4(aa[0], aa[1], aa[2], 0.0);
    const double un0 = (u1.x + dt * vv[0]) + hdt2 * aa[0];
    const double un1 = (u1.y + dt * vv[1]) + hdt2 * aa[1];
    const double un2 = (u1.z + dt * vv[2]) + hdt2 * aa[2];
    unext[k] = make_double4(un0, un1, un2, 0.0);
    if (!isfinite(u1.x) || !isfinite(u1.y) || !isfinite(u1.z) || !isfinite(vv[0]) || !isfinite(vv[1]) ||
        !isfinite(vv[2]) || !isfinite(aa[0]) || !isfinite(aa[1]) || !isfinite(aa[2])) {
        s.ctr[1] = 1;
        atomicMin(&s.ctr[2], (int32_t)k);
    }
}

// ------------------------------------------------------------------ a5: split pass (single block)
constexpr int kSplitThreads = 1024;
constexpr int kSortCap = 8192;

__global__ void __launch_bounds__(kSplitThreads) k_split(DevMesh m, DevState s, double4 *__restrict__ u_src,
                                                         double4 *__restrict__ u_dst, double hdt2, int advance) {
    __shared__ int32_t list[kSortCap];
    __shared__ int32_t n_sh;
    const int tid = threadIdx.x;
    const int32_t n = s.ctr[0];
    const int64_t step_no = *s.step + (advance ? 1 : 0);
    if (n == 0) {
        __syncthreads();
        if (tid == 0 && advance) *s.step = step_no;
        return;
    }
    int32_t cnt;
    int32_t *L;
    if (n <= kSortCap && n <= s.flag_cap) {
        // bitonic sort of the unordered flag list (ascending element id)
        int P = 1;
        while (P < n) P <<= 1;
        for (int i = tid; i < P; i += kSplitThreads) list[i] = i < n ? s.flag_list[i] : INT32_MAX;
        __syncthreads();
        for (int k = 2; k <= P; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < P; i += kSplitThreads) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const int32_t x = list[i], y = list[ixj];
                        const bool up = (i & k) == 0;
                        if ((x > y) == up) {
                            list[i] = y;
                            list[ixj] = x;
                        }
                    }
                }
                __syncthreads();
            }
        cnt = n;
        L = list;
    } else {
        // overflow: ordered scan of the flag bytes over all tets into flag_list (capacity E)
        if (tid == 0) n_sh = 0;
        __syncthreads();
        __shared__ int32_t warp_tot[32];
        for (int64_t base = 0; base < m.E; base += kSplitThreads) {
            const int64_t e = base + tid;
            const int f = (e < m.E) ? s.flag[e] : 0;
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            const int lane = tid & 31, w = tid >> 5;
            if (lane == 0) warp_tot[w] = __popc(bal);
            __syncthreads();
            int off = 0;
            for (int i = 0; i < w; ++i) off += warp_tot[i];
            const int pos = n_sh + off + __popc(bal & ((1u << lane) - 1u));
            if (f) s.flag_list[pos] = (int32_t)e;
            __syncthreads();
            if (tid == 0) {
                int tot = 0;
                for (int i = 0; i < 32; ++i) tot += warp_tot[i];
                n_sh += tot;
            }
            __syncthreads();
        }
        cnt = n_sh;
        L = s.flag_list;
    }
    __syncthreads();
    const int64_t r0 = *s.nrec;
    // deactivate + records (ascending element id)
    for (int i = tid; i < cnt; i += kSplitThreads) {
        const int32_t e = L[i];
        m.state[e] = 0;
        s.flag[e] = 0;
        s.rec_step[r0 + i] = step_no;
        s.rec_elem[r0 + i] = e;
        s.rec_cand[r0 + i] = s.flag_cand[e];
        s.rec_G[r0 + i] = s.flag_G[e];
        s.rec_area[r0 + i] = s.flag_area[e];
    }
    if (tid == 0) {
        double Ud = *s.Ud;
        for (int i = 0; i < cnt; ++i) {
            const int32_t e = L[i];
            Ud = Ud + m.gc[e] * s.flag_area[e];
        }
        *s.Ud = Ud;
    }
    __syncthreads();
    __threadfence_block();
    // lumped mass of the nodes of split tets, recomputed from the active incidences
    const double rho = m.rho, dt = m.dt;
    for (int i = tid; i < 4 * cnt; i += kSplitThreads) {
        const int32_t e = L[i >> 2];
        const int4 t = m.tet[e];
        const int32_t k = (i & 3) == 0 ? t.x : ((i & 3) == 1 ? t.y : ((i & 3) == 2 ? t.z : t.w));
        double acc = 0.0;
        for (int32_t j = m.node_off[k]; j < m.node_off[k + 1]; ++j) {
            const int32_t ee = m.node_ent[j] >> 2;
            if (!m.state[ee]) continue;
            acc = acc + (rho * m.geo[16 * (int64_t)ee]) / 4.0;
        }
        m.mass[k] = acc;
        if (acc == 0.0) {  // frozen node: v = a = 0, prediction restarts from u
            s.v[k] = make_double4(0.0, 0.0, 0.0, 0.0);
            s.a[k] = make_double4(0.0, 0.0, 0.0, 0.0);
            const double4 us = u_src[k];
            u_dst[k] = make_double4((us.x + dt * 0.0) + hdt2 * 0.0, (us.y + dt * 0.0) + hdt2 * 0.0,
                                    (us.z + dt * 0.0) + hdt2 * 0.0, 0.0);
        }
    }
    __syncthreads();
    if (tid == 0) {
        *s.nrec = r0 + cnt;
        s.ctr[0] = 0;
        if (advance) *s.step = step_no;
    }
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + kBlock - 1) / kBlock); }

}  // namespace

void launch_strain(const DevMesh &m, const DevState &s, int cur, cudaStream_t st) {
    k_strain<<<nblk(m.E), kBlock, 0, st>>>(m, s.u[cur ^ 1], s.tau);
}
void launch_edge(const DevMesh &m, const DevState &s, cudaStream_t st) {
    k_edge<<<nblk(m.S), kBlock, 0, st>>>(m, s.tau, s.sig);
}
void launch_force(const DevMesh &m, const DevState &s, int cur, int crack_every, cudaStream_t st) {
    k_force<<<nblk(m.E), kBlock, 0, st>>>(m, s, s.u[cur ^ 1], crack_every, 0);
}
void launch_node(const DevMesh &m, const DevState &s, int cur, cudaStream_t st) {
    const double hdt2 = 0.5 * m.dt * m.dt;
    k_node<<<nblk(m.N), kBlock, 0, st>>>(m, s, s.u[cur ^ 1], s.u[cur], hdt2);
}
void launch_split(const DevMesh &m, const DevState &s, int cur, int crack_every, int advance, cudaStream_t st) {
    (void)crack_every;
    const double hdt2 = 0.5 * m.dt * m.dt;
    // step mode: u_{n+1} lives in u[cur^1], u_{n+2} was written to u[cur]
    k_split<<<1, kSplitThreads, 0, st>>>(m, s, s.u[cur ^ 1], s.u[cur], hdt2, advance);
}

// criterion-only variant on the current state u_n = u[cur] (cem_crack_update)
void launch_crack_only(const DevMesh &m, const DevState &s, int cur, cudaStream_t st) {
    k_strain<<<nblk(m.E), kBlock, 0, st>>>(m, s.u[cur], s.tau);
    k_edge<<<nblk(m.S), kBlock, 0, st>>>(m, s.tau, s.sig);
    k_force<<<nblk(m.E), kBlock, 0, st>>>(m, s, s.u[cur], 1, 1);
    const double hdt2 = 0.5 * m.dt * m.dt;
    // a node frozen here restarts its prediction u_{n+1} (in u[cur^1]) from u_n (in u[cur])
    k_split<<<1, kSplitThreads, 0, st>>>(m, s, s.u[cur], s.u[cur ^ 1], hdt2, 0);
}

}  // namespace cem
