/*
 * cem_oracle_hex.c -- plain CPU oracle of the ES-H-FEM explicit step on trilinear hexahedra
 * (arXiv 2508.04076, §2.2: eq:hex_strain_discretization PAPER.md:L311-L338,
 * eq:hex_fint_discretization L368-L390).  TEST INFRASTRUCTURE ONLY (same rules as
 * cem_oracle.c): only tests/, __graft_entry__.smoke() and bench.py may load it; it shares no
 * code, header, table or helper with paper_2508_04076_b200/ (nor with cem_oracle.c).
 *
 * Readings (R23-R26; the paper writes dN_i/dx without a point for the trilinear
 * element):
 *  R23 the element strain of a hex is its volume-averaged compatible strain: the mean gradient
 *      B_i = (1/V_e) integral_e grad N_i dV = (1/V_e) sum_g cof(J_g) dN_i/dxi(xi_g) over the 2x2x2
 *      Gauss points (exact: the cofactors are quadratic, dN/dxi linear in each variable) -- the
 *      hex analogue of the constant-strain tet, which keeps the patch test on distorted hexes
 *      (sum_e V_e B_{e,a} = integral grad N_k = 0 at interior nodes); it is the centre value for a
 *      parallelepiped;
 *  R24 V_e = integral of det J over the element, 2x2x2 Gauss (exact for the trilinear map);
 *      lumped mass rho V_e / 8 per node;
 *  R25 time step dt = cfl * min_e (V_e / largest face area_e) / c_d, quad face area
 *      |(x_c - x_a) x (x_d - x_b)| / 2;
 *  R26 the smoothing-domain volume is (1/12) sum_j V_j (L385: each hex gives V/12 to each of its
 *      12 edges), so f_{e,a} = (V_e/12) B_a^T S_e with S_e = sum of the 12 edge stresses.
 * No crack patterns III-VI (L478-L540): hex meshes are run with Gc = infinity.
 *
 * Arithmetic: IEEE fp64, -ffp-contract=off, sequential sums in the order written.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define HX_API __attribute__((visibility("default")))

#include "exact_sum.h"

/* reference coordinates of the 8 nodes (bottom face 0-3 counter-clockwise, top 4-7 above) */
static const double XI[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                                {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
/* local edge l -> (p, q), p < q: bottom ring, top ring, verticals */
static const int HP[12] = {0, 1, 2, 0, 4, 5, 6, 4, 0, 1, 2, 3};
static const int HQ[12] = {1, 2, 3, 3, 5, 6, 7, 7, 4, 5, 6, 7};
/* faces (outward order irrelevant for areas) */
static const int HF[6][4] = {{0, 1, 2, 3}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};

typedef struct {
    int64_t N, E, S;
    double *X;            /* [N][3] */
    int32_t *hex;         /* [E][8] */
    uint8_t *active;      /* [E] */
    double *V;            /* [E] */
    double *grad;         /* [E][8][3] dN_a/dx at the centre */
    int32_t *elem_edge;   /* [E][12] */
    int64_t *inc_off;     /* [S+1] */
    int32_t *inc;         /* ascending element id */
    int64_t *nod_off;     /* [N+1] */
    int32_t *nod_ent;     /* 8e + a, ascending e */
    double *m, *fext;     /* [N], [N][3] */
    uint8_t *dir;         /* [N] prescribed-velocity mask */
    double *dir_v0;       /* [N][3] */
    double t0, lam, mu, l2m, rho, dt, gamma;
    double *u, *v, *a;    /* [N][3] */
    int64_t step;
    double *tau, *sig, *vhat, *fe, *fint;
} hx_sim;

static double dot3(const double *a, const double *b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
static void cross3(const double *a, const double *b, double *r) {
    r[0] = a[1] * b[2] - a[2] * b[1];
    r[1] = a[2] * b[0] - a[0] * b[2];
    r[2] = a[0] * b[1] - a[1] * b[0];
}
static void *xc(size_t n, size_t s) {
    void *p = calloc(n ? n : 1, s);
    if (!p) { fprintf(stderr, "hex oracle: out of memory\n"); abort(); }
    return p;
}

/* dN_i/dxi at (xi, eta, zeta) for N_i = (1 + xi xi_i)(1 + eta eta_i)(1 + zeta zeta_i) / 8 */
static void dshape(const double *p, int i, double *g) {
    const double a = 1.0 + p[0] * XI[i][0], b = 1.0 + p[1] * XI[i][1], c = 1.0 + p[2] * XI[i][2];
    g[0] = (XI[i][0] * b * c) / 8.0;
    g[1] = (a * XI[i][1] * c) / 8.0;
    g[2] = (a * b * XI[i][2]) / 8.0;
}

/* J[r][c] = dx_r / dxi_c = sum_i x_i,r dN_i/dxi_c (i ascending) */
static void jacobian(const double *X8, const double *p, double J[3][3]) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) J[r][c] = 0.0;
    for (int i = 0; i < 8; ++i) {
        double g[3];
        dshape(p, i, g);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) J[r][c] = J[r][c] + X8[3 * i + r] * g[c];
    }
}
static double det3(double J[3][3]) {
    double c0[3] = {J[0][0], J[1][0], J[2][0]}, c1[3] = {J[0][1], J[1][1], J[2][1]}, c2[3] = {J[0][2], J[1][2], J[2][2]};
    double x[3];
    cross3(c1, c2, x);
    return dot3(c0, x);
}

/* element geometry (R23, R24): V = sum_g det J_g and the mean gradients
 * grad[a] = (sum_g cof(J_g) dN_a/dxi(xi_g)) / V over the 2x2x2 Gauss points (g ascending,
 * xi_g = +-1/sqrt(3), weights 1), where cof(J) dN/dxi = det(J) J^-T dN/dxi: row c of det(J) J^-1 is
 * the cross product of the other two columns of J, so (cof dN)_r = sum_c (col_{c+1} x col_{c+2})_r
 * dN/dxi_c.  Returns 0 unless det J > 0 at the 8 corners. */
HX_API int hx_geometry(const double *X8, double *V, double *grad /*[8][3]*/) {
    for (int k = 0; k < 8; ++k) {  /* validity: positive Jacobian at the corners */
        double J[3][3];
        jacobian(X8, XI[k], J);
        if (!(det3(J) > 0.0)) return 0;
    }
    const double gp = 1.0 / sqrt(3.0);
    double vol = 0.0, acc[8][3];
    for (int a = 0; a < 8; ++a) acc[a][0] = acc[a][1] = acc[a][2] = 0.0;
    for (int k = 0; k < 8; ++k) {
        double p[3] = {XI[k][0] * gp, XI[k][1] * gp, XI[k][2] * gp}, J[3][3];
        jacobian(X8, p, J);
        vol = vol + det3(J);
        double c0[3] = {J[0][0], J[1][0], J[2][0]}, c1[3] = {J[0][1], J[1][1], J[2][1]}, c2[3] = {J[0][2], J[1][2], J[2][2]};
        double r0[3], r1[3], r2[3];
        cross3(c1, c2, r0);
        cross3(c2, c0, r1);
        cross3(c0, c1, r2);
        for (int a = 0; a < 8; ++a) {
            double g[3];
            dshape(p, a, g);
            for (int r = 0; r < 3; ++r) acc[a][r] = acc[a][r] + ((r0[r] * g[0] + r1[r] * g[1]) + r2[r] * g[2]);
        }
    }
    if (!(vol > 0.0)) return 0;
    const double inv = 1.0 / vol;
    for (int a = 0; a < 8; ++a)
        for (int r = 0; r < 3; ++r) grad[3 * a + r] = acc[a][r] * inv;
    *V = vol;
    return 1;
}

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}
static int64_t find_edge(const uint64_t *k, int64_t S, uint64_t key) {
    int64_t lo = 0, hi = S - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (k[mid] == key) return mid;
        if (k[mid] < key) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

static double node_mass(const hx_sim *s, int64_t k) {
    double acc = 0.0;
    for (int64_t j = s->nod_off[k]; j < s->nod_off[k + 1]; ++j) {
        int32_t e = s->nod_ent[j] >> 3;
        if (!s->active[e]) continue;
        acc = acc + (s->rho * s->V[e]) / 8.0;  /* R24 */
    }
    return acc;
}

HX_API void hx_destroy(hx_sim *s) {
    if (!s) return;
    free(s->X); free(s->hex); free(s->active); free(s->V); free(s->grad); free(s->elem_edge);
    free(s->inc_off); free(s->inc); free(s->nod_off); free(s->nod_ent); free(s->m); free(s->fext);
    free(s->dir); free(s->dir_v0); free(s->u); free(s->v); free(s->a); free(s->tau); free(s->sig);
    free(s->vhat); free(s->fe); free(s->fint);
    free(s);
}

/* element strain at the centre, tau = V eps (R23; eq:hex_strain_discretization, a = 0..7) */
static void stage_strain(hx_sim *s, const double *u) {
    for (int64_t e = 0; e < s->E; ++e) {
        double *t = s->tau + 6 * e;
        for (int c = 0; c < 6; ++c) t[c] = 0.0;
        if (!s->active[e]) continue;
        double ex = 0, ey = 0, ez = 0, gxy = 0, gyz = 0, gxz = 0;
        for (int a = 0; a < 8; ++a) {
            const double *g = s->grad + 24 * e + 3 * a, *ua = u + 3 * (int64_t)s->hex[8 * e + a];
            ex = ex + g[0] * ua[0];
            ey = ey + g[1] * ua[1];
            ez = ez + g[2] * ua[2];
            gxy = gxy + (g[1] * ua[0] + g[0] * ua[1]);
            gyz = gyz + (g[2] * ua[1] + g[1] * ua[2]);
            gxz = gxz + (g[2] * ua[0] + g[0] * ua[2]);
        }
        const double V = s->V[e];
        t[0] = V * ex; t[1] = V * ey; t[2] = V * ez; t[3] = V * gxy; t[4] = V * gyz; t[5] = V * gxz;
    }
}

/* edge smoothed strain and stress: Vhat = sum V, T = sum tau over active incident hexes in
 * ascending id, eps~ = T (1/Vhat), sigma = D eps~ */
static void stage_edge(hx_sim *s) {
    for (int64_t k = 0; k < s->S; ++k) {
        double Vh = 0.0, T[6] = {0, 0, 0, 0, 0, 0};
        for (int64_t j = s->inc_off[k]; j < s->inc_off[k + 1]; ++j) {
            int32_t e = s->inc[j];
            if (!s->active[e]) continue;
            Vh = Vh + s->V[e];
            for (int c = 0; c < 6; ++c) T[c] = T[c] + s->tau[6 * (int64_t)e + c];
        }
        s->vhat[k] = Vh;
        double *o = s->sig + 6 * k;
        if (Vh == 0.0) { for (int c = 0; c < 6; ++c) o[c] = 0.0; continue; }
        const double inv = 1.0 / Vh;
        const double e11 = T[0] * inv, e22 = T[1] * inv, e33 = T[2] * inv, g12 = T[3] * inv, g23 = T[4] * inv,
                     g13 = T[5] * inv;
        o[0] = s->l2m * e11 + s->lam * (e22 + e33);
        o[1] = s->l2m * e22 + s->lam * (e11 + e33);
        o[2] = s->l2m * e33 + s->lam * (e11 + e22);
        o[3] = s->mu * g12;
        o[4] = s->mu * g23;
        o[5] = s->mu * g13;
    }
}

/* element force (R26, eq:hex_fint_discretization): S = sum_{l=0..11} sigma_{s(e,l)}, c = V/12,
 * f_x = c((gx S11 + gy S12) + gz S13), f_y = c((gy S22 + gx S12) + gz S23), f_z = c((gz S33 + gy S23) + gx S13);
 * node force: sum over incidences in ascending e */
static void internal_force(hx_sim *s, const double *u) {
    stage_strain(s, u);
    stage_edge(s);
    for (int64_t e = 0; e < s->E; ++e) {
        double *f = s->fe + 24 * e;
        for (int i = 0; i < 24; ++i) f[i] = 0.0;
        if (!s->active[e]) continue;
        double S[6] = {0, 0, 0, 0, 0, 0};
        for (int l = 0; l < 12; ++l) {
            const double *sg = s->sig + 6 * (int64_t)s->elem_edge[12 * e + l];
            for (int c = 0; c < 6; ++c) S[c] = S[c] + sg[c];
        }
        const double c = s->V[e] / 12.0;
        for (int a = 0; a < 8; ++a) {
            const double *g = s->grad + 24 * e + 3 * a;
            f[3 * a] = c * ((g[0] * S[0] + g[1] * S[3]) + g[2] * S[5]);
            f[3 * a + 1] = c * ((g[1] * S[1] + g[0] * S[3]) + g[2] * S[4]);
            f[3 * a + 2] = c * ((g[2] * S[2] + g[1] * S[4]) + g[0] * S[5]);
        }
    }
    /* nodal assembly: exact sum rounded once (R27, exact_sum.h) */
    for (int64_t k = 0; k < s->N; ++k) {
        xsum acc[3];
        for (int c = 0; c < 3; ++c) xsum_init(&acc[c]);
        for (int64_t j = s->nod_off[k]; j < s->nod_off[k + 1]; ++j) {
            const int32_t ent = s->nod_ent[j];
            if (!s->active[ent >> 3]) continue;
            const double *x = s->fe + 24 * (int64_t)(ent >> 3) + 3 * (ent & 7);
            for (int c = 0; c < 3; ++c) xsum_add(&acc[c], x[c]);
        }
        for (int c = 0; c < 3; ++c) s->fint[3 * k + c] = xsum_round(&acc[c]);
    }
}

static void ramp(double t, double t0, double v0, double *v, double *acc) {
    if (t0 <= 0.0) { *v = v0; *acc = 0.0; return; }
    *v = (t <= t0) ? (t / t0) * v0 : v0;
    *acc = (t < t0) ? v0 / t0 : 0.0;
}

HX_API hx_sim *hx_create(int64_t n_nodes, const double *X, int64_t n_hex, const int32_t *hex, const uint8_t *state,
                         double E, double nu, double rho, int64_t n_tf, const int32_t *tface, const double *tface_t,
                         int64_t n_vbc, const int32_t *vbc_node, const uint8_t *vbc_mask, const double *vbc_v0,
                         double vbc_t0, double dt, double cfl, double gamma, const double *f_nodal,
                         const double *body, char *err, int errlen) {
    hx_sim *s = xc(1, sizeof(hx_sim));
    s->N = n_nodes; s->E = n_hex; s->rho = rho; s->gamma = gamma; s->t0 = vbc_t0;
    s->lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    s->mu = E / (2.0 * (1.0 + nu));
    s->l2m = s->lam + 2.0 * s->mu;
    s->X = xc(3 * n_nodes, sizeof(double)); memcpy(s->X, X, sizeof(double) * 3 * n_nodes);
    s->hex = xc(8 * n_hex, sizeof(int32_t)); memcpy(s->hex, hex, sizeof(int32_t) * 8 * n_hex);
    s->active = xc(n_hex, 1);
    s->V = xc(n_hex, sizeof(double));
    s->grad = xc(24 * n_hex, sizeof(double));
    for (int64_t e = 0; e < n_hex; ++e) {
        s->active[e] = state ? (state[e] != 0) : 1;
        double X8[24];
        for (int a = 0; a < 8; ++a) {
            int32_t n = hex[8 * e + a];
            if (n < 0 || n >= n_nodes) { snprintf(err, errlen, "hex %lld node out of range", (long long)e); hx_destroy(s); return NULL; }
            for (int c = 0; c < 3; ++c) X8[3 * a + c] = X[3 * (int64_t)n + c];
        }
        if (!hx_geometry(X8, s->V + e, s->grad + 24 * e)) {
            snprintf(err, errlen, "hex %lld: non-positive Jacobian", (long long)e); hx_destroy(s); return NULL;
        }
    }
    /* unique edges: sorted (min, max) node pairs; incidence in ascending element id */
    uint64_t *keys = xc(12 * n_hex, sizeof(uint64_t)), *uk = xc(12 * n_hex, sizeof(uint64_t));
    for (int64_t e = 0; e < n_hex; ++e)
        for (int l = 0; l < 12; ++l) {
            uint64_t i = (uint32_t)hex[8 * e + HP[l]], j = (uint32_t)hex[8 * e + HQ[l]];
            keys[12 * e + l] = (i < j ? i : j) << 32 | (i < j ? j : i);
        }
    memcpy(uk, keys, sizeof(uint64_t) * 12 * n_hex);
    qsort(uk, 12 * n_hex, sizeof(uint64_t), cmp_u64);
    int64_t S = 0;
    for (int64_t i = 0; i < 12 * n_hex; ++i)
        if (i == 0 || uk[i] != uk[i - 1]) uk[S++] = uk[i];
    s->S = S;
    s->elem_edge = xc(12 * n_hex, sizeof(int32_t));
    s->inc_off = xc(S + 1, sizeof(int64_t));
    for (int64_t i = 0; i < 12 * n_hex; ++i) {
        int64_t k = find_edge(uk, S, keys[i]);
        s->elem_edge[i] = (int32_t)k;
        s->inc_off[k + 1]++;
    }
    for (int64_t k = 0; k < S; ++k) s->inc_off[k + 1] += s->inc_off[k];
    s->inc = xc(12 * n_hex, sizeof(int32_t));
    int64_t *fill = xc(S, sizeof(int64_t));
    for (int64_t e = 0; e < n_hex; ++e)
        for (int l = 0; l < 12; ++l) {
            int64_t k = s->elem_edge[12 * e + l];
            s->inc[s->inc_off[k] + fill[k]++] = (int32_t)e;
        }
    free(fill); free(keys); free(uk);
    s->nod_off = xc(n_nodes + 1, sizeof(int64_t));
    for (int64_t e = 0; e < n_hex; ++e) for (int a = 0; a < 8; ++a) s->nod_off[hex[8 * e + a] + 1]++;
    for (int64_t k = 0; k < n_nodes; ++k) s->nod_off[k + 1] += s->nod_off[k];
    s->nod_ent = xc(8 * n_hex, sizeof(int32_t));
    fill = xc(n_nodes, sizeof(int64_t));
    for (int64_t e = 0; e < n_hex; ++e)
        for (int a = 0; a < 8; ++a) { int64_t k = hex[8 * e + a]; s->nod_ent[s->nod_off[k] + fill[k]++] = (int32_t)(8 * e + a); }
    free(fill);
    s->m = xc(n_nodes, sizeof(double));
    for (int64_t k = 0; k < n_nodes; ++k) s->m[k] = node_mass(s, k);
    /* external force as the tet oracle: body b (V/8) over active incident hexes ascending, then
     * traction triangles t (A/3), then nodal forces */
    s->fext = xc(3 * n_nodes, sizeof(double));
    if (body && (body[0] != 0.0 || body[1] != 0.0 || body[2] != 0.0))
        for (int64_t k = 0; k < n_nodes; ++k)
            for (int64_t j = s->nod_off[k]; j < s->nod_off[k + 1]; ++j) {
                int32_t e = s->nod_ent[j] >> 3;
                if (!s->active[e]) continue;
                double w = s->V[e] / 8.0;
                for (int c = 0; c < 3; ++c) s->fext[3 * k + c] = s->fext[3 * k + c] + body[c] * w;
            }
    for (int64_t f = 0; f < n_tf; ++f) {
        const int32_t *tri = tface + 3 * f;
        double d1[3], d2[3], cr[3];
        for (int c = 0; c < 3; ++c) {
            d1[c] = X[3 * (int64_t)tri[1] + c] - X[3 * (int64_t)tri[0] + c];
            d2[c] = X[3 * (int64_t)tri[2] + c] - X[3 * (int64_t)tri[0] + c];
        }
        cross3(d1, d2, cr);
        double w = (0.5 * sqrt(dot3(cr, cr))) / 3.0;
        for (int i = 0; i < 3; ++i)
            for (int c = 0; c < 3; ++c) s->fext[3 * (int64_t)tri[i] + c] = s->fext[3 * (int64_t)tri[i] + c] + tface_t[3 * f + c] * w;
    }
    if (f_nodal)
        for (int64_t i = 0; i < 3 * n_nodes; ++i) s->fext[i] = s->fext[i] + f_nodal[i];
    s->dir = xc(n_nodes, 1);
    s->dir_v0 = xc(3 * n_nodes, sizeof(double));
    for (int64_t b = 0; b < n_vbc; ++b) {
        int64_t k = vbc_node[b];
        s->dir[k] |= vbc_mask[b];
        for (int c = 0; c < 3; ++c) if (vbc_mask[b] >> c & 1) s->dir_v0[3 * k + c] = vbc_v0[3 * b + c];
    }
    if (dt <= 0.0) {  /* R25 */
        double cd = sqrt(s->l2m / rho), hmin = INFINITY;
        for (int64_t e = 0; e < n_hex; ++e) {
            if (!s->active[e]) continue;
            double amax = 0.0;
            for (int f = 0; f < 6; ++f) {
                const double *xa = X + 3 * (int64_t)hex[8 * e + HF[f][0]], *xb = X + 3 * (int64_t)hex[8 * e + HF[f][1]];
                const double *xcc = X + 3 * (int64_t)hex[8 * e + HF[f][2]], *xd = X + 3 * (int64_t)hex[8 * e + HF[f][3]];
                double d1[3], d2[3], cr[3];
                for (int c = 0; c < 3; ++c) { d1[c] = xcc[c] - xa[c]; d2[c] = xd[c] - xb[c]; }
                cross3(d1, d2, cr);
                double A = 0.5 * sqrt(dot3(cr, cr));
                if (A > amax) amax = A;
            }
            double h = s->V[e] / amax;
            if (h < hmin) hmin = h;
        }
        dt = (cfl * hmin) / cd;
    }
    s->dt = dt;
    s->u = xc(3 * n_nodes, sizeof(double)); s->v = xc(3 * n_nodes, sizeof(double)); s->a = xc(3 * n_nodes, sizeof(double));
    s->tau = xc(6 * n_hex, sizeof(double)); s->sig = xc(6 * S, sizeof(double)); s->vhat = xc(S, sizeof(double));
    s->fe = xc(24 * n_hex, sizeof(double)); s->fint = xc(3 * n_nodes, sizeof(double));
    internal_force(s, s->u);
    for (int64_t k = 0; k < n_nodes; ++k)
        for (int c = 0; c < 3; ++c) {
            int64_t i = 3 * k + c;
            if (s->m[k] == 0.0) { s->v[i] = 0.0; s->a[i] = 0.0; continue; }
            if (s->dir[k] >> c & 1) { double vv, aa; ramp(0.0, s->t0, s->dir_v0[i], &vv, &aa); s->v[i] = vv; s->a[i] = aa; continue; }
            s->a[i] = (s->fext[i] - s->fint[i]) / s->m[k];
        }
    return s;
}

/* one explicit step (the tet oracle's orc_run without the criterion) */
HX_API void hx_run(hx_sim *s, int64_t nsteps) {
    const double hdt2 = 0.5 * s->dt * s->dt;
    for (int64_t it = 0; it < nsteps; ++it) {
        const int64_t n1 = s->step + 1;
        const double t1 = (double)n1 * s->dt;
        for (int64_t i = 0; i < 3 * s->N; ++i) s->u[i] = (s->u[i] + s->dt * s->v[i]) + hdt2 * s->a[i];
        internal_force(s, s->u);
        for (int64_t k = 0; k < s->N; ++k)
            for (int c = 0; c < 3; ++c) {
                const int64_t i = 3 * k + c;
                if (s->m[k] == 0.0) { s->v[i] = 0.0; s->a[i] = 0.0; continue; }
                if (s->dir[k] >> c & 1) { double vv, aa; ramp(t1, s->t0, s->dir_v0[i], &vv, &aa); s->v[i] = vv; s->a[i] = aa; continue; }
                const double an = (s->fext[i] - s->fint[i]) / s->m[k];
                s->v[i] = s->v[i] + s->dt * ((1.0 - s->gamma) * s->a[i] + s->gamma * an);
                s->a[i] = an;
            }
        s->step = n1;
    }
}

HX_API int64_t hx_n_edges(const hx_sim *s) { return s->S; }
HX_API double hx_dt(const hx_sim *s) { return s->dt; }
HX_API void hx_get_state(const hx_sim *s, double *u, double *v, double *a, double *m) {
    if (u) memcpy(u, s->u, sizeof(double) * 3 * s->N);
    if (v) memcpy(v, s->v, sizeof(double) * 3 * s->N);
    if (a) memcpy(a, s->a, sizeof(double) * 3 * s->N);
    if (m) memcpy(m, s->m, sizeof(double) * s->N);
}
HX_API void hx_get_fext(const hx_sim *s, double *f) { memcpy(f, s->fext, sizeof(double) * 3 * s->N); }
HX_API void hx_get_geometry(const hx_sim *s, double *V, double *grad) {
    memcpy(V, s->V, sizeof(double) * s->E);
    memcpy(grad, s->grad, sizeof(double) * 24 * s->E);
}
HX_API void hx_edge_stress(hx_sim *s, const double *u, double *sigma, double *vhat, int32_t *edge_nodes) {
    stage_strain(s, u);
    stage_edge(s);
    if (sigma) memcpy(sigma, s->sig, sizeof(double) * 6 * s->S);
    if (vhat) memcpy(vhat, s->vhat, sizeof(double) * s->S);
    if (edge_nodes)  /* endpoints of each edge (from the first incident hex) */
        for (int64_t k = 0; k < s->S; ++k) {
            const int32_t e = s->inc[s->inc_off[k]];
            for (int l = 0; l < 12; ++l)
                if (s->elem_edge[12 * (int64_t)e + l] == (int32_t)k) {
                    int32_t i = s->hex[8 * (int64_t)e + HP[l]], j = s->hex[8 * (int64_t)e + HQ[l]];
                    edge_nodes[2 * k] = i < j ? i : j;
                    edge_nodes[2 * k + 1] = i < j ? j : i;
                    break;
                }
        }
}
HX_API void hx_internal_force(hx_sim *s, const double *u, double *f) {
    internal_force(s, u);
    memcpy(f, s->fint, sizeof(double) * 3 * s->N);
}
/* strain energy U = sum_s psi(eps~_s) Vhat_s / 12 (R26 smoothing-domain volume) */
HX_API double hx_strain_energy(hx_sim *s, const double *u) {
    stage_strain(s, u);
    stage_edge(s);
    double U = 0.0;
    for (int64_t k = 0; k < s->S; ++k) {
        if (s->vhat[k] == 0.0) continue;
        double T[6] = {0, 0, 0, 0, 0, 0};
        for (int64_t j = s->inc_off[k]; j < s->inc_off[k + 1]; ++j) {
            int32_t e = s->inc[j];
            if (!s->active[e]) continue;
            for (int c = 0; c < 6; ++c) T[c] = T[c] + s->tau[6 * (int64_t)e + c];
        }
        double inv = 1.0 / s->vhat[k];
        double e11 = T[0] * inv, e22 = T[1] * inv, e33 = T[2] * inv, g12 = T[3] * inv, g23 = T[4] * inv, g13 = T[5] * inv;
        double tr = e11 + e22 + e33;
        double ee = e11 * e11 + e22 * e22 + e33 * e33 + 0.5 * (g12 * g12 + g23 * g23 + g13 * g13);
        U += (0.5 * s->lam * tr * tr + s->mu * ee) * (s->vhat[k] / 12.0);
    }
    return U;
}
HX_API void hx_set_state(hx_sim *s, const double *u, const double *v, const double *a) {
    if (u) memcpy(s->u, u, sizeof(double) * 3 * s->N);
    if (v) memcpy(s->v, v, sizeof(double) * 3 * s->N);
    if (a) memcpy(s->a, a, sizeof(double) * 3 * s->N);
}
