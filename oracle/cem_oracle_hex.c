/*
 * cem_oracle_hex.c -- plain CPU oracle of the ES-H-FEM explicit step on trilinear hexahedra
 * (arXiv 2508.04076, §2.2: eq:hex_strain_discretization PAPER.md:L311-L338,
 * eq:hex_fint_discretization L368-L390).  TEST INFRASTRUCTURE ONLY (same rules as
 * cem_oracle.c): only tests/, __graft_entry__.smoke() and bench.py may load it; it shares no
 * code, header, table or helper with paper_2508_04076_b200/.  From cem_oracle.c (the same oracle
 * library) it calls the tet geometry, the principal-stress projection and the tet candidates.
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
 *  R28 crack patterns III-VI of the parallelepiped (L478-L540; the figure that defines them is
 *      missing): quadrature points G = edge midpoints; a crack front joins the points of two
 *      edges of one face -- opposite edges (patterns III, IV) or neighbouring edges meeting at a
 *      corner c (patterns V, VI); 84 candidates per hex (k tables below, R28).  III is
 *      the mid-plane (fully cracked: deactivated); IV, V and VI leave a remainder that becomes the
 *      half-hex triangular prism of original nodes on the far side of the parallel diagonal plane,
 *      split into three tets (A,B,C,A'), (B,C,A',B'), (C,A',B',C') (first two nodes swapped where
 *      the volume is negative).  III, IV, V follow eq:G-I, VI eq:G-II, with the tet readings
 *      R6 (H), R8 (sigma.n), R9 (sign), R10 (strict), R11/R11v, R14 (ties).
 *  R29 mixed edges (a remainder tet next to hexahedra): eps~_s = sum tau / sum V over the active
 *      elements of the edge (the paper's w = V_j / sum V, eq:strain_discretization), element force
 *      (V_e / n_e) B^T sum_l sigma_l with n_e = 12 (hex) or 6 (tet), mass rho V / 8 or rho V / 4;
 *      remainder tets take the tet criterion (24 candidates) and are deactivated when they split.
 *  Element order (sums over an edge's or a node's elements, records): hex e, then its remainder
 *  tets i = 0..2 (record id E + 3e + i); the two are never active together.
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
    int64_t S_h;          /* edges [0, S_h) are hex edges; [S_h, S) diagonals (remainder tets only) */
    int32_t *pair_edge;   /* [E][28] global edge of the local node pair (pair_id) */
    int32_t *inc_j;       /* [inc] local pair index of the edge in the incident hex */
    double *gc;           /* [E] */
    uint32_t flags;
    int8_t *rem;          /* [E] remainder prism (candidate k) or -1 */
    uint8_t *tact;        /* [E] bit i: remainder tet i active */
    uint8_t *tloc;        /* [E][3][4] local hex nodes of the remainder tets */
    double *tV, *tgrad, *ttau, *tfe;  /* [E][3], [E][3][4][3], [E][3][6], [E][3][4][3] */
    uint8_t *flag;        /* [E] this step: bit 0 hex splits, bit 1+i tet i splits */
    double *Gb, *Ab;      /* [E][4] chosen G, area (hex, tets) */
    int32_t *kb;          /* [E][4] chosen candidate */
    int64_t nrec, caprec;
    int64_t *rstep; int32_t *relem, *rcand; double *rG, *rA;
    double Ud;
    int nonfinite;
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

/* local node pair (a, b), a != b -> 0..27 in lexicographic order of (min, max) */
static int pair_id(int a, int b) {
    int p = a < b ? a : b, q = a < b ? b : a;
    return 7 * p - p * (p - 1) / 2 + (q - p - 1);
}
/* local hex edge of the pair (a, b), or -1 (a face or body diagonal) */
static int hex_edge(int a, int b) {
    int p = a < b ? a : b, q = a < b ? b : a;
    for (int l = 0; l < 12; ++l)
        if (HP[l] == p && HQ[l] == q) return l;
    return -1;
}
/* node x of face f -> the node joined to it by the hex edge that leaves the face */
static int partner(int f, int x) {
    for (int l = 0; l < 12; ++l) {
        int y = HP[l] == x ? HQ[l] : (HQ[l] == x ? HP[l] : -1);
        if (y < 0) continue;
        int in = 0;
        for (int i = 0; i < 4; ++i) in |= HF[f][i] == y;
        if (!in) return y;
    }
    return -1;
}
static int hex_edge_of_pair(int j) {
    static int tab[28], init = 0;
    if (!init) {
        for (int x = 0; x < 28; ++x) tab[x] = -1;
        for (int l = 0; l < 12; ++l) tab[pair_id(HP[l], HQ[l])] = l;
        init = 1;
    }
    return tab[j];
}
/* does remainder tet i of hex e contain the local pair j / the local node a */
static int tet_has_pair(const hx_sim *s, int64_t e, int i, int j) {
    const uint8_t *t = s->tloc + 12 * e + 4 * i;
    for (int x = 0; x < 4; ++x)
        for (int y = x + 1; y < 4; ++y)
            if (pair_id(t[x], t[y]) == j) return 1;
    return 0;
}
static int tet_has_node(const hx_sim *s, int64_t e, int i, int a) {
    const uint8_t *t = s->tloc + 12 * e + 4 * i;
    return t[0] == a || t[1] == a || t[2] == a || t[3] == a;
}

/* lumped mass (R24, R29): incidences (e, a) in ascending e -- the hex (rho V / 8) or its active
 * remainder tets holding node a (rho V_t / 4, i ascending) */
static double node_mass(const hx_sim *s, int64_t k) {
    double acc = 0.0;
    for (int64_t j = s->nod_off[k]; j < s->nod_off[k + 1]; ++j) {
        int32_t e = s->nod_ent[j] >> 3, a = s->nod_ent[j] & 7;
        if (s->active[e]) { acc = acc + (s->rho * s->V[e]) / 8.0; continue; }
        if (s->rem[e] < 0) continue;
        for (int i = 0; i < 3; ++i)
            if ((s->tact[e] >> i & 1) && tet_has_node(s, e, i, a)) acc = acc + (s->rho * s->tV[3 * (int64_t)e + i]) / 4.0;
    }
    return acc;
}

HX_API void hx_destroy(hx_sim *s) {
    if (!s) return;
    free(s->X); free(s->hex); free(s->active); free(s->V); free(s->grad); free(s->elem_edge);
    free(s->inc_off); free(s->inc); free(s->nod_off); free(s->nod_ent); free(s->m); free(s->fext);
    free(s->dir); free(s->dir_v0); free(s->u); free(s->v); free(s->a); free(s->tau); free(s->sig);
    free(s->vhat); free(s->fe); free(s->fint);
    free(s->pair_edge); free(s->inc_j); free(s->gc); free(s->rem); free(s->tact); free(s->tloc); free(s->tV);
    free(s->tgrad); free(s->ttau); free(s->tfe); free(s->flag); free(s->Gb); free(s->Ab); free(s->kb);
    free(s->rstep); free(s->relem); free(s->rcand); free(s->rG); free(s->rA);
    free(s);
}

/* element strain at the centre, tau = V eps (R23; eq:hex_strain_discretization, a = 0..7); remainder
 * tets (R28): tau = V_t eps_t over their 4 nodes, the same expression (eq:CSTet_strain_discretization) */
static void strain_of(const double *grad, int na, const int32_t *nodes, const double *u, double V, double *t) {
    double ex = 0, ey = 0, ez = 0, gxy = 0, gyz = 0, gxz = 0;
    for (int a = 0; a < na; ++a) {
        const double *g = grad + 3 * a, *ua = u + 3 * (int64_t)nodes[a];
        ex = ex + g[0] * ua[0];
        ey = ey + g[1] * ua[1];
        ez = ez + g[2] * ua[2];
        gxy = gxy + (g[1] * ua[0] + g[0] * ua[1]);
        gyz = gyz + (g[2] * ua[1] + g[1] * ua[2]);
        gxz = gxz + (g[2] * ua[0] + g[0] * ua[2]);
    }
    t[0] = V * ex; t[1] = V * ey; t[2] = V * ez; t[3] = V * gxy; t[4] = V * gyz; t[5] = V * gxz;
}
static void tet_nodes(const hx_sim *s, int64_t e, int i, int32_t *n4) {
    for (int a = 0; a < 4; ++a) n4[a] = s->hex[8 * e + s->tloc[12 * e + 4 * i + a]];
}
static void stage_strain(hx_sim *s, const double *u) {
    for (int64_t e = 0; e < s->E; ++e) {
        double *t = s->tau + 6 * e;
        for (int c = 0; c < 6; ++c) t[c] = 0.0;
        if (s->active[e]) strain_of(s->grad + 24 * e, 8, s->hex + 8 * e, u, s->V[e], t);
        if (s->rem[e] < 0) continue;
        for (int i = 0; i < 3; ++i) {
            double *tt = s->ttau + 18 * e + 6 * i;
            for (int c = 0; c < 6; ++c) tt[c] = 0.0;
            if (!(s->tact[e] >> i & 1)) continue;
            int32_t n4[4];
            tet_nodes(s, e, i, n4);
            strain_of(s->tgrad + 36 * e + 12 * i, 4, n4, u, s->tV[3 * e + i], tt);
        }
    }
}

/* edge smoothed strain and stress: Vhat = sum V, T = sum tau over the active elements of the edge
 * in element order (hex e, then its remainder tets), eps~ = T (1/Vhat), sigma = D eps~
 * (R29) */
static void stage_edge(hx_sim *s) {
    for (int64_t k = 0; k < s->S; ++k) {
        double Vh = 0.0, T[6] = {0, 0, 0, 0, 0, 0};
        for (int64_t j = s->inc_off[k]; j < s->inc_off[k + 1]; ++j) {
            int32_t e = s->inc[j], pj = s->inc_j[j];
            if (s->active[e]) {
                if (hex_edge_of_pair(pj) < 0) continue;
                Vh = Vh + s->V[e];
                for (int c = 0; c < 6; ++c) T[c] = T[c] + s->tau[6 * (int64_t)e + c];
                continue;
            }
            if (s->rem[e] < 0) continue;
            for (int i = 0; i < 3; ++i) {
                if (!(s->tact[e] >> i & 1) || !tet_has_pair(s, e, i, pj)) continue;
                Vh = Vh + s->tV[3 * (int64_t)e + i];
                for (int c = 0; c < 6; ++c) T[c] = T[c] + s->ttau[18 * (int64_t)e + 6 * i + c];
            }
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

/* f_a = c((gx S11 + gy S12) + gz S13, (gy S22 + gx S12) + gz S23, (gz S33 + gy S23) + gx S13) */
static void force_of(const double *grad, int na, const double *S, double c, double *f) {
    for (int a = 0; a < na; ++a) {
        const double *g = grad + 3 * a;
        f[3 * a] = c * ((g[0] * S[0] + g[1] * S[3]) + g[2] * S[5]);
        f[3 * a + 1] = c * ((g[1] * S[1] + g[0] * S[3]) + g[2] * S[4]);
        f[3 * a + 2] = c * ((g[2] * S[2] + g[1] * S[4]) + g[0] * S[5]);
    }
}
/* tet local edges (0,1),(0,2),(0,3),(1,2),(1,3),(2,3) */
static const int TP[6] = {0, 0, 0, 1, 1, 2}, TQ[6] = {1, 2, 3, 2, 3, 3};

/* element force (R26, eq:hex_fint_discretization): S = sum_{l=0..11} sigma_{s(e,l)}, c = V/12; remainder
 * tets (eq:CSTet_fint_discretization, R5, R29): S over the 6 tet edges, c = V_t/6.  Nodal assembly:
 * the exact sum of the active contributions rounded once (R27) */
static void internal_force(hx_sim *s, const double *u) {
    stage_strain(s, u);
    stage_edge(s);
    for (int64_t e = 0; e < s->E; ++e) {
        double *f = s->fe + 24 * e;
        for (int i = 0; i < 24; ++i) f[i] = 0.0;
        if (s->active[e]) {
            double S[6] = {0, 0, 0, 0, 0, 0};
            for (int l = 0; l < 12; ++l) {
                const double *sg = s->sig + 6 * (int64_t)s->elem_edge[12 * e + l];
                for (int c = 0; c < 6; ++c) S[c] = S[c] + sg[c];
            }
            force_of(s->grad + 24 * e, 8, S, s->V[e] / 12.0, f);
        }
        if (s->rem[e] < 0) continue;
        for (int i = 0; i < 3; ++i) {
            double *tf = s->tfe + 36 * e + 12 * i;
            for (int c = 0; c < 12; ++c) tf[c] = 0.0;
            if (!(s->tact[e] >> i & 1)) continue;
            const uint8_t *t = s->tloc + 12 * e + 4 * i;
            double S[6] = {0, 0, 0, 0, 0, 0};
            for (int l = 0; l < 6; ++l) {
                const double *sg = s->sig + 6 * (int64_t)s->pair_edge[28 * e + pair_id(t[TP[l]], t[TQ[l]])];
                for (int c = 0; c < 6; ++c) S[c] = S[c] + sg[c];
            }
            force_of(s->tgrad + 36 * e + 12 * i, 4, S, s->tV[3 * e + i] / 6.0, tf);
        }
    }
    for (int64_t k = 0; k < s->N; ++k) {
        xsum acc[3];
        for (int c = 0; c < 3; ++c) xsum_init(&acc[c]);
        for (int64_t j = s->nod_off[k]; j < s->nod_off[k + 1]; ++j) {
            const int32_t ent = s->nod_ent[j], e = ent >> 3, a = ent & 7;
            if (s->active[e]) {
                const double *x = s->fe + 24 * (int64_t)e + 3 * a;
                for (int c = 0; c < 3; ++c) xsum_add(&acc[c], x[c]);
                continue;
            }
            if (s->rem[e] < 0) continue;
            for (int i = 0; i < 3; ++i) {
                if (!(s->tact[e] >> i & 1)) continue;
                for (int b = 0; b < 4; ++b)
                    if (s->tloc[12 * (int64_t)e + 4 * i + b] == a) {
                        const double *x = s->tfe + 36 * (int64_t)e + 12 * i + 3 * b;
                        for (int c = 0; c < 3; ++c) xsum_add(&acc[c], x[c]);
                    }
            }
        }
        for (int c = 0; c < 3; ++c) s->fint[3 * k + c] = xsum_round(&acc[c]);
    }
}

static void ramp(double t, double t0, double v0, double *v, double *acc) {
    if (t0 <= 0.0) { *v = v0; *acc = 0.0; return; }
    *v = (t <= t0) ? (t / t0) * v0 : v0;
    *acc = (t < t0) ? v0 / t0 : 0.0;
}

/* ---------------------------------------------------------------- crack patterns III-VI (R28)
 * PAPER.md:L478-L540.  Quadrature point G_l = midpoint of hex edge l, sigma_{G_l} = sigma of that edge.
 * Face f = (v0, v1, v2, v3) cyclic (HF); x' = partner(f, x) is x's neighbour across the hex.
 *  opposite front j (0, 1) of face f: (a, b, c, d) = (v0, v1, v2, v3) or (v1, v2, v3, v0); front edges
 *    p = (a, b), q = (d, c); translates p' = (a', b'), q' = (d', c').
 *  m = (G_q - G_p) x (R - M), M = (G_p + G_q)/2 the front's midpoint and R the far side's point:
 *    III  k = 2f + j:           R = (G_p' + G_q')/2; G = 1/2 (S(p', m) Dd_p + S(q', m) Dd_q) / |m|^2,
 *                               area |m|; fully cracked (no remainder)
 *    IV   k = 12 + 4f + 2j + t: far edge g = (a', d') (t = 0) or (b', c') (t = 1), R = G_g; G = 1/2 (S(g, m) Dd_p + S(g, m) Dd_q) / |m|^2,
 *                               area |m|; remainder (b, b', a' | c, c', d') or (a, a', b' | d, d', c')
 *  neighbouring front at corner i of face f: c = v_i, x = v_{i+1}, z = v_{i+2}, y = v_{i+3}; p = (c, x),
 *    q = (c, y), r = (c, c'); p' = (c', x'), q' = (c', y').
 *    V    k = 36 + 4f + i:      R = (G_p' + G_q')/2; G = 1/2 (S(p', m) Dd_p + S(q', m) Dd_q) / |m|^2,
 *                               area |m|; remainder (x, z, y | x', z', y')
 *    VI   k = 60 + 4f + i:      R = G_r; G = 1/2 (S(r, m) (Dd_p + Dd_q)) / |m|^2,
 *                               area |m| / 2; remainder (x, z, y | x', z', y')
 * S(l, m) = sigma_{G_l} . m (R8), Dd_l = H_l ((u_q - u_p) . m) sgn((X_q - X_p) . m) over the edge's end
 * nodes (R6, R9); the R11v flag zeroes G unless H_p and H_q. */
double orc_sig_proj(const double *s6, const double *m);
void orc_tet_geometry(const double *X4, double *V, double *grad);
void orc_tet_cand_x(const double *X12, const double *u12, const double *s36, uint32_t flags, double *G24, double *A24);
#define HX_F_FRONT_BOTH_STRETCHED 0x40u

static double sgnd(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

typedef struct {
    double X[8][3], U[8][3], G[12][3];
    int H[12];
    const double *sg[12];
} hx_local;

static void local_of(const hx_sim *s, int64_t e, const double *u, hx_local *L) {
    for (int a = 0; a < 8; ++a)
        for (int c = 0; c < 3; ++c) {
            L->X[a][c] = s->X[3 * (int64_t)s->hex[8 * e + a] + c];
            L->U[a][c] = u[3 * (int64_t)s->hex[8 * e + a] + c];
        }
    for (int l = 0; l < 12; ++l) {
        double du[3], dX[3], w[3];
        for (int c = 0; c < 3; ++c) {
            L->G[l][c] = 0.5 * (L->X[HP[l]][c] + L->X[HQ[l]][c]);
            du[c] = L->U[HQ[l]][c] - L->U[HP[l]][c];
            dX[c] = L->X[HQ[l]][c] - L->X[HP[l]][c];
            w[c] = 2.0 * dX[c] + du[c];
        }
        L->H[l] = dot3(du, w) > 0.0;
        L->sg[l] = s->sig + 6 * (int64_t)s->elem_edge[12 * e + l];
    }
}
static double Dd_of(const hx_local *L, int l, const double *m) {
    if (!L->H[l]) return 0.0;
    double du[3], dX[3];
    for (int c = 0; c < 3; ++c) { du[c] = L->U[HQ[l]][c] - L->U[HP[l]][c]; dX[c] = L->X[HQ[l]][c] - L->X[HP[l]][c]; }
    return dot3(du, m) * sgnd(dot3(dX, m));
}
/* m = (Gq - Gp) x (R - M) with M = (Gp + Gq) / 2 the front's midpoint and R = Rm or (Rm + Rn) / 2 (Rn may
 * be NULL): symmetric in p <-> q (m changes sign exactly), so the candidate does not depend on the
 * labelling direction of the face */
static void mvec(const double *Gp, const double *Gq, const double *Rm, const double *Rn, double *m) {
    double d1[3], d2[3];
    for (int c = 0; c < 3; ++c) {
        const double M = 0.5 * (Gp[c] + Gq[c]), R = Rn ? 0.5 * (Rm[c] + Rn[c]) : Rm[c];
        d1[c] = Gq[c] - Gp[c];
        d2[c] = R - M;
    }
    cross3(d1, d2, m);
}

/* candidate k of a hex: G, area and the remainder prism (6 local nodes; returns 0 for none) */
static int hex_candidate(const hx_local *L, int k, uint32_t flags, double *G, double *area, int *P) {
    double m[3];
    int lp, lq, rem = 1;
    if (k < 36) {
        int f, j, t = 0;
        if (k < 12) { f = k / 2; j = k % 2; } else { f = (k - 12) / 4; j = ((k - 12) / 2) % 2; t = (k - 12) % 2; }
        const int *v = HF[f];
        int a = v[j], b = v[j + 1], c = v[(j + 2) % 4], d = v[(j + 3) % 4];
        int a1 = partner(f, a), b1 = partner(f, b), c1 = partner(f, c), d1 = partner(f, d);
        lp = hex_edge(a, b); lq = hex_edge(d, c);
        if (k < 12) {
            int lp1 = hex_edge(a1, b1), lq1 = hex_edge(d1, c1);
            mvec(L->G[lp], L->G[lq], L->G[lp1], L->G[lq1], m);
            double mm = dot3(m, m);
            double A1 = orc_sig_proj(L->sg[lp1], m) * Dd_of(L, lp, m);
            double A2 = orc_sig_proj(L->sg[lq1], m) * Dd_of(L, lq, m);
            *G = (0.5 * (A1 + A2)) / mm;
            *area = sqrt(mm);
            rem = 0;
        } else {
            int g = t == 0 ? hex_edge(a1, d1) : hex_edge(b1, c1);
            mvec(L->G[lp], L->G[lq], L->G[g], NULL, m);
            double mm = dot3(m, m);
            double A1 = orc_sig_proj(L->sg[g], m) * Dd_of(L, lp, m);
            double A2 = orc_sig_proj(L->sg[g], m) * Dd_of(L, lq, m);
            *G = (0.5 * (A1 + A2)) / mm;
            *area = sqrt(mm);
            if (t == 0) { P[0] = b; P[1] = b1; P[2] = a1; P[3] = c; P[4] = c1; P[5] = d1; }
            else { P[0] = a; P[1] = a1; P[2] = b1; P[3] = d; P[4] = d1; P[5] = c1; }
        }
    } else {
        int vi = k < 60 ? k - 36 : k - 60, f = vi / 4, i = vi % 4;
        const int *v = HF[f];
        int c = v[i], x = v[(i + 1) % 4], z = v[(i + 2) % 4], y = v[(i + 3) % 4];
        int c1 = partner(f, c), x1 = partner(f, x), z1 = partner(f, z), y1 = partner(f, y);
        lp = hex_edge(c, x); lq = hex_edge(c, y);
        int lr = hex_edge(c, c1);
        if (k < 60) {
            int lp1 = hex_edge(c1, x1), lq1 = hex_edge(c1, y1);
            mvec(L->G[lp], L->G[lq], L->G[lp1], L->G[lq1], m);
            double mm = dot3(m, m);
            double A1 = orc_sig_proj(L->sg[lp1], m) * Dd_of(L, lp, m);
            double A2 = orc_sig_proj(L->sg[lq1], m) * Dd_of(L, lq, m);
            *G = (0.5 * (A1 + A2)) / mm;
            *area = sqrt(mm);
        } else {
            mvec(L->G[lp], L->G[lq], L->G[lr], NULL, m);
            double mm = dot3(m, m);
            double Sg = orc_sig_proj(L->sg[lr], m);
            *G = (0.5 * (Sg * (Dd_of(L, lp, m) + Dd_of(L, lq, m)))) / mm;
            *area = sqrt(mm) / 2.0;
        }
        P[0] = x; P[1] = z; P[2] = y; P[3] = x1; P[4] = z1; P[5] = y1;
    }
    if ((flags & HX_F_FRONT_BOTH_STRETCHED) && !(L->H[lp] && L->H[lq])) *G = 0.0;
    return rem;
}

/* the remainder tets of prism P = (A, B, C | A', B', C'): (A,B,C,A'), (B,C,A',B'), (C,A',B',C'); a tet with
 * negative volume has its first two nodes swapped */
static void set_remainder(hx_sim *s, int64_t e, const int *P) {
    static const int TT[3][4] = {{0, 1, 2, 3}, {1, 2, 3, 4}, {2, 3, 4, 5}};
    for (int i = 0; i < 3; ++i) {
        uint8_t *t = s->tloc + 12 * e + 4 * i;
        for (int a = 0; a < 4; ++a) t[a] = (uint8_t)P[TT[i][a]];
        for (int pass = 0; pass < 2; ++pass) {
            double X4[12];
            for (int a = 0; a < 4; ++a)
                for (int c = 0; c < 3; ++c) X4[3 * a + c] = s->X[3 * (int64_t)s->hex[8 * e + t[a]] + c];
            orc_tet_geometry(X4, s->tV + 3 * e + i, s->tgrad + 36 * e + 12 * i);
            if (s->tV[3 * e + i] >= 0.0 || pass) break;
            uint8_t w = t[0]; t[0] = t[1]; t[1] = w;
        }
    }
    s->tact[e] = 7;
}

/* criterion on (u_{n+1}, sigma of this step) and split pass (R16, R18: decisions on the pre-split state;
 * ascending element order: hexes, then the remainder tets (e, i)); masses of the nodes of split
 * elements recomputed, m = 0 -> frozen (R15) */
static void hex_crack(hx_sim *s, int64_t step_no) {
    for (int64_t e = 0; e < s->E; ++e) {
        s->flag[e] = 0;
        if (s->active[e]) {
            hx_local L;
            local_of(s, e, s->u, &L);
            double Gb = 0.0, Ab = 0.0;
            int kb = -1;
            for (int k = 0; k < 84; ++k) {
                double G, A;
                int P[6];
                hex_candidate(&L, k, s->flags, &G, &A, P);
                if (kb < 0 || G > Gb || (G == Gb && A > Ab)) { Gb = G; Ab = A; kb = k; }
            }
            s->Gb[4 * e] = Gb; s->Ab[4 * e] = Ab; s->kb[4 * e] = kb;
            if (Gb > s->gc[e]) s->flag[e] |= 1;
            continue;
        }
        if (s->rem[e] < 0) continue;
        for (int i = 0; i < 3; ++i) {
            if (!(s->tact[e] >> i & 1)) continue;
            const uint8_t *t = s->tloc + 12 * e + 4 * i;
            double X12[12], u12[12], s36[36], G24[24], A24[24];
            for (int a = 0; a < 4; ++a)
                for (int c = 0; c < 3; ++c) {
                    X12[3 * a + c] = s->X[3 * (int64_t)s->hex[8 * e + t[a]] + c];
                    u12[3 * a + c] = s->u[3 * (int64_t)s->hex[8 * e + t[a]] + c];
                }
            for (int l = 0; l < 6; ++l)
                memcpy(s36 + 6 * l, s->sig + 6 * (int64_t)s->pair_edge[28 * e + pair_id(t[TP[l]], t[TQ[l]])], 48);
            orc_tet_cand_x(X12, u12, s36, s->flags, G24, A24);
            int best = 0;
            for (int k = 1; k < 24; ++k)
                if (G24[k] > G24[best] || (G24[k] == G24[best] && A24[k] > A24[best])) best = k;
            s->Gb[4 * e + 1 + i] = G24[best]; s->Ab[4 * e + 1 + i] = A24[best]; s->kb[4 * e + 1 + i] = best;
            if (G24[best] > s->gc[e]) s->flag[e] |= (uint8_t)(2 << i);
        }
    }
    int64_t n = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (int64_t e = 0; e < s->E; ++e)
            for (int i = pass ? 0 : -1; i < (pass ? 3 : 0); ++i) {
                if (!(s->flag[e] >> (i + 1) & 1)) continue;
                const int w = 4 * (int)e + 1 + i;
                if (s->nrec == s->caprec) {
                    s->caprec = s->caprec ? 2 * s->caprec : 256;
                    s->rstep = realloc(s->rstep, sizeof(int64_t) * s->caprec);
                    s->relem = realloc(s->relem, sizeof(int32_t) * s->caprec);
                    s->rcand = realloc(s->rcand, sizeof(int32_t) * s->caprec);
                    s->rG = realloc(s->rG, sizeof(double) * s->caprec);
                    s->rA = realloc(s->rA, sizeof(double) * s->caprec);
                }
                s->rstep[s->nrec] = step_no;
                s->relem[s->nrec] = i < 0 ? (int32_t)e : (int32_t)(s->E + 3 * e + i);
                s->rcand[s->nrec] = s->kb[w];
                s->rG[s->nrec] = s->Gb[w];
                s->rA[s->nrec] = s->Ab[w];
                s->nrec++;
                s->Ud = s->Ud + s->gc[e] * s->Ab[w];
                ++n;
                if (i < 0) {
                    s->active[e] = 0;
                    hx_local L;
                    double G, A;
                    int P[6];
                    local_of(s, e, s->u, &L);
                    if (hex_candidate(&L, s->kb[w], s->flags, &G, &A, P)) { s->rem[e] = (int8_t)s->kb[w]; set_remainder(s, e, P); }
                } else {
                    s->tact[e] &= (uint8_t)~(1u << i);
                }
            }
    if (!n) return;
    for (int64_t e = 0; e < s->E; ++e) {
        if (!s->flag[e]) continue;
        for (int a = 0; a < 8; ++a) {
            int touched = s->flag[e] & 1;
            for (int i = 0; i < 3; ++i)
                if ((s->flag[e] >> (i + 1) & 1) && tet_has_node(s, e, i, a)) touched = 1;
            if (!touched) continue;
            const int64_t k = s->hex[8 * e + a];
            s->m[k] = node_mass(s, k);
            if (s->m[k] == 0.0)
                for (int c = 0; c < 3; ++c) { s->v[3 * k + c] = 0.0; s->a[3 * k + c] = 0.0; }
        }
    }
}

HX_API hx_sim *hx_create(int64_t n_nodes, const double *X, int64_t n_hex, const int32_t *hex, const uint8_t *state,
                         double E, double nu, double rho, int64_t n_tf, const int32_t *tface, const double *tface_t,
                         int64_t n_vbc, const int32_t *vbc_node, const uint8_t *vbc_mask, const double *vbc_v0,
                         double vbc_t0, double dt, double cfl, double gamma, const double *f_nodal,
                         const double *body, const double *gc, uint32_t flags, char *err, int errlen) {
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
    /* edges: every node pair of every hex (28), as sorted (min, max) keys -- first the pairs that are
     * hex edges of some hex (the smoothing domains of the mesh, edges [0, S_h)), then the face and
     * body diagonals that only remainder tets can use (R28); incidence: (hex, local pair) in
     * ascending hex id */
    const int64_t K = 28 * n_hex;
    uint64_t *keys = xc(K, sizeof(uint64_t)), *uk = xc(K, sizeof(uint64_t)), *ud = xc(K, sizeof(uint64_t));
    int64_t nh = 0, nd = 0;
    for (int64_t e = 0; e < n_hex; ++e)
        for (int a = 0; a < 8; ++a)
            for (int b = a + 1; b < 8; ++b) {
                uint64_t i = (uint32_t)hex[8 * e + a], j = (uint32_t)hex[8 * e + b];
                uint64_t key = (i < j ? i : j) << 32 | (i < j ? j : i);
                keys[28 * e + pair_id(a, b)] = key;
                if (hex_edge(a, b) >= 0) uk[nh++] = key; else ud[nd++] = key;
            }
    qsort(uk, nh, sizeof(uint64_t), cmp_u64);
    int64_t S_h = 0;
    for (int64_t i = 0; i < nh; ++i)
        if (i == 0 || uk[i] != uk[i - 1]) uk[S_h++] = uk[i];
    qsort(ud, nd, sizeof(uint64_t), cmp_u64);
    int64_t S_d = 0;
    for (int64_t i = 0; i < nd; ++i)
        if ((i == 0 || ud[i] != ud[i - 1]) && find_edge(uk, S_h, ud[i]) < 0) ud[S_d++] = ud[i];
    const int64_t S = S_h + S_d;
    s->S = S; s->S_h = S_h;
    s->pair_edge = xc(K, sizeof(int32_t));
    s->elem_edge = xc(12 * n_hex, sizeof(int32_t));
    s->inc_off = xc(S + 1, sizeof(int64_t));
    for (int64_t i = 0; i < K; ++i) {
        int64_t k = find_edge(uk, S_h, keys[i]);
        if (k < 0) k = S_h + find_edge(ud, S_d, keys[i]);
        s->pair_edge[i] = (int32_t)k;
        s->inc_off[k + 1]++;
    }
    for (int64_t e = 0; e < n_hex; ++e)
        for (int l = 0; l < 12; ++l) s->elem_edge[12 * e + l] = s->pair_edge[28 * e + pair_id(HP[l], HQ[l])];
    for (int64_t k = 0; k < S; ++k) s->inc_off[k + 1] += s->inc_off[k];
    s->inc = xc(K, sizeof(int32_t));
    s->inc_j = xc(K, sizeof(int32_t));
    int64_t *fill = xc(S, sizeof(int64_t));
    for (int64_t e = 0; e < n_hex; ++e)
        for (int j = 0; j < 28; ++j) {
            int64_t k = s->pair_edge[28 * e + j], at = s->inc_off[k] + fill[k]++;
            s->inc[at] = (int32_t)e;
            s->inc_j[at] = j;
        }
    free(fill); free(keys); free(uk); free(ud);
    s->gc = xc(n_hex, sizeof(double));
    for (int64_t e = 0; e < n_hex; ++e) s->gc[e] = gc ? gc[e] : INFINITY;
    s->flags = flags;
    s->rem = xc(n_hex, 1);
    memset(s->rem, 0xff, n_hex);
    s->tact = xc(n_hex, 1);
    s->tloc = xc(12 * n_hex, 1);
    s->tV = xc(3 * n_hex, sizeof(double));
    s->tgrad = xc(36 * n_hex, sizeof(double));
    s->ttau = xc(18 * n_hex, sizeof(double));
    s->tfe = xc(36 * n_hex, sizeof(double));
    s->flag = xc(n_hex, 1);
    s->Gb = xc(4 * n_hex, sizeof(double));
    s->Ab = xc(4 * n_hex, sizeof(double));
    s->kb = xc(4 * n_hex, sizeof(int32_t));
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

/* explicit steps (the tet oracle's orc_run): predictor, internal force, node update, then every
 * crack_every-th step the criterion and split pass (R16).  Returns 1 on a non-finite state. */
HX_API int hx_run(hx_sim *s, int64_t nsteps, int32_t crack_every) {
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
        int bad = 0;
        for (int64_t i = 0; i < 3 * s->N; ++i)
            if (!isfinite(s->u[i]) || !isfinite(s->v[i]) || !isfinite(s->a[i])) bad = 1;
        if (crack_every > 0 && n1 % crack_every == 0) hex_crack(s, n1);
        s->step = n1;
        if (bad) { s->nonfinite = 1; return 1; }
    }
    return 0;
}

HX_API int64_t hx_n_edges(const hx_sim *s) { return s->S_h; }
HX_API int64_t hx_n_edges_all(const hx_sim *s) { return s->S; }
HX_API int64_t hx_n_records(const hx_sim *s) { return s->nrec; }
HX_API double hx_dissipated(const hx_sim *s) { return s->Ud; }
HX_API void hx_get_records(const hx_sim *s, int64_t *step, int32_t *elem, int32_t *cand, double *G, double *area) {
    for (int64_t i = 0; i < s->nrec; ++i) {
        step[i] = s->rstep[i]; elem[i] = s->relem[i]; cand[i] = s->rcand[i]; G[i] = s->rG[i]; area[i] = s->rA[i];
    }
}
/* element states: hex_active [E], tet_active [E][3] (remainder tets), tet nodes [E][3][4] (global ids,
 * -1 where the hex has no remainder), tet volumes [E][3] */
HX_API void hx_get_elements(const hx_sim *s, uint8_t *hex_active, uint8_t *tet_active, int32_t *tet_nodes, double *tV) {
    for (int64_t e = 0; e < s->E; ++e) {
        hex_active[e] = s->active[e];
        for (int i = 0; i < 3; ++i) {
            tet_active[3 * e + i] = s->rem[e] >= 0 ? (s->tact[e] >> i & 1) : 0;
            tV[3 * e + i] = s->rem[e] >= 0 ? s->tV[3 * e + i] : 0.0;
            for (int a = 0; a < 4; ++a)
                tet_nodes[12 * e + 4 * i + a] = s->rem[e] >= 0 ? s->hex[8 * e + s->tloc[12 * e + 4 * i + a]] : -1;
        }
    }
}
/* probe: the 84 candidates of hex e for the displacement u (sigma from u), and their remainder prisms
 * as local nodes [84][6] (-1 for pattern III) */
HX_API void hx_candidates(hx_sim *s, const double *u, int64_t e, double *G84, double *A84, int32_t *P84) {
    stage_strain(s, u);
    stage_edge(s);
    hx_local L;
    local_of(s, e, u, &L);
    for (int k = 0; k < 84; ++k) {
        int P[6];
        int r = hex_candidate(&L, k, s->flags, G84 + k, A84 + k, P);
        for (int i = 0; i < 6; ++i) P84[6 * k + i] = r ? P[i] : -1;
    }
}
/* probe: force a split of hex e by candidate k (the split pass's state change, no record) */
HX_API void hx_force_split(hx_sim *s, int64_t e, int32_t k) {
    hx_local L;
    double G, A;
    int P[6];
    local_of(s, e, s->u, &L);
    s->active[e] = 0;
    if (hex_candidate(&L, k, s->flags, &G, &A, P)) { s->rem[e] = (int8_t)k; set_remainder(s, e, P); }
    for (int a = 0; a < 8; ++a) {
        const int64_t n = s->hex[8 * e + a];
        s->m[n] = node_mass(s, n);
        if (s->m[n] == 0.0)
            for (int c = 0; c < 3; ++c) { s->v[3 * n + c] = 0.0; s->a[3 * n + c] = 0.0; }
    }
}
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
    if (sigma) memcpy(sigma, s->sig, sizeof(double) * 6 * s->S_h);
    if (vhat) memcpy(vhat, s->vhat, sizeof(double) * s->S_h);
    if (edge_nodes)  /* endpoints of each edge (from the first incident hex) */
        for (int64_t k = 0; k < s->S_h; ++k) {
            const int32_t e = s->inc[s->inc_off[k]], j = s->inc_j[s->inc_off[k]];
            for (int a = 0; a < 8; ++a)
                for (int b = a + 1; b < 8; ++b)
                    if (pair_id(a, b) == j) {
                        int32_t i = s->hex[8 * (int64_t)e + a], jj = s->hex[8 * (int64_t)e + b];
                        edge_nodes[2 * k] = i < jj ? i : jj;
                        edge_nodes[2 * k + 1] = i < jj ? jj : i;
                    }
        }
}
/* every edge incl. the diagonals of remainder tets: sigma [S][6], Vhat [S], endpoints [S][2] */
HX_API void hx_edge_stress_all(hx_sim *s, const double *u, double *sigma, double *vhat, int32_t *edge_nodes) {
    stage_strain(s, u);
    stage_edge(s);
    memcpy(sigma, s->sig, sizeof(double) * 6 * s->S);
    memcpy(vhat, s->vhat, sizeof(double) * s->S);
    for (int64_t k = 0; k < s->S; ++k) {
        const int32_t e = s->inc[s->inc_off[k]], j = s->inc_j[s->inc_off[k]];
        for (int a = 0; a < 8; ++a)
            for (int b = a + 1; b < 8; ++b)
                if (pair_id(a, b) == j) {
                    int32_t i = s->hex[8 * (int64_t)e + a], jj = s->hex[8 * (int64_t)e + b];
                    edge_nodes[2 * k] = i < jj ? i : jj;
                    edge_nodes[2 * k + 1] = i < jj ? jj : i;
                }
    }
}
HX_API void hx_internal_force(hx_sim *s, const double *u, double *f) {
    internal_force(s, u);
    memcpy(f, s->fint, sizeof(double) * 3 * s->N);
}
/* strain energy U = sum_s psi(eps~_s) Vhat_s / 12 (R26 smoothing-domain volume) */
/* strain energy U = sum_s psi(eps~_s) W_s with the smoothing-domain volume W_s = sum of V_j / n_j over the
 * active elements of the edge (R26: V/12 per hex, R5: V/6 per tet; R29), element order */
HX_API double hx_strain_energy(hx_sim *s, const double *u) {
    stage_strain(s, u);
    stage_edge(s);
    double U = 0.0;
    for (int64_t k = 0; k < s->S; ++k) {
        if (s->vhat[k] == 0.0) continue;
        double T[6] = {0, 0, 0, 0, 0, 0}, W = 0.0;
        for (int64_t j = s->inc_off[k]; j < s->inc_off[k + 1]; ++j) {
            int32_t e = s->inc[j], pj = s->inc_j[j];
            if (s->active[e]) {
                if (hex_edge_of_pair(pj) < 0) continue;
                W = W + s->V[e] / 12.0;
                for (int c = 0; c < 6; ++c) T[c] = T[c] + s->tau[6 * (int64_t)e + c];
                continue;
            }
            if (s->rem[e] < 0) continue;
            for (int i = 0; i < 3; ++i) {
                if (!(s->tact[e] >> i & 1) || !tet_has_pair(s, e, i, pj)) continue;
                W = W + s->tV[3 * (int64_t)e + i] / 6.0;
                for (int c = 0; c < 6; ++c) T[c] = T[c] + s->ttau[18 * (int64_t)e + 6 * i + c];
            }
        }
        double inv = 1.0 / s->vhat[k];
        double e11 = T[0] * inv, e22 = T[1] * inv, e33 = T[2] * inv, g12 = T[3] * inv, g23 = T[4] * inv, g13 = T[5] * inv;
        double tr = e11 + e22 + e33;
        double ee = e11 * e11 + e22 * e22 + e33 * e33 + 0.5 * (g12 * g12 + g23 * g23 + g13 * g13);
        U += (0.5 * s->lam * tr * tr + s->mu * ee) * W;
    }
    return U;
}
HX_API void hx_set_state(hx_sim *s, const double *u, const double *v, const double *a) {
    if (u) memcpy(s->u, u, sizeof(double) * 3 * s->N);
    if (v) memcpy(s->v, v, sizeof(double) * 3 * s->N);
    if (a) memcpy(s->a, a, sizeof(double) * 3 * s->N);
}
