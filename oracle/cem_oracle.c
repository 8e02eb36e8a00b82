/*
 * cem_oracle.c -- plain, slow, obviously-correct CPU oracle of the 3D Crack Element
 * Method explicit step (arXiv 2508.04076).  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * it.  It shares no code, header, table or helper with paper_2508_04076_b200/.
 *
 * Every function cites the PAPER.md passage it follows.  The readings of ambiguous or
 * garbled passages are DESIGN.md "Readings" R1..R21 (= SURVEY.md §8(c) Q1..Q21).
 *
 * Arithmetic: IEEE fp64, compiled with -O2 -ffp-contract=off -fno-fast-math, every sum
 * sequential in the order written here (the GPU path reproduces this order; the oracle
 * is the definition of that order) except the nodal
 * assembly sum, which is exact and rounded once (R27, exact_sum.h).  OpenMP only
 * parallelises loops over independent outputs, so results are identical at any
 * thread count.
 *
 * Pins: tests/test_oracle_*.py check this file against closed forms, invariants,
 * the literal assembled-B form (oracle/l0_literal.py), exact rationals and brute force.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

#include "exact_sum.h"

/* local edge l -> (p,q), p<q   (SURVEY.md §8(c) Init 2) */
static const int EP[6] = {0, 0, 0, 1, 1, 2};
static const int EQ[6] = {1, 2, 3, 2, 3, 3};

/* criterion variant (R11 / SURVEY.md §8(c) Q11): a candidate counts only when both edges of its
 * crack front (c-p and c-q) are stretched ("whose tensile stretches at two edges", PAPER.md:L459;
 * SPEC.md:L305 "front with both stretches nonzero"); other candidates get G = 0 */
#define ORC_F_FRONT_BOTH_STRETCHED 0x40u

static int local_edge(int a, int b) {
    int p = a < b ? a : b, q = a < b ? b : a;
    for (int l = 0; l < 6; ++l)
        if (EP[l] == p && EQ[l] == q) return l;
    return -1;
}

typedef struct {
    int64_t step; int32_t elem; int32_t cand; double G; double area;
} orc_record;

typedef struct { double lam[3], vec[9]; int32_t k1, deg; } eig_t;

typedef struct orc_sim {
    int64_t N, E, S, F, B;
    double *X;            /* [N][3] */
    int32_t *tet;         /* [E][4] */
    uint8_t *active;      /* [E] 1 active, 0 inactive */
    double *gc;           /* [E] */
    double *V;            /* [E] */
    double *grad;         /* [E][4][3] */
    int32_t *edge_nodes;  /* [S][2] */
    int32_t *elem_edge;   /* [E][6] */
    int64_t *inc_off;     /* [S+1] */
    int32_t *inc;         /* [6E] ascending element id */
    int64_t *nod_off;     /* [N+1] */
    int32_t *nod_ent;     /* [4E] packed 4e+a, ascending e */
    double *m;            /* [N] lumped mass */
    double *fext;         /* [N][3] */
    uint8_t *dir;         /* [N] Dirichlet mask bits */
    double *dir_v0;       /* [N][3] */
    double t0;
    uint32_t flags;       /* ORC_F_* (criterion variants) */
    double E_mod, nu, rho, lam, mu, l2m;
    double dt, gamma;
    /* state */
    double *u, *v, *a;    /* [N][3] */
    int64_t step;
    double Ud;
    /* energy ledger: reaction work of the prescribed dofs */
    double Wr;
    double *rprev;        /* [N][3] support force R at the previous step (prescribed dofs) */
    double *uold;         /* [N][3] u_n while step n -> n+1 runs */
    int has_dir;
    orc_record *rec; int64_t nrec, caprec;
    /* scratch */
    double *tau;          /* [E][6] */
    double *sig;          /* [S][6] */
    double *vhat;         /* [S] */
    double *fe;           /* [E][4][3] */
    double *fint;         /* [N][3] */
    void *eig;            /* [S] eig_t: principal decomposition of sigma_s */
    double *G;            /* [E] */
    int32_t *cand;        /* [E] */
    double *area;         /* [E] */
    uint8_t *flag;        /* [E] */
    int nonfinite;
} orc_sim;

/* ---------------------------------------------------------------- vectors */
static void sub3(const double *a, const double *b, double *r) { r[0] = a[0] - b[0]; r[1] = a[1] - b[1]; r[2] = a[2] - b[2]; }
static double dot3(const double *a, const double *b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
static void cross3(const double *a, const double *b, double *r) {
    r[0] = a[1] * b[2] - a[2] * b[1];
    r[1] = a[2] * b[0] - a[0] * b[2];
    r[2] = a[0] * b[1] - a[1] * b[0];
}

/* ---------------------------------------------------------------- geometry
 * Tet volume and constant shape-function gradients (PAPER.md:L283-L310,
 * eq:CSTet_strain_discretization; B_k^{V_j} built from dN_k/dx).
 *   d_i = X_i - X_0, det = d1.(d2 x d3), V = det/6,
 *   inv = 1/det, gradN1 = (d2 x d3) inv, gradN2 = (d3 x d1) inv, gradN3 = (d1 x d2) inv,
 *   gradN0 = -((gradN1 + gradN2) + gradN3).
 */
ORC_API void orc_tet_geometry(const double *X4 /*[4][3]*/, double *V, double *grad /*[4][3]*/) {
    double d1[3], d2[3], d3[3], c23[3], c31[3], c12[3];
    sub3(X4 + 3, X4, d1); sub3(X4 + 6, X4, d2); sub3(X4 + 9, X4, d3);
    cross3(d2, d3, c23); cross3(d3, d1, c31); cross3(d1, d2, c12);
    double det = dot3(d1, c23);
    *V = det / 6.0;
    double inv = 1.0 / det;
    for (int c = 0; c < 3; ++c) {
        grad[3 + c] = c23[c] * inv;
        grad[6 + c] = c31[c] * inv;
        grad[9 + c] = c12[c] * inv;
        grad[c] = -((grad[3 + c] + grad[6 + c]) + grad[9 + c]);
    }
}

/* Lame constants (standard isotropic relations; PAPER.md:L197-L202 names lambda, mu) */
ORC_API void orc_lame(double E, double nu, double *lam, double *mu) {
    *lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    *mu = E / (2.0 * (1.0 + nu));
}

/* ---------------------------------------------------------------- principal stress
 * Largest principal stress of a symmetric tensor ("maximum principal
 * stress at edge quadrature G") by cyclic Jacobi (R8).  s6 in Voigt order
 * (11,22,33,12,23,13) with tensor shears.  Outputs all eigenvalues lam[3], the
 * eigenvector matrix vec (column k = eigenvector of lam[k], vec[3*i+k]), k1 = index of
 * the largest eigenvalue (first on ties), degmask = bit k set iff
 * lam[k1] - lam[k] <= 1e-10 |lam[k1]| (degenerate top eigenspace, R8).
 */
ORC_API void orc_principal(const double *s6, double *lam, double *vec, int32_t *k1_out, int32_t *degmask_out) {
    double A[3][3] = {{s6[0], s6[3], s6[5]}, {s6[3], s6[1], s6[4]}, {s6[5], s6[4], s6[2]}};
    double Vm[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    static const int PP[3] = {0, 0, 1}, QQ[3] = {1, 2, 2}, RR[3] = {2, 1, 0};
    for (int sweep = 0; sweep < 8; ++sweep) {
        if (A[0][1] == 0.0 && A[0][2] == 0.0 && A[1][2] == 0.0) break;
        for (int r3 = 0; r3 < 3; ++r3) {
            int p = PP[r3], q = QQ[r3], r = RR[r3];
            double apq = A[p][q], app = A[p][p], aqq = A[q][q];
            if (fabs(apq) <= 0x1p-60 * (fabs(app) + fabs(aqq))) {
                A[p][q] = 0.0; A[q][p] = 0.0;
                continue;
            }
            double theta = (aqq - app) / (2.0 * apq);
            double t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
            if (theta < 0.0) t = -t;
            double c = 1.0 / sqrt(t * t + 1.0);
            double s = t * c;
            A[p][p] = app - t * apq;
            A[q][q] = aqq + t * apq;
            A[p][q] = 0.0; A[q][p] = 0.0;
            double arp = A[r][p], arq = A[r][q];
            A[r][p] = c * arp - s * arq; A[p][r] = A[r][p];
            A[r][q] = s * arp + c * arq; A[q][r] = A[r][q];
            for (int i = 0; i < 3; ++i) {
                double vip = Vm[i][p], viq = Vm[i][q];
                Vm[i][p] = c * vip - s * viq;
                Vm[i][q] = s * vip + c * viq;
            }
        }
    }
    lam[0] = A[0][0]; lam[1] = A[1][1]; lam[2] = A[2][2];
    int k1 = 0;
    if (lam[1] > lam[k1]) k1 = 1;
    if (lam[2] > lam[k1]) k1 = 2;
    int deg = 0;
    for (int k = 0; k < 3; ++k)
        if (lam[k1] - lam[k] <= 1e-10 * fabs(lam[k1])) deg |= 1 << k;
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) vec[3 * i + k] = Vm[i][k];
    *k1_out = k1; *degmask_out = deg;
}

/* sigma_G . m (unnormalised, R8): sigma1 * |e1.m|, or sigma1 * sqrt(sum_{k in D} (e_k.m)^2)
 * when the top eigenvalue is degenerate (D = degmask, >1 member). */
static double sig_proj(const double *lam, const double *vec, int k1, int deg, const double *m) {
    int cnt = (deg & 1) + ((deg >> 1) & 1) + ((deg >> 2) & 1);
    if (cnt == 1) {
        double e[3] = {vec[k1], vec[3 + k1], vec[6 + k1]};
        return lam[k1] * fabs(dot3(e, m));
    }
    double acc = 0.0;
    for (int k = 0; k < 3; ++k) {
        if (!(deg >> k & 1)) continue;
        double e[3] = {vec[k], vec[3 + k], vec[6 + k]};
        double d = dot3(e, m);
        acc = acc + d * d;
    }
    return lam[k1] * sqrt(acc);
}

/* probe (tests): sigma_G . m of the stress s6 for an unnormalised normal m (R8) */
ORC_API double orc_sig_proj(const double *s6, const double *m) {
    double lam[3], vec[9];
    int32_t k1, deg;
    orc_principal(s6, lam, vec, &k1, &deg);
    return sig_proj(lam, vec, k1, deg, m);
}

/* ---------------------------------------------------------------- topology */
static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

static int64_t find_edge(const uint64_t *keys, int64_t S, uint64_t k) {
    int64_t lo = 0, hi = S - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (keys[mid] == k) return mid;
        if (keys[mid] < k) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

static void *xcalloc(size_t n, size_t s) {
    void *p = calloc(n ? n : 1, s);
    if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return p;
}

/* lumped mass of node k: sum over active incident tets, ascending e, of (rho V_e)/4
 * (PAPER.md:L392-L407 eq:mass_discretization, diagonal; R2 row-sum lumping; R15). */
static double node_mass(const orc_sim *s, int64_t k) {
    double acc = 0.0;
    for (int64_t j = s->nod_off[k]; j < s->nod_off[k + 1]; ++j) {
        int32_t e = s->nod_ent[j] >> 2;
        if (!s->active[e]) continue;
        acc = acc + (s->rho * s->V[e]) / 4.0;
    }
    return acc;
}

static int dof_prescribed(const orc_sim *s, int64_t k, int c) { return (s->dir[k] >> c) & 1; }

/* prescribed velocity ramp: v = (t/t0) v0 for t <= t0, else v0;
 * acceleration v0/t0 for t < t0 else 0 (R17).  t0 <= 0: step, v = v0, a = 0. */
static void ramp(double t, double t0, double v0, double *v, double *acc) {
    if (t0 <= 0.0) { *v = v0; *acc = 0.0; return; }
    *v = (t <= t0) ? (t / t0) * v0 : v0;
    *acc = (t < t0) ? v0 / t0 : 0.0;
}

ORC_API void orc_destroy(orc_sim *s) {
    if (!s) return;
    free(s->X); free(s->tet); free(s->active); free(s->gc); free(s->V); free(s->grad);
    free(s->edge_nodes); free(s->elem_edge); free(s->inc_off); free(s->inc); free(s->nod_off);
    free(s->nod_ent); free(s->m); free(s->fext); free(s->dir); free(s->dir_v0);
    free(s->u); free(s->v); free(s->a); free(s->rec); free(s->tau); free(s->sig); free(s->vhat);
    free(s->fe); free(s->fint); free(s->eig); free(s->G); free(s->cand);
    free(s->area); free(s->flag); free(s->rprev); free(s->uold);
    free(s);
}

/* ---------------------------------------------------------------- stage 1: element strain
 * eps_e = sum_a B_a u_a in Voigt order (eps11, eps22, eps33, gam12, gam23, gam13),
 * PAPER.md:L278 eq:strain_discretization and L285-L307 eq:CSTet_strain_discretization;
 * tau_e = V_e eps_e (the volume weight w_j = V_j / sum V of PAPER.md:L281 is applied in
 * stage 2 as (sum_j V_j eps_j) / (sum_j V_j)).  Inactive tets are skipped. */
static void stage_strain(orc_sim *s, const double *u) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < s->E; ++e) {
        double *tau = s->tau + 6 * e;
        if (!s->active[e]) { for (int i = 0; i < 6; ++i) tau[i] = 0.0; continue; }
        const double *g = s->grad + 12 * e;
        double ex = 0.0, ey = 0.0, ez = 0.0, gxy = 0.0, gyz = 0.0, gxz = 0.0;
        for (int a = 0; a < 4; ++a) {
            const double *ua = u + 3 * (int64_t)s->tet[4 * e + a];
            const double gx = g[3 * a], gy = g[3 * a + 1], gz = g[3 * a + 2];
            ex = ex + gx * ua[0];
            ey = ey + gy * ua[1];
            ez = ez + gz * ua[2];
            gxy = gxy + (gy * ua[0] + gx * ua[1]);
            gyz = gyz + (gz * ua[1] + gy * ua[2]);
            gxz = gxz + (gz * ua[0] + gx * ua[2]);
        }
        const double V = s->V[e];
        tau[0] = V * ex; tau[1] = V * ey; tau[2] = V * ez;
        tau[3] = V * gxy; tau[4] = V * gyz; tau[5] = V * gxz;
    }
}

/* ---------------------------------------------------------------- stage 2: edge stress
 * Smoothed strain at edge quadrature point s:
 *   Vhat_s = sum_{active j in inc(s)} V_j,  eps~_s = (sum_j V_j eps_j) * (1/Vhat_s)
 * = sum_j w_j eps_j with w_j = V_j / sum V (L281).  Isotropic stress (PAPER.md:L197-L202,
 * R1): sigma_ii = (lam+2mu) eps_ii + lam (eps_jj + eps_kk), sigma_ij = mu gamma_ij.
 * Vhat_s = 0 (every incident tet inactive, R19) -> sigma_s = 0. */
static void stage_edge(orc_sim *s) {
    const double lam = s->lam, mu = s->mu, l2m = s->l2m;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < s->S; ++k) {
        double Vh = 0.0, T[6] = {0, 0, 0, 0, 0, 0};
        for (int64_t j = s->inc_off[k]; j < s->inc_off[k + 1]; ++j) {
            int32_t e = s->inc[j];
            if (!s->active[e]) continue;
            Vh = Vh + s->V[e];
            for (int i = 0; i < 6; ++i) T[i] = T[i] + s->tau[6 * (int64_t)e + i];
        }
        double *sg = s->sig + 6 * k;
        s->vhat[k] = Vh;
        if (Vh == 0.0) { for (int i = 0; i < 6; ++i) sg[i] = 0.0; continue; }
        double inv = 1.0 / Vh;
        double e11 = T[0] * inv, e22 = T[1] * inv, e33 = T[2] * inv;
        double g12 = T[3] * inv, g23 = T[4] * inv, g13 = T[5] * inv;
        sg[0] = l2m * e11 + lam * (e22 + e33);
        sg[1] = l2m * e22 + lam * (e11 + e33);
        sg[2] = l2m * e33 + lam * (e11 + e22);
        sg[3] = mu * g12;
        sg[4] = mu * g23;
        sg[5] = mu * g13;
    }
}

/* ---------------------------------------------------------------- stage 3: element force
 * f_int = A_j ( A_k [B_k^{V_j}]^T w_{V_j} sigma ) V_s with V_s = (1/6) sum_j V_j
 * (eq:fint_discretization / eq:CSTet_fint_discretization, R5).
 * Since w_j V_s = V_j / 6, element e receives (V_e/6) B_a^T S_e with
 * S_e = sum over its 6 edges (local order l = 0..5) of sigma_s (DESIGN.md identity I1;
 * pinned against the literal assembled form in tests/test_oracle_force.py). */
static void stage_element_force(orc_sim *s) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < s->E; ++e) {
        double *f = s->fe + 12 * e;
        if (!s->active[e]) { for (int i = 0; i < 12; ++i) f[i] = 0.0; continue; }
        double S[6] = {0, 0, 0, 0, 0, 0};
        for (int l = 0; l < 6; ++l) {
            const double *sg = s->sig + 6 * (int64_t)s->elem_edge[6 * e + l];
            for (int i = 0; i < 6; ++i) S[i] = S[i] + sg[i];
        }
        const double c = s->V[e] / 6.0;
        const double *g = s->grad + 12 * e;
        for (int a = 0; a < 4; ++a) {
            const double gx = g[3 * a], gy = g[3 * a + 1], gz = g[3 * a + 2];
            f[3 * a + 0] = c * ((gx * S[0] + gy * S[3]) + gz * S[5]);
            f[3 * a + 1] = c * ((gy * S[1] + gx * S[3]) + gz * S[4]);
            f[3 * a + 2] = c * ((gz * S[2] + gy * S[4]) + gx * S[5]);
        }
    }
}

/* ---------------------------------------------------------------- stage 4: node force
 * Assembly operator A over elements: f_int,k = sum over (e,a) in the
 * node's incidence list, active e only.  The sum is evaluated exactly and rounded once to
 * fp64 (reading R27, exact_sum.h): its value does not depend on the order of the terms. */
static void stage_node_force(orc_sim *s) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < s->N; ++k) {
        xsum acc[3];
        for (int c = 0; c < 3; ++c) xsum_init(&acc[c]);
        for (int64_t j = s->nod_off[k]; j < s->nod_off[k + 1]; ++j) {
            int32_t ent = s->nod_ent[j];
            int32_t e = ent >> 2, a = ent & 3;
            if (!s->active[e]) continue;
            const double *f = s->fe + 12 * (int64_t)e + 3 * a;
            for (int c = 0; c < 3; ++c) xsum_add(&acc[c], f[c]);
        }
        for (int c = 0; c < 3; ++c) s->fint[3 * k + c] = xsum_round(&acc[c]);
    }
}

/* probe (tests): the exact sum of n doubles rounded once (R27) */
ORC_API double orc_exact_sum(int64_t n, const double *x) {
    xsum acc;
    xsum_init(&acc);
    for (int64_t i = 0; i < n; ++i) xsum_add(&acc, x[i]);
    return xsum_round(&acc);
}

static void internal_force(orc_sim *s, const double *u) {
    stage_strain(s, u);
    stage_edge(s);
    stage_element_force(s);
    stage_node_force(s);
}

/* ---------------------------------------------------------------- Newmark (beta = 0)
 * PAPER.md:L414-L419:  a_{n+1} = M^-1 (f_ext - f_int(u_{n+1})),
 *                      v_{n+1} = v_n + [(1-gamma) a_n + gamma a_{n+1}] dt,
 *                      u_{n+1} = u_n + v_n dt + 1/2 a_n dt^2.
 * Free dofs only; exposed for the 1-dof pin (tests/test_oracle_newmark.py). */
ORC_API void orc_newmark_free(int64_t n, const double *m, const double *fext, const double *fint,
                              double *v, double *a, double dt, double gamma) {
    const double omg = 1.0 - gamma;
    for (int64_t i = 0; i < n; ++i) {
        double an = (fext[i] - fint[i]) / m[i];
        v[i] = v[i] + dt * (omg * a[i] + gamma * an);
        a[i] = an;
    }
}

ORC_API void orc_predict(int64_t n, double *u, const double *v, const double *a, double dt) {
    const double hdt2 = 0.5 * dt * dt;
    for (int64_t i = 0; i < n; ++i) u[i] = (u[i] + dt * v[i]) + hdt2 * a[i];
}

/* update of node k at t_{n+1} given f_int (stage 5).  frozen (m = 0, R15): v = a = 0. */
static void update_node(orc_sim *s, int64_t k, double t1) {
    const double omg = 1.0 - s->gamma;
    for (int c = 0; c < 3; ++c) {
        int64_t i = 3 * k + c;
        if (s->m[k] == 0.0) { s->v[i] = 0.0; s->a[i] = 0.0; continue; }
        if (dof_prescribed(s, k, c)) {
            double vv, aa; ramp(t1, s->t0, s->dir_v0[i], &vv, &aa);
            s->v[i] = vv; s->a[i] = aa;
            continue;
        }
        double an = (s->fext[i] - s->fint[i]) / s->m[k];
        s->v[i] = s->v[i] + s->dt * (omg * s->a[i] + s->gamma * an);
        s->a[i] = an;
    }
}

/* ---------------------------------------------------------------- criterion
 * Candidate crack patterns of a tet (PAPER.md:L426 + Fig.5 caption L455, Appendix I
 * L1628-L1654; R7): for corner c with other nodes o0<o1<o2, front f = {p,q} among
 * (o0,o1),(o0,o2),(o1,o2), r = the remaining node, candidate k = 6c + 2f + t.
 *   t=0 pattern I (quad through the midpoints of c-p, c-q, q-r, p-r):
 *       m = (X_q - X_p) x (X_r - X_c),  G_I = 1/2 [(sig_{pr}.n)(delta_{cp}.n) + (sig_{qr}.n)(delta_{cq}.n)]
 *       (eq:G-I; G1=mid(c,p), G2=mid(c,q), G3=mid(p,r), G4=mid(q,r)).
 *   t=1 pattern II (corner triangle through the midpoints of c-p, c-q, c-r):
 *       m = (X_q - X_p) x (X_r - X_p),  G_II = 1/2 (sig_{cr}.n)[(delta_{cp}.n) + (delta_{cq}.n)]
 *       (eq:G-II).
 * delta (eq:stretch-delta) of edge (a,b): (u_b-u_a) H(|x_b-x_a|/|X_b-X_a|-1),
 * H evaluated as du.(2dX+du) > 0 (R6); delta.n oriented to be positive on opening:
 * Dd = H ((u_b-u_a).m) sgn((X_b-X_a).m) (R9); sig.n = sig_proj (R8).  With n = m/|m|
 * G = (...)/|m|^2 (both factors scale with 1/|m|).  Areas: quad |m|/4, triangle |m|/8. */
static double sgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }


static void cand_core(double Xn[4][3], double un[4][3], const eig_t *eg /*[6] by local edge*/, uint32_t flags,
                      double *G24, double *A24) {
    int H[6];
    for (int l = 0; l < 6; ++l) {
        double du[3], dX[3], w[3];
        sub3(un[EQ[l]], un[EP[l]], du);
        sub3(Xn[EQ[l]], Xn[EP[l]], dX);
        for (int c = 0; c < 3; ++c) w[c] = 2.0 * dX[c] + du[c];
        H[l] = dot3(du, w) > 0.0;
    }
    for (int c = 0; c < 4; ++c) {
        int o[3], no = 0;
        for (int b = 0; b < 4; ++b) if (b != c) o[no++] = b;
        static const int FP[3] = {0, 0, 1}, FQ[3] = {1, 2, 2}, FR[3] = {2, 1, 0};
        for (int f = 0; f < 3; ++f) {
            int p = o[FP[f]], q = o[FQ[f]], r = o[FR[f]];
            /* Dd(c,x,m) for x in {p,q} */
            for (int t = 0; t < 2; ++t) {
                double m[3], d1[3], d2[3];
                sub3(Xn[q], Xn[p], d1);
                if (t == 0) sub3(Xn[r], Xn[c], d2); else sub3(Xn[r], Xn[p], d2);
                cross3(d1, d2, m);
                double mm = dot3(m, m);
                double Dd[2];
                int ends[2] = {p, q};
                for (int z = 0; z < 2; ++z) {
                    int b = ends[z];
                    int l = local_edge(c, b);
                    if (!H[l]) { Dd[z] = 0.0; continue; }
                    double du[3], dX[3];
                    sub3(un[b], un[c], du); sub3(Xn[b], Xn[c], dX);
                    Dd[z] = dot3(du, m) * sgn(dot3(dX, m));
                }
                double G, area;
                if (t == 0) {
                    const eig_t *e1 = &eg[local_edge(p, r)], *e2 = &eg[local_edge(q, r)];
                    double A1 = sig_proj(e1->lam, e1->vec, e1->k1, e1->deg, m) * Dd[0];
                    double A2 = sig_proj(e2->lam, e2->vec, e2->k1, e2->deg, m) * Dd[1];
                    G = (0.5 * (A1 + A2)) / mm;
                    area = sqrt(mm) / 4.0;
                } else {
                    const eig_t *e6 = &eg[local_edge(c, r)];
                    double Sg = sig_proj(e6->lam, e6->vec, e6->k1, e6->deg, m);
                    G = (0.5 * (Sg * (Dd[0] + Dd[1]))) / mm;
                    area = sqrt(mm) / 8.0;
                }
                if ((flags & ORC_F_FRONT_BOTH_STRETCHED) && !(H[local_edge(c, p)] && H[local_edge(c, q)]))
                    G = 0.0; /* R11 variant: the front is not stretched at both edges */
                int k = 6 * c + 2 * f + t;
                G24[k] = G; A24[k] = area;
            }
        }
    }
}

static void tet_candidates(const orc_sim *s, int64_t e, const double *u, const eig_t *eg /*[6] by local edge*/,
                           double *G24, double *A24) {
    double Xn[4][3], un[4][3];
    for (int a = 0; a < 4; ++a) {
        int64_t n = s->tet[4 * e + a];
        for (int c = 0; c < 3; ++c) { Xn[a][c] = s->X[3 * n + c]; un[a][c] = u[3 * n + c]; }
    }
    cand_core(Xn, un, eg, s->flags, G24, A24);
}

/* the 24 candidates of one tet from its node coordinates X12 [4][3], displacements u12 [4][3] and
 * the stresses s36 [6][6] of its local edges (EP/EQ order); flags: ORC_F_FRONT_BOTH_STRETCHED.
 * Used by the hexahedral oracle for the tets of a remainder prism (R28). */
ORC_API void orc_tet_cand_x(const double *X12, const double *u12, const double *s36, uint32_t flags, double *G24,
                            double *A24) {
    double Xn[4][3], un[4][3];
    for (int a = 0; a < 4; ++a)
        for (int c = 0; c < 3; ++c) { Xn[a][c] = X12[3 * a + c]; un[a][c] = u12[3 * a + c]; }
    eig_t eg[6];
    for (int l = 0; l < 6; ++l) {
        int32_t kk, dg;
        orc_principal(s36 + 6 * l, eg[l].lam, eg[l].vec, &kk, &dg);
        eg[l].k1 = kk; eg[l].deg = dg;
    }
    cand_core(Xn, un, eg, flags, G24, A24);
}

/* select: max G, ties -> larger area, then lower k (R14); split iff G > Gc (R10) */
static void criterion(orc_sim *s, const double *u) {
    eig_t *eig = (eig_t *)s->eig;
    /* the principal decomposition is a function of sigma_s alone: computed once per edge */
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < s->S; ++k)
        orc_principal(s->sig + 6 * k, eig[k].lam, eig[k].vec, &eig[k].k1, &eig[k].deg);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < s->E; ++e) {
        s->flag[e] = 0; s->G[e] = 0.0; s->cand[e] = -1; s->area[e] = 0.0;
        if (!s->active[e]) continue;
        eig_t eg[6];
        for (int l = 0; l < 6; ++l) eg[l] = eig[s->elem_edge[6 * e + l]];
        double G24[24], A24[24];
        tet_candidates(s, e, u, eg, G24, A24);
        int best = 0;
        for (int k = 1; k < 24; ++k)
            if (G24[k] > G24[best] || (G24[k] == G24[best] && A24[k] > A24[best])) best = k;
        s->G[e] = G24[best]; s->cand[e] = best; s->area[e] = A24[best];
        s->flag[e] = G24[best] > s->gc[e];
    }
}

/* split pass (the element is deactivated and excluded from
 * subsequent computations; irreversibility L208).  Ascending e; U_d += Gc_e * area
 * (R: dissipated energy = int_Gamma Gc dGamma); masses of the nodes of
 * split tets are recomputed; m = 0 -> frozen (v = a = 0). */
static int64_t split_pass(orc_sim *s, int64_t step_no) {
    int64_t n = 0;
    for (int64_t e = 0; e < s->E; ++e) {
        if (!s->flag[e]) continue;
        s->active[e] = 0;
        if (s->nrec == s->caprec) {
            s->caprec = s->caprec ? 2 * s->caprec : 1024;
            s->rec = realloc(s->rec, sizeof(orc_record) * s->caprec);
        }
        orc_record r = {step_no, (int32_t)e, s->cand[e], s->G[e], s->area[e]};
        s->rec[s->nrec++] = r;
        s->Ud = s->Ud + s->gc[e] * s->area[e];
        ++n;
    }
    if (!n) return 0;
    for (int64_t e = 0; e < s->E; ++e) {
        if (!s->flag[e]) continue;
        for (int a = 0; a < 4; ++a) {
            int64_t k = s->tet[4 * e + a];
            s->m[k] = node_mass(s, k);
            if (s->m[k] == 0.0)
                for (int c = 0; c < 3; ++c) { s->v[3 * k + c] = 0.0; s->a[3 * k + c] = 0.0; }
        }
    }
    return n;
}

/* ---------------------------------------------------------------- create */
ORC_API orc_sim *orc_create(int64_t n_nodes, const double *X, int64_t n_tets, const int32_t *tets,
                            const uint8_t *tet_state, const double *tet_gc, double E, double nu, double rho,
                            int64_t n_tf, const int32_t *tface, const double *tface_t,
                            int64_t n_vbc, const int32_t *vbc_node, const uint8_t *vbc_mask,
                            const double *vbc_v0, double vbc_t0, double dt, double cfl, double gamma,
                            const double *f_nodal, const double *body, uint32_t flags,
                            char *err, int errlen) {
    orc_sim *s = xcalloc(1, sizeof(orc_sim));
    s->N = n_nodes; s->E = n_tets; s->F = n_tf; s->B = n_vbc;
    s->E_mod = E; s->nu = nu; s->rho = rho; s->gamma = gamma; s->t0 = vbc_t0; s->flags = flags;
    orc_lame(E, nu, &s->lam, &s->mu);
    s->l2m = s->lam + 2.0 * s->mu;
    s->X = xcalloc(3 * n_nodes, sizeof(double)); memcpy(s->X, X, sizeof(double) * 3 * n_nodes);
    s->tet = xcalloc(4 * n_tets, sizeof(int32_t)); memcpy(s->tet, tets, sizeof(int32_t) * 4 * n_tets);
    s->active = xcalloc(n_tets, 1);
    s->gc = xcalloc(n_tets, sizeof(double));
    for (int64_t e = 0; e < n_tets; ++e) {
        s->active[e] = tet_state ? (tet_state[e] != 0) : 1;
        s->gc[e] = tet_gc ? tet_gc[e] : INFINITY;
    }
    /* geometry + validation */
    s->V = xcalloc(n_tets, sizeof(double));
    s->grad = xcalloc(12 * n_tets, sizeof(double));
    for (int64_t e = 0; e < n_tets; ++e) {
        double X4[12];
        for (int a = 0; a < 4; ++a) {
            int32_t n = tets[4 * e + a];
            if (n < 0 || n >= n_nodes) { snprintf(err, errlen, "tet %lld node out of range", (long long)e); orc_destroy(s); return NULL; }
            for (int c = 0; c < 3; ++c) X4[3 * a + c] = X[3 * (int64_t)n + c];
        }
        orc_tet_geometry(X4, s->V + e, s->grad + 12 * e);
        if (!(s->V[e] > 0.0)) { snprintf(err, errlen, "tet %lld non-positive volume", (long long)e); orc_destroy(s); return NULL; }
    }
    /* unique edges: sorted (min,max) pairs */
    uint64_t *keys = xcalloc(6 * n_tets, sizeof(uint64_t));
    for (int64_t e = 0; e < n_tets; ++e)
        for (int l = 0; l < 6; ++l) {
            uint64_t i = (uint32_t)tets[4 * e + EP[l]], j = (uint32_t)tets[4 * e + EQ[l]];
            uint64_t lo = i < j ? i : j, hi = i < j ? j : i;
            keys[6 * e + l] = lo << 32 | hi;
        }
    uint64_t *uk = xcalloc(6 * n_tets, sizeof(uint64_t));
    memcpy(uk, keys, sizeof(uint64_t) * 6 * n_tets);
    qsort(uk, 6 * n_tets, sizeof(uint64_t), cmp_u64);
    int64_t S = 0;
    for (int64_t i = 0; i < 6 * n_tets; ++i)
        if (i == 0 || uk[i] != uk[i - 1]) uk[S++] = uk[i];
    s->S = S;
    s->edge_nodes = xcalloc(2 * S, sizeof(int32_t));
    for (int64_t k = 0; k < S; ++k) { s->edge_nodes[2 * k] = (int32_t)(uk[k] >> 32); s->edge_nodes[2 * k + 1] = (int32_t)(uk[k] & 0xffffffffu); }
    s->elem_edge = xcalloc(6 * n_tets, sizeof(int32_t));
    s->inc_off = xcalloc(S + 1, sizeof(int64_t));
    for (int64_t i = 0; i < 6 * n_tets; ++i) {
        int64_t k = find_edge(uk, S, keys[i]);
        s->elem_edge[i] = (int32_t)k;
        s->inc_off[k + 1]++;
    }
    for (int64_t k = 0; k < S; ++k) s->inc_off[k + 1] += s->inc_off[k];
    s->inc = xcalloc(6 * n_tets, sizeof(int32_t));
    int64_t *fill = xcalloc(S, sizeof(int64_t));
    for (int64_t e = 0; e < n_tets; ++e)
        for (int l = 0; l < 6; ++l) {
            int64_t k = s->elem_edge[6 * e + l];
            for (int64_t j = s->inc_off[k]; j < s->inc_off[k] + fill[k]; ++j)
                if (s->inc[j] == e) { snprintf(err, errlen, "tet %lld repeats a node", (long long)e); free(fill); free(keys); free(uk); orc_destroy(s); return NULL; }
            s->inc[s->inc_off[k] + fill[k]++] = (int32_t)e;
        }
    free(fill); free(keys); free(uk);
    /* duplicate tets: same sorted node set */
    {
        uint64_t *tk = xcalloc(2 * n_tets, sizeof(uint64_t));
        for (int64_t e = 0; e < n_tets; ++e) {
            int32_t v[4]; memcpy(v, tets + 4 * e, sizeof v);
            for (int i = 0; i < 4; ++i) for (int j = i + 1; j < 4; ++j) if (v[j] < v[i]) { int32_t t = v[i]; v[i] = v[j]; v[j] = t; }
            tk[2 * e] = ((uint64_t)(uint32_t)v[0] << 32) | (uint32_t)v[1];
            tk[2 * e + 1] = ((uint64_t)(uint32_t)v[2] << 32) | (uint32_t)v[3];
        }
        /* edges-based check: two tets sharing all 6 edges -> sort pairs */
        int dup = 0;
        for (int64_t k = 0; k < S && !dup; ++k)
            for (int64_t i = s->inc_off[k]; i < s->inc_off[k + 1] && !dup; ++i)
                for (int64_t j = i + 1; j < s->inc_off[k + 1]; ++j) {
                    int32_t a = s->inc[i], b = s->inc[j];
                    if (tk[2 * a] == tk[2 * b] && tk[2 * a + 1] == tk[2 * b + 1]) { dup = 1; break; }
                }
        free(tk);
        if (dup) { snprintf(err, errlen, "duplicate tets"); orc_destroy(s); return NULL; }
    }
    /* node incidence */
    s->nod_off = xcalloc(n_nodes + 1, sizeof(int64_t));
    for (int64_t e = 0; e < n_tets; ++e) for (int a = 0; a < 4; ++a) s->nod_off[tets[4 * e + a] + 1]++;
    for (int64_t k = 0; k < n_nodes; ++k) s->nod_off[k + 1] += s->nod_off[k];
    s->nod_ent = xcalloc(4 * n_tets, sizeof(int32_t));
    fill = xcalloc(n_nodes, sizeof(int64_t));
    for (int64_t e = 0; e < n_tets; ++e)
        for (int a = 0; a < 4; ++a) { int64_t k = tets[4 * e + a]; s->nod_ent[s->nod_off[k] + fill[k]++] = (int32_t)(4 * e + a); }
    free(fill);
    /* mass */
    s->m = xcalloc(n_nodes, sizeof(double));
    for (int64_t k = 0; k < n_nodes; ++k) s->m[k] = node_mass(s, k);
    /* external force (f_ext = A_e [N^e] b A_e + A_e [N^e] t ell_e), constant
     * from t = 0 like the tractions:
     *  1. body force b (N/m^3, uniform): consistent lumping of the constant-b integral over each
     *     active tet, f_k += b (V_e / 4) per incidence, ascending e (R4b);
     *  2. traction t on triangle (x0,x1,x2), A = |(x1-x0)x(x2-x0)|/2, f_k += t (A/3) per node
     *     (R4), faces in the given order;
     *  3. nodal point forces f_nodal[k] added last (SURVEY.md §8(b) cem_load_in.f_ext). */
    s->fext = xcalloc(3 * n_nodes, sizeof(double));
    if (body && (body[0] != 0.0 || body[1] != 0.0 || body[2] != 0.0))
        for (int64_t k = 0; k < n_nodes; ++k)
            for (int64_t j = s->nod_off[k]; j < s->nod_off[k + 1]; ++j) {
                int32_t e = s->nod_ent[j] >> 2;
                if (!s->active[e]) continue;
                double w = s->V[e] / 4.0;
                for (int c = 0; c < 3; ++c) s->fext[3 * k + c] = s->fext[3 * k + c] + body[c] * w;
            }
    for (int64_t f = 0; f < n_tf; ++f) {
        const int32_t *tri = tface + 3 * f;
        double d1[3], d2[3], cr[3];
        sub3(X + 3 * (int64_t)tri[1], X + 3 * (int64_t)tri[0], d1);
        sub3(X + 3 * (int64_t)tri[2], X + 3 * (int64_t)tri[0], d2);
        cross3(d1, d2, cr);
        double A = 0.5 * sqrt(dot3(cr, cr));
        double w = A / 3.0;
        for (int i = 0; i < 3; ++i)
            for (int c = 0; c < 3; ++c) s->fext[3 * (int64_t)tri[i] + c] = s->fext[3 * (int64_t)tri[i] + c] + tface_t[3 * f + c] * w;
    }
    if (f_nodal)
        for (int64_t i = 0; i < 3 * n_nodes; ++i) s->fext[i] = s->fext[i] + f_nodal[i];
    /* Dirichlet */
    s->dir = xcalloc(n_nodes, 1);
    s->dir_v0 = xcalloc(3 * n_nodes, sizeof(double));
    for (int64_t b = 0; b < n_vbc; ++b) {
        int64_t k = vbc_node[b];
        s->dir[k] |= vbc_mask[b];
        for (int c = 0; c < 3; ++c) if (vbc_mask[b] >> c & 1) s->dir_v0[3 * k + c] = vbc_v0[3 * b + c];
    }
    /* time step (R12): dt = cfl * min_{active e} (3 V_e / max face area_e) / c_d */
    if (dt <= 0.0) {
        double cd = sqrt(s->l2m / rho);
        double altmin = INFINITY;
        static const int FA[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
        for (int64_t e = 0; e < n_tets; ++e) {
            if (!s->active[e]) continue;
            double amax = 0.0;
            for (int f = 0; f < 4; ++f) {
                const double *x0 = X + 3 * (int64_t)tets[4 * e + FA[f][0]];
                const double *x1 = X + 3 * (int64_t)tets[4 * e + FA[f][1]];
                const double *x2 = X + 3 * (int64_t)tets[4 * e + FA[f][2]];
                double d1[3], d2[3], cr[3];
                sub3(x1, x0, d1); sub3(x2, x0, d2); cross3(d1, d2, cr);
                double A = 0.5 * sqrt(dot3(cr, cr));
                if (A > amax) amax = A;
            }
            double alt = 3.0 * s->V[e] / amax;
            if (alt < altmin) altmin = alt;
        }
        dt = (cfl * altmin) / cd;
    }
    s->dt = dt;
    /* scratch + state */
    s->u = xcalloc(3 * n_nodes, sizeof(double)); s->v = xcalloc(3 * n_nodes, sizeof(double)); s->a = xcalloc(3 * n_nodes, sizeof(double));
    s->tau = xcalloc(6 * n_tets, sizeof(double)); s->sig = xcalloc(6 * S, sizeof(double)); s->vhat = xcalloc(S, sizeof(double));
    s->fe = xcalloc(12 * n_tets, sizeof(double)); s->fint = xcalloc(3 * n_nodes, sizeof(double));
    s->eig = xcalloc(S, sizeof(eig_t));
    s->G = xcalloc(n_tets, sizeof(double)); s->cand = xcalloc(n_tets, sizeof(int32_t)); s->area = xcalloc(n_tets, sizeof(double));
    s->flag = xcalloc(n_tets, 1);
    /* initial state (R17): u0 = v0 = 0; a0 = M^-1 (f_ext - f_int(0)) on free dofs,
     * prescribed dofs v = vbar(0), a = vbar'(0); frozen dofs 0 */
    internal_force(s, s->u);
    for (int64_t k = 0; k < n_nodes; ++k) {
        for (int c = 0; c < 3; ++c) {
            int64_t i = 3 * k + c;
            if (s->m[k] == 0.0) { s->v[i] = 0.0; s->a[i] = 0.0; continue; }
            if (dof_prescribed(s, k, c)) { double vv, aa; ramp(0.0, s->t0, s->dir_v0[i], &vv, &aa); s->v[i] = vv; s->a[i] = aa; continue; }
            s->a[i] = (s->fext[i] - s->fint[i]) / s->m[k];
        }
    }
    s->step = 0; s->Ud = 0.0;
    /* support force of the prescribed dofs at t = 0 (energy ledger) */
    s->rprev = xcalloc(3 * n_nodes, sizeof(double)); s->uold = xcalloc(3 * n_nodes, sizeof(double));
    s->Wr = 0.0; s->has_dir = 0;
    for (int64_t k = 0; k < n_nodes; ++k)
        for (int c = 0; c < 3; ++c)
            if (dof_prescribed(s, k, c)) {
                int64_t i = 3 * k + c;
                s->has_dir = 1;
                s->rprev[i] = s->m[k] * s->a[i] - (s->fext[i] - s->fint[i]);
            }
    return s;
}

/* ---------------------------------------------------------------- energy ledger (N1)
 * Support force of a prescribed dof at t_{n+1}: R = m a_{n+1} - (f_ext - f_int(u_{n+1}))
 * (the force the constraint applies, PAPER.md:L416 solved for the missing load); its work
 * over the step by the trapezoidal rule, W_R += 1/2 (R_n + R_{n+1}) (u_{n+1} - u_n)
 * (SPEC.md update_energy_ledger: "reaction work on Dirichlet dofs"; R22).
 * Sequential over k ascending, c = x, y, z. */
static void reaction_work(orc_sim *s) {
    for (int64_t k = 0; k < s->N; ++k)
        for (int c = 0; c < 3; ++c) {
            if (!dof_prescribed(s, k, c)) continue;
            const int64_t i = 3 * k + c;
            const double R = s->m[k] * s->a[i] - (s->fext[i] - s->fint[i]);
            s->Wr = s->Wr + 0.5 * (s->rprev[i] + R) * (s->u[i] - s->uold[i]);
            s->rprev[i] = R;
        }
}

/* ---------------------------------------------------------------- run
 * One explicit step n -> n+1: predictor u_{n+1}; f_int(u_{n+1});
 * a_{n+1}, v_{n+1} (+ BC, frozen); criterion on (u_{n+1}, sigma(u_{n+1})) every
 * crack_every steps (0 = never); split pass.  Returns 0, or 1 on a non-finite value. */
ORC_API int orc_run(orc_sim *s, int64_t nsteps, int32_t crack_every) {
    const double hdt2 = 0.5 * s->dt * s->dt;
    for (int64_t it = 0; it < nsteps; ++it) {
        const int64_t n1 = s->step + 1;
        const double t1 = (double)n1 * s->dt;
        if (s->has_dir) memcpy(s->uold, s->u, sizeof(double) * 3 * s->N);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < 3 * s->N; ++i) s->u[i] = (s->u[i] + s->dt * s->v[i]) + hdt2 * s->a[i];
        internal_force(s, s->u);
        int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
        for (int64_t k = 0; k < s->N; ++k) {
            update_node(s, k, t1);
            for (int c = 0; c < 3; ++c) {
                int64_t i = 3 * k + c;
                if (!isfinite(s->u[i]) || !isfinite(s->v[i]) || !isfinite(s->a[i])) bad = 1;
            }
        }
        if (s->has_dir) reaction_work(s);
        if (crack_every > 0 && n1 % crack_every == 0) {
            criterion(s, s->u);
            split_pass(s, n1);
        }
        s->step = n1;
        if (bad) { s->nonfinite = 1; return 1; }
    }
    return 0;
}

/* ---------------------------------------------------------------- probes / getters */
ORC_API int64_t orc_n_edges(const orc_sim *s) { return s->S; }
ORC_API double orc_dt(const orc_sim *s) { return s->dt; }
ORC_API int64_t orc_step_count(const orc_sim *s) { return s->step; }
ORC_API double orc_dissipated(const orc_sim *s) { return s->Ud; }
ORC_API int64_t orc_n_records(const orc_sim *s) { return s->nrec; }
ORC_API void orc_lame_of(const orc_sim *s, double *lam, double *mu) { *lam = s->lam; *mu = s->mu; }

ORC_API void orc_get_state(const orc_sim *s, double *u, double *v, double *a, uint8_t *state, double *m) {
    if (u) memcpy(u, s->u, sizeof(double) * 3 * s->N);
    if (v) memcpy(v, s->v, sizeof(double) * 3 * s->N);
    if (a) memcpy(a, s->a, sizeof(double) * 3 * s->N);
    if (state) memcpy(state, s->active, s->E);
    if (m) memcpy(m, s->m, sizeof(double) * s->N);
}

ORC_API void orc_get_records(const orc_sim *s, int64_t *step, int32_t *elem, int32_t *cand, double *G, double *area) {
    for (int64_t i = 0; i < s->nrec; ++i) {
        step[i] = s->rec[i].step; elem[i] = s->rec[i].elem; cand[i] = s->rec[i].cand;
        G[i] = s->rec[i].G; area[i] = s->rec[i].area;
    }
}

ORC_API void orc_get_fext(const orc_sim *s, double *f) { memcpy(f, s->fext, sizeof(double) * 3 * s->N); }
ORC_API void orc_get_geometry(const orc_sim *s, double *V, double *grad) {
    memcpy(V, s->V, sizeof(double) * s->E); memcpy(grad, s->grad, sizeof(double) * 12 * s->E);
}
ORC_API void orc_get_edges(const orc_sim *s, int32_t *edge_nodes, int64_t *inc_count) {
    memcpy(edge_nodes, s->edge_nodes, sizeof(int32_t) * 2 * s->S);
    if (inc_count) for (int64_t k = 0; k < s->S; ++k) inc_count[k] = s->inc_off[k + 1] - s->inc_off[k];
}

/* overwrite the kinematic state (tests: arbitrary u for force/criterion probes) */
ORC_API void orc_set_state(orc_sim *s, const double *u, const double *v, const double *a) {
    if (u) memcpy(s->u, u, sizeof(double) * 3 * s->N);
    if (v) memcpy(s->v, v, sizeof(double) * 3 * s->N);
    if (a) memcpy(s->a, a, sizeof(double) * 3 * s->N);
}

/* overwrite the active flags (tests: halo exchange of the multi-rank decomposition) */
ORC_API void orc_set_active(orc_sim *s, const uint8_t *state) {
    for (int64_t e = 0; e < s->E; ++e) s->active[e] = state[e] != 0;
}

ORC_API void orc_edge_stress(orc_sim *s, const double *u, double *sigma, double *vhat) {
    stage_strain(s, u); stage_edge(s);
    if (sigma) memcpy(sigma, s->sig, sizeof(double) * 6 * s->S);
    if (vhat) memcpy(vhat, s->vhat, sizeof(double) * s->S);
}

ORC_API void orc_internal_force(orc_sim *s, const double *u, double *f) {
    internal_force(s, u);
    memcpy(f, s->fint, sizeof(double) * 3 * s->N);
}

/* element contributions f_{e,a} [E][4][3] of the last internal_force evaluation (tests) */
ORC_API void orc_element_forces(const orc_sim *s, double *fe) { memcpy(fe, s->fe, sizeof(double) * 12 * s->E); }

/* strain energy U = sum_s psi(eps~_s) V_s, V_s = Vhat_s / 6, psi = 1/2 lam (tr eps)^2 + mu eps:eps
 * (PAPER.md:L197-L202 with R1; eps:eps = e11^2+e22^2+e33^2 + (g12^2+g23^2+g13^2)/2) */
ORC_API double orc_strain_energy(orc_sim *s, const double *u) {
    stage_strain(s, u); stage_edge(s);
    double U = 0.0;
    for (int64_t k = 0; k < s->S; ++k) {
        if (s->vhat[k] == 0.0) continue;
        double T[6] = {0, 0, 0, 0, 0, 0};
        for (int64_t j = s->inc_off[k]; j < s->inc_off[k + 1]; ++j) {
            int32_t e = s->inc[j];
            if (!s->active[e]) continue;
            for (int i = 0; i < 6; ++i) T[i] = T[i] + s->tau[6 * (int64_t)e + i];
        }
        double inv = 1.0 / s->vhat[k];
        double e11 = T[0] * inv, e22 = T[1] * inv, e33 = T[2] * inv, g12 = T[3] * inv, g23 = T[4] * inv, g13 = T[5] * inv;
        double tr = e11 + e22 + e33;
        double ee = e11 * e11 + e22 * e22 + e33 * e33 + 0.5 * (g12 * g12 + g23 * g23 + g13 * g13);
        double psi = 0.5 * s->lam * tr * tr + s->mu * ee;
        U += psi * (s->vhat[k] / 6.0);
    }
    return U;
}

/* energy ledger at the current step n (SPEC.md update_energy_ledger):
 *   out[0] kinetic  T = 1/2 sum_k m_k (v_k . v_k)          (lumped mass)
 *   out[1] strain   U = sum_s psi(eps~_s) Vhat_s / 6       (orc_strain_energy)
 *   out[2] external W = sum_k f_ext,k . u_k                (constant tractions from t = 0 and
 *                                                           u_0 = 0: the telescoped f.du sum, R22)
 *   out[3] reaction W_R (trapezoidal support-force work, reaction_work)
 *   out[4] dissipated U_d = sum Gc_e A_e over the splits   (R-U_d)
 * sums sequential over k (then x, y, z) ascending. */
ORC_API void orc_energy(orc_sim *s, double *out) {
    double T = 0.0, W = 0.0;
    for (int64_t k = 0; k < s->N; ++k) {
        const double *v = s->v + 3 * k, *u = s->u + 3 * k, *f = s->fext + 3 * k;
        T = T + s->m[k] * ((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
        W = W + ((f[0] * u[0] + f[1] * u[1]) + f[2] * u[2]);
    }
    out[0] = 0.5 * T;
    out[1] = orc_strain_energy(s, s->u);
    out[2] = W;
    out[3] = s->Wr;
    out[4] = s->Ud;
}

/* criterion on an arbitrary u (uses sigma(u)); outputs per tet G_e, candidate, area, flag */
ORC_API void orc_criterion(orc_sim *s, const double *u, double *G, int32_t *cand, double *area, uint8_t *flag) {
    stage_strain(s, u); stage_edge(s);
    criterion(s, u);
    if (G) memcpy(G, s->G, sizeof(double) * s->E);
    if (cand) memcpy(cand, s->cand, sizeof(int32_t) * s->E);
    if (area) memcpy(area, s->area, sizeof(double) * s->E);
    if (flag) memcpy(flag, s->flag, s->E);
}

/* all 24 candidates of tet e for an arbitrary u */
ORC_API void orc_candidates(orc_sim *s, const double *u, int64_t e, double *G24, double *A24) {
    stage_strain(s, u); stage_edge(s);
    eig_t eg[6];
    for (int l = 0; l < 6; ++l) {
        int32_t kk, dg;
        orc_principal(s->sig + 6 * (int64_t)s->elem_edge[6 * e + l], eg[l].lam, eg[l].vec, &kk, &dg);
        eg[l].k1 = kk; eg[l].deg = dg;
    }
    tet_candidates(s, e, u, eg, G24, A24);
}

/* bench.py's single-thread baseline: OpenMP threads of the following calls (results do not
 * depend on it: OpenMP only splits loops over independent outputs) */
ORC_API void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

ORC_API int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
