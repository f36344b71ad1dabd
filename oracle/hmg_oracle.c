/*
 * hmg_oracle.c -- plain, slow, obviously-correct CPU oracle for the pressure
 * Helmholtz solve of arXiv:1605.00492 (Mitchell & Mueller, "High level
 * implementation of geometric multigrid solvers for finite element problems:
 * applications in atmospheric modelling").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this code.  The
 * product path (paper_1605_00492_b200/) never links, imports or calls it, and
 * it shares no source with the CUDA path.
 *
 * Arithmetic: IEEE fp64, round-to-nearest, compiled with -O2
 * -ffp-contract=off (no FMA contraction, no -ffast-math).  Every expression is
 * written in the canonical left-to-right order of DESIGN.md "Readings" R1-R14
 * (= SURVEY.md section 8(c).2, O1-O10).  OpenMP is used only over independent
 * columns; dot products are plain sequential sums in index order, so results
 * do not depend on the thread count.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (the paper's LaTeX).
 *
 * Parity status of each function:
 *   mesh / geometry   pinned: counts, Euler characteristic, ref-0 closed forms
 *   assembly / apply  pinned: symmetry, row-sum identity, ref-0 spectrum
 *   thomas            pinned: dense LU, exact rational solves
 *   sweep             pinned: fixed point, w2=0 closed form, exact-solve case
 *   restrict/prolong  pinned: adjointness, RP = 4I, constants
 *   vcycle            pinned: dense two-grid matrix form, symmetry, linearity
 *   pcg               pinned: scipy.sparse.linalg.cg iteration count
 *   mixed system      pinned (NEXT-4, readings R15-R20): divergence theorem
 *   (Eq. 5, Eq. 6,    and adjointness of D, lumped Schur complement == the
 *    GMRES(30))       pinned apply above, RT0 exactness on constant fields,
 *                     P1 hat integrals, mass SPD, GMRES residual minimality
 *                     against dense least squares, Eq. 6 factorisation
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORA_OK 0
#define ORA_ERR_ARG 1
#define ORA_ERR_SINGULAR 4
#define ORA_ERR_NOT_CONVERGED 5
#define ORA_ERR_OOM 6

static char ora_msg[512];
const char* ora_last_error(void) { return ora_msg; }

/* ------------------------------------------------------------------ */
/* O1  Mesh: icosahedron refined by edge midpoints (P:234-235,        */
/*     P:282-297 "MeshHierarchy(UnitIcosahedralSphereMesh(r0), n)"). */
/* ------------------------------------------------------------------ */

typedef struct {
    int64_t nv, nf;
    double* v;      /* [nv][3] unit-sphere vertices */
    int32_t* f;     /* [nf][3] vertex ids, counter-clockwise from outside */
    int32_t* nbr;   /* [nf][3] cell across edge (v_j, v_{j+1 mod 3}) */
} ora_mesh;

/* v <- v / sqrt((x*x + y*y) + z*z), componentwise division (reading R1). */
static void normalise(double* v) {
    double r = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    v[0] = v[0] / r;
    v[1] = v[1] / r;
    v[2] = v[2] / r;
}

/* Base icosahedron: 12 vertices, 20 faces, orientation rule of reading R1. */
static int base_mesh(ora_mesh* m) {
    const double phi = (1.0 + sqrt(5.0)) / 2.0;
    double raw[12][3];
    int i = 0;
    for (int s1 = -1; s1 <= 1; s1 += 2)
        for (int s2 = -1; s2 <= 1; s2 += 2) {
            raw[i][0] = 0.0; raw[i][1] = (double)s1; raw[i][2] = s2 * phi; i++;
        }
    for (int s1 = -1; s1 <= 1; s1 += 2)
        for (int s2 = -1; s2 <= 1; s2 += 2) {
            raw[i][0] = (double)s1; raw[i][1] = s2 * phi; raw[i][2] = 0.0; i++;
        }
    for (int s1 = -1; s1 <= 1; s1 += 2)
        for (int s2 = -1; s2 <= 1; s2 += 2) {
            raw[i][0] = s2 * phi; raw[i][1] = 0.0; raw[i][2] = (double)s1; i++;
        }
    m->nv = 12;
    m->nf = 20;
    m->v = (double*)malloc(sizeof(double) * 36);
    m->f = (int32_t*)malloc(sizeof(int32_t) * 60);
    m->nbr = NULL;
    if (!m->v || !m->f) return ORA_ERR_OOM;
    /* adjacency: unnormalised distance 2 (squared 4); other distances are >= 2*phi */
    int adj[12][12];
    for (int a = 0; a < 12; a++)
        for (int b = 0; b < 12; b++) {
            double dx = raw[a][0] - raw[b][0], dy = raw[a][1] - raw[b][1], dz = raw[a][2] - raw[b][2];
            double d2 = dx * dx + dy * dy + dz * dz;
            adj[a][b] = (a != b) && fabs(d2 - 4.0) < 1e-9;
        }
    int nf = 0;
    for (int a = 0; a < 12; a++)
        for (int b = a + 1; b < 12; b++)
            for (int c = b + 1; c < 12; c++) {
                if (!(adj[a][b] && adj[b][c] && adj[a][c])) continue;
                double e1[3], e2[3], cr[3], s[3];
                for (int d = 0; d < 3; d++) {
                    e1[d] = raw[b][d] - raw[a][d];
                    e2[d] = raw[c][d] - raw[a][d];
                    s[d] = raw[a][d] + raw[b][d] + raw[c][d];
                }
                cr[0] = e1[1] * e2[2] - e1[2] * e2[1];
                cr[1] = e1[2] * e2[0] - e1[0] * e2[2];
                cr[2] = e1[0] * e2[1] - e1[1] * e2[0];
                double orient = cr[0] * s[0] + cr[1] * s[1] + cr[2] * s[2];
                m->f[3 * nf + 0] = a;
                if (orient > 0) { m->f[3 * nf + 1] = b; m->f[3 * nf + 2] = c; }
                else            { m->f[3 * nf + 1] = c; m->f[3 * nf + 2] = b; }
                nf++;
            }
    if (nf != 20) { snprintf(ora_msg, sizeof ora_msg, "base mesh: %d faces", nf); return ORA_ERR_ARG; }
    for (int a = 0; a < 12; a++) {
        for (int d = 0; d < 3; d++) m->v[3 * a + d] = raw[a][d];
        normalise(&m->v[3 * a]);
    }
    return ORA_OK;
}

/* Edge -> midpoint lookup: every vertex of a triangulated sphere has at most
 * 6 neighbours in this hierarchy (5 at the 12 original vertices). */
typedef struct { int32_t other[8]; int32_t mid[8]; int cnt; } edge_slot;

static int32_t get_mid(edge_slot* es, ora_mesh* fine, int64_t* nv, const double* pv, int32_t a, int32_t b) {
    edge_slot* s = &es[a];
    for (int i = 0; i < s->cnt; i++)
        if (s->other[i] == b) return s->mid[i];
    int32_t id = (int32_t)(*nv)++;
    /* m = (va + vb) * 0.5, then normalised (reading R1) */
    for (int d = 0; d < 3; d++) fine->v[3 * id + d] = (pv[3 * a + d] + pv[3 * b + d]) * 0.5;
    normalise(&fine->v[3 * id]);
    s->other[s->cnt] = b; s->mid[s->cnt] = id; s->cnt++;
    edge_slot* t = &es[b];
    t->other[t->cnt] = a; t->mid[t->cnt] = id; t->cnt++;
    return id;
}

/* Refinement (reading R1): parent p=(a,b,c) -> children
 *   4p+0=(a,m_ab,m_ca) 4p+1=(m_ab,b,m_bc) 4p+2=(m_ca,m_bc,c) 4p+3=(m_ab,m_bc,m_ca). */
static int refine(const ora_mesh* c, ora_mesh* f) {
    int64_t nv_max = c->nv + (c->nf * 3) / 2;
    f->nf = c->nf * 4;
    f->v = (double*)malloc(sizeof(double) * 3 * nv_max);
    f->f = (int32_t*)malloc(sizeof(int32_t) * 3 * f->nf);
    f->nbr = NULL;
    edge_slot* es = (edge_slot*)calloc((size_t)c->nv, sizeof(edge_slot));
    if (!f->v || !f->f || !es) { free(es); return ORA_ERR_OOM; }
    memcpy(f->v, c->v, sizeof(double) * 3 * c->nv);
    int64_t nv = c->nv;
    for (int64_t p = 0; p < c->nf; p++) {
        int32_t a = c->f[3 * p], b = c->f[3 * p + 1], cc = c->f[3 * p + 2];
        int32_t mab = get_mid(es, f, &nv, c->v, a, b);
        int32_t mbc = get_mid(es, f, &nv, c->v, b, cc);
        int32_t mca = get_mid(es, f, &nv, c->v, cc, a);
        int32_t* ch = &f->f[12 * p];
        ch[0] = a;   ch[1] = mab; ch[2] = mca;
        ch[3] = mab; ch[4] = b;   ch[5] = mbc;
        ch[6] = mca; ch[7] = mbc; ch[8] = cc;
        ch[9] = mab; ch[10] = mbc; ch[11] = mca;
    }
    free(es);
    f->nv = nv;
    return ORA_OK;
}

/* Neighbours: N[c][j] = the cell across edge (v_j, v_{(j+1)%3}).  Plain
 * approach: list all 3n half-edges keyed by (min, max) vertex id, sort, pair. */
typedef struct { int32_t lo, hi; int32_t cell; int32_t slot; } half_edge;

static int he_cmp(const void* A, const void* B) {
    const half_edge* a = (const half_edge*)A;
    const half_edge* b = (const half_edge*)B;
    if (a->lo != b->lo) return a->lo < b->lo ? -1 : 1;
    if (a->hi != b->hi) return a->hi < b->hi ? -1 : 1;
    return a->cell < b->cell ? -1 : (a->cell > b->cell);
}

static int build_neighbours(ora_mesh* m) {
    int64_t nh = 3 * m->nf;
    half_edge* he = (half_edge*)malloc(sizeof(half_edge) * nh);
    m->nbr = (int32_t*)malloc(sizeof(int32_t) * 3 * m->nf);
    if (!he || !m->nbr) { free(he); return ORA_ERR_OOM; }
    for (int64_t c = 0; c < m->nf; c++)
        for (int j = 0; j < 3; j++) {
            int32_t a = m->f[3 * c + j], b = m->f[3 * c + (j + 1) % 3];
            half_edge* h = &he[3 * c + j];
            h->lo = a < b ? a : b;
            h->hi = a < b ? b : a;
            h->cell = (int32_t)c;
            h->slot = j;
        }
    qsort(he, (size_t)nh, sizeof(half_edge), he_cmp);
    for (int64_t i = 0; i < nh; i += 2) {
        if (i + 1 >= nh || he[i].lo != he[i + 1].lo || he[i].hi != he[i + 1].hi ||
            (i + 2 < nh && he[i + 2].lo == he[i].lo && he[i + 2].hi == he[i].hi)) {
            free(he);
            snprintf(ora_msg, sizeof ora_msg, "mesh is not a closed 2-manifold");
            return ORA_ERR_ARG;
        }
        m->nbr[3 * he[i].cell + he[i].slot] = he[i + 1].cell;
        m->nbr[3 * he[i + 1].cell + he[i + 1].slot] = he[i].cell;
    }
    free(he);
    return ORA_OK;
}

/* ------------------------------------------------------------------ */
/* Hierarchy: per level geometry (O2), coefficients (O3), bands (O4).  */
/* ------------------------------------------------------------------ */

typedef struct {
    int ref;
    int64_t n;          /* cells at this level = 20 * 4^ref */
    ora_mesh mesh;
    double* area;       /* [n] */
    double* len;        /* [n][3] */
    double* cd;         /* [n][3] */
    double* lam;        /* [nz][n] */
    double* D;          /* [nz][n] */
    double* U;          /* [nz][n]  U[k] couples k and k+1; U[nz-1] = 0 */
    double* H;          /* [3][nz][n] */
    /* V-cycle work vectors, [nz][n] each */
    double *u, *b, *r, *t;
} ora_level;

typedef struct ora_h {
    int fine_ref, coarsest_ref, nz;
    double thickness, w2, dz;
    double sn;          /* 1 + omega_N^2 (reading R24; 1 without buoyancy) */
    ora_level lev[16];  /* indexed by ref */
} ora_h;

static void* zalloc(size_t bytes) { return calloc(bytes, 1); }

/* O2 geometry (reading R2): Euclidean quantities on the flat chordal
 * triangles; cross product with the usual component formulas. */
static void geometry(ora_level* L) {
    const double* V = L->mesh.v;
    const int32_t* F = L->mesh.f;
    int64_t n = L->n;
    double* cen = (double*)malloc(sizeof(double) * 3 * n);
    for (int64_t c = 0; c < n; c++) {
        const double* v0 = &V[3 * F[3 * c]];
        const double* v1 = &V[3 * F[3 * c + 1]];
        const double* v2 = &V[3 * F[3 * c + 2]];
        double e1x = v1[0] - v0[0], e1y = v1[1] - v0[1], e1z = v1[2] - v0[2];
        double e2x = v2[0] - v0[0], e2y = v2[1] - v0[1], e2z = v2[2] - v0[2];
        double cx = e1y * e2z - e1z * e2y;
        double cy = e1z * e2x - e1x * e2z;
        double cz = e1x * e2y - e1y * e2x;
        L->area[c] = 0.5 * sqrt((cx * cx + cy * cy) + cz * cz);
        for (int d = 0; d < 3; d++) cen[3 * c + d] = ((v0[d] + v1[d]) + v2[d]) / 3.0;
        const double* vs[3] = {v0, v1, v2};
        for (int j = 0; j < 3; j++) {
            const double* p = vs[j];
            const double* q = vs[(j + 1) % 3];
            double dx = q[0] - p[0], dy = q[1] - p[1], dzz = q[2] - p[2];
            L->len[3 * c + j] = sqrt((dx * dx + dy * dy) + dzz * dzz);
        }
    }
    for (int64_t c = 0; c < n; c++)
        for (int j = 0; j < 3; j++) {
            int32_t o = L->mesh.nbr[3 * c + j];
            double dx = cen[3 * c] - cen[3 * o];
            double dy = cen[3 * c + 1] - cen[3 * o + 1];
            double dzz = cen[3 * c + 2] - cen[3 * o + 2];
            L->cd[3 * c + j] = sqrt((dx * dx + dy * dy) + dzz * dzz);
        }
    free(cen);
}

/* O4 assembly (reading R4; Eq. 8 at P:598-606 with two-point lumped
 * couplings): vertical Vc = (((w2*area)*lamf)/dz)/(1 + omega_N^2) (the
 * buoyancy factor of Eq. 8, reading R24; exactly ((w2*area)*lamf)/dz for
 * omega_N = 0), horizontal
 * Hc_j = (((w2*len_j)*dz)*lamf)/cd_j, face factor lamf = 0.5*(lam_a+lam_b)
 * (reading R3), diagonal = vol + couplings, u.n = 0 at top/bottom. */
static void assemble(ora_h* h, ora_level* L) {
    int nz = h->nz;
    int64_t n = L->n;
    double w2 = h->w2, dz = h->dz;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; c++) {
        double vol = L->area[c] * dz;
        for (int k = 0; k < nz; k++) {
            double lam_kc = L->lam[(int64_t)k * n + c];
            double vc_dn = 0.0, vc_up = 0.0;
            if (k > 0) {
                double lamf = 0.5 * (L->lam[(int64_t)(k - 1) * n + c] + lam_kc);
                vc_dn = (((w2 * L->area[c]) * lamf) / dz) / h->sn;
            }
            if (k < nz - 1) {
                double lamf = 0.5 * (lam_kc + L->lam[(int64_t)(k + 1) * n + c]);
                vc_up = (((w2 * L->area[c]) * lamf) / dz) / h->sn;
            }
            double hc[3];
            for (int j = 0; j < 3; j++) {
                int32_t o = L->mesh.nbr[3 * c + j];
                double lamf = 0.5 * (lam_kc + L->lam[(int64_t)k * n + o]);
                hc[j] = (((w2 * L->len[3 * c + j]) * dz) * lamf) / L->cd[3 * c + j];
            }
            double d = vol;
            if (k > 0) d = d + vc_dn;
            if (k < nz - 1) d = d + vc_up;
            d = d + hc[0];
            d = d + hc[1];
            d = d + hc[2];
            L->D[(int64_t)k * n + c] = d;
            L->U[(int64_t)k * n + c] = (k < nz - 1) ? -vc_up : 0.0;
            for (int j = 0; j < 3; j++) L->H[((int64_t)j * nz + k) * n + c] = -hc[j];
        }
    }
}

void ora_free(ora_h* h) {
    if (!h) return;
    for (int r = 0; r < 16; r++) {
        ora_level* L = &h->lev[r];
        free(L->mesh.v); free(L->mesh.f); free(L->mesh.nbr);
        free(L->area); free(L->len); free(L->cd); free(L->lam);
        free(L->D); free(L->U); free(L->H);
        free(L->u); free(L->b); free(L->r); free(L->t);
    }
    free(h);
}

int ora_build_ex(int fine_ref, int coarsest_ref, int nz, double thickness, double w2, double omega_n,
                 const double* lam_fine, ora_h** out);

int ora_build(int fine_ref, int coarsest_ref, int nz, double thickness, double w2,
              const double* lam_fine, ora_h** out) {
    return ora_build_ex(fine_ref, coarsest_ref, nz, thickness, w2, 0.0, lam_fine, out);
}

/* omega_N = (dt/2) N, the buoyancy frequency term of Eq. 5. */
int ora_build_ex(int fine_ref, int coarsest_ref, int nz, double thickness, double w2, double omega_n,
                 const double* lam_fine, ora_h** out) {
    *out = NULL;
    if (fine_ref < 0 || fine_ref > 10) { snprintf(ora_msg, sizeof ora_msg, "fine_ref"); return ORA_ERR_ARG; }
    if (coarsest_ref < 0 || coarsest_ref > fine_ref) { snprintf(ora_msg, sizeof ora_msg, "coarsest_ref"); return ORA_ERR_ARG; }
    if (nz < 1) { snprintf(ora_msg, sizeof ora_msg, "nlayers"); return ORA_ERR_ARG; }
    if (!(thickness > 0)) { snprintf(ora_msg, sizeof ora_msg, "thickness"); return ORA_ERR_ARG; }
    if (!(w2 >= 0)) { snprintf(ora_msg, sizeof ora_msg, "w2"); return ORA_ERR_ARG; }
    if (!lam_fine) { snprintf(ora_msg, sizeof ora_msg, "lam"); return ORA_ERR_ARG; }
    if (!(omega_n >= 0) || !isfinite(omega_n)) { snprintf(ora_msg, sizeof ora_msg, "omega_n"); return ORA_ERR_ARG; }
    ora_h* h = (ora_h*)zalloc(sizeof(ora_h));
    if (!h) return ORA_ERR_OOM;
    h->fine_ref = fine_ref; h->coarsest_ref = coarsest_ref; h->nz = nz;
    h->thickness = thickness; h->w2 = w2;
    h->sn = 1.0 + omega_n * omega_n;
    h->dz = thickness / nz;
    int st = base_mesh(&h->lev[0].mesh);
    if (st) { ora_free(h); return st; }
    for (int r = 1; r <= fine_ref; r++) {
        st = refine(&h->lev[r - 1].mesh, &h->lev[r].mesh);
        if (st) { ora_free(h); return st; }
    }
    for (int r = 0; r <= fine_ref; r++) {
        ora_level* L = &h->lev[r];
        L->ref = r;
        L->n = L->mesh.nf;
        st = build_neighbours(&L->mesh);
        if (st) { ora_free(h); return st; }
        int64_t n = L->n, nn = (int64_t)nz * n;
        L->area = (double*)malloc(sizeof(double) * n);
        L->len = (double*)malloc(sizeof(double) * 3 * n);
        L->cd = (double*)malloc(sizeof(double) * 3 * n);
        L->lam = (double*)malloc(sizeof(double) * nn);
        L->D = (double*)malloc(sizeof(double) * nn);
        L->U = (double*)malloc(sizeof(double) * nn);
        L->H = (double*)malloc(sizeof(double) * 3 * nn);
        L->u = (double*)zalloc(sizeof(double) * nn);
        L->b = (double*)zalloc(sizeof(double) * nn);
        L->r = (double*)zalloc(sizeof(double) * nn);
        L->t = (double*)zalloc(sizeof(double) * nn);
        if (!L->area || !L->len || !L->cd || !L->lam || !L->D || !L->U || !L->H ||
            !L->u || !L->b || !L->r || !L->t) { ora_free(h); return ORA_ERR_OOM; }
        geometry(L);
    }
    /* O3 coefficients: fine lam given; coarse lam = 0.25*(((l0+l1)+l2)+l3) */
    ora_level* F = &h->lev[fine_ref];
    for (int64_t i = 0; i < (int64_t)nz * F->n; i++) {
        double v = lam_fine[i];
        if (!(v > 0) || !isfinite(v)) { snprintf(ora_msg, sizeof ora_msg, "lam"); ora_free(h); return ORA_ERR_ARG; }
        F->lam[i] = v;
    }
    for (int r = fine_ref - 1; r >= 0; r--) {
        ora_level* C = &h->lev[r];
        ora_level* Fi = &h->lev[r + 1];
        for (int k = 0; k < nz; k++)
            for (int64_t p = 0; p < C->n; p++) {
                const double* l = &Fi->lam[(int64_t)k * Fi->n + 4 * p];
                C->lam[(int64_t)k * C->n + p] = 0.25 * (((l[0] + l[1]) + l[2]) + l[3]);
            }
    }
    for (int r = 0; r <= fine_ref; r++) assemble(h, &h->lev[r]);
    *out = h;
    return ORA_OK;
}

int64_t ora_ncells(const ora_h* h, int ref) { return (ref >= 0 && ref <= h->fine_ref) ? h->lev[ref].n : -1; }
int64_t ora_nverts(const ora_h* h, int ref) { return (ref >= 0 && ref <= h->fine_ref) ? h->lev[ref].mesh.nv : -1; }

static int check_ref(const ora_h* h, int ref) {
    if (!h || ref < 0 || ref > h->fine_ref) { snprintf(ora_msg, sizeof ora_msg, "ref"); return 0; }
    return 1;
}

/* Export topology + geometry + bands of one level (any pointer may be NULL). */
int ora_export_level(const ora_h* h, int ref, double* verts, int32_t* faces, int32_t* nbr,
                     double* area, double* len, double* cd, double* lam,
                     double* D, double* U, double* H) {
    if (!check_ref(h, ref)) return ORA_ERR_ARG;
    const ora_level* L = &h->lev[ref];
    int64_t n = L->n, nn = (int64_t)h->nz * n;
    if (verts) memcpy(verts, L->mesh.v, sizeof(double) * 3 * L->mesh.nv);
    if (faces) memcpy(faces, L->mesh.f, sizeof(int32_t) * 3 * n);
    if (nbr) memcpy(nbr, L->mesh.nbr, sizeof(int32_t) * 3 * n);
    if (area) memcpy(area, L->area, sizeof(double) * n);
    if (len) memcpy(len, L->len, sizeof(double) * 3 * n);
    if (cd) memcpy(cd, L->cd, sizeof(double) * 3 * n);
    if (lam) memcpy(lam, L->lam, sizeof(double) * nn);
    if (D) memcpy(D, L->D, sizeof(double) * nn);
    if (U) memcpy(U, L->U, sizeof(double) * nn);
    if (H) memcpy(H, L->H, sizeof(double) * 3 * nn);
    return ORA_OK;
}

/* Test hook: overwrite the bands of one level (e.g. zero the horizontal
 * couplings) so that special cases of the method can be pinned. */
int ora_set_bands(ora_h* h, int ref, const double* D, const double* U, const double* H) {
    if (!check_ref(h, ref)) return ORA_ERR_ARG;
    ora_level* L = &h->lev[ref];
    int64_t nn = (int64_t)h->nz * L->n;
    if (D) memcpy(L->D, D, sizeof(double) * nn);
    if (U) memcpy(L->U, U, sizeof(double) * nn);
    if (H) memcpy(L->H, H, sizeof(double) * 3 * nn);
    return ORA_OK;
}

/* ------------------------------------------------------------------ */
/* O5 apply y = H^ x  ("v = H^ u = H^_z u + H^_h u")             */
/* y = ((((D x + U[k-1] x[k-1]) + U[k] x[k+1]) + H0 x[N0]) + H1 x[N1]) */
/*     + H2 x[N2], absent vertical terms skipped (reading R5).          */
/* ------------------------------------------------------------------ */
static void apply_level(const ora_h* h, const ora_level* L, const double* x, double* y) {
    int nz = h->nz;
    int64_t n = L->n;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; c++) {
        int32_t n0 = L->mesh.nbr[3 * c], n1 = L->mesh.nbr[3 * c + 1], n2 = L->mesh.nbr[3 * c + 2];
        for (int k = 0; k < nz; k++) {
            int64_t i = (int64_t)k * n + c;
            double acc = L->D[i] * x[i];
            if (k > 0) acc = acc + L->U[i - n] * x[i - n];
            if (k < nz - 1) acc = acc + L->U[i] * x[i + n];
            acc = acc + L->H[((int64_t)0 * nz + k) * n + c] * x[(int64_t)k * n + n0];
            acc = acc + L->H[((int64_t)1 * nz + k) * n + c] * x[(int64_t)k * n + n1];
            acc = acc + L->H[((int64_t)2 * nz + k) * n + c] * x[(int64_t)k * n + n2];
            y[i] = acc;
        }
    }
}

int ora_apply(const ora_h* h, int ref, const double* x, double* y) {
    if (!check_ref(h, ref)) return ORA_ERR_ARG;
    apply_level(h, &h->lev[ref], x, y);
    return ORA_OK;
}

/* ------------------------------------------------------------------ */
/* O6 Thomas algorithm (the textbook tridiagonal solve of   */
/* the cited Press et al. section 2.4), no pivoting.  Column of length */
/* nz with diagonal d[k*s], symmetric off-diagonal u[k*s] (coupling k, */
/* k+1), rhs r[k*s]; writes delta[k*s].  Work arrays g, z of length nz.*/
/* Returns 0, or 1 if a pivot den <= 0 or non-finite was met.          */
/* ------------------------------------------------------------------ */
static int thomas_col(int nz, int64_t s, const double* d, const double* u, const double* r,
                      double* delta, double* g, double* z) {
    double den = d[0];
    if (!(den > 0) || !isfinite(den)) return 1;
    z[0] = r[0] / den;
    for (int k = 1; k < nz; k++) {
        double ukm1 = u[(int64_t)(k - 1) * s];
        g[k - 1] = ukm1 / den;
        den = d[(int64_t)k * s] - ukm1 * g[k - 1];
        if (!(den > 0) || !isfinite(den)) return 1;
        z[k] = (r[(int64_t)k * s] - ukm1 * z[k - 1]) / den;
    }
    double dl = z[nz - 1];
    delta[(int64_t)(nz - 1) * s] = dl;
    for (int k = nz - 2; k >= 0; k--) {
        dl = z[k] - g[k] * dl;
        delta[(int64_t)k * s] = dl;
    }
    return 0;
}

/* Single contiguous column (for tests). */
int ora_thomas(int nz, const double* d, const double* u, const double* r, double* delta) {
    double* g = (double*)malloc(sizeof(double) * (nz + 1));
    double* z = (double*)malloc(sizeof(double) * (nz + 1));
    int bad = thomas_col(nz, 1, d, u, r, delta, g, z);
    free(g); free(z);
    if (bad) { snprintf(ora_msg, sizeof ora_msg, "singular column 0"); return ORA_ERR_SINGULAR; }
    return ORA_OK;
}

/* Column solve delta = T^{-1} rhs over all columns of a level; T = the
 * tridiagonal part of H^ (reading R6, Eq. 9 at P:607-615). */
static int tsolve_level(const ora_h* h, const ora_level* L, const double* rhs, double* delta, int64_t* bad_col) {
    int nz = h->nz;
    int64_t n = L->n;
    int64_t bad = -1;
#pragma omp parallel
    {
        double* g = (double*)malloc(sizeof(double) * (nz + 1));
        double* z = (double*)malloc(sizeof(double) * (nz + 1));
#pragma omp for schedule(static)
        for (int64_t c = 0; c < n; c++) {
            if (thomas_col(nz, n, &L->D[c], &L->U[c], &rhs[c], &delta[c], g, z)) {
#pragma omp critical
                { if (bad < 0 || c < bad) bad = c; }
            }
        }
        free(g); free(z);
    }
    if (bad >= 0) {
        if (bad_col) *bad_col = bad;
        snprintf(ora_msg, sizeof ora_msg, "singular column: ref %d column %lld", L->ref, (long long)bad);
        return ORA_ERR_SINGULAR;
    }
    return ORA_OK;
}

/* ------------------------------------------------------------------ */
/* O7 damped line-Jacobi sweep (Eq. 10 read with Eq. 13; */
/* reading R7): r = b - H^ u_old; delta = T^{-1} r; u_new = u_old +    */
/* omega*delta.  Zero-guess form: u_new = omega * T^{-1} b.            */
/* ------------------------------------------------------------------ */
static int sweep_level(const ora_h* h, ora_level* L, const double* b, double* u,
                       int nsweeps, double omega, int u_is_zero, int64_t* bad) {
    int64_t nn = (int64_t)h->nz * L->n;
    double* y = (double*)malloc(sizeof(double) * nn);
    double* r = (double*)malloc(sizeof(double) * nn);
    double* d = (double*)malloc(sizeof(double) * nn);
    int st = ORA_OK;
    for (int s = 0; s < nsweeps && st == ORA_OK; s++) {
        if (s == 0 && u_is_zero) {
            st = tsolve_level(h, L, b, d, bad);
            for (int64_t i = 0; i < nn; i++) u[i] = omega * d[i];
        } else {
            apply_level(h, L, u, y);
            for (int64_t i = 0; i < nn; i++) r[i] = b[i] - y[i];
            st = tsolve_level(h, L, r, d, bad);
            for (int64_t i = 0; i < nn; i++) u[i] = u[i] + omega * d[i];
        }
    }
    free(y); free(r); free(d);
    return st;
}

int ora_sweep(ora_h* h, int ref, const double* b, double* u, int nsweeps, double omega,
              int u_is_zero, int64_t* bad_col) {
    if (!check_ref(h, ref)) return ORA_ERR_ARG;
    return sweep_level(h, &h->lev[ref], b, u, nsweeps, omega, u_is_zero, bad_col);
}

/* Residual r = b - H^ u (elementwise b - y). */
int ora_residual(const ora_h* h, int ref, const double* b, const double* u, double* r) {
    if (!check_ref(h, ref)) return ORA_ERR_ARG;
    const ora_level* L = &h->lev[ref];
    int64_t nn = (int64_t)h->nz * L->n;
    double* y = (double*)malloc(sizeof(double) * nn);
    apply_level(h, L, u, y);
    for (int64_t i = 0; i < nn; i++) r[i] = b[i] - y[i];
    free(y);
    return ORA_OK;
}

/* ------------------------------------------------------------------ */
/* O8 transfers (reading R8): DG0 restriction = sum of the  */
/* 4 children ((r0+r1)+r2)+r3 (R = P^T, no 1/4); prolongation =        */
/* injection ("natural embedding") added to u.              */
/* ------------------------------------------------------------------ */
int ora_restrict(const ora_h* h, int fine_ref, const double* r, double* bc) {
    if (!check_ref(h, fine_ref) || fine_ref < 1) { snprintf(ora_msg, sizeof ora_msg, "fine_ref"); return ORA_ERR_ARG; }
    int64_t nf = h->lev[fine_ref].n, nc = h->lev[fine_ref - 1].n;
    for (int k = 0; k < h->nz; k++)
        for (int64_t p = 0; p < nc; p++) {
            const double* q = &r[(int64_t)k * nf + 4 * p];
            bc[(int64_t)k * nc + p] = ((q[0] + q[1]) + q[2]) + q[3];
        }
    return ORA_OK;
}

int ora_prolong_add(const ora_h* h, int fine_ref, const double* uc, double* uf) {
    if (!check_ref(h, fine_ref) || fine_ref < 1) { snprintf(ora_msg, sizeof ora_msg, "fine_ref"); return ORA_ERR_ARG; }
    int64_t nf = h->lev[fine_ref].n, nc = h->lev[fine_ref - 1].n;
    for (int k = 0; k < h->nz; k++)
        for (int64_t c = 0; c < nf; c++)
            uf[(int64_t)k * nf + c] = uf[(int64_t)k * nf + c] + uc[(int64_t)k * nc + c / 4];
    return ORA_OK;
}

/* ------------------------------------------------------------------ */
/* O9 V-cycle: Algorithm 1 applied recursively, correction */
/* scheme with zero initial guess on each level (reading R9):          */
/*   coarsest: u = 0, n_coarse sweeps                                  */
/*   else: u = 0; nu_pre sweeps (M1); b_c = R(b - H^u) (M2);           */
/*         u_c = V(l-1, b_c) (M3); u = u + P u_c (M4); nu_post (M5).   */
/* ------------------------------------------------------------------ */
static int vcycle_level(ora_h* h, int ref, int nu_pre, int nu_post, int n_coarse, double omega,
                        const double* b, double* u, int64_t* bad) {
    ora_level* L = &h->lev[ref];
    int64_t nn = (int64_t)h->nz * L->n;
    int st;
    for (int64_t i = 0; i < nn; i++) u[i] = 0.0;
    if (ref == h->coarsest_ref)
        return sweep_level(h, L, b, u, n_coarse, omega, 1, bad);
    st = sweep_level(h, L, b, u, nu_pre, omega, 1, bad);                        /* M1 */
    if (st) return st;
    ora_level* C = &h->lev[ref - 1];
    if (nu_pre > 0) {
        ora_residual(h, ref, b, u, L->r);                                        /* M2 */
    } else {
        for (int64_t i = 0; i < nn; i++) L->r[i] = b[i];
    }
    ora_restrict(h, ref, L->r, C->b);
    st = vcycle_level(h, ref - 1, nu_pre, nu_post, n_coarse, omega, C->b, C->u, bad); /* M3 */
    if (st) return st;
    ora_prolong_add(h, ref, C->u, u);                                            /* M4 */
    return sweep_level(h, L, b, u, nu_post, omega, 0, bad);                      /* M5 */
}

int ora_vcycle(ora_h* h, int nu_pre, int nu_post, int n_coarse, double omega, const double* b, double* z) {
    if (!h || nu_pre < 0 || nu_post < 0 || n_coarse < 1) { snprintf(ora_msg, sizeof ora_msg, "params"); return ORA_ERR_ARG; }
    int64_t bad = -1;
    return vcycle_level(h, h->fine_ref, nu_pre, nu_post, n_coarse, omega, b, z, &bad);
}

/* ------------------------------------------------------------------ */
/* O10 preconditioned conjugate gradients, x0 = 0 (reading R10/R12).   */
/* dot = plain sequential sum in index order.  precond: 0 = identity,  */
/* 1 = one V-cycle, 2 = single-level: nu_pre line-Jacobi sweeps from  */
/* zero on the fine level ("two iterations of Block-Jacobi").*/
/* ------------------------------------------------------------------ */
static double dot(int64_t n, const double* a, const double* b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s = s + a[i] * b[i];
    return s;
}

static int precond(ora_h* h, int kind, int nu_pre, int nu_post, int n_coarse, double omega,
                   const double* r, double* z) {
    int64_t nn = (int64_t)h->nz * h->lev[h->fine_ref].n;
    if (kind == 0) { memcpy(z, r, sizeof(double) * nn); return ORA_OK; }
    if (kind == 1) return ora_vcycle(h, nu_pre, nu_post, n_coarse, omega, r, z);
    int64_t bad = -1;
    return sweep_level(h, &h->lev[h->fine_ref], r, z, nu_pre, omega, 1, &bad);
}

int ora_pcg(ora_h* h, int kind, int nu_pre, int nu_post, int n_coarse, double omega,
            const double* b, double* x, double rtol, int maxit, int* iters, double* relres,
            double* hist /* [maxit+1] or NULL: ||r_k||/||b|| */) {
    int64_t nn = (int64_t)h->nz * h->lev[h->fine_ref].n;
    double* r = (double*)malloc(sizeof(double) * nn);
    double* z = (double*)malloc(sizeof(double) * nn);
    double* p = (double*)malloc(sizeof(double) * nn);
    double* q = (double*)malloc(sizeof(double) * nn);
    int st = ORA_OK;
    *iters = 0;
    for (int64_t i = 0; i < nn; i++) { x[i] = 0.0; r[i] = b[i]; }
    double bn = sqrt(dot(nn, b, b));
    *relres = 0.0;
    if (hist) hist[0] = bn == 0.0 ? 0.0 : 1.0;
    if (bn == 0.0) goto done;
    st = precond(h, kind, nu_pre, nu_post, n_coarse, omega, r, z);
    if (st) goto done;
    double rho = dot(nn, r, z);
    memcpy(p, z, sizeof(double) * nn);
    st = ORA_ERR_NOT_CONVERGED;
    for (int it = 1; it <= maxit; it++) {
        apply_level(h, &h->lev[h->fine_ref], p, q);
        double alpha = rho / dot(nn, p, q);
        for (int64_t i = 0; i < nn; i++) x[i] = x[i] + alpha * p[i];
        for (int64_t i = 0; i < nn; i++) r[i] = r[i] - alpha * q[i];
        double rn = sqrt(dot(nn, r, r));
        *iters = it;
        *relres = rn / bn;
        if (hist) hist[it] = rn / bn;
        if (rn <= rtol * bn) { st = ORA_OK; break; }
        int s2 = precond(h, kind, nu_pre, nu_post, n_coarse, omega, r, z);
        if (s2) { st = s2; break; }
        double rho_new = dot(nn, r, z);
        double beta = rho_new / rho;
        rho = rho_new;
        for (int64_t i = 0; i < nn; i++) p[i] = z[i] + beta * p[i];
    }
done:
    free(r); free(z); free(p); free(q);
    if (st == ORA_ERR_NOT_CONVERGED) snprintf(ora_msg, sizeof ora_msg, "not converged after %d iterations", maxit);
    return st;
}

/* ================================================================== */
/* NEXT-4: the mixed velocity-pressure system around    */
/* the V-cycle -- Eq. 5 with omega_N = 0, its Schur-       */
/* complement preconditioner (Eq. 6) with a lumped velocity */
/* mass, and restarted GMRES(30).  Readings R15-R20 of     */
/* DESIGN.md; every loop below is per (edge, layer), per (column,      */
/* interface) or per (cell, layer) in the canonical order stated.      */
/*                                                                    */
/* Unknowns (reading R15): U_h [nz][ne] normal flux through the        */
/* vertical face of edge e in layer k, positive from cell a to cell b  */
/* (a < b); U_z [nz-1][n] flux through interface i = 1..nz-1 of column */
/* c (row i-1), positive upward (u.n = 0 removes i = 0 and i = nz,     */
/* P:415-418); P [nz][n].  omega = sqrt(w2) (omega_c^2 = w2).          */
/*   A = [[M2, -omega D^T], [omega D, M3]]                              */
/* ================================================================== */

/* Edge table of the fine level (reading R16): edges in order of their  */
/* lower cell a, then a's slot j; b = nbr[a][j]; slot_b = the slot of b */
/* whose neighbour is a.  ce[c][j] = edge across slot j of cell c.      */
typedef struct {
    int64_t ne;
    int32_t *ec, *es, *ce;   /* [ne][2] cells (a, b), [ne][2] slots, [n][3] edges */
} ora_edges;

static void free_edges(ora_edges* E) { free(E->ec); free(E->es); free(E->ce); }

static int fine_edges(const ora_h* h, ora_edges* E) {
    const ora_level* L = &h->lev[h->fine_ref];
    int64_t n = L->n;
    E->ne = 3 * n / 2;
    E->ec = (int32_t*)malloc(sizeof(int32_t) * 2 * E->ne);
    E->es = (int32_t*)malloc(sizeof(int32_t) * 2 * E->ne);
    E->ce = (int32_t*)malloc(sizeof(int32_t) * 3 * n);
    if (!E->ec || !E->es || !E->ce) { free_edges(E); return ORA_ERR_OOM; }
    int64_t e = 0;
    for (int64_t c = 0; c < n; c++)
        for (int j = 0; j < 3; j++) {
            int32_t o = L->mesh.nbr[3 * c + j];
            if (c < o) {
                int jo = 0;
                while (L->mesh.nbr[3 * o + jo] != (int32_t)c) jo++;
                E->ec[2 * e] = (int32_t)c; E->ec[2 * e + 1] = o;
                E->es[2 * e] = j; E->es[2 * e + 1] = jo;
                E->ce[3 * c + j] = (int32_t)e;
                E->ce[3 * o + jo] = (int32_t)e;
                e++;
            }
        }
    return ORA_OK;
}

/* sigma_{c,j}: +1 if the flux of the edge across slot j leaves c (c is  */
/* the lower cell a), -1 otherwise.                                     */
static double edge_sign(const ora_level* L, int64_t c, int j) {
    return (c < L->mesh.nbr[3 * c + j]) ? 1.0 : -1.0;
}

/* Gram matrix of the outward flux-normalised RT0 functions of cell c    */
/* (reading R17): psi_j(x) = (x - P_{j+2}) / (2|T|) on the flat chordal  */
/* triangle (P_0, P_1, P_2), edge j = (P_j, P_{j+1}) opposite P_{j+2};    */
/* G_{jl} = int_T psi_j . psi_l dA by the edge-midpoint rule (exact for  */
/* quadratics): G_{jl} = ((s_0 + s_1) + s_2) / (12 |T|),                 */
/* s_q = (m_q - P_{j+2}) . (m_q - P_{l+2}), m_q = 0.5 (P_q + P_{q+1}).    */
static void rt0_gram(const ora_level* L, int64_t c, double G[3][3]) {
    const double* V = L->mesh.v;
    const int32_t* F = L->mesh.f;
    const double* Pv[3] = {&V[3 * F[3 * c]], &V[3 * F[3 * c + 1]], &V[3 * F[3 * c + 2]]};
    double m[3][3];
    for (int q = 0; q < 3; q++)
        for (int d = 0; d < 3; d++) m[q][d] = 0.5 * (Pv[q][d] + Pv[(q + 1) % 3][d]);
    for (int j = 0; j < 3; j++)
        for (int l = 0; l < 3; l++) {
            const double* A = Pv[(j + 2) % 3];
            const double* B = Pv[(l + 2) % 3];
            double s[3];
            for (int q = 0; q < 3; q++) {
                double ax = m[q][0] - A[0], ay = m[q][1] - A[1], az = m[q][2] - A[2];
                double bx = m[q][0] - B[0], by = m[q][1] - B[1], bz = m[q][2] - B[2];
                s[q] = (ax * bx + ay * by) + az * bz;
            }
            G[j][l] = ((s[0] + s[1]) + s[2]) / (12.0 * L->area[c]);
        }
}

/* Mixed-system parts (reading R18), used by the apply, the             */
/* preconditioner and the pins:                                          */
/*  div:   (D U)[k][c] = (((s0 U_h[E0] + s1 U_h[E1]) + s2 U_h[E2])       */
/*                        + U_z[k+1]) - U_z[k]   (absent U_z skipped)     */
/*  divT:  (D^T P)_h[k][e] = P[k][a] - P[k][b];                           */
/*         (D^T P)_z[i][c] = P[i-1][c] - P[i][c]                          */
/*  (with buoyancy, reading R24: the vertical mass times 1 + omega_N^2    */
/*   and its lumped inverse divided by it)                                 */
/*  mass:  (M2 U)_h[k][e] = t_a/(dz lam_a) + t_b/(dz lam_b),              */
/*         t_c = ((g0 U_h[E0] + g1 U_h[E1]) + g2 U_h[E2]),                */
/*         g_l = (s_j s_l) G^c_{j l}, j = the slot of e in c;              */
/*         (M2 U)_z[i] = ((dg W_i + lo W_{i-1}) + hi W_{i+1}),             */
/*         dg = ((dz/3)/(area lam_{i-1})) + ((dz/3)/(area lam_i)),          */
/*         lo = (dz/6)/(area lam_{i-1}), hi = (dz/6)/(area lam_i)           */
/*         (P1 vertical mass of unit-flux hats, weight 1/lam per cell)     */
/*  lumped inverse (reading R19, the two-point lumping whose Schur        */
/*  complement is BASELINE's H^): (L^-1 U)_h = U_h ((len dz) lamf)/cd,     */
/*  (L^-1 U)_z = U_z (area lamf)/dz, lamf = 0.5 (lam_a + lam_b).            */
static void mixed_div(const ora_h* h, const ora_edges* E, const double* Uh, const double* Uz, double* y) {
    const ora_level* L = &h->lev[h->fine_ref];
    int nz = h->nz;
    int64_t n = L->n, ne = E->ne;
    for (int k = 0; k < nz; k++)
        for (int64_t c = 0; c < n; c++) {
            double d = edge_sign(L, c, 0) * Uh[(int64_t)k * ne + E->ce[3 * c]];
            d = d + edge_sign(L, c, 1) * Uh[(int64_t)k * ne + E->ce[3 * c + 1]];
            d = d + edge_sign(L, c, 2) * Uh[(int64_t)k * ne + E->ce[3 * c + 2]];
            if (k + 1 <= nz - 1) d = d + Uz[(int64_t)k * n + c];         /* interface k+1: row k */
            if (k >= 1) d = d - Uz[(int64_t)(k - 1) * n + c];             /* interface k: row k-1 */
            y[(int64_t)k * n + c] = d;
        }
}

static void mixed_divT(const ora_h* h, const ora_edges* E, const double* P, double* yh, double* yz) {
    const ora_level* L = &h->lev[h->fine_ref];
    int nz = h->nz;
    int64_t n = L->n, ne = E->ne;
    for (int k = 0; k < nz; k++)
        for (int64_t e = 0; e < ne; e++)
            yh[(int64_t)k * ne + e] = P[(int64_t)k * n + E->ec[2 * e]] - P[(int64_t)k * n + E->ec[2 * e + 1]];
    for (int i = 1; i <= nz - 1; i++)
        for (int64_t c = 0; c < n; c++)
            yz[(int64_t)(i - 1) * n + c] = P[(int64_t)(i - 1) * n + c] - P[(int64_t)i * n + c];
}

static void mixed_mass(const ora_h* h, const ora_edges* E, const double* Uh, const double* Uz, double* yh,
                       double* yz) {
    const ora_level* L = &h->lev[h->fine_ref];
    int nz = h->nz;
    int64_t n = L->n, ne = E->ne;
    double dz = h->dz;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < ne; e++) {
        double G[2][3][3];
        rt0_gram(L, E->ec[2 * e], G[0]);
        rt0_gram(L, E->ec[2 * e + 1], G[1]);
        for (int k = 0; k < nz; k++) {
            double m[2];
            for (int s = 0; s < 2; s++) {
                int64_t c = E->ec[2 * e + s];
                int j = E->es[2 * e + s];
                double g[3];
                for (int l = 0; l < 3; l++) g[l] = (edge_sign(L, c, j) * edge_sign(L, c, l)) * G[s][j][l];
                double t = g[0] * Uh[(int64_t)k * ne + E->ce[3 * c]];
                t = t + g[1] * Uh[(int64_t)k * ne + E->ce[3 * c + 1]];
                t = t + g[2] * Uh[(int64_t)k * ne + E->ce[3 * c + 2]];
                m[s] = t / (dz * L->lam[(int64_t)k * n + c]);
            }
            yh[(int64_t)k * ne + e] = m[0] + m[1];
        }
    }
    for (int i = 1; i <= nz - 1; i++)
        for (int64_t c = 0; c < n; c++) {
            double slo = L->area[c] * L->lam[(int64_t)(i - 1) * n + c];
            double shi = L->area[c] * L->lam[(int64_t)i * n + c];
            double dg = ((dz / 3.0) / slo) + ((dz / 3.0) / shi);
            double v = dg * Uz[(int64_t)(i - 1) * n + c];
            if (i - 1 >= 1) v = v + ((dz / 6.0) / slo) * Uz[(int64_t)(i - 2) * n + c];
            if (i + 1 <= nz - 1) v = v + ((dz / 6.0) / shi) * Uz[(int64_t)i * n + c];
            yz[(int64_t)(i - 1) * n + c] = v * h->sn;   /* M~2z = (1 + omega_N^2) M2z (Eq. 5) */
        }
}

static void mixed_lumped_inv(const ora_h* h, const ora_edges* E, const double* Uh, const double* Uz, double* yh,
                             double* yz) {
    const ora_level* L = &h->lev[h->fine_ref];
    int nz = h->nz;
    int64_t n = L->n, ne = E->ne;
    double dz = h->dz;
    for (int k = 0; k < nz; k++)
        for (int64_t e = 0; e < ne; e++) {
            int64_t a = E->ec[2 * e], b = E->ec[2 * e + 1];
            int j = E->es[2 * e];
            double lamf = 0.5 * (L->lam[(int64_t)k * n + a] + L->lam[(int64_t)k * n + b]);
            double il = ((L->len[3 * a + j] * dz) * lamf) / L->cd[3 * a + j];
            yh[(int64_t)k * ne + e] = Uh[(int64_t)k * ne + e] * il;
        }
    for (int i = 1; i <= nz - 1; i++)
        for (int64_t c = 0; c < n; c++) {
            double lamf = 0.5 * (L->lam[(int64_t)(i - 1) * n + c] + L->lam[(int64_t)i * n + c]);
            double il = ((L->area[c] * lamf) / dz) / h->sn;      /* the lumping of M~2z */
            yz[(int64_t)(i - 1) * n + c] = Uz[(int64_t)(i - 1) * n + c] * il;
        }
}

int64_t ora_mixed_nedges(const ora_h* h) { return 3 * h->lev[h->fine_ref].n / 2; }

int ora_mixed_edges(const ora_h* h, int32_t* ec, int32_t* es, int32_t* ce) {
    ora_edges E;
    int st = fine_edges(h, &E);
    if (st) return st;
    int64_t n = h->lev[h->fine_ref].n;
    if (ec) memcpy(ec, E.ec, sizeof(int32_t) * 2 * E.ne);
    if (es) memcpy(es, E.es, sizeof(int32_t) * 2 * E.ne);
    if (ce) memcpy(ce, E.ce, sizeof(int32_t) * 3 * n);
    free_edges(&E);
    return ORA_OK;
}

/* One part of the mixed system: which = 0 div (Uh, Uz -> yp), 1 divT    */
/* (P -> yh, yz), 2 mass (Uh, Uz -> yh, yz), 3 lumped inverse,            */
/* 4 RT0 Gram matrices of all fine cells ([n][3][3] into yh).            */
int ora_mixed_part(const ora_h* h, int which, const double* Uh, const double* Uz, const double* P, double* yh,
                   double* yz, double* yp) {
    ora_edges E;
    int st = fine_edges(h, &E);
    if (st) return st;
    if (which == 0) mixed_div(h, &E, Uh, Uz, yp);
    else if (which == 1) mixed_divT(h, &E, P, yh, yz);
    else if (which == 2) mixed_mass(h, &E, Uh, Uz, yh, yz);
    else if (which == 3) mixed_lumped_inv(h, &E, Uh, Uz, yh, yz);
    else if (which == 4) {
        const ora_level* L = &h->lev[h->fine_ref];
        for (int64_t c = 0; c < L->n; c++) rt0_gram(L, c, (double(*)[3])&yh[9 * c]);
    } else st = ORA_ERR_ARG;
    free_edges(&E);
    return st;
}

/* y = A x (reading R18): y_h = M2h U_h - omega (D^T P)_h,                */
/* y_z = M2z U_z - omega (D^T P)_z, y_p = omega (D U) + vol P              */
/* (vol = area dz).  Vectors concatenated [U_h | U_z | P].                 */
static void mixed_apply(const ora_h* h, const ora_edges* E, const double* x, double* y, double* tmp) {
    const ora_level* L = &h->lev[h->fine_ref];
    int nz = h->nz;
    int64_t n = L->n, ne = E->ne;
    int64_t nh = (int64_t)nz * ne, nzz = (int64_t)(nz - 1) * n, np = (int64_t)nz * n;
    double om = sqrt(h->w2);
    const double *Uh = x, *Uz = x + nh, *P = x + nh + nzz;
    double *yh = y, *yz = y + nh, *yp = y + nh + nzz;
    double *th = tmp, *tz = tmp + nh, *tp = tmp + nh + nzz;
    mixed_mass(h, E, Uh, Uz, yh, yz);
    mixed_divT(h, E, P, th, tz);
    for (int64_t q = 0; q < nh; q++) yh[q] = yh[q] - om * th[q];
    for (int64_t q = 0; q < nzz; q++) yz[q] = yz[q] - om * tz[q];
    mixed_div(h, E, Uh, Uz, tp);
    for (int k = 0; k < nz; k++)
        for (int64_t c = 0; c < n; c++) {
            int64_t q = (int64_t)k * n + c;
            yp[q] = om * tp[q] + (L->area[c] * h->dz) * P[q];
        }
    (void)np;
}

int64_t ora_mixed_size(const ora_h* h) {
    int64_t n = h->lev[h->fine_ref].n;
    return (int64_t)h->nz * (3 * n / 2) + (int64_t)(h->nz - 1) * n + (int64_t)h->nz * n;
}

int ora_mixed_apply(const ora_h* h, const double* x, double* y) {
    ora_edges E;
    int st = fine_edges(h, &E);
    if (st) return st;
    double* tmp = (double*)malloc(sizeof(double) * ora_mixed_size(h));
    if (!tmp) { free_edges(&E); return ORA_ERR_OOM; }
    mixed_apply(h, &E, x, y, tmp);
    free(tmp);
    free_edges(&E);
    return ORA_OK;
}

/* Schur-complement preconditioner (Eq. 6 with M2^-1 -> L^-1 and H^-1 ->  */
/* one V-cycle; reading R19), applied right to left:                       */
/*   g_p = f_p - omega (D (L^-1 f_u));  x_p = V(g_p);                      */
/*   x_u = L^-1 (f_u + omega (D^T x_p)).                                   */
/* kind 1: V-cycle; kind 0: identity (no preconditioner).                  */
static int mixed_precond(ora_h* h, const ora_edges* E, int kind, int nu_pre, int nu_post, int n_coarse,
                         double omega_s, const double* f, double* x, double* tmp) {
    const ora_level* L = &h->lev[h->fine_ref];
    int nz = h->nz;
    int64_t n = L->n, ne = E->ne;
    int64_t nh = (int64_t)nz * ne, nzz = (int64_t)(nz - 1) * n, np = (int64_t)nz * n;
    if (kind == 0) { memcpy(x, f, sizeof(double) * (nh + nzz + np)); return ORA_OK; }
    double om = sqrt(h->w2);
    const double *fh = f, *fz = f + nh, *fp = f + nh + nzz;
    double *xh = x, *xz = x + nh, *xp = x + nh + nzz;
    double *th = tmp, *tz = tmp + nh, *tp = tmp + nh + nzz;
    mixed_lumped_inv(h, E, fh, fz, th, tz);
    mixed_div(h, E, th, tz, tp);
    for (int64_t q = 0; q < np; q++) tp[q] = fp[q] - om * tp[q];
    int st = ora_vcycle(h, nu_pre, nu_post, n_coarse, omega_s, tp, xp);
    if (st) return st;
    mixed_divT(h, E, xp, th, tz);
    for (int64_t q = 0; q < nh; q++) th[q] = fh[q] + om * th[q];
    for (int64_t q = 0; q < nzz; q++) tz[q] = fz[q] + om * tz[q];
    mixed_lumped_inv(h, E, th, tz, xh, xz);
    return ORA_OK;
}

int ora_mixed_precond(ora_h* h, int kind, int nu_pre, int nu_post, int n_coarse, double omega_s, const double* f,
                      double* x) {
    ora_edges E;
    int st = fine_edges(h, &E);
    if (st) return st;
    double* tmp = (double*)malloc(sizeof(double) * ora_mixed_size(h));
    if (!tmp) { free_edges(&E); return ORA_ERR_OOM; }
    st = mixed_precond(h, &E, kind, nu_pre, nu_post, n_coarse, omega_s, f, x, tmp);
    free(tmp);
    free_edges(&E);
    return st;
}

/* Restarted right-preconditioned GMRES(m) (reading R20; Saad & Schultz,  */
/* the paper's GMRES(30) to ||r||/||r_0|| < 1e-5), x0 = 0:       */
/*   r = F, beta = ||r||; per cycle: v_0 = r / beta, g = beta e_0;          */
/*   for j < m: w = A M^-1 v_j; classical Gram-Schmidt applied twice      */
/*   (CGS2): per pass c_i = <v_i, w> (i <= j, all against the same w), then */
/*   w = w - sum_i c_i v_i in order i; h_ij = c_i(pass 1) + c_i(pass 2);    */
/*   h_{j+1,j} = ||w||, v_{j+1} = w / h_{j+1,j}; previous Givens rotations  */
/*   applied to column j in order, new rotation (c, s) = (h_jj, h_{j+1,j})  */
/*   / sqrt(h_jj^2 + h_{j+1,j}^2); g_{j+1} = -s g_j, g_j = c g_j;            */
/*   stop the cycle when |g_{j+1}| <= rtol ||F|| (count = Arnoldi steps).   */
/*   Then y = H^-1 g (back substitution), x = x + M^-1 (sum_i y_i v_i);    */
/*   r = F - A x, beta = ||r||; converged when beta <= rtol ||F||.          */
/* dot = sequential sum in index order.                                    */
int ora_mixed_gmres(ora_h* h, int kind, int nu_pre, int nu_post, int n_coarse, double omega_s, int m, double rtol,
                    int maxit, int gs_passes, const double* F, double* X, int* iters, double* relres, double* hist,
                    double* orth) {
    ora_edges E;
    int st = fine_edges(h, &E);
    if (st) return st;
    int64_t N = ora_mixed_size(h);
    double* V = (double*)malloc(sizeof(double) * N * (m + 1));
    double* w = (double*)malloc(sizeof(double) * N);
    double* z = (double*)malloc(sizeof(double) * N);
    double* tmp = (double*)malloc(sizeof(double) * N);
    double* H = (double*)calloc((size_t)(m + 1) * m, sizeof(double));
    double* cs = (double*)malloc(sizeof(double) * m);
    double* sn = (double*)malloc(sizeof(double) * m);
    double* g = (double*)malloc(sizeof(double) * (m + 1));
    double* yv = (double*)malloc(sizeof(double) * m);
    if (!V || !w || !z || !tmp || !H || !cs || !sn || !g || !yv) { st = ORA_ERR_OOM; goto out; }
    *iters = 0;
    *relres = 0.0;
    if (orth) *orth = 0.0;
    if (gs_passes < 1) { st = ORA_ERR_ARG; snprintf(ora_msg, sizeof ora_msg, "gs_passes must be >= 1"); goto out; }
    for (int64_t q = 0; q < N; q++) X[q] = 0.0;
    double fn = sqrt(dot(N, F, F));
    if (hist) hist[0] = fn == 0.0 ? 0.0 : 1.0;
    if (fn == 0.0) { st = ORA_OK; goto out; }
    memcpy(w, F, sizeof(double) * N);
    double beta = fn;
    int total = 0;
    st = ORA_ERR_NOT_CONVERGED;
    while (total < maxit) {
        for (int64_t q = 0; q < N; q++) V[q] = w[q] / beta;
        for (int i = 0; i <= m; i++) g[i] = 0.0;
        g[0] = beta;
        int j, done = 0;
        for (j = 0; j < m && total < maxit; j++) {
            double* vj = V + (int64_t)j * N;
            int s2 = mixed_precond(h, &E, kind, nu_pre, nu_post, n_coarse, omega_s, vj, z, tmp);
            if (s2) { st = s2; goto out; }
            mixed_apply(h, &E, z, w, tmp);
            /* classical Gram-Schmidt, gs_passes times: 1 = CGS (PETSc's default,
               refinement "never"), 2 = CGS2 ("twice is enough"; reading R20) */
            for (int pass = 0; pass < gs_passes; pass++) {
                for (int i = 0; i <= j; i++) yv[i] = dot(N, V + (int64_t)i * N, w);
                for (int i = 0; i <= j; i++) {
                    const double* vi = V + (int64_t)i * N;
                    double hij = yv[i];
                    for (int64_t q = 0; q < N; q++) w[q] = w[q] - hij * vi[q];
                }
                for (int i = 0; i <= j; i++) H[i * m + j] = pass == 0 ? yv[i] : H[i * m + j] + yv[i];
            }
            double hn = sqrt(dot(N, w, w));
            H[(j + 1) * m + j] = hn;
            double* vn = V + (int64_t)(j + 1) * N;
            for (int64_t q = 0; q < N; q++) vn[q] = w[q] / hn;
            for (int i = 0; i < j; i++) {
                double a = H[i * m + j], b = H[(i + 1) * m + j];
                H[i * m + j] = cs[i] * a + sn[i] * b;
                H[(i + 1) * m + j] = -sn[i] * a + cs[i] * b;
            }
            double a = H[j * m + j], b = H[(j + 1) * m + j];
            double rr = sqrt(a * a + b * b);
            cs[j] = a / rr;
            sn[j] = b / rr;
            H[j * m + j] = rr;
            H[(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            total++;
            if (hist) hist[total] = fabs(g[j + 1]) / fn;
            if (fabs(g[j + 1]) <= rtol * fn) { j++; done = 1; break; }
        }
        if (orth) {   /* diagnostic: max |<v_a, v_b> - delta_ab| over the cycle's j + 1 basis vectors */
            for (int a2 = 0; a2 <= j; a2++)
                for (int b2 = 0; b2 <= a2; b2++) {
                    double e = dot(N, V + (int64_t)a2 * N, V + (int64_t)b2 * N) - (a2 == b2 ? 1.0 : 0.0);
                    if (fabs(e) > *orth) *orth = fabs(e);
                }
        }
        /* y = H^-1 g on the leading j x j block, x += M^-1 (V y) */
        for (int i = j - 1; i >= 0; i--) {
            double s = g[i];
            for (int l = i + 1; l < j; l++) s = s - H[i * m + l] * yv[l];
            yv[i] = s / H[i * m + i];
        }
        for (int64_t q = 0; q < N; q++) w[q] = 0.0;
        for (int i = 0; i < j; i++) {
            const double* vi = V + (int64_t)i * N;
            for (int64_t q = 0; q < N; q++) w[q] = w[q] + yv[i] * vi[q];
        }
        int s2 = mixed_precond(h, &E, kind, nu_pre, nu_post, n_coarse, omega_s, w, z, tmp);
        if (s2) { st = s2; goto out; }
        for (int64_t q = 0; q < N; q++) X[q] = X[q] + z[q];
        mixed_apply(h, &E, X, z, tmp);
        for (int64_t q = 0; q < N; q++) w[q] = F[q] - z[q];
        beta = sqrt(dot(N, w, w));
        *iters = total;
        *relres = beta / fn;
        if (beta <= rtol * fn) { st = ORA_OK; break; }
        (void)done;
    }
out:
    free(V); free(w); free(z); free(tmp); free(H); free(cs); free(sn); free(g); free(yv);
    free_edges(&E);
    if (st == ORA_ERR_NOT_CONVERGED) snprintf(ora_msg, sizeof ora_msg, "GMRES not converged after %d iterations", maxit);
    return st;
}

/* Thread count of the OpenMP column loops (results do not depend on it). */
void ora_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
