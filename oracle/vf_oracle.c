/*
 * vf_oracle.c -- FP64 CPU ORACLE for the view-factor hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header or constant generator with the product
 * library (paper_2209_07632_b200/csrc); neither includes the other.
 *
 * What it computes is the PLAIN DEFINITION of the paper's discrete
 * operator, written out (PAPER.md = "P:<line>"):
 *   - facet data A_i, x_i, n_i                         P:129 (§3)
 *   - visibility V_ij with back-face culling            P:164-173 (§3.2)
 *     (open segment, Moller-Trumbore, reading R-VIS)
 *   - F_ij = [n_i.(x_j-x_i)][n_j.(x_i-x_j)] V_ij A_j / (pi |x_i-x_j|^4)
 *                                                       P:134-136 eq. FF-def
 *   - insolation Q = S max(0, n_i.s) V_sun(x_i, s)     P:76-80 eq. insolation,
 *                                                       P:282 (§5.1)
 * Brute force over all triangles is the definition; the uniform xy grid
 * below is an independently written accelerator with the SAME
 * per-triangle predicate, pinned against brute force in
 * tests/test_oracle_pins.py (pin P7).
 *
 * No blocking, fusion or reordering beyond the definitions.  Rows are
 * independent, so OpenMP parallelises over rows i only.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_T_EPS 1e-9      /* open-segment parameter margin (R-VIS)        */
#define OR_DET_EPS 1e-300  /* |det| <= this: segment parallel to triangle  */

/* ------------------------------------------------------------ facet data */
/* "We denote the area, centroid, and surface normal of the ith
 * triangle by A_i, x_i, n_i".  x = (a+b+c)/3, n = (b-a)x(c-a)/|.|,
 * A = |(b-a)x(c-a)|/2.  orient_up != 0 flips n so that n_z > 0 (height
 * fields, reading R-ORIENT); 0 keeps the right-hand-rule normal.
 * Returns the number of degenerate (zero-area) faces found (A = 0 set). */
int or_facet_data(int64_t nf, const double* V, const int32_t* F, int orient_up,
                  double* x, double* n, double* A)
{
    int bad = 0;
    for (int64_t f = 0; f < nf; ++f) {
        const double* a = V + 3 * (int64_t)F[3 * f + 0];
        const double* b = V + 3 * (int64_t)F[3 * f + 1];
        const double* c = V + 3 * (int64_t)F[3 * f + 2];
        double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1],
                        e1[2] * e2[0] - e1[0] * e2[2],
                        e1[0] * e2[1] - e1[1] * e2[0]};
        double len = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
        for (int d = 0; d < 3; ++d) x[3 * f + d] = (a[d] + b[d] + c[d]) / 3.0;
        A[f] = 0.5 * len;
        if (len == 0.0) { ++bad; n[3 * f] = n[3 * f + 1] = n[3 * f + 2] = 0.0; continue; }
        double s = (orient_up && cr[2] < 0.0) ? -1.0 : 1.0;
        for (int d = 0; d < 3; ++d) n[3 * f + d] = s * cr[d] / len;
    }
    return bad;
}

/* --------------------------------------------------- segment vs triangle */
/* Moller-Trumbore: does P0 + t D, t in (tmin, tmax), meet triangle (a,b,c)?
 * Inclusive barycentrics u >= 0, v >= 0, u + v <= 1 (R-VIS). */
static int seg_hits_tri(const double* P0, const double* D,
                        const double* a, const double* b, const double* c,
                        double tmin, double tmax)
{
    double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    double p[3] = {D[1] * e2[2] - D[2] * e2[1],
                   D[2] * e2[0] - D[0] * e2[2],
                   D[0] * e2[1] - D[1] * e2[0]};
    double det = e1[0] * p[0] + e1[1] * p[1] + e1[2] * p[2];
    if (fabs(det) <= OR_DET_EPS) return 0;
    double inv = 1.0 / det;
    double s[3] = {P0[0] - a[0], P0[1] - a[1], P0[2] - a[2]};
    double u = (s[0] * p[0] + s[1] * p[1] + s[2] * p[2]) * inv;
    if (u < 0.0 || u > 1.0) return 0;
    double q[3] = {s[1] * e1[2] - s[2] * e1[1],
                   s[2] * e1[0] - s[0] * e1[2],
                   s[0] * e1[1] - s[1] * e1[0]};
    double v = (D[0] * q[0] + D[1] * q[1] + D[2] * q[2]) * inv;
    if (v < 0.0 || u + v > 1.0) return 0;
    double t = (e2[0] * q[0] + e2[1] * q[1] + e2[2] * q[2]) * inv;
    return t > tmin && t < tmax;
}

/* ------------------------------------------------------------ occluders */
typedef struct {
    int64_t nt;
    const double* V;
    const int32_t* T;
    /* uniform xy grid (NULL cells => brute force) */
    int nx, ny;
    double x0, y0, cw, ch, margin, zmax_all, diag;
    int64_t* cell_ptr;   /* nx*ny+1 */
    int32_t* cell_tri;
    double* cell_zmax;
} occ_t;

static const double* tv(const occ_t* o, int64_t t, int k) { return o->V + 3 * (int64_t)o->T[3 * t + k]; }

static int blocked_bf(const occ_t* o, const double* P0, const double* D, double tmin, double tmax,
                      int64_t skip1, int64_t skip2)
{
    for (int64_t t = 0; t < o->nt; ++t) {
        if (t == skip1 || t == skip2) continue;
        if (seg_hits_tri(P0, D, tv(o, t, 0), tv(o, t, 1), tv(o, t, 2), tmin, tmax)) return 1;
    }
    return 0;
}

/* Conservative supercover of the segment's xy projection: for every grid
 * column the segment's x-range crosses, visit all cells covering the
 * segment's y-range inside that column (expanded by a margin); triangles
 * are registered in every cell their (margin-expanded) xy bbox overlaps.
 * A cell is skipped only if the segment's lowest z over the column is
 * above every vertex in that cell. */
static int blocked_grid(const occ_t* o, const double* P0, const double* D, double tmin, double tmax,
                        int64_t skip1, int64_t skip2)
{
    double xa = P0[0] + tmin * D[0], xb = P0[0] + tmax * D[0];
    double lo_x = xa < xb ? xa : xb, hi_x = xa < xb ? xb : xa;
    int ix0 = (int)floor((lo_x - o->margin - o->x0) / o->cw);
    int ix1 = (int)floor((hi_x + o->margin - o->x0) / o->cw);
    if (ix0 < 0) ix0 = 0;
    if (ix1 > o->nx - 1) ix1 = o->nx - 1;
    for (int ix = ix0; ix <= ix1; ++ix) {
        /* parameter interval of the segment inside this column */
        double cx0 = o->x0 + ix * o->cw - o->margin, cx1 = o->x0 + (ix + 1) * o->cw + o->margin;
        double ta = tmin, tb = tmax;
        if (D[0] != 0.0) {
            double t0 = (cx0 - P0[0]) / D[0], t1 = (cx1 - P0[0]) / D[0];
            if (t0 > t1) { double tt = t0; t0 = t1; t1 = tt; }
            if (t0 > ta) ta = t0;
            if (t1 < tb) tb = t1;
            if (ta > tb) continue;
        }
        double ya = P0[1] + ta * D[1], yb = P0[1] + tb * D[1];
        double za = P0[2] + ta * D[2], zb = P0[2] + tb * D[2];
        double lo_y = ya < yb ? ya : yb, hi_y = ya < yb ? yb : ya;
        double zlo = za < zb ? za : zb;
        int iy0 = (int)floor((lo_y - o->margin - o->y0) / o->ch);
        int iy1 = (int)floor((hi_y + o->margin - o->y0) / o->ch);
        if (iy0 < 0) iy0 = 0;
        if (iy1 > o->ny - 1) iy1 = o->ny - 1;
        for (int iy = iy0; iy <= iy1; ++iy) {
            int64_t c = (int64_t)ix * o->ny + iy;
            if (zlo > o->cell_zmax[c] + o->margin) continue;
            for (int64_t k = o->cell_ptr[c]; k < o->cell_ptr[c + 1]; ++k) {
                int64_t t = o->cell_tri[k];
                if (t == skip1 || t == skip2) continue;
                if (seg_hits_tri(P0, D, tv(o, t, 0), tv(o, t, 1), tv(o, t, 2), tmin, tmax)) return 1;
            }
        }
    }
    return 0;
}

static int blocked(const occ_t* o, const double* P0, const double* D, double tmin, double tmax,
                   int64_t s1, int64_t s2)
{
    return o->cell_ptr ? blocked_grid(o, P0, D, tmin, tmax, s1, s2)
                       : blocked_bf(o, P0, D, tmin, tmax, s1, s2);
}

static void occ_init(occ_t* o, int64_t nv, const double* V, int64_t nt, const int32_t* T, int grid_cells)
{
    memset(o, 0, sizeof(*o));
    o->nt = nt; o->V = V; o->T = T;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t v = 0; v < nv; ++v)
        for (int d = 0; d < 3; ++d) {
            if (V[3 * v + d] < lo[d]) lo[d] = V[3 * v + d];
            if (V[3 * v + d] > hi[d]) hi[d] = V[3 * v + d];
        }
    if (nv == 0) { for (int d = 0; d < 3; ++d) lo[d] = hi[d] = 0.0; }
    o->diag = sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                   (hi[2] - lo[2]) * (hi[2] - lo[2]));
    o->zmax_all = hi[2];
    if (grid_cells <= 0 || nt == 0) return;
    o->nx = o->ny = grid_cells;
    o->margin = 1e-9 * (o->diag > 0 ? o->diag : 1.0);
    o->x0 = lo[0]; o->y0 = lo[1];
    o->cw = (hi[0] - lo[0]) / o->nx; if (o->cw <= 0) o->cw = 1.0;
    o->ch = (hi[1] - lo[1]) / o->ny; if (o->ch <= 0) o->ch = 1.0;
    int64_t nc = (int64_t)o->nx * o->ny;
    o->cell_ptr = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    o->cell_zmax = (double*)malloc((size_t)nc * sizeof(double));
    for (int64_t c = 0; c < nc; ++c) o->cell_zmax[c] = -INFINITY;
    for (int pass = 0; pass < 2; ++pass) {
        int64_t* fill = NULL;
        if (pass == 1) {
            for (int64_t c = 0; c < nc; ++c) o->cell_ptr[c + 1] += o->cell_ptr[c];
            o->cell_tri = (int32_t*)malloc((size_t)(o->cell_ptr[nc] > 0 ? o->cell_ptr[nc] : 1) * sizeof(int32_t));
            fill = (int64_t*)malloc((size_t)nc * sizeof(int64_t));
            memcpy(fill, o->cell_ptr, (size_t)nc * sizeof(int64_t));
        }
        for (int64_t t = 0; t < nt; ++t) {
            double bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
            for (int k = 0; k < 3; ++k)
                for (int d = 0; d < 3; ++d) {
                    double v = tv(o, t, k)[d];
                    if (v < bl[d]) bl[d] = v;
                    if (v > bh[d]) bh[d] = v;
                }
            int ix0 = (int)floor((bl[0] - o->margin - o->x0) / o->cw), ix1 = (int)floor((bh[0] + o->margin - o->x0) / o->cw);
            int iy0 = (int)floor((bl[1] - o->margin - o->y0) / o->ch), iy1 = (int)floor((bh[1] + o->margin - o->y0) / o->ch);
            if (ix0 < 0) ix0 = 0;
            if (iy0 < 0) iy0 = 0;
            if (ix1 > o->nx - 1) ix1 = o->nx - 1;
            if (iy1 > o->ny - 1) iy1 = o->ny - 1;
            for (int ix = ix0; ix <= ix1; ++ix)
                for (int iy = iy0; iy <= iy1; ++iy) {
                    int64_t c = (int64_t)ix * o->ny + iy;
                    if (pass == 0) { o->cell_ptr[c + 1]++; if (bh[2] > o->cell_zmax[c]) o->cell_zmax[c] = bh[2]; }
                    else o->cell_tri[fill[c]++] = (int32_t)t;
                }
        }
        free(fill);
    }
}

static void occ_free(occ_t* o)
{
    free(o->cell_ptr); free(o->cell_tri); free(o->cell_zmax);
    memset(o, 0, sizeof(*o));
}

/* ------------------------------------------------------------- V_ij, F_ij */
/* V_ij = 1 iff n_i.d_ij > 0 and n_j.d_ji > 0 and the open segment
 * (x_i, x_j) meets no triangle other than i and j.  Facet index f maps to
 * occluder triangle index tri_of[f] (or f itself when tri_of == NULL; -1 =
 * facet is not an occluder, e.g. sphere-exact facet data). */
static int vis_pair(const occ_t* o, const double* x, const double* n, const int64_t* tri_of,
                    int64_t i, int64_t j, int cull_only)
{
    const double* xi = x + 3 * i;
    const double* xj = x + 3 * j;
    double d[3] = {xj[0] - xi[0], xj[1] - xi[1], xj[2] - xi[2]};
    double ci = n[3 * i] * d[0] + n[3 * i + 1] * d[1] + n[3 * i + 2] * d[2];
    double cj = -(n[3 * j] * d[0] + n[3 * j + 1] * d[1] + n[3 * j + 2] * d[2]);
    if (!(ci > 0.0) || !(cj > 0.0)) return 0;
    if (cull_only || o == NULL || o->nt == 0) return 1;
    int64_t ti = tri_of ? tri_of[i] : i, tj = tri_of ? tri_of[j] : j;
    return !blocked(o, xi, d, OR_T_EPS, 1.0 - OR_T_EPS, ti, tj);
}

/* P:134-136 eq. FF-def (value for a visible pair). */
static double ff_entry(const double* x, const double* n, const double* A, int64_t i, int64_t j)
{
    const double* xi = x + 3 * i;
    const double* xj = x + 3 * j;
    double d[3] = {xj[0] - xi[0], xj[1] - xi[1], xj[2] - xi[2]};
    double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    double ni_d = n[3 * i] * d[0] + n[3 * i + 1] * d[1] + n[3 * i + 2] * d[2];
    double nj_md = -(n[3 * j] * d[0] + n[3 * j + 1] * d[1] + n[3 * j + 2] * d[2]);
    return ni_d * nj_md / (M_PI * r2 * r2) * A[j];
}

/* Visibility matrix rows (uint8, nrows x N) for rows[], all columns. */
void or_visibility_rows(int64_t N, const double* x, const double* n,
                        int64_t nv, const double* V, int64_t nt, const int32_t* T,
                        const int64_t* tri_of, int cull_only, int grid_cells,
                        int64_t nrows, const int64_t* rows, uint8_t* out)
{
    occ_t o;
    occ_init(&o, nv, V, nt, T, grid_cells);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        for (int64_t j = 0; j < N; ++j)
            out[r * N + j] = (j == i) ? 0 : (uint8_t)vis_pair(&o, x, n, tri_of, i, j, cull_only);
    }
    occ_free(&o);
}

/* Dense F (row-major N x N).  F_ii = 0. */
void or_viewfactor_dense(int64_t N, const double* x, const double* n, const double* A,
                         int64_t nv, const double* V, int64_t nt, const int32_t* T,
                         const int64_t* tri_of, int cull_only, int grid_cells, double* Fout)
{
    occ_t o;
    occ_init(&o, nv, V, nt, T, grid_cells);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = 0; i < N; ++i) {
        double* row = Fout + i * N;
        for (int64_t j = 0; j < N; ++j)
            row[j] = (j != i && vis_pair(&o, x, n, tri_of, i, j, cull_only)) ? ff_entry(x, n, A, i, j) : 0.0;
    }
    occ_free(&o);
}

/* Exact CSR rows of F for rows[] (Alg. 1, "emit ... row by row").
 * Returns an opaque result; fetch with or_csr_fetch, release with or_csr_free. */
typedef struct { int64_t nrows, nnz; int64_t* cnt; int64_t** cols; double** vals; } or_csr_t;

void* or_viewfactor_csr_rows(int64_t N, const double* x, const double* n, const double* A,
                             int64_t nv, const double* V, int64_t nt, const int32_t* T,
                             const int64_t* tri_of, int cull_only, int grid_cells,
                             int64_t nrows, const int64_t* rows)
{
    occ_t o;
    occ_init(&o, nv, V, nt, T, grid_cells);
    or_csr_t* R = (or_csr_t*)calloc(1, sizeof(or_csr_t));
    R->nrows = nrows;
    R->cnt = (int64_t*)calloc((size_t)(nrows > 0 ? nrows : 1), sizeof(int64_t));
    R->cols = (int64_t**)calloc((size_t)(nrows > 0 ? nrows : 1), sizeof(int64_t*));
    R->vals = (double**)calloc((size_t)(nrows > 0 ? nrows : 1), sizeof(double*));
#pragma omp parallel
    {
        int64_t* bc = (int64_t*)malloc((size_t)(N > 0 ? N : 1) * sizeof(int64_t));
        double* bv = (double*)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
#pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < nrows; ++r) {
            int64_t i = rows[r], c = 0;
            for (int64_t j = 0; j < N; ++j)
                if (j != i && vis_pair(&o, x, n, tri_of, i, j, cull_only)) { bc[c] = j; bv[c] = ff_entry(x, n, A, i, j); ++c; }
            R->cnt[r] = c;
            R->cols[r] = (int64_t*)malloc((size_t)(c > 0 ? c : 1) * sizeof(int64_t));
            R->vals[r] = (double*)malloc((size_t)(c > 0 ? c : 1) * sizeof(double));
            memcpy(R->cols[r], bc, (size_t)c * sizeof(int64_t));
            memcpy(R->vals[r], bv, (size_t)c * sizeof(double));
        }
        free(bc); free(bv);
    }
    for (int64_t r = 0; r < nrows; ++r) R->nnz += R->cnt[r];
    occ_free(&o);
    return R;
}

int64_t or_csr_nnz(void* h) { return ((or_csr_t*)h)->nnz; }

void or_csr_fetch(void* h, int64_t* rowptr, int64_t* cols, double* vals)
{
    or_csr_t* R = (or_csr_t*)h;
    rowptr[0] = 0;
    for (int64_t r = 0; r < R->nrows; ++r) {
        memcpy(cols + rowptr[r], R->cols[r], (size_t)R->cnt[r] * sizeof(int64_t));
        memcpy(vals + rowptr[r], R->vals[r], (size_t)R->cnt[r] * sizeof(double));
        rowptr[r + 1] = rowptr[r] + R->cnt[r];
    }
}

void or_csr_free(void* h)
{
    or_csr_t* R = (or_csr_t*)h;
    for (int64_t r = 0; r < R->nrows; ++r) { free(R->cols[r]); free(R->vals[r]); }
    free(R->cnt); free(R->cols); free(R->vals); free(R);
}

/* ------------------------------------------------------------ insolation */
/* P:76-80 eq. insolation with R_sun = 1 AU: Q_ij = S max(0, n_i.s_j) V_sun.
 * sin(e) relative to the facet's tangent plane = n_i.s (reading R-SUN).
 * V_sun: the ray x_i + t s, t > 1e-9 * diag, meets no triangle but i.
 * Output column-major N x k. */
void or_insolation(int64_t N, const double* x, const double* n,
                   int64_t nv, const double* V, int64_t nt, const int32_t* T,
                   const int64_t* tri_of, int grid_cells,
                   int64_t k, const double* suns, double S, double* Q)
{
    occ_t o;
    occ_init(&o, nv, V, nt, T, grid_cells);
    double tmin = 1e-9 * (o.diag > 0 ? o.diag : 1.0);
    /* any ray leaving the mesh bbox can no longer hit it: bound t by
     * 2 * diag (the ray starts inside the bbox). */
    double tmax = 2.0 * (o.diag > 0 ? o.diag : 1.0) + 1.0;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < N; ++i) {
        for (int64_t c = 0; c < k; ++c) {
            const double* s = suns + 3 * c;
            double mu = n[3 * i] * s[0] + n[3 * i + 1] * s[1] + n[3 * i + 2] * s[2];
            double q = 0.0;
            if (mu > 0.0) {
                int64_t ti = tri_of ? tri_of[i] : i;
                if (!blocked(&o, x + 3 * i, s, tmin, tmax, ti, -1)) q = S * mu;
            }
            Q[c * N + i] = q;
        }
    }
    occ_free(&o);
}

/* ---------------------------------------------------------------- apply */
/* Y = F X for dense row-major F (N x N), X/Y column-major N x k.  Row by
 * row, j ascending (the plain sum of eq. FF-def's discrete operator). */
void or_apply_dense(int64_t N, const double* F, int64_t k, const double* X, double* Y)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i)
        for (int64_t c = 0; c < k; ++c) {
            double s = 0.0;
            const double* row = F + i * N;
            const double* xc = X + c * N;
            for (int64_t j = 0; j < N; ++j) s += row[j] * xc[j];
            Y[c * N + i] = s;
        }
}

/* Y = F X for CSR F (rowptr/cols int64), X/Y column-major N x k. */
void or_apply_csr(int64_t nrows, const int64_t* rowptr, const int64_t* cols, const double* vals,
                  int64_t N, int64_t k, const double* X, double* Y)
{
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t c = 0; c < k; ++c) {
            double s = 0.0;
            for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) s += vals[e] * X[c * N + cols[e]];
            Y[c * nrows + i] = s;
        }
}
