// vf_build.cpp -- host-side assembly of the compressed view-factor matrix
// F-hat (PAPER.md = "P:<line>").  Untimed support for the hot path:
//   facet data, BVH ray casting for V_ij, Alg. 1 CSR
//   blocks, Alg. 2 quadtree, Alg. 3 rank estimation
//   (vf_svd.cpp), Alg. 4 dynamic-programming assembly, and the
//   insolation used as input generation.
// Readings of the paper (A1..A26, R-*) are listed in DESIGN.md.
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include "vf_internal.h"

namespace vf {
namespace {

constexpr double kTEps = 1e-9;      // open-segment margin (reading R-VIS / A18)
constexpr double kDetEps = 1e-300;  // parallel ray/triangle
constexpr int64_t kNodeOverhead = 64;

// ------------------------------------------------------------------ BVH
struct Bvh {
    struct NodeB { double lo[3], hi[3]; int32_t left, right, first, count; };
    std::vector<NodeB> nodes;
    std::vector<int32_t> order;      // triangle ids in leaf order
    const double* V = nullptr;
    const int32_t* F = nullptr;
    double margin = 0, diag = 0;

    void build(const double* Vp, int64_t nv, const int32_t* Fp, int64_t nt) {
        V = Vp; F = Fp;
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t v = 0; v < nv; ++v)
            for (int d = 0; d < 3; ++d) { lo[d] = std::min(lo[d], V[3 * v + d]); hi[d] = std::max(hi[d], V[3 * v + d]); }
        diag = nv ? std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                              (hi[2] - lo[2]) * (hi[2] - lo[2])) : 0.0;
        margin = 1e-9 * (diag > 0 ? diag : 1.0);
        order.resize(nt);
        std::iota(order.begin(), order.end(), 0);
        nodes.clear();
        if (nt == 0) return;
        std::vector<double> cen(3 * nt);
        for (int64_t t = 0; t < nt; ++t)
            for (int d = 0; d < 3; ++d)
                cen[3 * t + d] = (V[3 * F[3 * t] + d] + V[3 * F[3 * t + 1] + d] + V[3 * F[3 * t + 2] + d]) / 3.0;
        nodes.reserve(2 * nt);
        split(0, (int32_t)nt, cen, 0);
    }
    int32_t split(int32_t first, int32_t count, const std::vector<double>& cen, int depth) {
        int32_t id = (int32_t)nodes.size();
        nodes.push_back(NodeB{});
        NodeB nb;
        for (int d = 0; d < 3; ++d) { nb.lo[d] = INFINITY; nb.hi[d] = -INFINITY; }
        double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int32_t k = first; k < first + count; ++k) {
            int32_t t = order[k];
            for (int c = 0; c < 3; ++c)
                for (int d = 0; d < 3; ++d) {
                    double v = V[3 * F[3 * t + c] + d];
                    nb.lo[d] = std::min(nb.lo[d], v); nb.hi[d] = std::max(nb.hi[d], v);
                }
            for (int d = 0; d < 3; ++d) { clo[d] = std::min(clo[d], cen[3 * t + d]); chi[d] = std::max(chi[d], cen[3 * t + d]); }
        }
        for (int d = 0; d < 3; ++d) { nb.lo[d] -= margin; nb.hi[d] += margin; }
        nb.left = nb.right = -1; nb.first = first; nb.count = count;
        if (count > 4 && depth < 60) {
            int ax = 0;
            for (int d = 1; d < 3; ++d) if (chi[d] - clo[d] > chi[ax] - clo[ax]) ax = d;
            if (chi[ax] > clo[ax]) {
                int32_t mid = first + count / 2;
                std::nth_element(order.begin() + first, order.begin() + mid, order.begin() + first + count,
                                 [&](int32_t a, int32_t b) { return cen[3 * a + ax] < cen[3 * b + ax]; });
                nb.left = split(first, mid - first, cen, depth + 1);
                nb.right = split(mid, first + count - mid, cen, depth + 1);
                nb.count = 0;
            }
        }
        nodes[id] = nb;
        return id;
    }
    // Moller-Trumbore, inclusive barycentrics, t in (tmin, tmax)
    bool hit_tri(const double* P, const double* D, int32_t t, double tmin, double tmax) const {
        const double* a = V + 3 * F[3 * t];
        const double* b = V + 3 * F[3 * t + 1];
        const double* c = V + 3 * F[3 * t + 2];
        double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        double p[3] = {D[1] * e2[2] - D[2] * e2[1], D[2] * e2[0] - D[0] * e2[2], D[0] * e2[1] - D[1] * e2[0]};
        double det = e1[0] * p[0] + e1[1] * p[1] + e1[2] * p[2];
        if (std::fabs(det) <= kDetEps) return false;
        double inv = 1.0 / det;
        double s[3] = {P[0] - a[0], P[1] - a[1], P[2] - a[2]};
        double u = (s[0] * p[0] + s[1] * p[1] + s[2] * p[2]) * inv;
        if (u < 0.0 || u > 1.0) return false;
        double q[3] = {s[1] * e1[2] - s[2] * e1[1], s[2] * e1[0] - s[0] * e1[2], s[0] * e1[1] - s[1] * e1[0]};
        double v = (D[0] * q[0] + D[1] * q[1] + D[2] * q[2]) * inv;
        if (v < 0.0 || u + v > 1.0) return false;
        double tt = (e2[0] * q[0] + e2[1] * q[1] + e2[2] * q[2]) * inv;
        return tt > tmin && tt < tmax;
    }
    static bool hit_box(const NodeB& nb, const double* P, const double* inv, double tmin, double tmax) {
        for (int d = 0; d < 3; ++d) {
            if (std::isinf(inv[d])) {
                if (P[d] < nb.lo[d] || P[d] > nb.hi[d]) return false;
                continue;
            }
            double t0 = (nb.lo[d] - P[d]) * inv[d], t1 = (nb.hi[d] - P[d]) * inv[d];
            if (t0 > t1) std::swap(t0, t1);
            tmin = std::max(tmin, t0);
            tmax = std::min(tmax, t1);
            if (tmin > tmax) return false;
        }
        return true;
    }
    // any triangle except skip1/skip2 met by P + t D, t in (tmin, tmax)?
    bool occluded(const double* P, const double* D, double tmin, double tmax, int64_t skip1, int64_t skip2) const {
        if (nodes.empty()) return false;
        double inv[3];
        for (int d = 0; d < 3; ++d) inv[d] = 1.0 / D[d];
        int32_t stack[128];
        int sp = 0;
        stack[sp++] = 0;
        while (sp) {
            const NodeB& nb = nodes[stack[--sp]];
            if (!hit_box(nb, P, inv, tmin * (1 - 1e-12) - margin, tmax * (1 + 1e-12) + margin)) continue;
            if (nb.left < 0) {
                for (int32_t k = nb.first; k < nb.first + nb.count; ++k) {
                    int32_t t = order[k];
                    if (t == skip1 || t == skip2) continue;
                    if (hit_tri(P, D, t, tmin, tmax)) return true;
                }
            } else {
                stack[sp++] = nb.left;
                stack[sp++] = nb.right;
            }
        }
        return false;
    }
};

// ------------------------------------------------------------- quadtree
struct QNode { int64_t start, stop; int depth; std::vector<int> kids; };

struct QuadTree {
    std::vector<QNode> nodes;
    std::vector<int32_t> perm;
    // Alg. 2, readings A1 (split at the midpoint, ties to the
    // upper half), A2 (one root), A3 (stop at max_depth or <= min_leaf).
    int build(const double* x, std::vector<int32_t> idx, int depth, int max_depth, int min_leaf) {
        int id = (int)nodes.size();
        nodes.push_back(QNode{(int64_t)perm.size(), 0, depth, {}});
        if (depth >= max_depth || (int64_t)idx.size() <= min_leaf) {
            std::sort(idx.begin(), idx.end());
            perm.insert(perm.end(), idx.begin(), idx.end());
            nodes[id].stop = (int64_t)perm.size();
            return id;
        }
        double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
        for (int32_t i : idx) {
            xmin = std::min(xmin, x[3 * i]); xmax = std::max(xmax, x[3 * i]);
            ymin = std::min(ymin, x[3 * i + 1]); ymax = std::max(ymax, x[3 * i + 1]);
        }
        double xmid = 0.5 * (xmin + xmax), ymid = 0.5 * (ymin + ymax);
        std::vector<int32_t> part[4];
        for (int32_t i : idx) {
            bool hx = x[3 * i] >= xmid, hy = x[3 * i + 1] >= ymid;
            part[(hx ? 2 : 0) + (hy ? 1 : 0)].push_back(i);     // I1..I4 of step 4
        }
        for (int c = 0; c < 4; ++c)
            if (!part[c].empty()) {
                int k = build(x, std::move(part[c]), depth + 1, max_depth, min_leaf);
                nodes[id].kids.push_back(k);
            }
        nodes[id].stop = (int64_t)perm.size();
        return id;
    }
};

// ------------------------------------------------------------- CSR blocks
struct Csr {                        // rows [0,m), local cols [0,n)
    int64_t m = 0, n = 0;
    std::vector<int64_t> rowptr;
    std::vector<int32_t> cols;
    std::vector<double> vals;
    int64_t nnz() const { return rowptr.empty() ? 0 : rowptr.back(); }
    Csr slice(int64_t r0, int64_t r1, int64_t c0, int64_t c1) const {
        Csr s;
        s.m = r1 - r0; s.n = c1 - c0;
        s.rowptr.assign(s.m + 1, 0);
        for (int64_t i = r0; i < r1; ++i) {
            auto b = cols.begin() + rowptr[i], e = cols.begin() + rowptr[i + 1];
            auto lo = std::lower_bound(b, e, (int32_t)c0), hi = std::lower_bound(b, e, (int32_t)c1);
            for (auto it = lo; it != hi; ++it) {
                s.cols.push_back((int32_t)(*it - c0));
                s.vals.push_back(vals[it - cols.begin()]);
            }
            s.rowptr[i - r0 + 1] = (int64_t)s.cols.size();
        }
        return s;
    }
};

int64_t bytes_dense(int64_t m, int64_t n, int w) { return (int64_t)w * m * n; }
int64_t bytes_csr(int64_t m, int64_t nnz, int w) { return 8 * (m + 1) + 4 * nnz + (int64_t)w * nnz; }
int64_t bytes_svd(int64_t q, int64_t mu, int64_t nv, int w) {
    return (int64_t)w * q * (mu + nv) + (int64_t)w * q + 4 * (mu + nv);
}

struct TreeBlock {                   // result of Alg. 4 for one block pair
    Leaf leaf;                       // kind K_ZERO/DENSE/CSR/SVD, or K_SUB
    std::vector<TreeBlock> kids;
    int64_t nbytes = 0;
};

struct Builder {
    const double* x; const double* nrm; const double* A;
    int64_t N;
    const Bvh* bvh;
    const int64_t* tri_of;
    bool cull_only;
    double tol;
    int w;
    int dtype;
    int64_t min_block;
    int k0;
    uint64_t seed;
    const QuadTree* qt;
    int64_t visible = 0;

    double rnd(double v) const { return dtype == VF_F32 ? (double)(float)v : v; }

    // Alg. 1 for rows I x cols J (tree order), CSR with local cols.
    Csr assemble_csr(const QNode& I, const QNode& J) {
        Csr c;
        c.m = I.stop - I.start; c.n = J.stop - J.start;
        std::vector<std::vector<int32_t>> rc(c.m);
        std::vector<std::vector<double>> rv(c.m);
#pragma omp parallel for schedule(dynamic, 8)
        for (int64_t r = 0; r < c.m; ++r) {
            int64_t i = qt->perm[I.start + r];
            const double* xi = x + 3 * i;
            const double* ni = nrm + 3 * i;
            for (int64_t cc = 0; cc < c.n; ++cc) {
                int64_t j = qt->perm[J.start + cc];
                if (j == i) continue;
                const double* xj = x + 3 * j;
                const double* nj = nrm + 3 * j;
                double d[3] = {xj[0] - xi[0], xj[1] - xi[1], xj[2] - xi[2]};
                double ci = ni[0] * d[0] + ni[1] * d[1] + ni[2] * d[2];
                double cj = -(nj[0] * d[0] + nj[1] * d[1] + nj[2] * d[2]);
                if (!(ci > 0.0) || !(cj > 0.0)) continue;          // culling
                if (!cull_only &&
                    bvh->occluded(xi, d, kTEps, 1.0 - kTEps, tri_of ? tri_of[i] : i, tri_of ? tri_of[j] : j))
                    continue;
                double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
                rc[r].push_back((int32_t)cc);                      // eq. FF-def
                rv[r].push_back(ci * cj / (M_PI * r2 * r2) * A[j]);
            }
        }
        c.rowptr.assign(c.m + 1, 0);
        for (int64_t r = 0; r < c.m; ++r) c.rowptr[r + 1] = c.rowptr[r] + (int64_t)rc[r].size();
        c.cols.reserve(c.nnz());
        c.vals.reserve(c.nnz());
        for (int64_t r = 0; r < c.m; ++r) {
            c.cols.insert(c.cols.end(), rc[r].begin(), rc[r].end());
            c.vals.insert(c.vals.end(), rv[r].begin(), rv[r].end());
        }
        return c;
    }

    Leaf make_leaf(int kind, const QNode& I, const QNode& J, const Csr& c, int level) {
        Leaf L;
        L.kind = kind; L.level = level;
        L.row0 = I.start; L.m = c.m; L.col0 = J.start; L.n = c.n;
        if (kind == K_DENSE) {
            L.a.assign(c.m * c.n, 0.0);
            for (int64_t r = 0; r < c.m; ++r)
                for (int64_t e = c.rowptr[r]; e < c.rowptr[r + 1]; ++e) L.a[r * c.n + c.cols[e]] = rnd(c.vals[e]);
            L.nbytes = bytes_dense(c.m, c.n, w);
        } else if (kind == K_CSR) {
            L.rowptr = c.rowptr;
            L.idx_a = c.cols;
            L.a.resize(c.vals.size());
            for (size_t e = 0; e < c.vals.size(); ++e) L.a[e] = rnd(c.vals[e]);
            L.nbytes = bytes_csr(c.m, c.nnz(), w);
        }
        return L;
    }

    // Alg. 4.
    TreeBlock assemble(int Ii, int Jj, const Csr& c, int level) {
        const QNode& I = qt->nodes[Ii];
        const QNode& J = qt->nodes[Jj];
        TreeBlock out;
        const int64_t m = c.m, n = c.n, nnz = c.nnz();
        if (nnz == 0) {                                            // A11: zero block
            out.leaf.kind = K_ZERO; out.leaf.level = level;
            out.leaf.row0 = I.start; out.leaf.m = m; out.leaf.col0 = J.start; out.leaf.n = n;
            return out;
        }
        const int64_t b_csr = bytes_csr(m, nnz, w), b_den = bytes_dense(m, n, w);
        const int best_leaf = b_csr <= b_den ? K_CSR : K_DENSE;   // tie -> CSR (A25)
        if (m * n < min_block || I.kids.empty() || J.kids.empty()) {  // step 2
            out.leaf = make_leaf(best_leaf, I, J, c, level);
            out.nbytes = out.leaf.nbytes;
            return out;
        }
        // step 3: rank estimate on the block restricted to nonzero rows/cols (A8)
        std::vector<int32_t> urows, vrows, cmap(n, -1);
        for (int64_t r = 0; r < m; ++r)
            if (c.rowptr[r + 1] > c.rowptr[r]) urows.push_back((int32_t)r);
        {
            std::vector<char> used(n, 0);
            for (int32_t cc : c.cols) used[cc] = 1;
            for (int64_t j = 0; j < n; ++j)
                if (used[j]) { cmap[j] = (int32_t)vrows.size(); vrows.push_back((int32_t)j); }
        }
        const int64_t mu = (int64_t)urows.size(), nv = (int64_t)vrows.size();
        std::vector<int64_t> crp(mu + 1, 0);
        std::vector<int32_t> ccol;
        std::vector<double> cval;
        ccol.reserve(nnz); cval.reserve(nnz);
        for (int64_t k = 0; k < mu; ++k) {
            int64_t r = urows[k];
            for (int64_t e = c.rowptr[r]; e < c.rowptr[r + 1]; ++e) { ccol.push_back(cmap[c.cols[e]]); cval.push_back(c.vals[e]); }
            crp[k + 1] = (int64_t)ccol.size();
        }
        std::vector<double> dense;
        if ((double)nnz > 0.25 * (double)mu * (double)nv) {
            dense.assign(mu * nv, 0.0);
            for (int64_t k = 0; k < mu; ++k)
                for (int64_t e = crp[k]; e < crp[k + 1]; ++e) dense[k * nv + ccol[e]] = cval[e];
        }
        uint64_t bseed = seed ^ (0x9e3779b97f4a7c15ull * (uint64_t)(I.start * 1000003 + J.start * 7919 + m * 31 + n));
        SvdResult svd = estimate_rank(mu, nv, dense.empty() ? nullptr : dense.data(), crp.data(), ccol.data(),
                                      cval.data(), tol, w, k0, b_csr, m, n, bseed);
        // step 4: recurse on the children pairs, slicing the CSR (never re-ray-tracing)
        std::vector<TreeBlock> kids;
        int64_t b_sub = kNodeOverhead;
        for (int ci : I.kids)
            for (int cj : J.kids) {
                const QNode& Ic = qt->nodes[ci];
                const QNode& Jc = qt->nodes[cj];
                Csr s = c.slice(Ic.start - I.start, Ic.stop - I.start, Jc.start - J.start, Jc.stop - J.start);
                kids.push_back(assemble(ci, cj, s, level + 1));
                b_sub += kids.back().nbytes;
            }
        // step 5: fewest bytes (ties in the order CSR < dense < SVD < subdivided)
        int kind = K_CSR;
        int64_t best = b_csr;
        if (b_den < best) { best = b_den; kind = K_DENSE; }
        int64_t b_svd = svd.q ? bytes_svd(svd.q, mu, nv, w) : INT64_MAX;
        if (b_svd < best) { best = b_svd; kind = K_SVD; }
        if (b_sub < best) { best = b_sub; kind = K_SUB; }
        if (kind == K_SVD) {
            Leaf& L = out.leaf;
            L.kind = K_SVD; L.level = level;
            L.row0 = I.start; L.m = m; L.col0 = J.start; L.n = n;
            L.q = svd.q;
            L.idx_a = urows; L.idx_b = vrows;
            L.s.resize(svd.q); L.a.resize(svd.U.size()); L.b.resize(svd.V.size());
            for (int64_t p = 0; p < svd.q; ++p) L.s[p] = rnd(svd.S[p]);
            for (size_t e = 0; e < svd.U.size(); ++e) L.a[e] = rnd(svd.U[e]);
            for (size_t e = 0; e < svd.V.size(); ++e) L.b[e] = rnd(svd.V[e]);
            L.nbytes = b_svd;
            out.nbytes = b_svd;
            return out;
        }
        if (kind == K_CSR || kind == K_DENSE) {
            out.leaf = make_leaf(kind, I, J, c, level);
            out.nbytes = out.leaf.nbytes;
            return out;
        }
        // step 6: coalesce all-CSR (or all-dense) children; Zero fits either (A10)
        bool any_csr = false, any_den = false, other = false;
        for (auto& k : kids) {
            int kk = k.leaf.kind;
            if (kk == K_CSR) any_csr = true;
            else if (kk == K_DENSE) any_den = true;
            else if (kk != K_ZERO) other = true;
        }
        if (!other && any_csr && !any_den) { out.leaf = make_leaf(K_CSR, I, J, c, level); out.nbytes = out.leaf.nbytes; return out; }
        if (!other && any_den && !any_csr) { out.leaf = make_leaf(K_DENSE, I, J, c, level); out.nbytes = out.leaf.nbytes; return out; }
        out.leaf.kind = K_SUB; out.leaf.level = level;
        out.leaf.row0 = I.start; out.leaf.m = m; out.leaf.col0 = J.start; out.leaf.n = n;
        out.kids = std::move(kids);
        out.nbytes = b_sub;
        return out;
    }
};

void flatten(const TreeBlock& b, std::vector<Leaf>& out) {
    if (b.leaf.kind == K_SUB) {
        for (auto& k : b.kids) flatten(k, out);
    } else if (b.leaf.kind != K_ZERO) {
        out.push_back(b.leaf);
    }
}

}  // namespace

int64_t leaf_nbytes(const Leaf& L, int w) {
    switch (L.kind) {
        case K_DENSE: return bytes_dense(L.m, L.n, w);
        case K_CSR: return bytes_csr(L.m, (int64_t)L.idx_a.size(), w);
        case K_SVD: return bytes_svd(L.q, (int64_t)L.idx_a.size(), (int64_t)L.idx_b.size(), w);
        default: return 0;
    }
}

int build_handle(Handle* h, int64_t N, const double* x, const double* n, const double* A,
                 const double* occV, int64_t nv, const int32_t* occF, int64_t nt,
                 const int64_t* tri_of, double tol, const vf_build_opts& o) {
    auto t0 = std::chrono::steady_clock::now();
    if (o.threads > 0) omp_set_num_threads(o.threads);
    h->N = N;
    h->dtype = o.dtype;
    h->tol = tol;
    h->x.assign(x, x + 3 * N);
    h->nrm.assign(n, n + 3 * N);
    h->A.assign(A, A + N);
    if (occV && occF && nt > 0) {
        h->occ_V.assign(occV, occV + 3 * nv);
        h->occ_F.assign(occF, occF + 3 * nt);
    }
    if (tri_of) h->tri_of.assign(tri_of, tri_of + N);
    h->has_mesh = true;

    Bvh bvh;
    bvh.build(h->occ_V.data(), nv, h->occ_F.data(), (int64_t)h->occ_F.size() / 3);

    QuadTree qt;
    std::vector<int32_t> all(N);
    std::iota(all.begin(), all.end(), 0);
    qt.nodes.reserve(4 * N / std::max(1, o.min_leaf) + 16);
    qt.build(h->x.data(), std::move(all), 0, o.max_depth, o.min_leaf);
    h->perm = qt.perm;

    Builder B{h->x.data(), h->nrm.data(), h->A.data(), N, &bvh,
              h->tri_of.empty() ? nullptr : h->tri_of.data(),
              o.visibility == VF_VIS_CULL_ONLY || h->occ_F.empty(), tol,
              o.dtype == VF_F32 ? 4 : 8, o.dtype, o.min_block, o.k0, o.seed, &qt};
    // Alg. 4 on the first-level block pairs (<= 16 for a quadtree),
    // one at a time so only one first-level CSR block is ever held.
    std::vector<int> level1 = qt.nodes[0].kids;
    if (level1.empty()) level1.push_back(0);
    h->leaves.clear();
    for (int I : level1)
        for (int J : level1) {
            Csr c = B.assemble_csr(qt.nodes[I], qt.nodes[J]);
            B.visible += c.nnz();
            TreeBlock tb = B.assemble(I, J, c, 1);
            flatten(tb, h->leaves);
        }
    h->visible_pairs = B.visible;
    h->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return VF_OK;
}

// P:76-80 eq. insolation, R_sun = 1 AU: Q = S max(0, n.s) V_sun (reading R-SUN).
int insolation(const Handle* h, const double* suns, int k, double S, double* Q) {
    if (!h->has_mesh) return set_error(VF_EUNSUPPORTED, "vf_insolation: handle has no mesh (loaded from file)");
    Bvh bvh;
    int64_t nt = (int64_t)h->occ_F.size() / 3;
    bvh.build(h->occ_V.data(), (int64_t)h->occ_V.size() / 3, h->occ_F.data(), nt);
    const double tmin = 1e-9 * (bvh.diag > 0 ? bvh.diag : 1.0);
    const double tmax = 2.0 * (bvh.diag > 0 ? bvh.diag : 1.0) + 1.0;
    const int64_t N = h->N;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < N; ++i) {
        for (int c = 0; c < k; ++c) {
            const double* s = suns + 3 * c;
            const double* ni = h->nrm.data() + 3 * i;
            double mu = ni[0] * s[0] + ni[1] * s[1] + ni[2] * s[2];
            double q = 0.0;
            if (mu > 0.0) {
                int64_t ti = h->tri_of.empty() ? i : h->tri_of[i];
                if (!bvh.occluded(h->x.data() + 3 * i, s, tmin, tmax, ti, -1)) q = S * mu;
            }
            Q[(int64_t)c * N + i] = q;
        }
    }
    return VF_OK;
}

}  // namespace vf
