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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include "vf_bvh.h"
#include "vf_internal.h"

namespace vf {
namespace {

constexpr int64_t kNodeOverhead = 64;

// ------------------------------------------------------------- quadtree
struct QNode { int64_t start, stop; int depth; std::vector<int> kids; };

struct QuadTree {
    std::vector<QNode> nodes;
    std::vector<int32_t> perm;
    // Alg. 2, readings A1 (split at the midpoint, ties to the
    // upper half), A2 (one root), A3 (stop at max_depth or <= min_leaf).
    // dims = 3: the octree, split also at z_mid; children ordered
    // by (x, y, z) half with x slowest (reading A1 in 3D).
    int dims = 2;
    int build(const double* x, std::vector<int32_t> idx, int depth, int max_depth, int min_leaf) {
        int id = (int)nodes.size();
        nodes.push_back(QNode{(int64_t)perm.size(), 0, depth, {}});
        if (depth >= max_depth || (int64_t)idx.size() <= min_leaf) {
            std::sort(idx.begin(), idx.end());
            perm.insert(perm.end(), idx.begin(), idx.end());
            nodes[id].stop = (int64_t)perm.size();
            return id;
        }
        double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY, zmin = INFINITY, zmax = -INFINITY;
        for (int32_t i : idx) {
            xmin = std::min(xmin, x[3 * i]); xmax = std::max(xmax, x[3 * i]);
            ymin = std::min(ymin, x[3 * i + 1]); ymax = std::max(ymax, x[3 * i + 1]);
            zmin = std::min(zmin, x[3 * i + 2]); zmax = std::max(zmax, x[3 * i + 2]);
        }
        double xmid = 0.5 * (xmin + xmax), ymid = 0.5 * (ymin + ymax), zmid = 0.5 * (zmin + zmax);
        std::vector<int32_t> part[8];
        for (int32_t i : idx) {
            bool hx = x[3 * i] >= xmid, hy = x[3 * i + 1] >= ymid;
            if (dims == 3) part[(hx ? 4 : 0) + (hy ? 2 : 0) + (x[3 * i + 2] >= zmid ? 1 : 0)].push_back(i);
            else part[(hx ? 2 : 0) + (hy ? 1 : 0)].push_back(i);     // I1..I4 of step 4
        }
        for (int c = 0; c < (dims == 3 ? 8 : 4); ++c)
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
        // steps 3 and 4 are independent: the rank estimate of this block and
        // the recursion on its children pairs (slicing the CSR, never
        // re-ray-tracing) run as concurrent OpenMP tasks.
        // Alg. 3's byte test is against nbytes(F_IJ) as CSR (eq. nbytes-comparison);
        // the doubling is cut at min(CSR, dense) bytes instead: step 5 takes the
        // SVD only below both, and the smallest passing q is reached either way,
        // so the chosen leaves are identical while dense, not-low-rank blocks
        // stop doubling at k ~ min(m', n')/2 instead of running to a full SVD.
        SvdResult svd;
        const int64_t b_svd_cap = std::min(b_csr, b_den);
#pragma omp task shared(svd, dense, crp, ccol, cval) if (m * n >= 16 * min_block)
        svd = estimate_rank(mu, nv, dense.empty() ? nullptr : dense.data(), crp.data(), ccol.data(), cval.data(), tol,
                            w, k0, b_svd_cap, m, n, bseed);
        std::vector<TreeBlock> kids(I.kids.size() * J.kids.size());
        for (size_t a = 0; a < I.kids.size(); ++a)
            for (size_t b = 0; b < J.kids.size(); ++b) {
                const int ci = I.kids[a], cj = J.kids[b];
                const QNode& Ic = qt->nodes[ci];
                const QNode& Jc = qt->nodes[cj];
#pragma omp task shared(kids, c) if ((Ic.stop - Ic.start) * (Jc.stop - Jc.start) >= 16 * min_block)
                {
                    Csr s = c.slice(Ic.start - I.start, Ic.stop - I.start, Jc.start - J.start, Jc.stop - J.start);
                    kids[a * J.kids.size() + b] = assemble(ci, cj, s, level + 1);
                }
            }
#pragma omp taskwait
        int64_t b_sub = kNodeOverhead;
        for (auto& k : kids) b_sub += k.nbytes;
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
    qt.dims = o.tree == VF_TREE_OCT ? 3 : 2;
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
    // Alg. 1 for all pairs on the device (NEXT-2) when a device is given:
    // one tree-order CSR of the exact F, sliced per block below.
    const bool on_gpu = o.evaluator == VF_EVAL_DEVICE || (o.evaluator == VF_EVAL_AUTO && o.device >= 0);
    Csr global;
    if (on_gpu) {
        if (o.device < 0) return set_error(VF_EINVAL, "evaluator VF_EVAL_DEVICE needs opts.device >= 0");
        std::vector<double> xt(3 * N), nt(3 * N), At(N);
        std::vector<int64_t> tt(N);
        for (int64_t r = 0; r < N; ++r) {
            const int64_t i = qt.perm[r];
            for (int d = 0; d < 3; ++d) { xt[3 * r + d] = h->x[3 * i + d]; nt[3 * r + d] = h->nrm[3 * i + d]; }
            At[r] = h->A[i];
            tt[r] = h->tri_of.empty() ? i : h->tri_of[i];
        }
        global.m = global.n = N;
        int rc = gpu_exact_csr(o.device, N, xt.data(), nt.data(), At.data(), tt.data(), B.cull_only ? nullptr : &bvh,
                               global.rowptr, global.cols, global.vals);
        if (rc) return rc;
        if (getenv("VF_BUILD_PROFILE"))
            fprintf(stderr, "[vf build] device evaluator: N %ld nnz %ld, %.2f s since start\n", (long)N,
                    (long)global.cols.size(),
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    // Alg. 1 per first-level pair (host rays are parallel over rows inside),
    // then Alg. 3-4 on the pairs in parallel (largest first; each pair's
    // randomized SVDs are seeded by the block, so the result does not depend
    // on the schedule); leaves are emitted in pair order.
    std::vector<std::pair<int, int>> pairs;
    for (int I : level1)
        for (int J : level1) pairs.push_back({I, J});
    std::vector<Csr> blocks(pairs.size());
    for (size_t p = 0; p < pairs.size(); ++p) {
        const QNode& In = qt.nodes[pairs[p].first];
        const QNode& Jn = qt.nodes[pairs[p].second];
        blocks[p] = on_gpu ? global.slice(In.start, In.stop, Jn.start, Jn.stop) : B.assemble_csr(In, Jn);
        B.visible += blocks[p].nnz();
    }
    { Csr().rowptr.swap(global.rowptr); std::vector<int32_t>().swap(global.cols); std::vector<double>().swap(global.vals); }
    std::vector<size_t> order(pairs.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        return blocks[a].m * blocks[a].n > blocks[b].m * blocks[b].n;
    });
    std::vector<TreeBlock> result(pairs.size());
    g_svd_device = on_gpu ? o.device : -1;          // large rank searches on the device
#pragma omp parallel
#pragma omp single
    for (size_t k = 0; k < order.size(); ++k) {
        const size_t p = order[k];
#pragma omp task shared(result, blocks, pairs)
        {
            auto tp = std::chrono::steady_clock::now();
            result[p] = B.assemble(pairs[p].first, pairs[p].second, blocks[p], 1);
            if (getenv("VF_BUILD_PROFILE"))
                fprintf(stderr, "[vf build] pair %zu (%ld x %ld, nnz %ld): %.2f s, done at %.2f s\n", p,
                        (long)blocks[p].m, (long)blocks[p].n, (long)blocks[p].nnz(),
                        std::chrono::duration<double>(std::chrono::steady_clock::now() - tp).count(),
                        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
            Csr().rowptr.swap(blocks[p].rowptr);
        }
    }
    for (auto& tb : result) flatten(tb, h->leaves);
    h->visible_pairs = B.visible;
    svd_profile_report();
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
