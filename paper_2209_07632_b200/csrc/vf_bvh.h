// vf_bvh.h -- FP64 bounding-volume hierarchy over the occluder triangles and
// the visibility predicate V_ij of P:164-173 (§3.2), reading R-VIS / A18:
// Moller-Trumbore in FP64, t in (1e-9, 1 - 1e-9) of the segment x_i -> x_j,
// inclusive barycentrics, |det| <= 1e-300 = parallel, triangles of i and j
// excluded.  Used by the host build (vf_build.cpp) and, flattened, by the
// device evaluator (vf_build_gpu.cu), which repeats hit_tri's arithmetic
// operation for operation so both builds take identical decisions.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

namespace vf {

constexpr double kTEps = 1e-9;      // open-segment margin (reading R-VIS / A18)
constexpr double kDetEps = 1e-300;  // parallel ray/triangle

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


}  // namespace vf
