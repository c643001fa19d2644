// vf_svd.cpp -- numerical-rank estimation of a view-factor block (Alg. 3,
// PAPER.md P:219-232) for the host-side build.  Not on the timed path.
//
// The paper computes k-term truncated sparse SVDs with ARPACK and doubles k
// (P:222-230).  Here the k-term truncated SVD is a seeded randomized
// range finder with two power iterations (Halko-Martinsson-Tropp) on the
// block restricted to its nonzero rows/columns (reading A8), finished by a
// one-sided Jacobi SVD of the small projected matrix.  Because randomized
// singular values can be slightly low, an accepted rank q is VERIFIED: the
// spectral norm of the residual A - U_q S_q V_q^T is estimated by power
// iteration and q is raised until it is below eps * sigma_1 (DESIGN.md,
// "differences from the paper").  Small blocks (min dimension <= 48) get an
// exact one-sided Jacobi SVD instead.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "vf_internal.h"

namespace vf {
namespace {

struct Rng {
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed ? seed : 0x9e3779b97f4a7c15ull) {}
    uint64_t next() {  // splitmix64
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return ((next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
    double normal() {
        double u1 = uniform(), u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
};

// The compact block as an operator (dense row-major or CSR).
struct Op {
    int64_t m, n;
    const double* dense;
    const int64_t* rowptr;
    const int32_t* cols;
    const double* vals;
    // Y (m x l, row-major) = A X (n x l row-major)
    void mul(const double* X, int64_t l, double* Y) const {
        std::fill(Y, Y + m * l, 0.0);
        for (int64_t i = 0; i < m; ++i) {
            double* y = Y + i * l;
            if (dense) {
                const double* a = dense + i * n;
                for (int64_t j = 0; j < n; ++j) {
                    double v = a[j];
                    if (v == 0.0) continue;
                    const double* x = X + j * l;
                    for (int64_t c = 0; c < l; ++c) y[c] += v * x[c];
                }
            } else {
                for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                    double v = vals[e];
                    const double* x = X + (int64_t)cols[e] * l;
                    for (int64_t c = 0; c < l; ++c) y[c] += v * x[c];
                }
            }
        }
    }
    // Z (n x l) = A^T Y (m x l)
    void tmul(const double* Y, int64_t l, double* Z) const {
        std::fill(Z, Z + n * l, 0.0);
        for (int64_t i = 0; i < m; ++i) {
            const double* y = Y + i * l;
            if (dense) {
                const double* a = dense + i * n;
                for (int64_t j = 0; j < n; ++j) {
                    double v = a[j];
                    if (v == 0.0) continue;
                    double* z = Z + j * l;
                    for (int64_t c = 0; c < l; ++c) z[c] += v * y[c];
                }
            } else {
                for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                    double v = vals[e];
                    double* z = Z + (int64_t)cols[e] * l;
                    for (int64_t c = 0; c < l; ++c) z[c] += v * y[c];
                }
            }
        }
    }
};

// Orthonormalise the l columns of Y (m x l row-major) in place: classical
// Gram-Schmidt applied twice; columns that vanish are zeroed.
void orthonormalize(double* Y, int64_t m, int64_t l) {
    std::vector<double> col(m), dots(l);
    for (int64_t j = 0; j < l; ++j) {
        for (int64_t i = 0; i < m; ++i) col[i] = Y[i * l + j];
        double n0 = 0;
        for (int64_t i = 0; i < m; ++i) n0 += col[i] * col[i];
        n0 = std::sqrt(n0);
        for (int pass = 0; pass < 2; ++pass) {
            for (int64_t p = 0; p < j; ++p) {
                double d = 0;
                for (int64_t i = 0; i < m; ++i) d += Y[i * l + p] * col[i];
                dots[p] = d;
            }
            for (int64_t p = 0; p < j; ++p)
                for (int64_t i = 0; i < m; ++i) col[i] -= dots[p] * Y[i * l + p];
        }
        double nn = 0;
        for (int64_t i = 0; i < m; ++i) nn += col[i] * col[i];
        nn = std::sqrt(nn);
        double inv = (nn > 1e-13 * n0 && nn > 0) ? 1.0 / nn : 0.0;
        for (int64_t i = 0; i < m; ++i) Y[i * l + j] = col[i] * inv;
    }
}

// One-sided Jacobi SVD of G (m x l row-major, m >= 1): on return G holds
// U*Sigma's columns normalised to U (m x l), sig the singular values and W
// (l x l row-major) the right singular vectors, sorted descending.
void jacobi_svd(std::vector<double>& G, int64_t m, int64_t l, std::vector<double>& sig,
                std::vector<double>& W) {
    W.assign(l * l, 0.0);
    for (int64_t j = 0; j < l; ++j) W[j * l + j] = 1.0;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0;
        for (int64_t p = 0; p < l - 1; ++p)
            for (int64_t q = p + 1; q < l; ++q) {
                double a = 0, b = 0, c = 0;
                for (int64_t i = 0; i < m; ++i) {
                    double gp = G[i * l + p], gq = G[i * l + q];
                    a += gp * gp; b += gq * gq; c += gp * gq;
                }
                if (c == 0.0 || std::fabs(c) <= 1e-15 * std::sqrt(a * b)) continue;
                off = std::max(off, std::fabs(c) / std::sqrt(a * b));
                double zeta = (b - a) / (2.0 * c);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
                for (int64_t i = 0; i < m; ++i) {
                    double gp = G[i * l + p], gq = G[i * l + q];
                    G[i * l + p] = cs * gp - sn * gq;
                    G[i * l + q] = sn * gp + cs * gq;
                }
                for (int64_t i = 0; i < l; ++i) {
                    double wp = W[i * l + p], wq = W[i * l + q];
                    W[i * l + p] = cs * wp - sn * wq;
                    W[i * l + q] = sn * wp + cs * wq;
                }
            }
        if (off <= 1e-15) break;
    }
    sig.assign(l, 0.0);
    for (int64_t j = 0; j < l; ++j) {
        double s = 0;
        for (int64_t i = 0; i < m; ++i) s += G[i * l + j] * G[i * l + j];
        sig[j] = std::sqrt(s);
    }
    std::vector<int64_t> ord(l);
    for (int64_t j = 0; j < l; ++j) ord[j] = j;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return sig[a] > sig[b]; });
    std::vector<double> G2(m * l), W2(l * l), s2(l);
    for (int64_t jj = 0; jj < l; ++jj) {
        int64_t j = ord[jj];
        s2[jj] = sig[j];
        double inv = sig[j] > 0 ? 1.0 / sig[j] : 0.0;
        for (int64_t i = 0; i < m; ++i) G2[i * l + jj] = G[i * l + j] * inv;
        for (int64_t i = 0; i < l; ++i) W2[i * l + jj] = W[i * l + j];
    }
    G.swap(G2); W.swap(W2); sig.swap(s2);
}

struct Trunc {
    std::vector<double> U;   // m x l row-major
    std::vector<double> S;   // l
    std::vector<double> V;   // n x l row-major
    int64_t l = 0;
    bool exact = false;
};

Trunc exact_svd(const Op& A) {
    // dense copy, transpose so that rows >= cols
    Trunc T;
    bool tr = A.m < A.n;
    int64_t m = tr ? A.n : A.m, l = tr ? A.m : A.n;
    std::vector<double> G(m * l, 0.0);
    for (int64_t i = 0; i < A.m; ++i) {
        if (A.dense) {
            for (int64_t j = 0; j < A.n; ++j) {
                double v = A.dense[i * A.n + j];
                if (tr) G[j * l + i] = v; else G[i * l + j] = v;
            }
        } else {
            for (int64_t e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e) {
                int64_t j = A.cols[e];
                if (tr) G[j * l + i] = A.vals[e]; else G[i * l + j] = A.vals[e];
            }
        }
    }
    std::vector<double> sig, W;
    jacobi_svd(G, m, l, sig, W);
    T.l = l; T.S = sig; T.exact = true;
    if (tr) { T.U = W; T.V = G; } else { T.U = G; T.V = W; }
    return T;
}

Trunc randomized_svd(const Op& A, int64_t l, Rng& rng) {
    Trunc T;
    T.l = l;
    std::vector<double> Om(A.n * l), Y(A.m * l), Z(A.n * l);
    for (auto& v : Om) v = rng.normal();
    A.mul(Om.data(), l, Y.data());
    for (int it = 0; it < 2; ++it) {       // power iterations
        orthonormalize(Y.data(), A.m, l);
        A.tmul(Y.data(), l, Z.data());
        orthonormalize(Z.data(), A.n, l);
        A.mul(Z.data(), l, Y.data());
    }
    orthonormalize(Y.data(), A.m, l);      // Q
    A.tmul(Y.data(), l, Z.data());         // B^T = A^T Q   (n x l)
    std::vector<double> sig, W;
    jacobi_svd(Z, A.n, l, sig, W);         // B^T = V S W^T
    T.S = sig;
    T.V = Z;
    T.U.assign(A.m * l, 0.0);              // U = Q W
    for (int64_t i = 0; i < A.m; ++i)
        for (int64_t p = 0; p < l; ++p) {
            double qv = Y[i * l + p];
            if (qv == 0.0) continue;
            for (int64_t j = 0; j < l; ++j) T.U[i * l + j] += qv * W[p * l + j];
        }
    return T;
}

// Spectral norm estimate of A - U_q S_q V_q^T by power iteration.
double residual_norm(const Op& A, const Trunc& T, int64_t q, Rng& rng) {
    std::vector<double> x(A.n), y(A.m), z(A.n), c(q);
    for (auto& v : x) v = rng.normal();
    double est = 0;
    for (int it = 0; it < 24; ++it) {
        double nx = 0;
        for (double v : x) nx += v * v;
        nx = std::sqrt(nx);
        if (nx == 0) return 0;
        for (auto& v : x) v /= nx;
        A.mul(x.data(), 1, y.data());                       // y = R x
        for (int64_t p = 0; p < q; ++p) {
            double d = 0;
            for (int64_t j = 0; j < A.n; ++j) d += T.V[j * T.l + p] * x[j];
            c[p] = d * T.S[p];
        }
        for (int64_t i = 0; i < A.m; ++i) {
            double s = 0;
            for (int64_t p = 0; p < q; ++p) s += T.U[i * T.l + p] * c[p];
            y[i] -= s;
        }
        double ny = 0;
        for (double v : y) ny += v * v;
        est = std::sqrt(ny);
        A.tmul(y.data(), 1, z.data());                      // z = R^T y
        for (int64_t p = 0; p < q; ++p) {
            double d = 0;
            for (int64_t i = 0; i < A.m; ++i) d += T.U[i * T.l + p] * y[i];
            c[p] = d * T.S[p];
        }
        for (int64_t j = 0; j < A.n; ++j) {
            double s = 0;
            for (int64_t p = 0; p < q; ++p) s += T.V[j * T.l + p] * c[p];
            z[j] -= s;
        }
        x.swap(z);
    }
    return est;
}

}  // namespace

SvdResult estimate_rank(int64_t mu, int64_t nv, const double* dense, const int64_t* rowptr,
                        const int32_t* cols, const double* vals, double eps, int w, int k0,
                        int64_t target_bytes, int64_t, int64_t, uint64_t seed) {
    SvdResult R;
    Op A{mu, nv, dense, rowptr, cols, vals};
    const int64_t r = std::min(mu, nv);
    Rng rng(seed);
    auto svd_bytes = [&](int64_t q) { return (int64_t)w * q * (mu + nv) + (int64_t)w * q + 4 * (mu + nv); };
    Trunc full;
    bool have_full = false;
    if (r <= 48) { full = exact_svd(A); have_full = true; }
    for (int64_t k = k0;; k *= 2) {                          // Alg. 3 steps 2-6
        Trunc T;
        if (have_full) T = full;
        else if (std::min<int64_t>(k + 8, r) >= r) { full = exact_svd(A); have_full = true; T = full; }
        else T = randomized_svd(A, std::min<int64_t>(k + 8, r), rng);
        const int64_t kk = std::min<int64_t>(k, T.l);
        const bool complete = T.exact && kk == r;             // sigma_{r+1} = 0
        const double s1 = T.S[0];
        if (!(s1 > 0)) return R;
        int64_t q = 0;
        for (int64_t qq = 1; qq <= kk; ++qq) {                // smallest q: sigma_{q+1}/sigma_1 < eps
            double nxt;
            if (qq < kk) nxt = T.S[qq];
            else if (complete) nxt = 0.0;
            else break;
            if (nxt / s1 < eps) { q = qq; break; }
        }
        if (q > 0 && !T.exact) {                              // verify the randomized truncation
            while (q < kk && 1.2 * residual_norm(A, T, q, rng) >= eps * s1) ++q;
            if (1.2 * residual_norm(A, T, q, rng) >= eps * s1) q = 0;
        }
        if (q > 0) {
            if (svd_bytes(q) >= target_bytes) return R;         // eq. nbytes-comparison fails
            R.q = q;
            R.S.assign(T.S.begin(), T.S.begin() + q);
            R.U.resize(mu * q);
            R.V.resize(nv * q);
            for (int64_t i = 0; i < mu; ++i)
                for (int64_t p = 0; p < q; ++p) R.U[i * q + p] = T.U[i * T.l + p];
            for (int64_t j = 0; j < nv; ++j)
                for (int64_t p = 0; p < q; ++p) R.V[j * q + p] = T.V[j * T.l + p];
            return R;
        }
        // reading A5: stop once k >= min(m,n)/2 or w k (m+n) >= nbytes(F_IJ)
        if (2 * k >= r || (int64_t)w * k * (mu + nv) >= target_bytes || complete) return R;
    }
}

}  // namespace vf
