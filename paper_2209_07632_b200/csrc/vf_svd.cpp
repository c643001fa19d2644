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
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "vf_internal.h"

namespace vf {
namespace {

// optional build profile (VF_BUILD_PROFILE=1): seconds per SVD stage
std::atomic<long long> g_ns[8];
std::atomic<long long> g_cnt[8];
struct Prof {
    int i;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit Prof(int k) : i(k) {}
    ~Prof() {
        g_ns[i] += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
        g_cnt[i]++;
    }
};


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

// The compact block as an operator (dense row-major or CSR) and its
// transpose (built once per block), so that both A X and A^T Y are row-
// parallel products over row-major X (l contiguous values per row).
constexpr int64_t kParWork = 1 << 15;    // multiply-adds below which loops stay serial
constexpr int64_t kGpuSvdWork = 1ll << 25; // nnz x l above which the SVD runs on the device

struct Op {
    int64_t m, n;
    const double* dense;
    const int64_t* rowptr;
    const int32_t* cols;
    const double* vals;
    // transpose (n x m)
    std::vector<double> dT;
    std::vector<int64_t> rpT;
    std::vector<int32_t> colT;
    std::vector<double> valT;

    void build_transpose() {
        if (dense) {
            dT.resize(m * n);
            for (int64_t i = 0; i < m; ++i)
                for (int64_t j = 0; j < n; ++j) dT[j * m + i] = dense[i * n + j];
            return;
        }
        const int64_t nnz = rowptr[m];
        rpT.assign(n + 1, 0);
        for (int64_t e = 0; e < nnz; ++e) rpT[cols[e] + 1]++;
        for (int64_t j = 0; j < n; ++j) rpT[j + 1] += rpT[j];
        colT.resize(nnz);
        valT.resize(nnz);
        std::vector<int64_t> pos(rpT.begin(), rpT.end() - 1);
        for (int64_t i = 0; i < m; ++i)
            for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                const int64_t q = pos[cols[e]]++;
                colT[q] = (int32_t)i;
                valT[q] = vals[e];
            }
    }
    static void spmm(int64_t rows, int64_t ncols, const double* dn, const int64_t* rp, const int32_t* ci,
                     const double* vv, const double* X, int64_t l, double* Y) {
        const int64_t work = (dn ? rows * ncols : (rp ? rp[rows] : 0)) * l;
#pragma omp parallel for schedule(dynamic, 64) if (work > kParWork)
        for (int64_t i = 0; i < rows; ++i) {
            double* y = Y + i * l;
            for (int64_t c = 0; c < l; ++c) y[c] = 0.0;
            if (dn) {
                const double* a = dn + i * ncols;
                for (int64_t j = 0; j < ncols; ++j) {
                    const double v = a[j];
                    if (v == 0.0) continue;
                    const double* x = X + j * l;
                    for (int64_t c = 0; c < l; ++c) y[c] += v * x[c];
                }
            } else {
                for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
                    const double v = vv[e];
                    const double* x = X + (int64_t)ci[e] * l;
                    for (int64_t c = 0; c < l; ++c) y[c] += v * x[c];
                }
            }
        }
    }
    // Y (m x l, row-major) = A X (n x l row-major)
    void mul(const double* X, int64_t l, double* Y) const { Prof p(4); spmm(m, n, dense, rowptr, cols, vals, X, l, Y); }
    // Z (n x l) = A^T Y (m x l)
    void tmul(const double* Y, int64_t l, double* Z) const {
        Prof p(4);
        if (dense) spmm(n, m, dT.data(), nullptr, nullptr, nullptr, Y, l, Z);
        else spmm(n, m, nullptr, rpT.data(), colT.data(), valT.data(), Y, l, Z);
    }
};

// row-major (rows x l) <-> column-major
void to_cm(const double* rm, int64_t rows, int64_t l, double* cm) {
#pragma omp parallel for if (rows * l > kParWork)
    for (int64_t c = 0; c < l; ++c)
        for (int64_t i = 0; i < rows; ++i) cm[c * rows + i] = rm[i * l + c];
}
void to_rm(const double* cm, int64_t rows, int64_t l, double* rm) {
#pragma omp parallel for if (rows * l > kParWork)
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t c = 0; c < l; ++c) rm[i * l + c] = cm[c * rows + i];
}

// Orthonormalise the l columns of the COLUMN-MAJOR m x l matrix Y in place
// (classical Gram-Schmidt applied twice; a column that vanishes relative to
// its original norm is zeroed).  If R is given (l x l column-major) it
// receives the upper-triangular factor, Y_in = Q R.
void orthonormalize_cm(double* Y, int64_t m, int64_t l, double* R) {
    Prof prof(5);
    std::vector<double> dots(l);
    if (R) std::fill(R, R + l * l, 0.0);
    constexpr int64_t RB = 512;
    for (int64_t j = 0; j < l; ++j) {
        double* y = Y + j * m;
        double n0 = 0;
#pragma omp simd reduction(+ : n0)
        for (int64_t i = 0; i < m; ++i) n0 += y[i] * y[i];
        n0 = std::sqrt(n0);
        for (int pass = 0; pass < 2 && j > 0; ++pass) {
#pragma omp parallel for if (m * j > kParWork)
            for (int64_t p = 0; p < j; ++p) {
                const double* qp = Y + p * m;
                double d = 0;
#pragma omp simd reduction(+ : d)
                for (int64_t i = 0; i < m; ++i) d += qp[i] * y[i];
                dots[p] = d;
            }
#pragma omp parallel for if (m * j > kParWork)
            for (int64_t i0 = 0; i0 < m; i0 += RB) {
                const int64_t i1 = std::min(m, i0 + RB);
                for (int64_t p = 0; p < j; ++p) {
                    const double dp = dots[p];
                    const double* qp = Y + p * m;
                    for (int64_t i = i0; i < i1; ++i) y[i] -= dp * qp[i];
                }
            }
            if (R)
                for (int64_t p = 0; p < j; ++p) R[j * l + p] += dots[p];
        }
        double nn = 0;
#pragma omp simd reduction(+ : nn)
        for (int64_t i = 0; i < m; ++i) nn += y[i] * y[i];
        nn = std::sqrt(nn);
        const double inv = (nn > 1e-13 * n0 && nn > 0) ? 1.0 / nn : 0.0;
        for (int64_t i = 0; i < m; ++i) y[i] *= inv;
        if (R) R[j * l + j] = inv > 0 ? nn : 0.0;
    }
}

// One-sided Jacobi SVD of the COLUMN-MAJOR rows x l matrix G: on return G's
// columns are the left singular vectors (zero where sigma = 0), sig the
// singular values and W (l x l column-major) the right singular vectors,
// sorted descending: G_in = G diag(sig) W^T.
void jacobi_svd_cm(std::vector<double>& G, int64_t rows, int64_t l, std::vector<double>& sig,
                   std::vector<double>& W) {
    W.assign(l * l, 0.0);
    for (int64_t j = 0; j < l; ++j) W[j * l + j] = 1.0;
    // round-robin (tournament) ordering: a round rotates lp/2 disjoint column
    // pairs, in parallel; a sweep is lp - 1 rounds (every pair once).
    const int64_t lp = l + (l & 1);
    std::vector<int64_t> ring(lp);
    std::iota(ring.begin(), ring.end(), 0);
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0;
        for (int64_t round = 0; round < lp - 1; ++round) {
#pragma omp parallel for reduction(max : off) if (rows * l > 8192)
            for (int64_t k = 0; k < lp / 2; ++k) {
                int64_t p = ring[k], q = ring[lp - 1 - k];
                if (p > q) std::swap(p, q);
                if (q >= l) continue;                               // padding slot
                double* gp = G.data() + p * rows;
                double* gq = G.data() + q * rows;
                double a = 0, b = 0, c = 0;
#pragma omp simd reduction(+ : a, b, c)
                for (int64_t i = 0; i < rows; ++i) { a += gp[i] * gp[i]; b += gq[i] * gq[i]; c += gp[i] * gq[i]; }
                if (c == 0.0 || std::fabs(c) <= 1e-15 * std::sqrt(a * b)) continue;
                off = std::max(off, std::fabs(c) / std::sqrt(a * b));
                const double zeta = (b - a) / (2.0 * c);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
                for (int64_t i = 0; i < rows; ++i) {
                    const double x = gp[i], y = gq[i];
                    gp[i] = cs * x - sn * y;
                    gq[i] = sn * x + cs * y;
                }
                double* wp = W.data() + p * l;
                double* wq = W.data() + q * l;
                for (int64_t i = 0; i < l; ++i) {
                    const double x = wp[i], y = wq[i];
                    wp[i] = cs * x - sn * y;
                    wq[i] = sn * x + cs * y;
                }
            }
            std::rotate(ring.begin() + 1, ring.end() - 1, ring.end());   // ring[0] stays
        }
        if (off <= 1e-15) break;
    }
    sig.assign(l, 0.0);
    for (int64_t j = 0; j < l; ++j) {
        double s = 0;
        const double* g = G.data() + j * rows;
        for (int64_t i = 0; i < rows; ++i) s += g[i] * g[i];
        sig[j] = std::sqrt(s);
    }
    std::vector<int64_t> ord(l);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return sig[a] > sig[b]; });
    std::vector<double> G2(rows * l), W2(l * l), s2(l);
    for (int64_t jj = 0; jj < l; ++jj) {
        const int64_t j = ord[jj];
        s2[jj] = sig[j];
        const double inv = sig[j] > 0 ? 1.0 / sig[j] : 0.0;
        for (int64_t i = 0; i < rows; ++i) G2[jj * rows + i] = G[j * rows + i] * inv;
        for (int64_t i = 0; i < l; ++i) W2[jj * l + i] = W[j * l + i];
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

// C (rows x l, row-major) = Acm (rows x l column-major) * Wcm (l x l column-major)
void mul_cm_small(const double* Acm, int64_t rows, int64_t l, const double* Wcm, double* Crm) {
#pragma omp parallel for if (rows * l * l > kParWork)
    for (int64_t i = 0; i < rows; ++i) {
        double* c = Crm + i * l;
        for (int64_t j = 0; j < l; ++j) c[j] = 0.0;
        for (int64_t p = 0; p < l; ++p) {
            const double a = Acm[p * rows + i];
            if (a == 0.0) continue;
            const double* w = Wcm + p;   // row p of W: W[j * l + p]
            for (int64_t j = 0; j < l; ++j) c[j] += a * w[j * l];
        }
    }
}

Trunc exact_svd(const Op& A) {
    // dense column-major copy, transposed so that rows >= cols
    Prof prof(0);
    Trunc T;
    const bool tr = A.m < A.n;
    const int64_t rows = tr ? A.n : A.m, l = tr ? A.m : A.n;
    std::vector<double> G(rows * l, 0.0);                  // column-major rows x l
    auto put = [&](int64_t i, int64_t j, double v) {
        if (tr) G[i * rows + j] = v; else G[j * rows + i] = v;
    };
    for (int64_t i = 0; i < A.m; ++i) {
        if (A.dense) {
            for (int64_t j = 0; j < A.n; ++j) put(i, j, A.dense[i * A.n + j]);
        } else {
            for (int64_t e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e) put(i, A.cols[e], A.vals[e]);
        }
    }
    std::vector<double> sig, W;
    jacobi_svd_cm(G, rows, l, sig, W);
    T.l = l; T.S = sig; T.exact = true;
    std::vector<double> Grm(rows * l), Wrm(l * l);
    to_rm(G.data(), rows, l, Grm.data());
    to_rm(W.data(), l, l, Wrm.data());
    if (tr) { T.U = Wrm; T.V = Grm; } else { T.U = Grm; T.V = Wrm; }
    return T;
}

// Randomized k-term SVD (range finder with 2 power iterations), then
// Z = A^T Q = Qz R (QR) and a one-sided Jacobi SVD of the small l x l R:
// R = Ur S W^T  =>  A ~ Q B = (Q W) S (Qz Ur)^T.
Trunc randomized_svd(const Op& A, int64_t l, Rng& rng) {
    Prof prof(1);
    auto t0 = std::chrono::steady_clock::now();
    struct Rep { const Op& A; int64_t l; std::chrono::steady_clock::time_point t0;
        ~Rep() { if (getenv("VF_BUILD_PROFILE") && atoi(getenv("VF_BUILD_PROFILE")) > 1) {
            double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (dt > 0.5) fprintf(stderr, "  rsvd m %ld n %ld nnz %ld l %ld: %.3f s\n", (long)A.m, (long)A.n,
                                   (long)(A.dense ? A.m * A.n : A.rowptr[A.m]), (long)l, dt); } } } rep{A, l, t0};
    Trunc T;
    T.l = l;
    std::vector<double> Om(A.n * l);
    for (auto& v : Om) v = rng.normal();
    // large blocks: the same algorithm on the device (vf_svd_gpu.cu)
    const int64_t nnz = A.dense ? A.m * A.n : A.rowptr[A.m];
    if (nnz * l >= kGpuSvdWork && g_svd_device >= 0) {
        Prof pg(7);
        if (gpu_randomized_svd(A.m, A.n, A.rowptr, A.cols, A.vals, A.dense, Om.data(), l, T.U, T.S, T.V)) return T;
    }
    if (false &&
        gpu_randomized_svd(A.m, A.n, A.rowptr, A.cols, A.vals, A.dense, Om.data(), l, T.U, T.S, T.V))
        return T;
    std::vector<double> Y(A.m * l), Z(A.n * l), Ycm(A.m * l), Zcm(A.n * l);
    A.mul(Om.data(), l, Y.data());
    for (int it = 0; it < 2; ++it) {       // power iterations
        to_cm(Y.data(), A.m, l, Ycm.data());
        orthonormalize_cm(Ycm.data(), A.m, l, nullptr);
        to_rm(Ycm.data(), A.m, l, Y.data());
        A.tmul(Y.data(), l, Z.data());
        to_cm(Z.data(), A.n, l, Zcm.data());
        orthonormalize_cm(Zcm.data(), A.n, l, nullptr);
        to_rm(Zcm.data(), A.n, l, Z.data());
        A.mul(Z.data(), l, Y.data());
    }
    to_cm(Y.data(), A.m, l, Ycm.data());
    orthonormalize_cm(Ycm.data(), A.m, l, nullptr);      // Q (column-major)
    to_rm(Ycm.data(), A.m, l, Y.data());
    A.tmul(Y.data(), l, Z.data());                       // Z = A^T Q  (n x l)
    to_cm(Z.data(), A.n, l, Zcm.data());
    std::vector<double> R(l * l);
    orthonormalize_cm(Zcm.data(), A.n, l, R.data());     // Z = Qz R
    std::vector<double> sig, W;
    { Prof pj(6); jacobi_svd_cm(R, l, l, sig, W); }      // R = Ur S W^T (R now holds Ur)
    T.S = sig;
    T.V.resize(A.n * l);
    mul_cm_small(Zcm.data(), A.n, l, R.data(), T.V.data());   // V = Qz Ur
    T.U.resize(A.m * l);
    mul_cm_small(Ycm.data(), A.m, l, W.data(), T.U.data());   // U = Q W
    return T;
}

// Spectral norm estimate of A - U_q S_q V_q^T by power iteration.
double residual_norm(const Op& A, const Trunc& T, int64_t q, Rng& rng) {
    Prof prof(2);
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

void small_jacobi_svd(std::vector<double>& R, int64_t l, std::vector<double>& sig, std::vector<double>& W) {
    jacobi_svd_cm(R, l, l, sig, W);
}

void svd_profile_report() {
    if (!getenv("VF_BUILD_PROFILE")) return;
    const char* nm[8] = {"exact_svd", "randomized_svd", "residual_norm", "estimate_rank", "spmm", "orth", "jacobi", "gpu_rsvd"};
    for (int i = 0; i < 8; ++i)
        fprintf(stderr, "[vf build] %-15s calls %8lld  %9.3f s\n", nm[i], (long long)g_cnt[i], g_ns[i] * 1e-9);
}

SvdResult estimate_rank(int64_t mu, int64_t nv, const double* dense, const int64_t* rowptr,
                        const int32_t* cols, const double* vals, double eps, int w, int k0,
                        int64_t target_bytes, int64_t, int64_t, uint64_t seed) {
    SvdResult R;
    Prof prof_all(3);
    Op A{mu, nv, dense, rowptr, cols, vals, {}, {}, {}, {}};
    A.build_transpose();
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
            // smallest q' in [q, kk] whose residual passes (the residual norm is
            // non-increasing in q'): exponential probe, then bisection
            auto pass = [&](int64_t qq) { return 1.2 * residual_norm(A, T, qq, rng) < eps * s1; };
            if (!pass(q)) {
                int64_t lo = q, hi = -1, step = 1;           // lo fails
                while (hi < 0) {
                    const int64_t c = std::min<int64_t>(kk, lo + step);
                    if (pass(c)) hi = c;
                    else if (c == kk) break;
                    else { lo = c; step *= 2; }
                }
                if (hi < 0) q = 0;
                else {
                    while (hi - lo > 1) {
                        const int64_t mid = (lo + hi) / 2;
                        if (pass(mid)) hi = mid; else lo = mid;
                    }
                    q = hi;
                }
            }
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
        // reading A5: the doubling stops once w k (m'+n') >= nbytes(F_IJ) (then every
        // q > k fails eq. nbytes-comparison) or the spectrum is complete (k >= rank)
        if ((int64_t)w * k * (mu + nv) >= target_bytes || complete) return R;
    }
}

}  // namespace vf
