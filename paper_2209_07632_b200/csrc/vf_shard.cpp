// vf_shard.cpp -- block-row sharding of F-hat for single-RHS multi-GPU solves
// (SURVEY §8(e) "ROWS", §8(a) row a6).  Host side, untimed.
//
// The paper has no parallelism ("we do not focus on parallelism"); the
// operator it parallelises over here is its own Alg. 5: the
// product Y = F-hat X decomposes by output rows, Y_I = sum_J F_IJ X_J, so a
// rank that owns a contiguous range of tree-order rows [lo, hi) needs exactly
// the leaf rows that fall in that range:
//   dense / CSR leaves   -> their rows in [lo, hi);
//   SVD leaves U S V^T   -> the rows of U in [lo, hi); V and S duplicated (a
//                           block that spans two ranks is split through U).
// Every rank keeps the full X (B) and exchanges its rows of the new iterate
// by an allgather each Jacobi iteration (vf_device.cu, rows_* kernels).
//
// The cut points balance the per-row F-hat bytes an apply streams (A7/A8
// accounting: dense n w, CSR nnz (w+4) + 8, SVD U row q w plus the block's V
// bytes spread over its stored rows), so every rank moves about the same
// number of HBM bytes per iteration.
#include <algorithm>
#include <cmath>
#include <vector>

#include "vf_internal.h"

namespace vf {

std::vector<double> row_costs(const Handle* h) {
    const int w = h->dtype == VF_F32 ? 4 : 8;
    std::vector<double> c(h->N, 0.0);
    for (const Leaf& L : h->leaves) {
        if (L.kind == K_DENSE) {
            for (int64_t r = 0; r < L.m; ++r) c[L.row0 + r] += (double)w * L.n;
        } else if (L.kind == K_CSR) {
            for (int64_t r = 0; r < L.m; ++r)
                c[L.row0 + r] += (double)(w + 4) * (L.rowptr[r + 1] - L.rowptr[r]) + 8.0;
        } else if (L.kind == K_SVD) {
            const int64_t mu = (int64_t)L.idx_a.size(), nv = (int64_t)L.idx_b.size();
            const double vshare = mu ? (double)w * L.q * nv / (double)mu : 0.0;
            for (int32_t r : L.idx_a) c[L.row0 + r] += (double)w * L.q + vshare;
        }
    }
    return c;
}

// bounds[0] = 0 <= bounds[1] <= ... <= bounds[world] = N; rank g owns rows
// [bounds[g], bounds[g+1]).  Cut g is the first row whose cost prefix reaches
// g/world of the total (ties and empty operators: equal row counts).
int row_partition(const Handle* h, int world, std::vector<int64_t>& bounds) {
    if (world < 1) return set_error(VF_EINVAL, "world must be >= 1");
    const int64_t N = h->N;
    bounds.assign(world + 1, 0);
    bounds[world] = N;
    std::vector<double> c = row_costs(h);
    std::vector<double> pre(N + 1, 0.0);
    for (int64_t i = 0; i < N; ++i) pre[i + 1] = pre[i] + c[i];
    const double tot = pre[N];
    for (int g = 1; g < world; ++g) {
        if (!(tot > 0)) { bounds[g] = N * g / world; continue; }
        const double target = tot * g / world;
        int64_t cut = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
        // pick the closer of the two rows around the crossing
        if (cut > 0 && target - pre[cut - 1] < pre[cut] - target) --cut;
        bounds[g] = std::max(bounds[g - 1], std::min<int64_t>(cut, N));
    }
    return VF_OK;
}

// Replace h->leaves by their restriction to tree rows [lo, hi).
void restrict_leaves(Handle* h, int64_t lo, int64_t hi) {
    std::vector<Leaf> out;
    for (Leaf& L : h->leaves) {
        if (L.kind == K_DENSE || L.kind == K_CSR) {
            const int64_t r0 = std::max(L.row0, lo), r1 = std::min(L.row0 + L.m, hi);
            if (r0 >= r1) continue;
            Leaf S;
            S.kind = L.kind; S.level = L.level;
            S.row0 = r0; S.m = r1 - r0; S.col0 = L.col0; S.n = L.n;
            const int64_t a = r0 - L.row0, b = r1 - L.row0;
            if (L.kind == K_DENSE) {
                S.a.assign(L.a.begin() + a * L.n, L.a.begin() + b * L.n);
            } else {
                const int64_t e0 = L.rowptr[a], e1 = L.rowptr[b];
                if (e1 == e0) continue;
                S.rowptr.resize(S.m + 1);
                for (int64_t r = 0; r <= S.m; ++r) S.rowptr[r] = L.rowptr[a + r] - e0;
                S.idx_a.assign(L.idx_a.begin() + e0, L.idx_a.begin() + e1);
                S.a.assign(L.a.begin() + e0, L.a.begin() + e1);
            }
            S.nbytes = leaf_nbytes(S, h->dtype == VF_F32 ? 4 : 8);
            out.push_back(std::move(S));
        } else if (L.kind == K_SVD) {
            std::vector<int64_t> keep;
            for (int64_t r = 0; r < (int64_t)L.idx_a.size(); ++r) {
                const int64_t row = L.row0 + L.idx_a[r];
                if (row >= lo && row < hi) keep.push_back(r);
            }
            if (keep.empty()) continue;
            Leaf S = L;
            if ((int64_t)keep.size() != (int64_t)L.idx_a.size()) {
                S.idx_a.clear();
                S.a.clear();
                for (int64_t r : keep) {
                    S.idx_a.push_back(L.idx_a[r]);
                    S.a.insert(S.a.end(), L.a.begin() + r * L.q, L.a.begin() + (r + 1) * L.q);
                }
            }
            S.nbytes = leaf_nbytes(S, h->dtype == VF_F32 ? 4 : 8);
            out.push_back(std::move(S));
        }
    }
    h->leaves.swap(out);
}

std::vector<uint8_t> active_rows_of(const Handle* h) {
    std::vector<uint8_t> act(h->N, 0);
    for (const Leaf& L : h->leaves) {
        if (L.kind == K_DENSE) {
            for (int64_t r = 0; r < L.m; ++r) act[L.row0 + r] = 1;
        } else if (L.kind == K_CSR) {
            for (int64_t r = 0; r < L.m; ++r) if (L.rowptr[r + 1] > L.rowptr[r]) act[L.row0 + r] = 1;
        } else if (L.kind == K_SVD) {
            for (int32_t r : L.idx_a) act[L.row0 + r] = 1;
        }
    }
    return act;
}

int shard_rows(Handle* h, int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) return set_error(VF_EINVAL, "vf_shard_rows: bad rank/world");
    if (h->world > 1 || h->sharded) return set_error(VF_EINVAL, "vf_shard_rows: handle is already sharded");
    std::vector<int64_t> b;
    int rc = row_partition(h, world, b);
    if (rc) return rc;
    h->active_global = active_rows_of(h);
    h->row_bounds = b;
    h->rank = rank;
    h->world = world;
    h->row_lo = b[rank];
    h->row_hi = b[rank + 1];
    restrict_leaves(h, h->row_lo, h->row_hi);
    h->sharded = true;
    return VF_OK;
}

}  // namespace vf
