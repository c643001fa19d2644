// vf_io.cpp -- HVFM v1 container (layout documented in include/vf.h).
// The compressed matrix is geometric and reused across runs,
// so it is saved once per mesh / tolerance / dtype and reloaded.
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

#include "vf_internal.h"

namespace vf {
namespace {

struct File {
    FILE* f = nullptr;
    explicit File(FILE* p) : f(p) {}
    ~File() { if (f) fclose(f); }
};

bool wr(FILE* f, const void* p, size_t n) { return n == 0 || fwrite(p, 1, n, f) == n; }
bool rd(FILE* f, void* p, size_t n) { return n == 0 || fread(p, 1, n, f) == n; }

bool wr_vals(FILE* f, const std::vector<double>& v, int dtype) {
    if (dtype == VF_F64) return wr(f, v.data(), v.size() * 8);
    std::vector<float> t(v.size());
    for (size_t i = 0; i < v.size(); ++i) t[i] = (float)v[i];
    return wr(f, t.data(), t.size() * 4);
}

bool rd_vals(FILE* f, std::vector<double>& v, int64_t n, int dtype) {
    if (n < 0) return false;
    v.resize(n);
    if (dtype == VF_F64) return rd(f, v.data(), (size_t)n * 8);
    std::vector<float> t(n);
    if (!rd(f, t.data(), (size_t)n * 4)) return false;
    for (int64_t i = 0; i < n; ++i) v[i] = t[i];
    return true;
}

}  // namespace

int save_hvfm(const Handle* h, const char* path) {
    File F(fopen(path, "wb"));
    if (!F.f) return set_error(VF_EIO, std::string("vf_save: cannot open ") + path);
    uint32_t hdr[4] = {1u, (uint32_t)h->dtype, 0u, 0u};
    int64_t N = h->N, nl = (int64_t)h->leaves.size();
    bool ok = wr(F.f, "HVFM", 4) && wr(F.f, hdr, 12) && wr(F.f, &N, 8) && wr(F.f, &h->tol, 8) &&
              wr(F.f, &nl, 8) && wr(F.f, h->perm.data(), (size_t)N * 4);
    for (const Leaf& L : h->leaves) {
        if (!ok) break;
        int32_t kl[2] = {L.kind, L.level};
        int64_t rng[4] = {L.row0, L.m, L.col0, L.n};
        ok = wr(F.f, kl, 8) && wr(F.f, rng, 32);
        if (L.kind == K_DENSE) {
            ok = ok && wr_vals(F.f, L.a, h->dtype);
        } else if (L.kind == K_CSR) {
            int64_t nnz = (int64_t)L.idx_a.size();
            ok = ok && wr(F.f, &nnz, 8) && wr(F.f, L.rowptr.data(), (size_t)(L.m + 1) * 8) &&
                 wr(F.f, L.idx_a.data(), (size_t)nnz * 4) && wr_vals(F.f, L.a, h->dtype);
        } else {
            int64_t qmn[3] = {L.q, (int64_t)L.idx_a.size(), (int64_t)L.idx_b.size()};
            ok = ok && wr(F.f, qmn, 24) && wr(F.f, L.idx_a.data(), L.idx_a.size() * 4) &&
                 wr(F.f, L.idx_b.data(), L.idx_b.size() * 4) && wr_vals(F.f, L.s, h->dtype) &&
                 wr_vals(F.f, L.a, h->dtype) && wr_vals(F.f, L.b, h->dtype);
        }
    }
    if (!ok) return set_error(VF_EIO, std::string("vf_save: write failed: ") + path);
    return VF_OK;
}

int load_hvfm(Handle* h, const char* path) {
    File F(fopen(path, "rb"));
    if (!F.f) return set_error(VF_EIO, std::string("vf_load: cannot open ") + path);
    char magic[4];
    uint32_t hdr[3];
    int64_t N, nl;
    double tol;
    if (!rd(F.f, magic, 4) || memcmp(magic, "HVFM", 4) != 0) return set_error(VF_EIO, "vf_load: bad magic");
    if (!rd(F.f, hdr, 12) || hdr[0] != 1u) return set_error(VF_EIO, "vf_load: unsupported version");
    if (hdr[1] != (uint32_t)VF_F64 && hdr[1] != (uint32_t)VF_F32) return set_error(VF_EIO, "vf_load: bad dtype");
    if (!rd(F.f, &N, 8) || !rd(F.f, &tol, 8) || !rd(F.f, &nl, 8) || N < 0 || nl < 0 || N > (int64_t)1 << 31)
        return set_error(VF_EIO, "vf_load: truncated header");
    h->N = N;
    h->dtype = (int)hdr[1];
    h->tol = tol;
    h->perm.resize(N);
    if (!rd(F.f, h->perm.data(), (size_t)N * 4)) return set_error(VF_EIO, "vf_load: truncated permutation");
    {
        std::vector<char> seen(N, 0);
        for (int32_t p : h->perm) {
            if (p < 0 || p >= N || seen[p]) return set_error(VF_EIO, "vf_load: permutation is not a bijection");
            seen[p] = 1;
        }
    }
    h->leaves.clear();
    h->leaves.reserve(nl);
    for (int64_t b = 0; b < nl; ++b) {
        Leaf L;
        int32_t kl[2];
        int64_t rng[4];
        if (!rd(F.f, kl, 8) || !rd(F.f, rng, 32)) return set_error(VF_EIO, "vf_load: truncated block header");
        L.kind = kl[0]; L.level = kl[1];
        L.row0 = rng[0]; L.m = rng[1]; L.col0 = rng[2]; L.n = rng[3];
        if (L.m < 0 || L.n < 0 || L.row0 < 0 || L.col0 < 0 || L.row0 + L.m > N || L.col0 + L.n > N)
            return set_error(VF_EIO, "vf_load: block range out of bounds");
        if (L.kind == K_DENSE) {
            if (!rd_vals(F.f, L.a, L.m * L.n, h->dtype)) return set_error(VF_EIO, "vf_load: truncated dense block");
        } else if (L.kind == K_CSR) {
            int64_t nnz;
            if (!rd(F.f, &nnz, 8) || nnz < 0) return set_error(VF_EIO, "vf_load: truncated csr block");
            L.rowptr.resize(L.m + 1);
            L.idx_a.resize(nnz);
            if (!rd(F.f, L.rowptr.data(), (size_t)(L.m + 1) * 8) || !rd(F.f, L.idx_a.data(), (size_t)nnz * 4) ||
                !rd_vals(F.f, L.a, nnz, h->dtype))
                return set_error(VF_EIO, "vf_load: truncated csr block");
            if (L.rowptr[0] != 0 || L.rowptr[L.m] != nnz) return set_error(VF_EIO, "vf_load: bad csr rowptr");
            for (int64_t r = 0; r < L.m; ++r)
                if (L.rowptr[r + 1] < L.rowptr[r]) return set_error(VF_EIO, "vf_load: bad csr rowptr");
            for (int32_t c : L.idx_a)
                if (c < 0 || c >= L.n) return set_error(VF_EIO, "vf_load: csr column out of range");
        } else if (L.kind == K_SVD) {
            int64_t qmn[3];
            if (!rd(F.f, qmn, 24) || qmn[0] < 0 || qmn[1] < 0 || qmn[2] < 0) return set_error(VF_EIO, "vf_load: truncated svd block");
            L.q = qmn[0];
            L.idx_a.resize(qmn[1]);
            L.idx_b.resize(qmn[2]);
            if (!rd(F.f, L.idx_a.data(), (size_t)qmn[1] * 4) || !rd(F.f, L.idx_b.data(), (size_t)qmn[2] * 4) ||
                !rd_vals(F.f, L.s, L.q, h->dtype) || !rd_vals(F.f, L.a, qmn[1] * L.q, h->dtype) ||
                !rd_vals(F.f, L.b, qmn[2] * L.q, h->dtype))
                return set_error(VF_EIO, "vf_load: truncated svd block");
            for (int32_t r : L.idx_a) if (r < 0 || r >= L.m) return set_error(VF_EIO, "vf_load: svd row out of range");
            for (int32_t c : L.idx_b) if (c < 0 || c >= L.n) return set_error(VF_EIO, "vf_load: svd col out of range");
        } else {
            return set_error(VF_EIO, "vf_load: unknown block kind");
        }
        L.nbytes = leaf_nbytes(L, h->dtype == VF_F32 ? 4 : 8);
        h->leaves.push_back(std::move(L));
    }
    h->has_mesh = false;
    return VF_OK;
}

}  // namespace vf
