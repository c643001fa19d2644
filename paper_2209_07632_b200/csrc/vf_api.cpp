// vf_api.cpp -- the extern "C" boundary of libvf (declared in include/vf.h).
// Argument checking, error mapping and handle ownership only; the build is in
// vf_build.cpp, the hot path in vf_device.cu.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <vector>
#include <new>
#include <string>

#include <cuda_runtime.h>

#include "vf_internal.h"

namespace vf {
static thread_local std::string g_err;
int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int64_t device_alg_bytes(const Handle* h);
int64_t device_alg_flops(const Handle* h);
int64_t device_active_rows(const Handle* h);
void device_phase_info(const Handle* h, int64_t* out16);
}  // namespace vf

using namespace vf;

#define GUARD(...)                                                            \
    try {                                                                     \
        __VA_ARGS__                                                           \
    } catch (const std::bad_alloc&) {                                         \
        return set_error(VF_ENOMEM, "host allocation failed");               \
    } catch (const std::exception& e) {                                       \
        return set_error(VF_EINVAL, std::string("internal error: ") + e.what()); \
    }

extern "C" {

void vf_default_opts(vf_build_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->dtype = VF_F64;
    o->max_depth = 16;
    o->min_leaf = 16;
    o->min_block = 16384;
    o->k0 = 8;
    o->visibility = VF_VIS_RAYCAST;
    o->orient_up = 1;
    o->device = 0;
    o->threads = 0;
    o->seed = 0x5eedull;
}

static int check_opts(const vf_build_opts& o, double tol) {
    if (o.dtype != VF_F64 && o.dtype != VF_F32) return set_error(VF_EINVAL, "opts.dtype must be VF_F64 or VF_F32");
    if (!(tol > 0.0) || !(tol < 1.0)) return set_error(VF_EINVAL, "tol must be in (0, 1)");
    if (o.max_depth < 0 || o.min_leaf < 1 || o.min_block < 1 || o.k0 < 1)
        return set_error(VF_EINVAL, "bad tree/rank options");
    return VF_OK;
}

static int finish(Handle* h, int device, vf_handle* out) {
    if (device >= 0) {
        int rc = device_upload(h, device);
        if (rc) { delete h; return rc; }
    }
    *out = reinterpret_cast<vf_handle>(h);
    return VF_OK;
}

// Facet data of P:129: centroid, unit normal (right-hand rule, n_z > 0 when
// orient_up: reading R-ORIENT), area.
static int facet_data(const vf_mesh* mesh, int orient_up, std::vector<double>& x, std::vector<double>& n,
                      std::vector<double>& A) {
    const int64_t N = mesh->nf;
    x.resize(3 * N); n.resize(3 * N); A.resize(N);
    for (int64_t f = 0; f < N; ++f) {
        int32_t ia = mesh->F[3 * f], ib = mesh->F[3 * f + 1], ic = mesh->F[3 * f + 2];
        if (ia < 0 || ib < 0 || ic < 0 || ia >= mesh->nv || ib >= mesh->nv || ic >= mesh->nv)
            return set_error(VF_EINVAL, "mesh: face index out of range");
        const double* a = mesh->V + 3 * (int64_t)ia;
        const double* b = mesh->V + 3 * (int64_t)ib;
        const double* c = mesh->V + 3 * (int64_t)ic;
        double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
        double len = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
        if (!(len > 0.0)) return set_error(VF_EINVAL, "mesh: zero-area face " + std::to_string(f));
        double sgn = (orient_up && cr[2] < 0.0) ? -1.0 : 1.0;
        for (int d = 0; d < 3; ++d) {
            x[3 * f + d] = (a[d] + b[d] + c[d]) / 3.0;
            n[3 * f + d] = sgn * cr[d] / len;
        }
        A[f] = 0.5 * len;
    }
    return VF_OK;
}

int vf_build(const vf_mesh* mesh, double tol, const vf_build_opts* opts, vf_handle* out) {
    GUARD({
        if (!mesh || !out || !mesh->V || !mesh->F || mesh->nf <= 0 || mesh->nv <= 0)
            return set_error(VF_EINVAL, "vf_build: null or empty mesh");
        vf_build_opts o;
        if (opts) o = *opts; else vf_default_opts(&o);
        int rc = check_opts(o, tol);
        if (rc) return rc;
        const int64_t N = mesh->nf;
        std::vector<double> x, n, A;
        if ((rc = facet_data(mesh, o.orient_up, x, n, A))) return rc;
        Handle* h = new Handle();
        rc = build_handle(h, N, x.data(), n.data(), A.data(), mesh->V, mesh->nv, mesh->F, N, nullptr, tol, o);
        if (rc) { delete h; return rc; }
        return finish(h, o.device, out);
    })
}

int vf_build_facets(int64_t N, const double* x, const double* n, const double* A, const vf_mesh* occ, double tol,
                    const vf_build_opts* opts, vf_handle* out) {
    GUARD({
        if (N <= 0 || !x || !n || !A || !out) return set_error(VF_EINVAL, "vf_build_facets: bad arguments");
        vf_build_opts o;
        if (opts) o = *opts; else vf_default_opts(&o);
        int rc = check_opts(o, tol);
        if (rc) return rc;
        Handle* h = new Handle();
        std::vector<int64_t> tri_of(N, -1);
        if (occ && occ->nf == N) for (int64_t i = 0; i < N; ++i) tri_of[i] = i;
        if (occ && o.visibility == VF_VIS_RAYCAST)
            rc = build_handle(h, N, x, n, A, occ->V, occ->nv, occ->F, occ->nf, tri_of.data(), tol, o);
        else
            rc = build_handle(h, N, x, n, A, nullptr, 0, nullptr, 0, tri_of.data(), tol, o);
        if (rc) { delete h; return rc; }
        return finish(h, o.device, out);
    })
}

int vf_load(const char* path, int device, vf_handle* out) {
    GUARD({
        if (!path || !out) return set_error(VF_EINVAL, "vf_load: null argument");
        Handle* h = new Handle();
        int rc = load_hvfm(h, path);
        if (rc) { delete h; return rc; }
        return finish(h, device, out);
    })
}

int vf_save(vf_handle hh, const char* path) {
    GUARD({
        if (!hh || !path) return set_error(VF_EINVAL, "vf_save: null argument");
        return save_hvfm(reinterpret_cast<Handle*>(hh), path);
    })
}

int vf_upload(vf_handle hh, int device) {
    GUARD({
        if (!hh) return set_error(VF_EINVAL, "vf_upload: null handle");
        return device_upload(reinterpret_cast<Handle*>(hh), device);
    })
}

int vf_free(vf_handle hh) {
    if (!hh) return VF_OK;
    Handle* h = reinterpret_cast<Handle*>(hh);
    comm_destroy(h);
    device_free(h);
    delete h;
    return VF_OK;
}

int vf_set_stream(vf_handle hh, void* stream) {
    if (!hh) return set_error(VF_EINVAL, "vf_set_stream: null handle");
    reinterpret_cast<Handle*>(hh)->stream = stream;
    return VF_OK;
}

static int need_dev(Handle* h) {
    if (!h) return set_error(VF_EINVAL, "null handle");
    if (!h->dev) return set_error(VF_ENODEV, "handle has no device copy (built with device = -1 or no GPU)");
    return VF_OK;
}

int vf_matvec(vf_handle hh, const void* X, void* Y, int nrhs) {
    GUARD({
        Handle* h = reinterpret_cast<Handle*>(hh);
        int rc = need_dev(h);
        if (rc) return rc;
        if (!X || !Y || nrhs <= 0) return set_error(VF_EINVAL, "vf_matvec: bad arguments");
        if (X == Y) return set_error(VF_EINVAL, "vf_matvec: X aliases Y");
        return device_matvec(h, X, Y, nrhs);
    })
}

int vf_solve_radiosity(vf_handle hh, const void* E, const void* rho, void* B, int nrhs, int iters, double tol,
                       int clamp) {
    GUARD({
        Handle* h = reinterpret_cast<Handle*>(hh);
        int rc = need_dev(h);
        if (rc) return rc;
        if (!E || !rho || !B || nrhs <= 0 || iters < 0 || !(tol >= 0))
            return set_error(VF_EINVAL, "vf_solve_radiosity: bad arguments");
        return device_solve_radiosity(h, E, rho, B, nrhs, iters, tol, clamp);
    })
}

int vf_solve_thermal(vf_handle hh, const void* Qdir, const void* albedo, const void* emiss, void* T, void* Qvis,
                     void* Qir, int nrhs, int iters, double tol) {
    GUARD({
        Handle* h = reinterpret_cast<Handle*>(hh);
        int rc = need_dev(h);
        if (rc) return rc;
        if (!Qdir || !albedo || !emiss || !T || nrhs <= 0 || iters < 0 || !(tol >= 0))
            return set_error(VF_EINVAL, "vf_solve_thermal: bad arguments");
        return device_solve_thermal(h, Qdir, albedo, emiss, T, Qvis, Qir, nrhs, iters, tol);
    })
}

int vf_ts_create(vf_handle hh, int nscen, int M, double depth, double ratio, double k_th, double rho_c, double H,
                 const void* albedo, const void* emiss, const void* Qdir0, const void* T0, vf_tstate* out) {
    GUARD({
        Handle* h = reinterpret_cast<Handle*>(hh);
        int rc = need_dev(h);
        if (rc) return rc;
        if (!out || !albedo || !emiss || !Qdir0 || !T0 || nscen <= 0 || M < 1 || M > 128 || !(depth > 0) ||
            !(ratio > 0) || !(k_th > 0) || !(rho_c > 0))
            return set_error(VF_EINVAL, "vf_ts_create: bad arguments");
        TState* S = nullptr;
        rc = device_ts_create(h, nscen, M, depth, ratio, k_th, rho_c, H, albedo, emiss, Qdir0, T0, &S);
        *out = reinterpret_cast<vf_tstate>(S);
        return rc;
    })
}

int vf_ts_step(vf_tstate s, const void* Qdir, double dt, void* Tsurf) {
    GUARD({
        if (!s || !Qdir || !(dt > 0)) return set_error(VF_EINVAL, "vf_ts_step: bad arguments");
        return device_ts_step(reinterpret_cast<TState*>(s), Qdir, dt, Tsurf);
    })
}

int vf_ts_get(vf_tstate s, void* Qrefl, void* Qir, void* Qabs, void* Tsurf) {
    GUARD({
        if (!s) return set_error(VF_EINVAL, "vf_ts_get: null state");
        return device_ts_get(reinterpret_cast<TState*>(s), Qrefl, Qir, Qabs, Tsurf);
    })
}

int vf_selftest_rows_exchange(int world, int kp, int k, int64_t N, const int64_t* bounds, const double* xrank,
                              const double* part, int nblk, const double* enorm2, double tol, int iters, int iter0,
                              double* xout, double* resid, int* iter_after, int* done_after) {
    GUARD({
        if (world < 1 || kp < 1 || k < 1 || k > kp || N < 1 || !bounds || !xrank || !part || nblk < 1 || !enorm2 ||
            !xout || !resid || !iter_after || !done_after)
            return set_error(VF_EINVAL, "vf_selftest_rows_exchange: bad arguments");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { cudaGetLastError(); return set_error(VF_ENODEV, "no device"); }
        return selftest_rows_exchange(world, kp, k, N, bounds, xrank, part, nblk, enorm2, tol, iters, iter0, xout,
                                      resid, iter_after, done_after);
    })
}

int vf_ts_free(vf_tstate s) {
    device_ts_free(reinterpret_cast<TState*>(s));
    return VF_OK;
}

int vf_last_solve_stats(vf_handle hh, int* it1, double* r1, int* it2, double* r2) {
    if (!hh) return set_error(VF_EINVAL, "null handle");
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (it1) *it1 = h->iters1;
    if (r1) *r1 = h->resid1;
    if (it2) *it2 = h->iters2;
    if (r2) *r2 = h->resid2;
    return VF_OK;
}

int vf_insolation(vf_handle hh, const double* suns, int k, double S, double* Q) {
    GUARD({
        if (!hh || !suns || !Q || k <= 0) return set_error(VF_EINVAL, "vf_insolation: bad arguments");
        return insolation(reinterpret_cast<Handle*>(hh), suns, k, S, Q);
    })
}

int vf_insolation_sum(vf_handle hh, const double* dirs, const double* w, int k, int P, double S, double* Q) {
    GUARD({
        if (!hh || !dirs || !w || !Q || k <= 0 || P <= 0) return set_error(VF_EINVAL, "vf_insolation_sum: bad arguments");
        Handle* h = reinterpret_cast<Handle*>(hh);
        const int64_t N = h->N;
        std::vector<double> Qp((size_t)N * P);
        std::fill(Q, Q + (size_t)N * k, 0.0);
        for (int c = 0; c < k; ++c) {
            const int rc = insolation(h, dirs + (size_t)3 * c * P, P, S, Qp.data());   // N x P
            if (rc) return rc;
            double* q = Q + (size_t)c * N;
            for (int p = 0; p < P; ++p)
                for (int64_t i = 0; i < N; ++i) q[i] += w[p] * Qp[(size_t)p * N + i];
        }
        return VF_OK;
    })
}

int vf_info(vf_handle hh, vf_info_t* out) {
    if (!hh || !out) return set_error(VF_EINVAL, "vf_info: null argument");
    Handle* h = reinterpret_cast<Handle*>(hh);
    std::memset(out, 0, sizeof(*out));
    out->N = h->N;
    out->dtype = h->dtype;
    out->tol = h->tol;
    const int w = h->dtype == VF_F32 ? 4 : 8;
    std::vector<char> act(h->N, 0);
    int64_t fl = 0;
    for (const Leaf& L : h->leaves) {
        int64_t b = leaf_nbytes(L, w);
        if (L.kind == K_DENSE) {
            out->n_dense++; out->bytes_dense += b; fl += 2 * L.m * L.n;
            for (int64_t r = 0; r < L.m; ++r) act[L.row0 + r] = 1;
        } else if (L.kind == K_CSR) {
            out->n_csr++; out->bytes_csr += b; out->nnz_csr += (int64_t)L.idx_a.size(); fl += 2 * (int64_t)L.idx_a.size();
            for (int64_t r = 0; r < L.m; ++r) if (L.rowptr[r + 1] > L.rowptr[r]) act[L.row0 + r] = 1;
        } else if (L.kind == K_SVD) {
            out->n_svd++; out->bytes_svd += b; out->sum_rank += L.q;
            out->max_rank = std::max<int64_t>(out->max_rank, L.q);
            fl += 2 * L.q * ((int64_t)L.idx_a.size() + (int64_t)L.idx_b.size()) + L.q;
            for (int32_t r : L.idx_a) act[L.row0 + r] = 1;
        }
    }
    for (char a : act) out->active_rows += a;
    out->alg_flops_per_col = fl;
    out->device_bytes = device_bytes(h);
    out->alg_bytes = h->dev ? device_alg_bytes(h) : (out->bytes_dense + out->bytes_csr + out->bytes_svd);
    out->visible_pairs = h->visible_pairs;
    out->build_seconds = h->build_seconds;
    out->device = h->dev ? h->device : -1;
    int64_t ph[17];
    device_phase_info(h, ph);
    out->groups1 = ph[7]; out->groups2 = ph[8];
    out->t_rows = ph[0]; out->p1_bytes = ph[1]; out->p2_bytes = ph[2]; out->p1_src_rows = ph[3];
    out->p2_src_rows = ph[4]; out->p1_flops_per_col = ph[5]; out->p2_flops_per_col = ph[6];
    out->resident = ph[9];
    out->stream_payload_bytes = ph[10]; out->stream_meta_bytes = ph[11]; out->stream_chunks = ph[12];
    out->tiles = ph[13]; out->tile_sources = ph[14]; out->k1_payload_bytes = ph[15];
    out->k1_kernel = ph[16];
    return VF_OK;
}

int vf_enable_kernel_timing(vf_handle hh, int on) {
    if (!hh) return set_error(VF_EINVAL, "null handle");
    reinterpret_cast<Handle*>(hh)->timing = on != 0;
    return VF_OK;
}

int vf_kernel_timing(vf_handle hh, double* ms2, int* l2, double* ms1, int* l1, int* lt) {
    if (!hh) return set_error(VF_EINVAL, "null handle");
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (ms2) *ms2 = h->ms_p2;
    if (l2) *l2 = h->launches_p2;
    if (ms1) *ms1 = h->ms_p1;
    if (l1) *l1 = h->launches_p1;
    if (lt) *lt = h->launches_total;
    return VF_OK;
}

int vf_set_mesh(vf_handle hh, const vf_mesh* mesh, int orient_up) {
    GUARD({
        if (!hh || !mesh || !mesh->V || !mesh->F) return set_error(VF_EINVAL, "vf_set_mesh: null argument");
        Handle* h = reinterpret_cast<Handle*>(hh);
        if (mesh->nf != h->N) return set_error(VF_EINVAL, "vf_set_mesh: mesh has a different facet count");
        std::vector<double> x, n, A;
        int rc = facet_data(mesh, orient_up, x, n, A);
        if (rc) return rc;
        h->x.swap(x); h->nrm.swap(n); h->A.swap(A);
        h->occ_V.assign(mesh->V, mesh->V + 3 * mesh->nv);
        h->occ_F.assign(mesh->F, mesh->F + 3 * mesh->nf);
        h->tri_of.clear();
        h->has_mesh = true;
        return VF_OK;
    })
}

int vf_row_partition(vf_handle hh, int world, int64_t* bounds) {
    GUARD({
        if (!hh || !bounds || world < 1) return set_error(VF_EINVAL, "vf_row_partition: bad arguments");
        Handle* h = reinterpret_cast<Handle*>(hh);
        if (h->sharded) {
            if (world != h->world) return set_error(VF_EINVAL, "vf_row_partition: handle is sharded for another world");
            std::copy(h->row_bounds.begin(), h->row_bounds.end(), bounds);
            return VF_OK;
        }
        std::vector<int64_t> b;
        int rc = row_partition(h, world, b);
        if (rc) return rc;
        std::copy(b.begin(), b.end(), bounds);
        return VF_OK;
    })
}

int vf_shard_rows(vf_handle hh, int rank, int world) {
    GUARD({
        if (!hh) return set_error(VF_EINVAL, "vf_shard_rows: null handle");
        Handle* h = reinterpret_cast<Handle*>(hh);
        int rc = shard_rows(h, rank, world);
        if (rc) return rc;
        if (h->dev) return device_upload(h, h->device);    // re-flatten the shard
        return VF_OK;
    })
}

int vf_row_range(vf_handle hh, int64_t* lo, int64_t* hi) {
    if (!hh || !lo || !hi) return set_error(VF_EINVAL, "vf_row_range: null argument");
    Handle* h = reinterpret_cast<Handle*>(hh);
    *lo = h->sharded ? h->row_lo : 0;
    *hi = h->sharded ? h->row_hi : h->N;
    return VF_OK;
}

int vf_get_nccl_id(void* id128) {
    GUARD({
        if (!id128) return set_error(VF_EINVAL, "vf_get_nccl_id: null argument");
        return comm_get_id(id128);
    })
}

int vf_comm_init(vf_handle hh, int rank, int world, const void* id128) {
    GUARD({
        if (!hh || !id128) return set_error(VF_EINVAL, "vf_comm_init: null argument");
        Handle* h = reinterpret_cast<Handle*>(hh);
        if (!h->dev) return set_error(VF_ENODEV, "vf_comm_init: handle has no device copy");
        if (!h->sharded) return set_error(VF_EINVAL, "vf_comm_init: call vf_shard_rows first");
        if (rank != h->rank || world != h->world)
            return set_error(VF_EINVAL, "vf_comm_init: rank/world differ from vf_shard_rows");
        return comm_init(h, rank, world, id128);
    })
}

const char* vf_last_error(void) { return g_err.c_str(); }

}  // extern "C"
