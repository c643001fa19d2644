// vf_internal.h -- host-side data structures of libvf (not part of the ABI).
// PAPER.md = "P:<line>".  See include/vf.h for the operation and DESIGN.md for
// the device layout.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/vf.h"

namespace vf {

enum LeafKind : int { K_ZERO = 0, K_DENSE = 1, K_CSR = 2, K_SVD = 3, K_SUB = 4 };

// One leaf block of F-hat (Alg. 4 output), tree-order ranges.  Values are
// kept in double on the host; for VF_F32 handles they are already rounded to
// float (so save/load and upload see exactly the stored values).
struct Leaf {
    int kind = K_ZERO;
    int level = 0;
    int64_t row0 = 0, m = 0, col0 = 0, n = 0;
    // dense: a = m*n row-major
    // csr:   rowptr (m+1), idx_a = local cols, a = values
    // svd:   q; idx_a = urows (mu), idx_b = vrows (nv); s = S (q);
    //        a = U (mu*q row-major), b = V (nv*q row-major)
    int64_t q = 0;
    std::vector<int64_t> rowptr;
    std::vector<int32_t> idx_a, idx_b;
    std::vector<double> a, b, s;
    int64_t nbytes = 0;
};

// Device copy of the flattened F-hat (see vf_device.cu).
struct DeviceHMat;

struct Handle {
    int64_t N = 0;
    int dtype = VF_F64;
    double tol = 0;
    std::vector<int32_t> perm;       // perm[r] = caller facet at tree position r
    std::vector<Leaf> leaves;        // Alg. 5 order
    // geometry kept for vf_insolation (empty for loaded handles)
    std::vector<double> x, nrm, A;
    std::vector<double> occ_V;
    std::vector<int32_t> occ_F;
    std::vector<int64_t> tri_of;     // facet -> occluder triangle (-1 none)
    bool has_mesh = false;
    int64_t visible_pairs = 0;
    double build_seconds = 0;
    int device = -1;
    void* stream = nullptr;
    DeviceHMat* dev = nullptr;
    // last-solve stats
    int iters1 = 0, iters2 = 0;
    double resid1 = 0, resid2 = 0;
    // kernel timing
    bool timing = false;
    double ms_p2 = 0, ms_p1 = 0;
    int launches_p2 = 0, launches_p1 = 0, launches_total = 0;
    double ms_comm = 0;                  // allgather time of the last call (ROWS mode)
    // block-row sharding (vf_shard.cpp; SURVEY §8(e) ROWS): this handle holds
    // the leaf rows of tree rows [row_lo, row_hi) only.
    bool sharded = false;
    int rank = 0, world = 1;
    int64_t row_lo = 0, row_hi = 0;
    std::vector<int64_t> row_bounds;     // world + 1 cut points
    std::vector<uint8_t> active_global;  // rows of the UNSHARDED F-hat with a stored entry
    void* comm = nullptr;                // ncclComm_t (vf_comm.cpp) or null
};

// error reporting (thread-local message)
int set_error(int code, const std::string& msg);

// host build (vf_build.cpp)
int build_handle(Handle* h, int64_t N, const double* x, const double* n, const double* A,
                 const double* occV, int64_t nv, const int32_t* occF, int64_t nt,
                 const int64_t* tri_of, double tol, const vf_build_opts& o);
int insolation(const Handle* h, const double* suns, int k, double S, double* Q);
int64_t leaf_nbytes(const Leaf& L, int w);

// block-row sharding (vf_shard.cpp)
int row_partition(const Handle* h, int world, std::vector<int64_t>& bounds);
int shard_rows(Handle* h, int rank, int world);
std::vector<uint8_t> active_rows_of(const Handle* h);

// NCCL (vf_comm.cpp; libnccl is dlopen'ed, sharing the process's copy)
int comm_get_id(void* id128);
int comm_init(Handle* h, int rank, int world, const void* id128);
void comm_destroy(Handle* h);
int comm_allgather(Handle* h, const void* send, void* recv, size_t bytes_per_rank, void* stream);

// HVFM io (vf_io.cpp)
int save_hvfm(const Handle* h, const char* path);
int load_hvfm(Handle* h, const char* path);

// device (vf_device.cu)
int device_upload(Handle* h, int device);
void device_free(Handle* h);
int device_matvec(Handle* h, const void* X, void* Y, int nrhs);
int device_solve_radiosity(Handle* h, const void* E, const void* rho, void* B, int nrhs,
                           int iters, double tol, int clamp);
int device_solve_thermal(Handle* h, const void* Qdir, const void* alb, const void* emi, void* T,
                         void* Qvis, void* Qir, int nrhs, int iters, double tol);
int64_t device_bytes(const Handle* h);
// Alg. 6 time stepping (vf_device.cu)
struct TState;
int device_ts_create(Handle* h, int ns, int M, double depth, double ratio, double k_th, double rho_c, double H,
                     const void* albedo, const void* emiss, const void* Qdir0, const void* T0, TState** out);
int device_ts_step(TState* S, const void* Qdir, double dt, void* Tsurf);
int device_ts_get(TState* S, void* Qrefl, void* Qir, void* Qabs, void* Tsurf);
void device_ts_free(TState* S);
int selftest_rows_exchange(int world, int kp, int k, int64_t N, const int64_t* bounds, const double* xrank,
                           const double* part, int nblk, const double* enorm2, double tol, int iters, int iter0,
                           double* xout, double* resid, int* iter_after, int* done_after);

// truncated SVD (vf_svd.cpp)
struct SvdResult {
    int64_t q = 0;              // accepted rank (0 = failure)
    std::vector<double> U;      // mu x q row-major
    std::vector<double> S;      // q
    std::vector<double> V;      // nv x q row-major
};
// Rank estimation of Alg. 3 on the compact (nonzero rows/cols) block given as
// a dense row-major mu x nv matrix or a CSR (rowptr/cols/vals with local
// compact columns).  target_bytes = nbytes(F_IJ) of eq. nbytes-comparison.
SvdResult estimate_rank(int64_t mu, int64_t nv, const double* dense, const int64_t* rowptr,
                        const int32_t* cols, const double* vals, double eps, int w, int k0,
                        int64_t target_bytes, int64_t m_full, int64_t n_full, uint64_t seed);

void svd_profile_report();
// large-block randomized SVD on the device (vf_svd_gpu.cu); false = not done
extern int g_svd_device;
bool gpu_randomized_svd(int64_t m, int64_t n, const int64_t* rowptr, const int32_t* cols, const double* vals,
                        const double* dense, const double* Om_rm, int64_t l, std::vector<double>& U_rm,
                        std::vector<double>& S, std::vector<double>& V_rm);
// one-sided Jacobi SVD of a small l x l column-major R (vf_svd.cpp): R <- Ur
void small_jacobi_svd(std::vector<double>& R, int64_t l, std::vector<double>& sig, std::vector<double>& W);

// device evaluator of the exact F for the build (vf_build_gpu.cu)
struct Bvh;
int gpu_exact_csr(int device, int64_t N, const double* x, const double* n, const double* A, const int64_t* tri,
                  const Bvh* bvh, std::vector<int64_t>& rowptr, std::vector<int32_t>& cols,
                  std::vector<double>& vals);

}  // namespace vf
