// vf_device.cu -- device layout of F-hat and the sm_100a hot path.
// PAPER.md = "P:<line>".  DESIGN.md §"Device layout" / §"Kernels".
//
// Alg. 5 is flattened into two launches of ONE segmented-row
// kernel over a single source buffer XT = [Xp ; T] (tree-order rows, k
// contiguous per row):
//   phase 1  (a2)  T_t = S_b[l] * sum_j V_b[j,l] Xp[col0_b + vrow_j]     for
//                  every rank-1 term t = (b, l) of every SVD block, blocks
//                  sorted by tree level (low-rank phase 1, "U(Sigma(V^T x))",
//                  S:276);
//   phase 2  (a3+a4) for every active tree row i: Y_i = sum over its
//                  segments: dense-leaf row (contiguous X rows), U_b row
//                  (contiguous T rows), merged CSR row (gathered X rows);
//                  followed by the fused Jacobi epilogue (clamp P:237,
//                  B' = E + rho Q, residual partials, B'/Q stores).
// Every output row is owned by one warp; segments are summed in a fixed
// order and per-CTA residual partials are reduced in a fixed order, so
// results are bitwise reproducible (no float atomics).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "vf_internal.h"

namespace vf {

namespace {

constexpr int kWarps = 8;               // warps per CTA (256 threads)
constexpr int kCtasPerSm = 6;
constexpr int kNumSms = 148;            // B200
constexpr double kSigmaSB = 5.670374419e-8;

struct Seg {                            // one run of a row's terms
    int64_t val_off;                    // first value in vals[]
    int64_t src;                        // kind 0: first XT row; kind 1: offset into idx[]
    int32_t len;
    int32_t kind;                       // 0 contiguous, 1 gather
};

struct Ctl {                            // device-side loop control
    int iter;                           // completed iterations
    int done;
    int pad[2];
};

enum Mode { M_PHASE1 = 0, M_MATVEC = 1, M_SOLVE = 2 };

#define CK(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return set_error(VF_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <typename T, int VEC>
struct VecIO;
template <>
struct VecIO<double, 1> {
    static __device__ __forceinline__ void ld(const double* p, double* v) { v[0] = __ldg(p); }
    static __device__ __forceinline__ void st(double* p, const double* v) { p[0] = v[0]; }
};
template <>
struct VecIO<double, 2> {
    static __device__ __forceinline__ void ld(const double* p, double* v) {
        double2 a = __ldg(reinterpret_cast<const double2*>(p)); v[0] = a.x; v[1] = a.y;
    }
    static __device__ __forceinline__ void st(double* p, const double* v) { *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]); }
};
template <>
struct VecIO<double, 4> {
    static __device__ __forceinline__ void ld(const double* p, double* v) {
        double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
    static __device__ __forceinline__ void st(double* p, const double* v) {
        reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
    }
};
template <>
struct VecIO<float, 1> {
    static __device__ __forceinline__ void ld(const float* p, float* v) { v[0] = __ldg(p); }
    static __device__ __forceinline__ void st(float* p, const float* v) { p[0] = v[0]; }
};
template <>
struct VecIO<float, 2> {
    static __device__ __forceinline__ void ld(const float* p, float* v) {
        float2 a = __ldg(reinterpret_cast<const float2*>(p)); v[0] = a.x; v[1] = a.y;
    }
    static __device__ __forceinline__ void st(float* p, const float* v) { *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]); }
};
template <>
struct VecIO<float, 4> {
    static __device__ __forceinline__ void ld(const float* p, float* v) {
        float4 a = __ldg(reinterpret_cast<const float4*>(p)); v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
    static __device__ __forceinline__ void st(float* p, const float* v) { *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]); }
};

struct RowArgs {
    const int64_t* segptr;    // [nrows + 1]
    const Seg* segs;
    const int32_t* rows;      // output row id per row (phase 2: tree row; phase 1: t)
    int64_t nrows;
    const void* vals;
    const int32_t* idx;
    const void* scale;        // phase 1: S per T row
    const void* xt;           // source rows (XT[cur])
    void* out;                // phase 1: XT[cur] (T region written at row N+t); matvec: Yp; solve: XT[next]
    const void* E;            // solve
    const void* rho;          // solve (nullptr => rho = 1)
    void* Q;                  // solve: last Q
    double* partial;          // solve: [gridDim.x][kp] residual partial sums
    const Ctl* ctl;
    int64_t N;                // rows of Xp (T region starts at N)
    int kp;
    int clamp;
};

// Segmented-row kernel.  One warp per output row; lane = (group g, sub-lane c):
// KC sub-lanes cover KC*VEC consecutive columns, the 32/KC groups split the
// row's terms; groups are combined by a fixed xor-shuffle tree.
template <typename T, int KC, int VEC, int MODE>
__global__ void __launch_bounds__(kWarps * 32)
segrow_kernel(RowArgs a) {
    constexpr int G = 32 / KC;
    constexpr int CW = KC * VEC;
    if (a.ctl && a.ctl->done) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / KC, c = lane % KC;
    const int col = blockIdx.y * CW + c * VEC;
    const bool col_ok = col < a.kp;
    const int64_t kp = a.kp;
    const T* __restrict__ vals = static_cast<const T*>(a.vals);
    const T* __restrict__ xt = static_cast<const T*>(a.xt);
    int cur = a.ctl ? (a.ctl->iter & 1) : 0;
    (void)cur;
    double part[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) part[v] = 0.0;

    const int64_t wstride = (int64_t)gridDim.x * kWarps;
    for (int64_t r = (int64_t)blockIdx.x * kWarps + warp; r < a.nrows; r += wstride) {
        T acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = T(0);
        const int64_t s0 = a.segptr[r], s1 = a.segptr[r + 1];
        for (int64_t s = s0; s < s1; ++s) {
            const Seg sg = a.segs[s];
            const T* __restrict__ vp = vals + sg.val_off;
            if (sg.kind == 0) {
                const T* __restrict__ xp = xt + sg.src * kp + col;
#pragma unroll 4
                for (int e = g; e < sg.len; e += G) {
                    const T w = __ldg(vp + e);
                    if (col_ok) {
                        T x[VEC];
                        VecIO<T, VEC>::ld(xp + (int64_t)e * kp, x);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] = fma(w, x[v], acc[v]);
                    }
                }
            } else {
                const int32_t* __restrict__ ip = a.idx + sg.src;
#pragma unroll 4
                for (int e = g; e < sg.len; e += G) {
                    const T w = __ldg(vp + e);
                    const int64_t xr = __ldg(ip + e);
                    if (col_ok) {
                        T x[VEC];
                        VecIO<T, VEC>::ld(xt + xr * kp + col, x);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] = fma(w, x[v], acc[v]);
                    }
                }
            }
        }
#pragma unroll
        for (int off = KC; off < 32; off <<= 1)
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], off);
        if (g != 0 || !col_ok) continue;
        const int64_t orow = a.rows[r];
        if (MODE == M_PHASE1) {
            const T s = static_cast<const T*>(a.scale)[orow];
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] *= s;
            VecIO<T, VEC>::st(static_cast<T*>(a.out) + (a.N + orow) * kp + col, acc);
        } else if (MODE == M_MATVEC) {
            VecIO<T, VEC>::st(static_cast<T*>(a.out) + orow * kp + col, acc);
        } else {
            const int64_t o = orow * kp + col;
            T e[VEC], bo[VEC], bn[VEC];
            VecIO<T, VEC>::ld(static_cast<const T*>(a.E) + o, e);
            VecIO<T, VEC>::ld(xt + o, bo);
            const T rh = a.rho ? static_cast<const T*>(a.rho)[orow] : T(1);
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                if (a.clamp) acc[v] = acc[v] > T(0) ? acc[v] : T(0);
                bn[v] = e[v] + rh * acc[v];                               // eq. (1)
                const double d = (double)bn[v] - (double)bo[v];
                if (col + v < a.kp) part[v] += d * d;
            }
            VecIO<T, VEC>::st(static_cast<T*>(a.out) + o, bn);
            VecIO<T, VEC>::st(static_cast<T*>(a.Q) + o, acc);
        }
    }
    if (MODE == M_SOLVE) {
        // CTA-level fixed-order reduction of residual partials: [warp][CW]
        __shared__ double red[kWarps][32 * 4];
        if (g == 0) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) red[warp][c * VEC + v] = part[v];
        }
        __syncthreads();
        for (int cc = threadIdx.x; cc < CW; cc += blockDim.x) {
            double s = 0.0;
            for (int w = 0; w < kWarps; ++w) s += red[w][cc];
            const int gc = blockIdx.y * CW + cc;
            if (gc < a.kp) a.partial[(int64_t)blockIdx.x * kp + gc] = s;
        }
    }
}

// Per-column sums of partial[nblk][kp] in block order -> r_c, loop control.
__global__ void reduce_kernel(const double* partial, int nblk, int kp, int k, const double* enorm2,
                              double* resid, Ctl* ctl, int iters, double tol) {
    if (ctl->done) return;
    __shared__ int ok;
    if (threadIdx.x == 0) ok = 1;
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < nblk; ++b) s += partial[(int64_t)b * kp + c];
        const double en = enorm2[c];
        const double r = en > 0.0 ? sqrt(s) / sqrt(en) : 0.0;
        resid[c] = r;
        if (!(r <= tol)) atomicAnd(&ok, 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int it = ctl->iter + 1;
        ctl->iter = it;
        if (ok || it >= iters) ctl->done = 1;
    }
}

// Column sums of squares of V (tree order, N x kp): per-CTA partials.
template <typename T>
__global__ void colnorm_partial_kernel(const T* V, int64_t N, int kp, double* partial) {
    extern __shared__ double sh[];
    for (int c = threadIdx.x; c < kp; c += blockDim.x) sh[c] = 0.0;
    __syncthreads();
    // each CTA owns a contiguous row range; thread t handles column t % kp
    const int64_t rows_per = (N + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(N, r0 + rows_per);
    const int lanes_per_col = max(1, (int)blockDim.x / kp);
    const int c = threadIdx.x % kp, j = threadIdx.x / kp;
    double s = 0.0;
    if (j < lanes_per_col && threadIdx.x < lanes_per_col * kp)
        for (int64_t r = r0 + j; r < r1; r += lanes_per_col) {
            const double v = (double)V[r * kp + c];
            s += v * v;
        }
    // fixed-order combine: sh[c] += s for j = 0..lanes_per_col-1 in order
    for (int jj = 0; jj < lanes_per_col; ++jj) {
        __syncthreads();
        if (j == jj && threadIdx.x < lanes_per_col * kp) sh[c] += s;
    }
    __syncthreads();
    for (int cc = threadIdx.x; cc < kp; cc += blockDim.x) partial[(int64_t)blockIdx.x * kp + cc] = sh[cc];
}

__global__ void colnorm_final_kernel(const double* partial, int nblk, int kp, int k, double* out) {
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < nblk; ++b) s += partial[(int64_t)b * kp + c];
        out[c] = s;
    }
}

// Caller order (column-major N x k, ld N) -> tree order (N x kp, row-major):
// dst[r, c] = src[perm[r] + c N] * (mul ? mul[perm[r]] : 1); padding columns 0.
// Writes up to three destinations (for E/B initialisation).
template <typename T>
__global__ void permute_in_kernel(const T* src, const int32_t* perm, int64_t N, int k, int kp,
                                  const T* mul, T* d0, T* d1, T* d2, T* raw) {
    __shared__ T tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    // load: threads over rows (gather through perm), loop over 32 columns
    for (int cc = threadIdx.y; cc < 32; cc += blockDim.y) {
        const int64_t r = r0 + threadIdx.x;
        const int c = c0 + cc;
        T v = T(0);
        if (r < N && c < k) {
            const int64_t p = perm[r];
            v = src[p + (int64_t)c * N];
        }
        tile[threadIdx.x][cc] = v;
    }
    __syncthreads();
    for (int rr = threadIdx.y; rr < 32; rr += blockDim.y) {
        const int64_t r = r0 + rr;
        const int c = c0 + threadIdx.x;
        if (r < N && c < kp) {
            T v = tile[rr][threadIdx.x];
            if (raw) raw[r * kp + c] = v;
            if (mul) v *= mul[perm[r]];
            if (d0) d0[r * kp + c] = v;
            if (d1) d1[r * kp + c] = v;
            if (d2) d2[r * kp + c] = v;
        }
    }
}

// tree order (N x kp) -> caller order (N x k): dst[perm[r] + c N] = active[r] ? src : 0
template <typename T>
__global__ void permute_out_kernel(const T* src, const int32_t* perm, const uint8_t* active, int64_t N, int k,
                                   int kp, T* dst) {
    __shared__ T tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    for (int rr = threadIdx.y; rr < 32; rr += blockDim.y) {
        const int64_t r = r0 + rr;
        const int c = c0 + threadIdx.x;
        T v = T(0);
        if (r < N && c < k && (!active || active[r])) v = src[r * kp + c];
        tile[rr][threadIdx.x] = v;
    }
    __syncthreads();
    for (int cc = threadIdx.y; cc < 32; cc += blockDim.y) {
        const int64_t r = r0 + threadIdx.x;
        const int c = c0 + cc;
        if (r < N && c < k) dst[(int64_t)perm[r] + (int64_t)c * N] = tile[threadIdx.x][cc];
    }
}

// length-N parameter vector, caller order -> tree order
template <typename T>
__global__ void gather_vec_kernel(const T* src, const int32_t* perm, int64_t N, T* dst) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x)
        dst[r] = src[perm[r]];
}

// Thermal stage change (a7): Qvis = Qdir + Qrefl (Qrefl = last Q, 0 on
// inactive rows); E2 = (1 - alpha) Qvis into E and both XT buffers.
template <typename T>
__global__ void thermal_mid_kernel(const T* Qdir, const T* Q, const uint8_t* active, const T* alpha, int64_t N,
                                   int k, int kp, T* Qvis, T* E, T* x0, T* x1) {
    const int64_t tot = N * kp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / kp;
        const int c = (int)(i - r * kp);
        T qv = T(0), e = T(0);
        if (c < k) {
            qv = Qdir[i] + (active[r] ? Q[i] : T(0));
            e = (T(1) - alpha[r]) * qv;
        }
        Qvis[i] = qv;
        E[i] = e;
        x0[i] = e;
        x1[i] = e;
    }
}

// T = (((1 - alpha) Qvis + eps Qir) / (eps sigma))^(1/4)   (eq. 3d-equilbr)
template <typename T>
__global__ void thermal_T_kernel(const T* Qvis, const T* Q, const uint8_t* active, const T* alpha, const T* emis,
                                 int64_t N, int k, int kp, T* Tout, T* Qir) {
    const int64_t tot = N * kp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / kp;
        const int c = (int)(i - r * kp);
        if (c >= k) { Tout[i] = T(0); Qir[i] = T(0); continue; }
        const T qir = active[r] ? Q[i] : T(0);
        const T qabs = (T(1) - alpha[r]) * Qvis[i] + emis[r] * qir;
        Tout[i] = (T)sqrt(sqrt((double)qabs / ((double)emis[r] * kSigmaSB)));
        Qir[i] = qir;
    }
}

}  // namespace

// --------------------------------------------------------------- layout
struct DeviceHMat {
    int64_t N = 0, NT = 0;              // tree rows, T rows (sum of ranks)
    int w = 8;
    int dtype = VF_F64;
    // F-hat
    void* vals = nullptr;
    int32_t* idx = nullptr;
    Seg* segs = nullptr;
    int64_t* p1_segptr = nullptr;
    int32_t* p1_rows = nullptr;
    void* p1_scale = nullptr;
    int64_t n_p1 = 0;
    int64_t* p2_segptr = nullptr;
    int32_t* p2_rows = nullptr;
    int64_t n_p2 = 0;
    int32_t* perm = nullptr;
    uint8_t* active = nullptr;
    int64_t bytes = 0;
    int64_t alg_bytes = 0;
    int64_t alg_flops_per_col = 0;
    int64_t p1_bytes = 0, p2_bytes = 0, p1_src = 0, p2_src = 0, p1_flops = 0, p2_flops = 0;
    // kernel timing: event pool, pairs recorded around phase launches
    std::vector<cudaEvent_t> evpool;
    std::vector<int> evwhich;     // phase of pair i (1 or 2)
    int evused = 0;
    // scratch (grown by kp)
    int kp_cap = 0;
    void* xt[2] = {nullptr, nullptr};
    void* Ep = nullptr;
    void* Qp = nullptr;       // last Q
    void* Qdp = nullptr;      // Qdir (tree)
    void* Qvp = nullptr;      // Qvis (tree)
    void* Yp = nullptr;       // matvec result / T (tree)
    void* Qip = nullptr;      // Qir (tree)
    void* pv[3] = {nullptr, nullptr, nullptr};   // rho/alpha, emis (tree), spare
    double* partial = nullptr;
    double* enorm2 = nullptr;
    double* resid = nullptr;
    int64_t partial_cap = 0;
    Ctl* ctl = nullptr;
    Ctl* ctl_host = nullptr;  // pinned
    double* resid_host = nullptr;
    int resid_host_cap = 0;
    // staging for host pointers
    void* stage[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    size_t stage_cap[6] = {0, 0, 0, 0, 0, 0};
};

namespace {

int grid_rows(int64_t nrows) {
    int64_t g = (nrows + kWarps - 1) / kWarps;
    g = std::min<int64_t>(g, (int64_t)kNumSms * kCtasPerSm);
    return (int)std::max<int64_t>(g, 1);
}

template <typename T>
int upload_impl(Handle* h, DeviceHMat* D) {
    const int64_t N = h->N;
    D->N = N;
    D->w = sizeof(T);
    D->dtype = h->dtype;
    // order SVD leaves by tree level (stable) for phase 1
    std::vector<int> svd_ids;
    for (int b = 0; b < (int)h->leaves.size(); ++b)
        if (h->leaves[b].kind == K_SVD) svd_ids.push_back(b);
    std::stable_sort(svd_ids.begin(), svd_ids.end(),
                     [&](int a, int b) { return h->leaves[a].level < h->leaves[b].level; });
    std::vector<int64_t> toff(h->leaves.size(), -1);
    int64_t NT = 0;
    for (int b : svd_ids) { toff[b] = NT; NT += h->leaves[b].q; }
    D->NT = NT;

    std::vector<T> vals;
    std::vector<int32_t> idx;
    std::vector<Seg> segs;
    auto push_vals = [&](const double* p, int64_t n) {
        int64_t off = (int64_t)vals.size();
        for (int64_t i = 0; i < n; ++i) vals.push_back((T)p[i]);
        // keep every segment start 16-byte aligned
        while ((vals.size() * sizeof(T)) % 16) vals.push_back(T(0));
        return off;
    };
    int64_t alg_bytes = 0, alg_flops = 0;

    // ---- phase 1 rows: t = (b, l) ----
    std::vector<int64_t> p1_segptr(1, 0);
    std::vector<int32_t> p1_rows;
    std::vector<T> p1_scale;
    for (int b : svd_ids) {
        const Leaf& L = h->leaves[b];
        const int64_t nv = (int64_t)L.idx_b.size(), q = L.q;
        bool contig = true;
        for (int64_t j = 1; j < nv; ++j) contig = contig && (L.idx_b[j] == L.idx_b[0] + j);
        int64_t ioff = -1;
        if (!contig) {
            ioff = (int64_t)idx.size();
            for (int64_t j = 0; j < nv; ++j) idx.push_back((int32_t)(L.col0 + L.idx_b[j]));
            alg_bytes += 4 * nv;
        }
        std::vector<double> col(nv);
        for (int64_t l = 0; l < q; ++l) {
            for (int64_t j = 0; j < nv; ++j) col[j] = L.b[j * q + l];
            int64_t voff = push_vals(col.data(), nv);
            Seg s;
            s.val_off = voff;
            s.len = (int32_t)nv;
            if (contig) { s.kind = 0; s.src = L.col0 + (nv ? L.idx_b[0] : 0); }
            else { s.kind = 1; s.src = ioff; }
            segs.push_back(s);
            p1_segptr.push_back((int64_t)segs.size() - 0);
            p1_rows.push_back((int32_t)(toff[b] + l));
            p1_scale.push_back((T)L.s[l]);
        }
        alg_bytes += (int64_t)sizeof(T) * (q * nv + q);
        alg_flops += 2 * q * nv + q;
    }
    const int64_t p1_seg_count = (int64_t)segs.size();
    D->p1_bytes = alg_bytes;
    D->p1_flops = alg_flops;
    {
        std::vector<char> used(N, 0);
        for (int b : svd_ids) {
            const Leaf& L = h->leaves[b];
            for (int32_t j : L.idx_b) used[L.col0 + j] = 1;
        }
        D->p1_src = std::count(used.begin(), used.end(), 1);
    }

    // ---- phase 2 rows: per tree row, its segments ----
    std::vector<std::vector<Seg>> rowsegs(N);
    // CSR leaves merged per row: collect (global col, value)
    std::vector<std::vector<std::pair<int32_t, double>>> csr_rows(N);
    for (int b = 0; b < (int)h->leaves.size(); ++b) {
        const Leaf& L = h->leaves[b];
        if (L.kind == K_DENSE) {
            for (int64_t r = 0; r < L.m; ++r) {
                Seg s;
                s.val_off = push_vals(L.a.data() + r * L.n, L.n);
                s.src = L.col0; s.len = (int32_t)L.n; s.kind = 0;
                rowsegs[L.row0 + r].push_back(s);
            }
            alg_bytes += (int64_t)sizeof(T) * L.m * L.n;
            alg_flops += 2 * L.m * L.n;
        } else if (L.kind == K_SVD) {
            const int64_t mu = (int64_t)L.idx_a.size();
            for (int64_t r = 0; r < mu; ++r) {
                Seg s;
                s.val_off = push_vals(L.a.data() + r * L.q, L.q);
                s.src = N + toff[b]; s.len = (int32_t)L.q; s.kind = 0;
                rowsegs[L.row0 + L.idx_a[r]].push_back(s);
            }
            alg_bytes += (int64_t)sizeof(T) * L.q * mu + 4 * mu;
            alg_flops += 2 * L.q * mu;
        } else if (L.kind == K_CSR) {
            for (int64_t r = 0; r < L.m; ++r)
                for (int64_t e = L.rowptr[r]; e < L.rowptr[r + 1]; ++e)
                    csr_rows[L.row0 + r].push_back({(int32_t)(L.col0 + L.idx_a[e]), L.a[e]});
            const int64_t nnz = (int64_t)L.idx_a.size();
            alg_bytes += (int64_t)(sizeof(T) + 4) * nnz + 8 * (L.m + 1);
            alg_flops += 2 * nnz;
        }
    }
    std::vector<int64_t> p2_segptr(1, p1_seg_count);
    std::vector<int32_t> p2_rows;
    std::vector<uint8_t> active(N, 0);
    std::vector<double> cv;
    for (int64_t i = 0; i < N; ++i) {
        auto& cr = csr_rows[i];
        if (rowsegs[i].empty() && cr.empty()) continue;
        for (auto& s : rowsegs[i]) segs.push_back(s);
        if (!cr.empty()) {
            std::stable_sort(cr.begin(), cr.end(), [](auto& a, auto& b) { return a.first < b.first; });
            Seg s;
            s.src = (int64_t)idx.size();
            for (auto& p : cr) idx.push_back(p.first);
            while (idx.size() % 4) idx.push_back(0);
            cv.resize(cr.size());
            for (size_t e = 0; e < cr.size(); ++e) cv[e] = cr[e].second;
            s.val_off = push_vals(cv.data(), (int64_t)cv.size());
            s.len = (int32_t)cr.size(); s.kind = 1;
            segs.push_back(s);
        }
        p2_segptr.push_back((int64_t)segs.size());
        p2_rows.push_back((int32_t)i);
        active[i] = 1;
        std::vector<std::pair<int32_t, double>>().swap(cr);
    }
    if (vals.empty()) vals.push_back(T(0));
    if (idx.empty()) idx.push_back(0);
    if (segs.empty()) segs.push_back(Seg{0, 0, 0, 0});
    D->n_p1 = (int64_t)p1_rows.size();
    D->n_p2 = (int64_t)p2_rows.size();
    D->alg_bytes = alg_bytes;
    D->alg_flops_per_col = alg_flops;
    D->p2_bytes = alg_bytes - D->p1_bytes;
    D->p2_flops = alg_flops - D->p1_flops;
    {
        std::vector<char> used(N + NT, 0);
        for (int64_t r = 0; r < (int64_t)p2_rows.size(); ++r)
            for (int64_t s = p2_segptr[r]; s < p2_segptr[r + 1]; ++s) {
                const Seg& sg = segs[s];
                for (int32_t e = 0; e < sg.len; ++e) used[sg.kind == 0 ? sg.src + e : idx[sg.src + e]] = 1;
            }
        D->p2_src = std::count(used.begin(), used.end(), 1);
    }

    auto up = [&](void** dst, const void* src, size_t bytes) -> int {
        if (bytes == 0) bytes = 16;
        CK(cudaMalloc(dst, bytes));
        D->bytes += (int64_t)bytes;
        if (src) CK(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
        return VF_OK;
    };
    int rc;
    if ((rc = up(&D->vals, vals.data(), vals.size() * sizeof(T)))) return rc;
    if ((rc = up((void**)&D->idx, idx.data(), idx.size() * 4))) return rc;
    if ((rc = up((void**)&D->segs, segs.data(), segs.size() * sizeof(Seg)))) return rc;
    if ((rc = up((void**)&D->p1_segptr, p1_segptr.data(), p1_segptr.size() * 8))) return rc;
    if ((rc = up((void**)&D->p1_rows, p1_rows.data(), p1_rows.size() * 4))) return rc;
    if ((rc = up(&D->p1_scale, p1_scale.data(), p1_scale.size() * sizeof(T)))) return rc;
    if ((rc = up((void**)&D->p2_segptr, p2_segptr.data(), p2_segptr.size() * 8))) return rc;
    if ((rc = up((void**)&D->p2_rows, p2_rows.data(), p2_rows.size() * 4))) return rc;
    if ((rc = up((void**)&D->perm, h->perm.data(), h->perm.size() * 4))) return rc;
    if ((rc = up((void**)&D->active, active.data(), active.size()))) return rc;
    CK(cudaMalloc((void**)&D->ctl, sizeof(Ctl)));
    CK(cudaMallocHost((void**)&D->ctl_host, sizeof(Ctl)));
    D->evpool.resize(2048);
    D->evwhich.resize(1024);
    for (auto& e : D->evpool) CK(cudaEventCreate(&e));
    return VF_OK;
}

int ensure_scratch(DeviceHMat* D, int kp) {
    if (kp <= D->kp_cap) return VF_OK;
    void** bufs[] = {&D->xt[0], &D->xt[1], &D->Ep, &D->Qp, &D->Qdp, &D->Qvp, &D->Yp, &D->Qip};
    for (void** b : bufs) if (*b) { cudaFree(*b); *b = nullptr; }
    for (void*& b : D->pv) if (b) { cudaFree(b); b = nullptr; }
    const size_t rows_x = (size_t)(D->N + D->NT), rows = (size_t)D->N;
    for (int i = 0; i < 2; ++i) {
        CK(cudaMalloc(&D->xt[i], std::max<size_t>(16, rows_x * kp * D->w)));
        CK(cudaMemset(D->xt[i], 0, std::max<size_t>(16, rows_x * kp * D->w)));
    }
    void** vbufs[] = {&D->Ep, &D->Qp, &D->Qdp, &D->Qvp, &D->Yp, &D->Qip};
    for (void** b : vbufs) {
        CK(cudaMalloc(b, std::max<size_t>(16, rows * kp * D->w)));
        CK(cudaMemset(*b, 0, std::max<size_t>(16, rows * kp * D->w)));
    }
    for (void*& b : D->pv) CK(cudaMalloc(&b, std::max<size_t>(16, rows * D->w)));
    const int64_t nblk = (int64_t)kNumSms * kCtasPerSm;
    if (D->partial) cudaFree(D->partial);
    CK(cudaMalloc((void**)&D->partial, (size_t)nblk * kp * 8));
    CK(cudaMemset(D->partial, 0, (size_t)nblk * kp * 8));
    if (D->enorm2) cudaFree(D->enorm2);
    if (D->resid) cudaFree(D->resid);
    CK(cudaMalloc((void**)&D->enorm2, (size_t)kp * 8));
    CK(cudaMalloc((void**)&D->resid, (size_t)kp * 8));
    if (D->resid_host) cudaFreeHost(D->resid_host);
    CK(cudaMallocHost((void**)&D->resid_host, (size_t)kp * 8));
    D->kp_cap = kp;
    return VF_OK;
}

int pad_k(int k) {
    if (k <= 2) return k;
    return (k + 3) & ~3;
}

// ---------------------------------------------------------- launching
template <typename T, int MODE>
void launch_segrow(const RowArgs& a, int kp, cudaStream_t st, int* nblk_out) {
    const int grid = grid_rows(a.nrows);
    if (nblk_out) *nblk_out = grid;
    auto go = [&](auto kern, int cw) {
        dim3 g(grid, (kp + cw - 1) / cw);
        kern<<<g, kWarps * 32, 0, st>>>(a);
    };
    if (kp == 1) go(segrow_kernel<T, 1, 1, MODE>, 1);
    else if (kp == 2) go(segrow_kernel<T, 1, 2, MODE>, 2);
    else if (kp <= 4) go(segrow_kernel<T, 1, 4, MODE>, 4);
    else if (kp <= 8) go(segrow_kernel<T, 2, 4, MODE>, 8);
    else if (kp <= 16) go(segrow_kernel<T, 4, 4, MODE>, 16);
    else if (kp <= 32) go(segrow_kernel<T, 8, 4, MODE>, 32);
    else if (kp <= 64) go(segrow_kernel<T, 16, 4, MODE>, 64);
    else go(segrow_kernel<T, 32, 4, MODE>, 128);
}

// Records a CUDA event pair around one phase launch on the launching stream
// (no synchronisation); collect_timing() reads them after the call's final sync.
struct Timer {
    Handle* h;
    cudaStream_t st;
    int idx = -1;
    Timer(Handle* hh, cudaStream_t s, int which) : h(hh), st(s) {
        DeviceHMat* D = h->dev;
        if (!h->timing || D->evused + 2 > (int)D->evpool.size()) return;
        idx = D->evused;
        D->evused += 2;
        D->evwhich[idx / 2] = which;
        cudaEventRecord(D->evpool[idx], st);
    }
    ~Timer() {
        if (idx >= 0) cudaEventRecord(h->dev->evpool[idx + 1], st);
    }
};

void collect_timing(Handle* h) {
    DeviceHMat* D = h->dev;
    for (int i = 0; i + 1 < D->evused; i += 2) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, D->evpool[i], D->evpool[i + 1]) != cudaSuccess) { cudaGetLastError(); continue; }
        if (D->evwhich[i / 2] == 2) { h->ms_p2 += ms; h->launches_p2++; }
        else { h->ms_p1 += ms; h->launches_p1++; }
    }
    D->evused = 0;
}

void reset_counters(Handle* h) {
    h->ms_p1 = h->ms_p2 = 0;
    h->launches_p1 = h->launches_p2 = h->launches_total = 0;
    h->dev->evused = 0;
}

// One F-hat apply of XT[src] (phases 1 and 2).
template <typename T, int MODE>
int apply_once(Handle* h, int src, int kp, cudaStream_t st, void* out, const void* E, const void* rho, int clamp,
               int* nblk2) {
    DeviceHMat* D = h->dev;
    if (D->n_p1 > 0) {
        RowArgs a{};
        a.segptr = D->p1_segptr; a.segs = D->segs; a.rows = D->p1_rows; a.nrows = D->n_p1;
        a.vals = D->vals; a.idx = D->idx; a.scale = D->p1_scale;
        a.xt = D->xt[src]; a.out = D->xt[src];
        a.ctl = D->ctl; a.N = D->N; a.kp = kp;
        Timer tm(h, st, 1);
        launch_segrow<T, M_PHASE1>(a, kp, st, nullptr);
        h->launches_total++;
    }
    RowArgs a{};
    a.segptr = D->p2_segptr; a.segs = D->segs; a.rows = D->p2_rows; a.nrows = D->n_p2;
    a.vals = D->vals; a.idx = D->idx;
    a.xt = D->xt[src]; a.out = out;
    a.E = E; a.rho = rho; a.Q = D->Qp; a.partial = D->partial;
    a.ctl = D->ctl; a.N = D->N; a.kp = kp; a.clamp = clamp;
    {
        Timer tm(h, st, 2);
        launch_segrow<T, MODE>(a, kp, st, nblk2);
    }
    h->launches_total++;
    return VF_OK;
}

int stream_of(Handle* h, cudaStream_t* st) {
    *st = (cudaStream_t)h->stream;
    CK(cudaSetDevice(h->device));
    return VF_OK;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Stage a host pointer into a handle buffer (slot) when needed.
int stage_in(Handle* h, int slot, const void* p, size_t bytes, cudaStream_t st, const void** out) {
    if (!p || is_device_ptr(p)) { *out = p; return VF_OK; }
    DeviceHMat* D = h->dev;
    if (D->stage_cap[slot] < bytes) {
        if (D->stage[slot]) cudaFree(D->stage[slot]);
        CK(cudaMalloc(&D->stage[slot], bytes));
        D->stage_cap[slot] = bytes;
    }
    CK(cudaMemcpyAsync(D->stage[slot], p, bytes, cudaMemcpyHostToDevice, st));
    *out = D->stage[slot];
    return VF_OK;
}

int stage_out_buf(Handle* h, int slot, void* p, size_t bytes, void** out) {
    if (!p || is_device_ptr(p)) { *out = p; return VF_OK; }
    DeviceHMat* D = h->dev;
    if (D->stage_cap[slot] < bytes) {
        if (D->stage[slot]) cudaFree(D->stage[slot]);
        CK(cudaMalloc(&D->stage[slot], bytes));
        D->stage_cap[slot] = bytes;
    }
    *out = D->stage[slot];
    return VF_OK;
}

int stage_out_copy(void* host, const void* dev, size_t bytes, cudaStream_t st) {
    if (!host || host == dev) return VF_OK;
    CK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st));
    return VF_OK;
}

template <typename T>
void launch_permute_in(Handle* h, const void* src, int k, int kp, const void* mul, void* d0, void* d1, void* d2,
                       void* raw, cudaStream_t st) {
    DeviceHMat* D = h->dev;
    dim3 g((unsigned)((D->N + 31) / 32), (unsigned)((kp + 31) / 32));
    permute_in_kernel<T><<<g, dim3(32, 8), 0, st>>>((const T*)src, D->perm, D->N, k, kp, (const T*)mul, (T*)d0,
                                                    (T*)d1, (T*)d2, (T*)raw);
    h->launches_total++;
}

template <typename T>
void launch_permute_out(Handle* h, const void* src, int k, int kp, bool use_active, void* dst, cudaStream_t st) {
    DeviceHMat* D = h->dev;
    dim3 g((unsigned)((D->N + 31) / 32), (unsigned)((kp + 31) / 32));
    permute_out_kernel<T><<<g, dim3(32, 8), 0, st>>>((const T*)src, D->perm, use_active ? D->active : nullptr, D->N,
                                                     k, kp, (T*)dst);
    h->launches_total++;
}

template <typename T>
void launch_colnorm(Handle* h, const void* V, int k, int kp, cudaStream_t st) {
    DeviceHMat* D = h->dev;
    const int nblk = 148;
    colnorm_partial_kernel<T><<<nblk, 256, kp * sizeof(double), st>>>((const T*)V, D->N, kp, D->partial);
    colnorm_final_kernel<<<1, 256, 0, st>>>(D->partial, nblk, kp, k, D->enorm2);
    h->launches_total += 2;
}

// Jacobi iterations on the current XT/E/rho state until ctl->done.
template <typename T>
int iterate(Handle* h, int k, int kp, const void* rho, int clamp, int iters, double tol, cudaStream_t st,
            int* iters_done, double* max_resid) {
    DeviceHMat* D = h->dev;
    CK(cudaMemsetAsync(D->ctl, 0, sizeof(Ctl), st));
    *iters_done = 0;
    *max_resid = 0;
    if (iters <= 0) return VF_OK;
    int enq = 0, chunk = 2;
    while (true) {
        for (int c = 0; c < chunk && enq < iters; ++c, ++enq) {
            const int src = enq & 1;     // == ctl->iter & 1 while not done
            int nblk = 1;
            int rc = apply_once<T, M_SOLVE>(h, src, kp, st, D->xt[src ^ 1], D->Ep, rho, clamp, &nblk);
            if (rc) return rc;
            reduce_kernel<<<1, 256, 0, st>>>(D->partial, nblk, kp, k, D->enorm2, D->resid, D->ctl, iters, tol);
            h->launches_total++;
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(D->ctl_host, D->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (D->ctl_host->done || enq >= iters) break;
        chunk = std::min(chunk * 2, 16);
    }
    *iters_done = D->ctl_host->iter;
    CK(cudaMemcpyAsync(D->resid_host, D->resid, (size_t)k * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double mr = 0;
    for (int c = 0; c < k; ++c) mr = std::max(mr, D->resid_host[c]);
    *max_resid = mr;
    return VF_OK;
}

template <typename T>
int matvec_impl(Handle* h, const void* X, void* Y, int nrhs) {
    DeviceHMat* D = h->dev;
    cudaStream_t st;
    int rc;
    if ((rc = stream_of(h, &st))) return rc;
    const int kp = pad_k(nrhs);
    if ((rc = ensure_scratch(D, kp))) return rc;
    reset_counters(h);
    const size_t vb = (size_t)D->N * nrhs * sizeof(T);
    const void* Xd;
    void* Yd;
    if ((rc = stage_in(h, 0, X, vb, st, &Xd))) return rc;
    if ((rc = stage_out_buf(h, 1, Y, vb, &Yd))) return rc;
    CK(cudaMemsetAsync(D->ctl, 0, sizeof(Ctl), st));
    launch_permute_in<T>(h, Xd, nrhs, kp, nullptr, D->xt[0], nullptr, nullptr, nullptr, st);
    if ((rc = apply_once<T, M_MATVEC>(h, 0, kp, st, D->Yp, nullptr, nullptr, 0, nullptr))) return rc;
    launch_permute_out<T>(h, D->Yp, nrhs, kp, true, Yd, st);
    CK(cudaGetLastError());
    if ((rc = stage_out_copy(Y, Yd, vb, st))) return rc;
    if (Yd != Y || h->timing) CK(cudaStreamSynchronize(st));
    if (h->timing) collect_timing(h);
    return VF_OK;
}

template <typename T>
int radiosity_impl(Handle* h, const void* E, const void* rho, void* B, int nrhs, int iters, double tol, int clamp) {
    DeviceHMat* D = h->dev;
    cudaStream_t st;
    int rc;
    if ((rc = stream_of(h, &st))) return rc;
    const int kp = pad_k(nrhs);
    if ((rc = ensure_scratch(D, kp))) return rc;
    reset_counters(h);
    const size_t vb = (size_t)D->N * nrhs * sizeof(T);
    const void *Ed, *rd;
    void* Bd;
    if ((rc = stage_in(h, 0, E, vb, st, &Ed))) return rc;
    if ((rc = stage_in(h, 1, rho, (size_t)D->N * sizeof(T), st, &rd))) return rc;
    if ((rc = stage_out_buf(h, 2, B, vb, &Bd))) return rc;
    gather_vec_kernel<T><<<148, 256, 0, st>>>((const T*)rd, D->perm, D->N, (T*)D->pv[0]);
    h->launches_total++;
    launch_permute_in<T>(h, Ed, nrhs, kp, nullptr, D->Ep, D->xt[0], D->xt[1], nullptr, st);
    launch_colnorm<T>(h, D->Ep, nrhs, kp, st);
    int it = 0;
    double res = 0;
    if ((rc = iterate<T>(h, nrhs, kp, D->pv[0], clamp, iters, tol, st, &it, &res))) return rc;
    h->iters1 = it; h->resid1 = res; h->iters2 = 0; h->resid2 = 0;
    launch_permute_out<T>(h, D->xt[it & 1], nrhs, kp, false, Bd, st);
    CK(cudaGetLastError());
    if ((rc = stage_out_copy(B, Bd, vb, st))) return rc;
    CK(cudaStreamSynchronize(st));
    if (h->timing) collect_timing(h);
    if (iters > 0 && !(res <= tol)) return set_error(VF_ENOCONV, "vf_solve_radiosity: no convergence within iters");
    return VF_OK;
}

template <typename T>
int thermal_impl(Handle* h, const void* Qdir, const void* alb, const void* emi, void* Tout, void* Qvis, void* Qir,
                 int nrhs, int iters, double tol) {
    DeviceHMat* D = h->dev;
    cudaStream_t st;
    int rc;
    if ((rc = stream_of(h, &st))) return rc;
    const int kp = pad_k(nrhs);
    if ((rc = ensure_scratch(D, kp))) return rc;
    reset_counters(h);
    const size_t vb = (size_t)D->N * nrhs * sizeof(T), pb = (size_t)D->N * sizeof(T);
    const void *Qd, *ad, *ed;
    void *Td, *Qvd, *Qid;
    if ((rc = stage_in(h, 0, Qdir, vb, st, &Qd))) return rc;
    if ((rc = stage_in(h, 1, alb, pb, st, &ad))) return rc;
    if ((rc = stage_in(h, 2, emi, pb, st, &ed))) return rc;
    if ((rc = stage_out_buf(h, 3, Tout, vb, &Td))) return rc;
    if ((rc = stage_out_buf(h, 4, Qvis, vb, &Qvd))) return rc;
    if ((rc = stage_out_buf(h, 5, Qir, vb, &Qid))) return rc;
    T* alpha = (T*)D->pv[0];
    T* emis = (T*)D->pv[1];
    gather_vec_kernel<T><<<148, 256, 0, st>>>((const T*)ad, D->perm, D->N, alpha);
    gather_vec_kernel<T><<<148, 256, 0, st>>>((const T*)ed, D->perm, D->N, emis);
    h->launches_total += 2;
    // stage 1: E = alpha Qdir, rho = alpha (reading R-A14)
    launch_permute_in<T>(h, Qd, nrhs, kp, ad, D->Ep, D->xt[0], D->xt[1], D->Qdp, st);
    launch_colnorm<T>(h, D->Ep, nrhs, kp, st);
    int it1 = 0, it2 = 0;
    double r1 = 0, r2 = 0;
    if ((rc = iterate<T>(h, nrhs, kp, alpha, 1, iters, tol, st, &it1, &r1))) return rc;
    // stage 2: Qvis = Qdir + Qrefl, E = (1 - alpha) Qvis, rho = 1
    const int64_t tot = D->N * kp;
    const int gb = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
    thermal_mid_kernel<T><<<std::max(gb, 1), 256, 0, st>>>((const T*)D->Qdp, (const T*)D->Qp, D->active, alpha, D->N,
                                                          nrhs, kp, (T*)D->Qvp, (T*)D->Ep, (T*)D->xt[0],
                                                          (T*)D->xt[1]);
    h->launches_total++;
    launch_colnorm<T>(h, D->Ep, nrhs, kp, st);
    if ((rc = iterate<T>(h, nrhs, kp, nullptr, 1, iters, tol, st, &it2, &r2))) return rc;
    thermal_T_kernel<T><<<std::max(gb, 1), 256, 0, st>>>((const T*)D->Qvp, (const T*)D->Qp, D->active, alpha, emis,
                                                        D->N, nrhs, kp, (T*)D->Yp, (T*)D->Qip);
    h->launches_total++;
    launch_permute_out<T>(h, D->Yp, nrhs, kp, false, Td, st);
    if (Qvd) launch_permute_out<T>(h, D->Qvp, nrhs, kp, false, Qvd, st);
    if (Qid) launch_permute_out<T>(h, D->Qip, nrhs, kp, false, Qid, st);
    CK(cudaGetLastError());
    if ((rc = stage_out_copy(Tout, Td, vb, st))) return rc;
    if ((rc = stage_out_copy(Qvis, Qvd, vb, st))) return rc;
    if ((rc = stage_out_copy(Qir, Qid, vb, st))) return rc;
    CK(cudaStreamSynchronize(st));
    if (h->timing) collect_timing(h);
    h->iters1 = it1; h->resid1 = r1; h->iters2 = it2; h->resid2 = r2;
    if (iters > 0 && (!(r1 <= tol) || !(r2 <= tol)))
        return set_error(VF_ENOCONV, "vf_solve_thermal: no convergence within iters");
    return VF_OK;
}

}  // namespace

int device_upload(Handle* h, int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_error(VF_ENODEV, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return set_error(VF_ENODEV, "device index out of range");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return set_error(VF_ENODEV, "libvf is built for sm_100a (B200); device is not sm_100");
    CK(cudaSetDevice(device));
    if (h->dev) device_free(h);
    h->dev = new DeviceHMat();
    h->device = device;
    int rc = h->dtype == VF_F64 ? upload_impl<double>(h, h->dev) : upload_impl<float>(h, h->dev);
    if (rc) { device_free(h); h->device = -1; }
    return rc;
}

void device_free(Handle* h) {
    DeviceHMat* D = h->dev;
    if (!D) return;
    cudaSetDevice(h->device);
    void* ptrs[] = {D->vals, D->idx, D->segs, D->p1_segptr, D->p1_rows, D->p1_scale, D->p2_segptr, D->p2_rows,
                    D->perm, D->active, D->xt[0], D->xt[1], D->Ep, D->Qp, D->Qdp, D->Qvp, D->Yp, D->Qip,
                    D->pv[0], D->pv[1], D->pv[2], D->partial, D->enorm2, D->resid, D->ctl,
                    D->stage[0], D->stage[1], D->stage[2], D->stage[3], D->stage[4], D->stage[5]};
    for (void* p : ptrs) if (p) cudaFree(p);
    if (D->ctl_host) cudaFreeHost(D->ctl_host);
    if (D->resid_host) cudaFreeHost(D->resid_host);
    for (auto& e : D->evpool) if (e) cudaEventDestroy(e);
    delete D;
    h->dev = nullptr;
}

int device_matvec(Handle* h, const void* X, void* Y, int nrhs) {
    return h->dtype == VF_F64 ? matvec_impl<double>(h, X, Y, nrhs) : matvec_impl<float>(h, X, Y, nrhs);
}

int device_solve_radiosity(Handle* h, const void* E, const void* rho, void* B, int nrhs, int iters, double tol,
                           int clamp) {
    return h->dtype == VF_F64 ? radiosity_impl<double>(h, E, rho, B, nrhs, iters, tol, clamp)
                              : radiosity_impl<float>(h, E, rho, B, nrhs, iters, tol, clamp);
}

int device_solve_thermal(Handle* h, const void* Qdir, const void* alb, const void* emi, void* T, void* Qvis,
                         void* Qir, int nrhs, int iters, double tol) {
    return h->dtype == VF_F64 ? thermal_impl<double>(h, Qdir, alb, emi, T, Qvis, Qir, nrhs, iters, tol)
                              : thermal_impl<float>(h, Qdir, alb, emi, T, Qvis, Qir, nrhs, iters, tol);
}

int64_t device_bytes(const Handle* h) { return h->dev ? h->dev->bytes : 0; }
int64_t device_alg_bytes(const Handle* h) { return h->dev ? h->dev->alg_bytes : -1; }
int64_t device_alg_flops(const Handle* h) { return h->dev ? h->dev->alg_flops_per_col : -1; }
int64_t device_active_rows(const Handle* h) { return h->dev ? h->dev->n_p2 : -1; }
void device_phase_info(const Handle* h, int64_t* out7) {
    const DeviceHMat* D = h->dev;
    if (!D) { for (int i = 0; i < 7; ++i) out7[i] = 0; return; }
    out7[0] = D->NT; out7[1] = D->p1_bytes; out7[2] = D->p2_bytes; out7[3] = D->p1_src; out7[4] = D->p2_src;
    out7[5] = D->p1_flops; out7[6] = D->p2_flops;
}

}  // namespace vf
