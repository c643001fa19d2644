// vf_build_gpu.cu -- device evaluator of the exact view-factor matrix for the
// build: Alg. 1 for ALL facet pairs at once,
//   F_ij = [n_i.(x_j-x_i)][n_j.(x_i-x_j)] / (pi |x_i-x_j|^4) V_ij A_j   (eq. FF-def,
//   P:134-136), V_ij = culling and the ray-cast predicate of P:166
//   (reading R-VIS / A18, vf_bvh.h),
// returned as one tree-order CSR from which Alg. 4 slices its blocks.  Not
// on the timed path: it replaces the host ray caster when a device is given,
// because a 131k-facet terrain needs ~4e9 ray casts (hard part 2).
//
// Design: rows are processed in chunks; a warp owns one row i and its 32
// lanes test consecutive columns j (coherent rays from the same origin), each
// lane walking the FP64 BVH with a private stack.  Pass 1 writes the
// visibility bit-matrix of the chunk (one __ballot_sync word per 32
// columns) and per-row counts; the host scans the counts; pass 2 expands the
// bits into sorted column indices and F_ij values.  Every floating-point
// operation of the culling, the triangle test and F_ij is an explicit
// round-to-nearest intrinsic (no FMA contraction) in the order of the host
// code, so the device and host builds take bit-identical decisions and
// values.
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "vf_bvh.h"
#include "vf_internal.h"

namespace vf {
namespace {

#define CKB(call)                                                                         \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return set_error(VF_ECUDA, std::string("build: ") + #call + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DevNode { double lo[3], hi[3]; int32_t left, right, first, count; };
static_assert(sizeof(DevNode) == sizeof(Bvh::NodeB), "node layout");

struct DevBvh {
    const DevNode* nodes;
    const int32_t* order;
    const double* V;
    const int32_t* F;
    int32_t nnodes;
    double margin;
};

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return add(add(mul(a[0], b[0]), mul(a[1], b[1])), mul(a[2], b[2]));
}

// Bvh::hit_tri, operation for operation.
__device__ bool hit_tri(const DevBvh& B, const double* P, const double* D, int32_t t, double tmin, double tmax) {
    const double* a = B.V + 3 * (int64_t)B.F[3 * t];
    const double* b = B.V + 3 * (int64_t)B.F[3 * t + 1];
    const double* c = B.V + 3 * (int64_t)B.F[3 * t + 2];
    const double e1[3] = {sub(b[0], a[0]), sub(b[1], a[1]), sub(b[2], a[2])};
    const double e2[3] = {sub(c[0], a[0]), sub(c[1], a[1]), sub(c[2], a[2])};
    const double p[3] = {sub(mul(D[1], e2[2]), mul(D[2], e2[1])), sub(mul(D[2], e2[0]), mul(D[0], e2[2])),
                         sub(mul(D[0], e2[1]), mul(D[1], e2[0]))};
    const double det = dot3(e1, p);
    if (fabs(det) <= kDetEps) return false;
    const double inv = __ddiv_rn(1.0, det);
    const double s[3] = {sub(P[0], a[0]), sub(P[1], a[1]), sub(P[2], a[2])};
    const double u = mul(dot3(s, p), inv);
    if (u < 0.0 || u > 1.0) return false;
    const double q[3] = {sub(mul(s[1], e1[2]), mul(s[2], e1[1])), sub(mul(s[2], e1[0]), mul(s[0], e1[2])),
                         sub(mul(s[0], e1[1]), mul(s[1], e1[0]))};
    const double v = mul(dot3(D, q), inv);
    if (v < 0.0 || add(u, v) > 1.0) return false;
    const double tt = mul(dot3(e2, q), inv);
    return tt > tmin && tt < tmax;
}

// Bvh::hit_box (conservative: the box is padded by `margin`, the t range widened).
__device__ bool hit_box(const DevNode& nb, const double* P, const double* inv, double tmin, double tmax) {
    for (int d = 0; d < 3; ++d) {
        if (isinf(inv[d])) {
            if (P[d] < nb.lo[d] || P[d] > nb.hi[d]) return false;
            continue;
        }
        double t0 = mul(sub(nb.lo[d], P[d]), inv[d]), t1 = mul(sub(nb.hi[d], P[d]), inv[d]);
        if (t0 > t1) { const double x = t0; t0 = t1; t1 = x; }
        tmin = fmax(tmin, t0);
        tmax = fmin(tmax, t1);
        if (tmin > tmax) return false;
    }
    return true;
}

__device__ bool occluded(const DevBvh& B, const double* P, const double* D, double tmin, double tmax, int64_t skip1,
                         int64_t skip2) {
    if (B.nnodes == 0) return false;
    double inv[3];
    for (int d = 0; d < 3; ++d) inv[d] = __ddiv_rn(1.0, D[d]);
    const double blo = sub(mul(tmin, sub(1.0, 1e-12)), B.margin);
    const double bhi = add(mul(tmax, add(1.0, 1e-12)), B.margin);
    int32_t stack[128];
    int sp = 0;
    stack[sp++] = 0;
    while (sp) {
        const DevNode nb = B.nodes[stack[--sp]];
        if (!hit_box(nb, P, inv, blo, bhi)) continue;
        if (nb.left < 0) {
            for (int32_t k = nb.first; k < nb.first + nb.count; ++k) {
                const int32_t t = B.order[k];
                if (t == skip1 || t == skip2) continue;
                if (hit_tri(B, P, D, t, tmin, tmax)) return true;
            }
        } else {
            stack[sp++] = nb.left;
            stack[sp++] = nb.right;
        }
    }
    return false;
}

// culling + visibility of the pair (i, j), i != j, tree order
__device__ __forceinline__ bool pair_visible(const DevBvh& B, bool cull_only, const double* X, const double* Nn,
                                             const int64_t* tri, int64_t i, int64_t j, double* dd, double* ci,
                                             double* cj) {
    const double* xi = X + 3 * i;
    const double* xj = X + 3 * j;
    const double d[3] = {sub(xj[0], xi[0]), sub(xj[1], xi[1]), sub(xj[2], xi[2])};
    const double a = dot3(Nn + 3 * i, d);
    const double b = -dot3(Nn + 3 * j, d);
    dd[0] = d[0]; dd[1] = d[1]; dd[2] = d[2];
    *ci = a; *cj = b;
    if (!(a > 0.0) || !(b > 0.0)) return false;
    if (cull_only) return true;
    return !occluded(B, xi, d, kTEps, 1.0 - kTEps, tri[i], tri[j]);
}

// pass 1: bit-matrix of the chunk's rows [r0, r0 + R) and per-row counts
__global__ void vis_mask_kernel(DevBvh B, bool cull_only, const double* X, const double* Nn, const int64_t* tri,
                                int64_t N, int64_t r0, int64_t R, int64_t W, uint32_t* mask, int32_t* cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t rr = warp; rr < R; rr += nwarp) {
        const int64_t i = r0 + rr;
        int32_t c = 0;
        for (int64_t w = 0; w < W; ++w) {
            const int64_t j = w * 32 + lane;
            bool vis = false;
            if (j < N && j != i) {
                double d[3], ci, cj;
                vis = pair_visible(B, cull_only, X, Nn, tri, i, j, d, &ci, &cj);
            }
            const uint32_t word = __ballot_sync(0xffffffffu, vis);
            if (lane == 0) mask[rr * W + w] = word;
            c += __popc(word);
        }
        if (lane == 0) cnt[rr] = c;
    }
}

// pass 2: bits -> sorted columns and F_ij (eq. FF-def, the host's operation order)
__global__ void vis_fill_kernel(const double* X, const double* Nn, const double* A, int64_t N, int64_t r0, int64_t R,
                                int64_t W, const uint32_t* mask, const int64_t* off, int32_t* cols, double* vals) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double kPi = 3.14159265358979323846;
    for (int64_t rr = warp; rr < R; rr += nwarp) {
        const int64_t i = r0 + rr;
        int64_t base = off[rr];
        const double* xi = X + 3 * i;
        const double* ni = Nn + 3 * i;
        for (int64_t w = 0; w < W; ++w) {
            const uint32_t word = mask[rr * W + w];
            if (!word) continue;
            if ((word >> lane) & 1u) {
                const int64_t j = w * 32 + lane;
                const double* xj = X + 3 * j;
                const double d[3] = {sub(xj[0], xi[0]), sub(xj[1], xi[1]), sub(xj[2], xi[2])};
                const double ci = dot3(ni, d);
                const double cj = -dot3(Nn + 3 * j, d);
                const double r2 = add(add(mul(d[0], d[0]), mul(d[1], d[1])), mul(d[2], d[2]));
                const int64_t pos = base + __popc(word & ((1u << lane) - 1u));
                cols[pos] = (int32_t)j;
                vals[pos] = mul(__ddiv_rn(mul(ci, cj), mul(mul(kPi, r2), r2)), A[j]);
            }
            base += __popc(word);
        }
    }
}

struct DevBuf {
    std::vector<void*> p;
    ~DevBuf() { for (void* q : p) cudaFree(q); }
    template <typename T>
    int alloc(T** out, size_t n) {
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
        if (e != cudaSuccess) return set_error(VF_ENOMEM, std::string("build: cudaMalloc: ") + cudaGetErrorString(e));
        p.push_back(q);
        *out = static_cast<T*>(q);
        return VF_OK;
    }
};

}  // namespace

// The exact F in tree order as CSR (rows = tree rows, sorted tree columns).
// x, n, A, tri: tree-order facet data and the occluder triangle of each facet
// (excluded from its own rays; -1 none).  bvh == nullptr: culling only.
int gpu_exact_csr(int device, int64_t N, const double* x, const double* n, const double* A, const int64_t* tri,
                  const Bvh* bvh, std::vector<int64_t>& rowptr, std::vector<int32_t>& cols,
                  std::vector<double>& vals) {
    CKB(cudaSetDevice(device));
    DevBuf mem;
    double *dX, *dN, *dA;
    int64_t* dT;
    int rc;
    if ((rc = mem.alloc(&dX, 3 * N)) || (rc = mem.alloc(&dN, 3 * N)) || (rc = mem.alloc(&dA, N)) ||
        (rc = mem.alloc(&dT, N)))
        return rc;
    CKB(cudaMemcpy(dX, x, 3 * N * 8, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(dN, n, 3 * N * 8, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(dA, A, N * 8, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(dT, tri, N * 8, cudaMemcpyHostToDevice));
    DevBvh B{};
    const bool cull_only = bvh == nullptr || bvh->nodes.empty();
    if (!cull_only) {
        DevNode* nodes;
        int32_t *order, *F;
        double* V;
        const size_t nt = bvh->order.size();
        size_t nv = 0;
        for (size_t t = 0; t < 3 * nt; ++t) nv = std::max<size_t>(nv, (size_t)bvh->F[t] + 1);
        if ((rc = mem.alloc(&nodes, bvh->nodes.size())) || (rc = mem.alloc(&order, nt)) ||
            (rc = mem.alloc(&F, 3 * nt)) || (rc = mem.alloc(&V, 3 * nv)))
            return rc;
        CKB(cudaMemcpy(nodes, bvh->nodes.data(), bvh->nodes.size() * sizeof(DevNode), cudaMemcpyHostToDevice));
        CKB(cudaMemcpy(order, bvh->order.data(), nt * 4, cudaMemcpyHostToDevice));
        CKB(cudaMemcpy(F, bvh->F, 3 * nt * 4, cudaMemcpyHostToDevice));
        CKB(cudaMemcpy(V, bvh->V, 3 * nv * 8, cudaMemcpyHostToDevice));
        B = DevBvh{nodes, order, V, F, (int32_t)bvh->nodes.size(), bvh->margin};
    }
    const int64_t W = (N + 31) / 32;
    const int64_t R = std::max<int64_t>(1, std::min<int64_t>(N, (int64_t)(1ll << 30) / (W * 4)));   // <= 1 GiB of bits
    uint32_t* mask;
    int32_t* cnt;
    int64_t* off;
    if ((rc = mem.alloc(&mask, (size_t)R * W)) || (rc = mem.alloc(&cnt, R)) || (rc = mem.alloc(&off, R))) return rc;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    rowptr.assign(N + 1, 0);
    cols.clear();
    vals.clear();
    std::vector<int32_t> hc(R);
    std::vector<int64_t> ho(R);
    int32_t* dcols = nullptr;
    double* dvals = nullptr;
    size_t cap = 0;
    DevBuf vbuf;
    for (int64_t r0 = 0; r0 < N; r0 += R) {
        const int64_t Rc = std::min<int64_t>(R, N - r0);
        const int grid = (int)std::min<int64_t>((Rc + 7) / 8, (int64_t)nsm * 16);
        vis_mask_kernel<<<grid, 256>>>(B, cull_only, dX, dN, dT, N, r0, Rc, W, mask, cnt);
        CKB(cudaGetLastError());
        CKB(cudaMemcpy(hc.data(), cnt, Rc * 4, cudaMemcpyDeviceToHost));
        int64_t s = 0;
        for (int64_t r = 0; r < Rc; ++r) { ho[r] = s; s += hc[r]; rowptr[r0 + r + 1] = rowptr[r0 + r] + hc[r]; }
        if ((size_t)s > cap) {
            for (void* q : vbuf.p) cudaFree(q);
            vbuf.p.clear();
            cap = (size_t)s;
            if ((rc = vbuf.alloc(&dcols, cap)) || (rc = vbuf.alloc(&dvals, cap))) return rc;
        }
        CKB(cudaMemcpy(off, ho.data(), Rc * 8, cudaMemcpyHostToDevice));
        if (s > 0) {
            vis_fill_kernel<<<grid, 256>>>(dX, dN, dA, N, r0, Rc, W, mask, off, dcols, dvals);
            CKB(cudaGetLastError());
            const size_t old = cols.size();
            cols.resize(old + s);
            vals.resize(old + s);
            CKB(cudaMemcpy(cols.data() + old, dcols, s * 4, cudaMemcpyDeviceToHost));
            CKB(cudaMemcpy(vals.data() + old, dvals, s * 8, cudaMemcpyDeviceToHost));
        }
    }
    CKB(cudaDeviceSynchronize());
    return VF_OK;
}

}  // namespace vf
