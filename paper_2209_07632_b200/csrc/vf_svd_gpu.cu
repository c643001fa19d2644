// vf_svd_gpu.cu -- the randomized k-term truncated SVD of Alg. 3
// for LARGE blocks on the device, with library primitives (cuSPARSE SpMM,
// cuSOLVER Householder QR, cuBLAS DGEMM).  Build-time only, never on the
// timed path (the rank search is what makes a 131k-facet
// build O(hours) on the host).  Same algorithm as randomized_svd() in
// vf_svd.cpp: Y = A Omega, two power iterations with re-orthonormalisation,
// Q = orth(Y), Z = A^T Q = Qz R, R = Ur S W^T (small one-sided Jacobi SVD on
// the host), U = Q W, V = Qz Ur.
//
// One device context (stream, library handles, buffers) per build thread, so
// the rank searches of concurrently processed blocks overlap on the GPU; the
// block's CSR is uploaded once and reused across the k-doubling steps.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cusparse.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "vf_internal.h"

namespace vf {
namespace {

struct Ctx {
    int device = -1;
    bool ok = false;
    cudaStream_t st = nullptr;
    cublasHandle_t blas = nullptr;
    cusolverDnHandle_t sol = nullptr;
    cusparseHandle_t sp = nullptr;
    // cached block
    const void* key0 = nullptr;
    const void* key1 = nullptr;
    int64_t km = -1, kn = -1, knnz = -1;
    int32_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* vv = nullptr;
    cusparseSpMatDescr_t A = nullptr;
    // work buffers (grown)
    double *Om = nullptr, *Y = nullptr, *Z = nullptr, *tau = nullptr, *work = nullptr, *W = nullptr, *Ur = nullptr,
           *U = nullptr, *V = nullptr;
    void* spbuf = nullptr;
    size_t cap_m = 0, cap_n = 0, cap_l = 0, cap_work = 0, cap_sp = 0;
    int* info = nullptr;
};

thread_local Ctx g_ctx;

bool cu(cudaError_t e) { return e == cudaSuccess; }

template <typename T>
bool grow(T** p, size_t& cap, size_t n) {
    if (n <= cap && *p) return true;
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (!cu(cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T)))) { cap = 0; return false; }
    cap = n;
    return true;
}

bool init(int device) {
    Ctx& c = g_ctx;
    if (c.ok && c.device == device) return true;
    if (c.device >= 0) return false;              // one device per thread
    c.device = device;
    if (!cu(cudaSetDevice(device)) || !cu(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking))) return false;
    if (cublasCreate(&c.blas) != CUBLAS_STATUS_SUCCESS || cusolverDnCreate(&c.sol) != CUSOLVER_STATUS_SUCCESS ||
        cusparseCreate(&c.sp) != CUSPARSE_STATUS_SUCCESS)
        return false;
    cublasSetStream(c.blas, c.st);
    cusolverDnSetStream(c.sol, c.st);
    cusparseSetStream(c.sp, c.st);
    if (!cu(cudaMalloc((void**)&c.info, sizeof(int)))) return false;
    c.ok = true;
    return true;
}

bool upload_block(int64_t m, int64_t n, const int64_t* rowptr, const int32_t* cols, const double* vals,
                  const double* dense) {
    Ctx& c = g_ctx;
    const void* k0 = dense ? (const void*)dense : (const void*)rowptr;
    const void* k1 = dense ? nullptr : (const void*)vals;
    const int64_t nnz = dense ? -1 : rowptr[m];
    if (c.A && c.key0 == k0 && c.key1 == k1 && c.km == m && c.kn == n && c.knnz == nnz) return true;
    if (c.A) { cusparseDestroySpMat(c.A); c.A = nullptr; }
    if (c.rp) cudaFree(c.rp);
    if (c.ci) cudaFree(c.ci);
    if (c.vv) cudaFree(c.vv);
    c.rp = nullptr; c.ci = nullptr; c.vv = nullptr;
    std::vector<int32_t> hrp(m + 1), hci;
    std::vector<double> hvv;
    if (dense) {
        for (int64_t i = 0; i < m; ++i) {
            for (int64_t j = 0; j < n; ++j)
                if (dense[i * n + j] != 0.0) { hci.push_back((int32_t)j); hvv.push_back(dense[i * n + j]); }
            hrp[i + 1] = (int32_t)hci.size();
        }
    } else {
        for (int64_t i = 0; i <= m; ++i) hrp[i] = (int32_t)rowptr[i];
    }
    const int64_t z = dense ? (int64_t)hci.size() : rowptr[m];
    if (!cu(cudaMalloc((void**)&c.rp, (m + 1) * 4)) || !cu(cudaMalloc((void**)&c.ci, std::max<int64_t>(z, 1) * 4)) ||
        !cu(cudaMalloc((void**)&c.vv, std::max<int64_t>(z, 1) * 8)))
        return false;
    cudaMemcpyAsync(c.rp, hrp.data(), (m + 1) * 4, cudaMemcpyHostToDevice, c.st);
    cudaMemcpyAsync(c.ci, dense ? hci.data() : cols, z * 4, cudaMemcpyHostToDevice, c.st);
    cudaMemcpyAsync(c.vv, dense ? hvv.data() : vals, z * 8, cudaMemcpyHostToDevice, c.st);
    if (!cu(cudaStreamSynchronize(c.st))) return false;
    if (cusparseCreateCsr(&c.A, m, n, z, c.rp, c.ci, c.vv, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                          CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F) != CUSPARSE_STATUS_SUCCESS)
        return false;
    c.key0 = k0; c.key1 = k1; c.km = m; c.kn = n; c.knnz = nnz;
    return true;
}

// C (rows_out x l, col-major) = op(A) B (col-major)
bool spmm(bool trans, const double* B, int64_t rows_in, int64_t rows_out, int64_t l, double* C) {
    Ctx& c = g_ctx;
    cusparseDnMatDescr_t mb, mc;
    cusparseCreateDnMat(&mb, rows_in, l, rows_in, (void*)B, CUDA_R_64F, CUSPARSE_ORDER_COL);
    cusparseCreateDnMat(&mc, rows_out, l, rows_out, C, CUDA_R_64F, CUSPARSE_ORDER_COL);
    const double one = 1.0, zero = 0.0;
    const cusparseOperation_t op = trans ? CUSPARSE_OPERATION_TRANSPOSE : CUSPARSE_OPERATION_NON_TRANSPOSE;
    size_t bs = 0;
    bool ok = cusparseSpMM_bufferSize(c.sp, op, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, c.A, mb, &zero, mc, CUDA_R_64F,
                                      CUSPARSE_SPMM_ALG_DEFAULT, &bs) == CUSPARSE_STATUS_SUCCESS;
    ok = ok && grow((char**)&c.spbuf, c.cap_sp, bs);
    ok = ok && cusparseSpMM(c.sp, op, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, c.A, mb, &zero, mc, CUDA_R_64F,
                            CUSPARSE_SPMM_ALG_DEFAULT, c.spbuf) == CUSPARSE_STATUS_SUCCESS;
    cusparseDestroyDnMat(mb);
    cusparseDestroyDnMat(mc);
    return ok;
}

// Householder QR of the col-major rows x l matrix M in place -> Q; if Rout,
// the l x l upper triangle R (col-major) is copied out first.
bool qr(double* M, int64_t rows, int64_t l, double* Rout_host) {
    Ctx& c = g_ctx;
    int lw1 = 0, lw2 = 0;
    if (cusolverDnDgeqrf_bufferSize(c.sol, (int)rows, (int)l, M, (int)rows, &lw1) != CUSOLVER_STATUS_SUCCESS) return false;
    if (cusolverDnDorgqr_bufferSize(c.sol, (int)rows, (int)l, (int)l, M, (int)rows, c.tau, &lw2) !=
        CUSOLVER_STATUS_SUCCESS)
        return false;
    if (!grow(&c.work, c.cap_work, (size_t)std::max(lw1, lw2))) return false;
    if (cusolverDnDgeqrf(c.sol, (int)rows, (int)l, M, (int)rows, c.tau, c.work, std::max(lw1, lw2), c.info) !=
        CUSOLVER_STATUS_SUCCESS)
        return false;
    if (Rout_host) {
        std::vector<double> tmp(l * l);
        if (!cu(cudaMemcpy2DAsync(tmp.data(), l * 8, M, rows * 8, l * 8, l, cudaMemcpyDeviceToHost, c.st)) ||
            !cu(cudaStreamSynchronize(c.st)))
            return false;
        for (int64_t j = 0; j < l; ++j)
            for (int64_t i = 0; i < l; ++i) Rout_host[j * l + i] = i <= j ? tmp[j * l + i] : 0.0;
    }
    return cusolverDnDorgqr(c.sol, (int)rows, (int)l, (int)l, M, (int)rows, c.tau, c.work, std::max(lw1, lw2),
                            c.info) == CUSOLVER_STATUS_SUCCESS;
}

}  // namespace

int g_svd_device = -1;      // set by the build when a device is available

bool gpu_randomized_svd(int64_t m, int64_t n, const int64_t* rowptr, const int32_t* cols, const double* vals,
                        const double* dense, const double* Om_rm, int64_t l, std::vector<double>& U_rm,
                        std::vector<double>& S, std::vector<double>& V_rm) {
    if (g_svd_device < 0) return false;
    Ctx& c = g_ctx;
    if (!init(g_svd_device)) return false;
    cudaSetDevice(c.device);
    if (!upload_block(m, n, rowptr, cols, vals, dense)) return false;
    const size_t mx = (size_t)std::max(m, n);
    if (!grow(&c.Om, c.cap_n, (size_t)n * l) || !grow(&c.Y, c.cap_m, mx * l) || !grow(&c.Z, c.cap_l, mx * l))
        return false;
    static thread_local size_t cap_tau = 0, cap_w = 0, cap_ur = 0, cap_u = 0, cap_v = 0;
    if (!grow(&c.tau, cap_tau, (size_t)l) || !grow(&c.W, cap_w, (size_t)l * l) || !grow(&c.Ur, cap_ur, (size_t)l * l) ||
        !grow(&c.U, cap_u, (size_t)m * l) || !grow(&c.V, cap_v, (size_t)n * l))
        return false;
    const double one = 1.0, zero = 0.0;
    // Omega: row-major n x l on the host = col-major l x n; transpose on the device
    if (!cu(cudaMemcpyAsync(c.Z, Om_rm, (size_t)n * l * 8, cudaMemcpyHostToDevice, c.st)) ||
        cublasDgeam(c.blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)n, (int)l, &one, c.Z, (int)l, &zero, c.Z, (int)n, c.Om,
                    (int)n) != CUBLAS_STATUS_SUCCESS)
        return false;
    if (!spmm(false, c.Om, n, m, l, c.Y)) return false;                 // Y = A Omega
    for (int it = 0; it < 2; ++it) {                                     // power iterations
        if (!qr(c.Y, m, l, nullptr) || !spmm(true, c.Y, m, n, l, c.Z) || !qr(c.Z, n, l, nullptr) ||
            !spmm(false, c.Z, n, m, l, c.Y))
            return false;
    }
    if (!qr(c.Y, m, l, nullptr) || !spmm(true, c.Y, m, n, l, c.Z)) return false;   // Q; Z = A^T Q
    std::vector<double> R(l * l);
    if (!qr(c.Z, n, l, R.data())) return false;                          // Z = Qz R
    std::vector<double> sig;
    cublasOperation_t wop = CUBLAS_OP_N;
    if (l <= 64) {                                                       // small: host one-sided Jacobi
        std::vector<double> W;
        small_jacobi_svd(R, l, sig, W);                                  // R = Ur S W^T (R <- Ur)
        if (!cu(cudaMemcpyAsync(c.W, W.data(), l * l * 8, cudaMemcpyHostToDevice, c.st)) ||
            !cu(cudaMemcpyAsync(c.Ur, R.data(), l * l * 8, cudaMemcpyHostToDevice, c.st)))
            return false;
    } else {                                                             // cuSOLVER: R = Ur S VT, W = VT^T
        static thread_local size_t cap_s = 0, cap_rw = 0, cap_gw = 0;
        static thread_local double *dS = nullptr, *dRW = nullptr, *dGW = nullptr;
        int lw = 0;
        if (cusolverDnDgesvd_bufferSize(c.sol, (int)l, (int)l, &lw) != CUSOLVER_STATUS_SUCCESS ||
            !grow(&dS, cap_s, (size_t)l) || !grow(&dRW, cap_rw, (size_t)l) || !grow(&dGW, cap_gw, (size_t)lw))
            return false;
        if (!cu(cudaMemcpyAsync(c.U, R.data(), l * l * 8, cudaMemcpyHostToDevice, c.st)) ||
            cusolverDnDgesvd(c.sol, 'A', 'A', (int)l, (int)l, c.U, (int)l, dS, c.Ur, (int)l, c.W, (int)l, dGW, lw, dRW,
                             c.info) != CUSOLVER_STATUS_SUCCESS)
            return false;
        sig.resize(l);
        if (!cu(cudaMemcpyAsync(sig.data(), dS, l * 8, cudaMemcpyDeviceToHost, c.st))) return false;
        wop = CUBLAS_OP_T;
    }
    if (cublasDgemm(c.blas, CUBLAS_OP_N, wop, (int)m, (int)l, (int)l, &one, c.Y, (int)m, c.W, (int)l, &zero,
                    c.U, (int)m) != CUBLAS_STATUS_SUCCESS ||
        cublasDgemm(c.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n, (int)l, (int)l, &one, c.Z, (int)n, c.Ur, (int)l, &zero,
                    c.V, (int)n) != CUBLAS_STATUS_SUCCESS)
        return false;
    // row-major results = col-major l x m / l x n: transpose on the device (into Y, Om)
    if (cublasDgeam(c.blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)l, (int)m, &one, c.U, (int)m, &zero, c.U, (int)l, c.Y,
                    (int)l) != CUBLAS_STATUS_SUCCESS ||
        cublasDgeam(c.blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)l, (int)n, &one, c.V, (int)n, &zero, c.V, (int)l, c.Om,
                    (int)l) != CUBLAS_STATUS_SUCCESS)
        return false;
    U_rm.resize(m * l);
    V_rm.resize(n * l);
    if (!cu(cudaMemcpyAsync(U_rm.data(), c.Y, U_rm.size() * 8, cudaMemcpyDeviceToHost, c.st)) ||
        !cu(cudaMemcpyAsync(V_rm.data(), c.Om, V_rm.size() * 8, cudaMemcpyDeviceToHost, c.st)) ||
        !cu(cudaStreamSynchronize(c.st)))
        return false;
    S = sig;
    return true;
}

}  // namespace vf
