// Dev probe: one tcgen05.mma.kind::tf32 tile (M = 128, N = 16, K = 16 as two
// K = 8 steps) with both operands MN-major, SWIZZLE_NONE core matrices
// (8 K-rows x 16 B), accumulator in TMEM, read back with tcgen05.ld.
// Checks the descriptor / layout conventions used by bt_tc_kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tc_probe tools/tc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 16, K = 16;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// MN-major SWIZZLE_NONE: element (mn, k) at (mn/4)*SBO + (k/8)*LBO + (k%8)*16 + (mn%4)*4 bytes
__device__ __forceinline__ int off_mn(int mn, int k, int sbo, int lbo) {
    return (mn >> 2) * sbo + (k >> 3) * lbo + (k & 7) * 16 + (mn & 3) * 4;
}
// K-major SWIZZLE_NONE: element (mn, k) at (mn/8)*SBO + (k/4)*LBO + (mn%8)*16 + (k%4)*4 bytes
__device__ __forceinline__ int off_k(int mn, int k, int sbo, int lbo) {
    return (mn >> 3) * sbo + (k >> 2) * lbo + (mn & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ uint64_t sdesc(unsigned addr, unsigned lbo, unsigned sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;                 // version (sm_100)
    return d;                               // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__global__ void probe(const float* A /*M x K row-major*/, const float* B /*K x N row-major*/, float* D /*M x N*/,
                      int mode) {
    __shared__ __align__(1024) unsigned char sa[M * K * 4];
    __shared__ __align__(1024) unsigned char sb[N * K * 4];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const bool kmaj = mode >= 2;
    // MN-major: SBO = (K/8)*128 (all K rows of a 4-wide MN group), LBO = 128 (next 8 K rows)
    // K-major:  SBO = 128 (next 8 MN rows), LBO = (MN/8)*128 (next 4 K elements)
    const int sboA = kmaj ? 128 : (K / 8) * 128, lboA = kmaj ? (M / 8) * 128 : 128;
    const int sboB = kmaj ? 128 : (K / 8) * 128, lboB = kmaj ? (N / 8) * 128 : 128;
    for (int i = t; i < M * K; i += blockDim.x) {
        const int m = i / K, k = i % K;
        *reinterpret_cast<float*>(sa + (kmaj ? off_k(m, k, sboA, lboA) : off_mn(m, k, sboA, lboA))) = A[m * K + k];
    }
    for (int i = t; i < N * K; i += blockDim.x) {
        const int n = i / K, k = i % K;
        *reinterpret_cast<float*>(sb + (kmaj ? off_k(n, k, sboB, lboB) : off_mn(n, k, sboB, lboB))) = B[k * N + n];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tm = tbase;
    // idesc: c_format F32 (bit 4), a/b format TF32 (2 at bits 7 and 10), a/b MN-major (bits 15, 16),
    // N >> 3 at bit 17, M >> 4 at bit 24
    const uint32_t mj = kmaj ? 0u : 1u;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (mj << 15) | (mj << 16) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);
    if (mode == 4 && warp < 4) {          // tcgen05.st / ld round trip
        uint32_t v = 1000u + (unsigned)(warp * 32 + lane);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(tm + ((uint32_t)(warp * 32) << 16)), "r"(v));
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    if (t == 0 && mode != 4) {
        for (int ks = 0; ks < K / 8; ++ks) {
            // K step of 8: MN-major -> next 8-row K group (+LBO); K-major -> 2 K chunks of 4 (+2 LBO)
            const unsigned ka = kmaj ? 2 * ks * lboA : ks * lboA, kb = kmaj ? 2 * ks * lboB : ks * lboB;
            const bool sw = (mode & 1) != 0;
            const uint64_t da = !sw ? sdesc(smem_u32(sa) + ka, lboA, sboA) : sdesc(smem_u32(sa) + ka, sboA, lboA);
            const uint64_t db = !sw ? sdesc(smem_u32(sb) + kb, lboB, sboB) : sdesc(smem_u32(sb) + kb, sboB, lboB);
            const uint32_t acc = ks > 0 ? 1u : 0u;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
    }
    if (t == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                     : "memory");
    // wait for the MMAs
    {
        unsigned ok = 0;
        while (!ok) {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp < 4) {
        uint32_t r[16];
        const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        const int m = warp * 32 + lane;
        for (int n = 0; n < N; ++n) D[m * N + n] = __uint_as_float(r[n]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tm));
}

int main() {
    std::vector<float> A(M * K), B(K * N), D(M * N, -1.f), R(M * N, 0.f);
    for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7 + 3) % 17 - 8) / 8.0f;
    for (int i = 0; i < K * N; ++i) B[i] = (float)((i * 5 + 1) % 13 - 6) / 4.0f;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[k * N + n];
            R[m * N + n] = (float)s;
        }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    int anybad = 0;
    for (int mode = 0; mode < 5; ++mode) {
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 256>>>(dA, dB, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d kernel: %s\n", mode, cudaGetErrorString(e));
        if (e != cudaSuccess) return 2;
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double mx = 0;
        int bad = 0;
        for (int i = 0; i < M * N; ++i) { mx = fmax(mx, fabs(D[i] - R[i])); bad += fabs(D[i] - R[i]) > 1e-4; }
        printf("mode %d: max abs err %g, bad %d of %d; D[0..3] %g %g %g %g ref %g %g %g %g\n", mode, mx, bad, M * N,
               D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
        if (mode == 4) printf("st/ld round trip: D[0] %g (expect bits of 1000 -> %g)\n", D[0], __builtin_bit_cast(float, 1000u));
        anybad |= mode == 0 && bad;
    }
    return anybad;
}
