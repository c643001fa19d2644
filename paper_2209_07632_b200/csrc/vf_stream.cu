// vf_stream.cu -- the nrhs = 1 compressed apply Y = F-hat X as a bulk-copy
// chunk stream (SURVEY §8(a) a2 + a3; Alg. 5, applied as
// "U(Sigma(V^T x))").  DESIGN.md §7 "stream_k1_kernel".
//
// One persistent cooperative launch, one CTA of NW warps per SM.  Work items
// (vf_stream.h) come from two global queues in longest-first order: phase-1
// items (T_t = S_t sum_j V[j,t] x_{J_b[j]} for up to 16 rank terms t of one
// SVD block over a part of its V rows) and phase-2 items (one output row:
// y_i = sum of its dense-leaf row, U_b rows applied to T, and merged CSR row).
// Each warp owns a ring of NS shared-memory slots: lane 0 copies the chunks of
// its items into the ring with cp.async.bulk (complete_tx on one mbarrier per
// slot, L2 evict-first policy: F-hat is read once), the warp consumes a slot
// when its mbarrier phase completes and lane 0 refills it.  The x gathers are
// the only global loads of the consumers.  Between the phases a warp-granular
// grid barrier (per-CTA aggregated arrival counter): a warp arrives when its
// last phase-1 chunk is consumed and waits only before consuming its first
// phase-2 chunk -- its producer keeps prefetching phase-2 chunks meanwhile.
// Every item is summed by one warp in the fixed lane order of its chunks and
// multi-part phase-1 groups are combined in part order: bitwise reproducible.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "vf_internal.h"
#include "vf_stream.h"

#ifndef VF_SK1_U
#define VF_SK1_U 2       // phase-2 quads (4 terms) in flight per lane
#endif

namespace vf {
namespace stream {

namespace {

__host__ __device__ constexpr int pad16(int b) { return (b + 15) & ~15; }

// ---- PTX wrappers: mbarrier + bulk copy (sm_90+; UBLKCP / SYNCS in SASS)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    unsigned long long spins = 0;
    while (!mbar_try_wait(bar, parity))
        if (++spins > (1ull << 22)) __trap();          // a lost copy: fail loudly instead of hanging
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// 4 consecutive chunk values from shared memory (16-B aligned: quads start at 4q)
template <typename T> struct Quad;
template <> struct Quad<double> {
    static __device__ __forceinline__ void ld(const double* p, double* v) {
        const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
};
template <> struct Quad<float> {
    static __device__ __forceinline__ void ld(const float* p, float* v) {
        const float4 a = *reinterpret_cast<const float4*>(p);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
};

template <typename T>
struct SArgs {
    const unsigned char* bytes;
    const int64_t* coff;
    const int32_t* ic0;
    const P1Item* p1;
    int32_t n1, n2;
    T* XT;               // [x (N rows, read-only) | T rows (N + t, written in phase 1)]
    T* Y;                // tree-order y
    double* pscr;        // [scratch rows][16] part sums of multi-part phase-1 groups
    int32_t* pcnt;       // [group] parts finished (reset by the finisher)
    int32_t* ctr;        // [0] phase-1 queue, [1] phase-2 queue, [2] CTAs past phase 1
};

template <typename T, int NW, int NS>
__global__ void __launch_bounds__(NW * 32, 1) stream_k1_kernel(SArgs<T> a) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ int cta_arrived;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr unsigned FULL = 0xffffffffu;
    unsigned char* ring = sm + (size_t)warp * NS * kSlot;
    // per warp: piece records [32] (int4) + start bitmap [kMaxTerms / 32] words
    int4* prec = reinterpret_cast<int4*>(sm + (size_t)NW * NS * kSlot) + warp * kMaxPieces;
    unsigned* pw = reinterpret_cast<unsigned*>(sm + (size_t)NW * NS * kSlot + (size_t)NW * kMaxPieces * 16) +
                   warp * (kMaxTerms / 32);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)NW * NS * kSlot + (size_t)NW * kMaxPieces * 16 +
                                                (size_t)NW * (kMaxTerms / 32) * 4) + warp * NS;
    if (threadIdx.x == 0) cta_arrived = 0;
    if (lane == 0)
        for (int s = 0; s < NS; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    const T* __restrict__ XT = a.XT;

    // ---- producer (lane 0): item cursor over the two queues
    const uint64_t pol = evict_first_policy();
    int pphase = 1;
    int32_t pc = 0, pce = 0;
    auto issue = [&](int slot) -> int {            // lane 0 only; 1 if a chunk was issued
        while (pc == pce) {
            if (pphase == 1) {
                const int t = atomicAdd(a.ctr + 0, 1);
                if (t < a.n1) { pc = a.ic0[t]; pce = a.ic0[t + 1]; break; }
                pphase = 2;
            } else {
                const int t = atomicAdd(a.ctr + 1, 1);
                if (t < a.n2) { pc = a.ic0[a.n1 + t]; pce = a.ic0[a.n1 + t + 1]; break; }
                return 0;
            }
        }
        const int64_t off = a.coff[pc];
        const unsigned sz = (unsigned)(a.coff[pc + 1] - off);
        mbar_expect_tx(bar + slot, sz);
        bulk_g2s(ring + (size_t)slot * kSlot, a.bytes + off, sz, bar + slot, pol);
        ++pc;
        return 1;
    };
    int issued = 0;
    for (int s = 0; s < NS; ++s) {
        int ok = lane == 0 ? issue(s) : 0;
        ok = __shfl_sync(FULL, ok, 0);
        if (!ok) break;
        ++issued;
    }

    // warp-granular grid barrier between the phases
    bool arrived = false, passed = false;
    auto arrive = [&]() {
        __syncwarp();
        if (lane == 0) {
            __threadfence();                                     // this warp's T / scratch stores
            if (atomicAdd(&cta_arrived, 1) == NW - 1) atomicAdd(a.ctr + 2, 1);
        }
        arrived = true;
    };

    T acc = T(0);                 // phase 2: this lane's part of the current row
    T acc1[16];                   // phase 1: this lane's part of the group's 16 T rows
#pragma unroll
    for (int t = 0; t < 16; ++t) acc1[t] = T(0);

    for (int consumed = 0; consumed < issued; ++consumed) {
        const int slot = consumed % NS;
        mbar_wait(bar + slot, (unsigned)(consumed / NS) & 1u);
        const unsigned char* ch = ring + (size_t)slot * kSlot;
        const Hdr h = *reinterpret_cast<const Hdr*>(ch);
        if (h.flags & 2) {
            // ---- phase 1: T_t += sum_j V[j, t] x_j over this chunk's V rows
            const int G = h.n, nj = h.nterm;
            const unsigned char* p = ch + sizeof(Hdr);
            const int32_t* rows = nullptr;
            if (h.src < 0) {
                rows = reinterpret_cast<const int32_t*>(p);
                p += pad16(4 * nj);
            }
            const T* V = reinterpret_cast<const T*>(p);
            for (int jj = lane; jj < nj; jj += 32) {
                const T x = XT[rows ? rows[jj] : h.src + jj];
#pragma unroll
                for (int t = 0; t < 16; ++t)
                    if (t < G) acc1[t] = fma(V[t * nj + jj], x, acc1[t]);
            }
            if (h.flags & 1) {                                   // last chunk of the item
                const P1Item it = a.p1[h.item];
                double mine = 0.0;
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    T s = acc1[t];
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
                    if (lane == t) mine = (double)s;
                    acc1[t] = T(0);
                }
                bool finish = it.np == 1;
                if (!finish) {
                    // part sums meet in scratch; the last part to finish adds them in part order
                    if (lane < G) a.pscr[((int64_t)it.sbase + it.pidx) * 16 + lane] = mine;
                    __threadfence();
                    __syncwarp();
                    int last = 0;
                    if (lane == 0) {
                        last = atomicAdd(a.pcnt + it.group, 1) + 1 == it.np;
                        if (last) atomicExch(a.pcnt + it.group, 0);     // ready for the next launch
                    }
                    finish = __shfl_sync(FULL, last, 0) != 0;
                    if (finish) {
                        __threadfence();
                        mine = 0.0;
                        if (lane < G)
                            for (int q = 0; q < it.np; ++q) mine += __ldcg(a.pscr + ((int64_t)it.sbase + q) * 16 + lane);
                    }
                }
                if (finish && lane < G) a.XT[it.t0 + lane] = (T)mine;      // S_t is folded into V
            }
        } else {
            // ---- phase 2
            if (!passed) {
                if (!arrived) arrive();
                if (lane == 0) {
                    unsigned long long spins = 0;
                    while (ld_acquire(a.ctr + 2) < (int)gridDim.x) {
                        __nanosleep(100);
                        if (++spins > (1ull << 25)) __trap();
                    }
                }
                __syncwarp();
                passed = true;
            }
            const int np = h.n, nt = h.nterm;
            const Piece* pcs = reinterpret_cast<const Piece*>(ch + sizeof(Hdr));
            const T* vals = reinterpret_cast<const T*>(ch + sizeof(Hdr) + pad16(8 * np));
            const uint16_t* ix =
                reinterpret_cast<const uint16_t*>(reinterpret_cast<const unsigned char*>(vals) + pad16((int)sizeof(T) * nt));
            Piece my{0, 0, 0, 0};
            if (lane < np) my = pcs[lane];
            const int len = my.len, clen = my.kind ? len : 0;
            int incl = len, cincl = clen;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int v = __shfl_up_sync(FULL, incl, off), cv = __shfl_up_sync(FULL, cincl, off);
                if (lane >= off) { incl += v; cincl += cv; }
            }
            const int excl = incl - len, cexcl = cincl - clen;
            // piece lookup without a search: a bitmap of piece starts over the
            // chunk's terms (word w covers terms 32w .. 32w+31); the piece of term
            // t = 32w + l is (pieces starting before wave w) + popc(word_w up to
            // bit l) - 1.  Piece records (src, first term, first u16 slot, kind) in smem.
            constexpr int NWORD = kMaxTerms / 32;
            if (lane < NWORD) pw[lane] = 0u;
            __syncwarp();
            if (lane < np) {
                atomicOr(pw + (excl >> 5), 1u << (excl & 31));
                prec[lane] = make_int4(my.src, excl, cexcl, (int)my.kind);
            }
            __syncwarp();
            const unsigned wl = lane < NWORD ? pw[lane] : 0u;
            int wcnt = __popc(wl), wincl = wcnt;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int v = __shfl_up_sync(FULL, wincl, off);
                if (lane >= off) wincl += v;
            }
            const int wexcl = wincl - wcnt;             // pieces starting before wave `lane`
            // lane l takes quads q = 32 i + l of 4 consecutive terms (a warp covers 128
            // consecutive terms per round: neighbouring lanes gather neighbouring
            // columns); one bitmap lookup per quad, a piece boundary inside the quad
            // advances to the next record
            const int nq = (nt + 3) >> 2;
            constexpr int UQ = VF_SK1_U;
            for (int q0 = 0; q0 < nq; q0 += 32 * UQ) {
                T v[UQ][4], x[UQ][4];
#pragma unroll
                for (int u = 0; u < UQ; ++u) {
                    const int q = q0 + 32 * u + lane;
                    const int t0 = 4 * q;
                    const int wi = min(t0 >> 5, NWORD - 1);
                    const unsigned word = pw[wi];
                    const int base = __shfl_sync(FULL, wexcl, wi);
#pragma unroll
                    for (int j = 0; j < 4; ++j) { v[u][j] = T(0); x[u][j] = T(0); }
                    if (t0 < nt) {
                        const int b = t0 & 31;
                        int p = base + __popc(word & ((2u << b) - 1u)) - 1;
                        const unsigned inner = (word >> (b + 1)) & 7u;
                        Quad<T>::ld(vals + t0, v[u]);
                        int4 pr = prec[p];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if (j > 0 && ((inner >> (j - 1)) & 1u)) pr = prec[++p];
                            const int t = t0 + j;
                            if (t < nt) {
                                const int e = t - pr.y;
                                x[u][j] = XT[pr.x + (pr.w ? (int)ix[pr.z + e] : e)];
                            } else {
                                v[u][j] = T(0);
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < UQ; ++u)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc = fma(v[u][j], x[u][j], acc);
            }
            if (h.flags & 1) {
                T s = acc;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
                if (lane == 0) a.Y[h.item] = s;
                acc = T(0);
            }
        }
        __syncwarp();
        int ok = 0;
        if (lane == 0) {
            fence_proxy_async();            // generic-proxy reads of the slot before the async refill
            ok = issue(slot);
        }
        ok = __shfl_sync(FULL, ok, 0);
        issued += ok;
    }
    if (!arrived) arrive();
}

}  // namespace

#ifndef VF_SK1_WARPS
#define VF_SK1_WARPS 16
#endif
#ifndef VF_SK1_STAGES
#define VF_SK1_STAGES 3
#endif
constexpr int kNW = VF_SK1_WARPS;    // warps per CTA (one CTA per SM)
constexpr int kNS = VF_SK1_STAGES;   // ring slots per warp

size_t smem_bytes() {
    return (size_t)kNW * kNS * kSlot + (size_t)kNW * kMaxPieces * 16 + (size_t)kNW * (kMaxTerms / 32) * 4 +
           (size_t)kNW * kNS * 8;
}

#define SCK(call)                                                                        \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return set_error(VF_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int upload(const HostLayout& L, int w, int64_t NT, DevLayout* D) {
    auto up = [&](void** dst, const void* src, size_t bytes) -> int {
        if (bytes == 0) bytes = 16;
        SCK(cudaMalloc(dst, bytes));
        D->device_bytes += (int64_t)bytes;
        if (src) SCK(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
        else SCK(cudaMemset(*dst, 0, bytes));
        return VF_OK;
    };
    int rc;
    std::vector<P1Item> p1 = L.p1;
    if (p1.empty()) p1.resize(1);
    std::vector<int32_t> pc(std::max<int64_t>(L.ngroups, 1), 0);
    if ((rc = up((void**)&D->bytes, L.bytes.data(), L.bytes.size())) ||
        (rc = up((void**)&D->coff, L.coff.data(), L.coff.size() * 8)) ||
        (rc = up((void**)&D->ic0, L.ic0.data(), L.ic0.size() * 4)) ||
        (rc = up((void**)&D->p1, p1.data(), p1.size() * sizeof(P1Item))) ||
        (rc = up((void**)&D->pscr, nullptr, (size_t)std::max<int64_t>(L.nscratch, 1) * 16 * 8)) ||
        (rc = up((void**)&D->pcnt, pc.data(), pc.size() * 4)) ||
        (rc = up((void**)&D->ctr, nullptr, 16)))
        return rc;
    (void)NT;
    D->n1 = L.n1;
    D->n2 = L.n2;
    D->w = w;
    D->stream_bytes = (int64_t)L.bytes.size();
    D->payload_bytes = L.payload_bytes;
    D->meta_bytes = L.meta_bytes;
    D->nchunks = (int64_t)L.coff.size() - 1;
    D->ok = true;
    return VF_OK;
}

void free_dev(DevLayout* D) {
    void* ps[] = {D->bytes, D->coff, D->ic0, D->p1, D->pscr, D->pcnt, D->ctr};
    for (void* p : ps) if (p) cudaFree(p);
    *D = DevLayout{};
}

template <typename T>
static int launch_t(const DevLayout& D, void* XT, void* Y, cudaStream_t st, int* grid_out) {
    auto fn = stream_k1_kernel<T, kNW, kNS>;
    const size_t smem = smem_bytes();
    SCK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kNW * 32, smem));
    if (per_sm < 1) return set_error(VF_ECUDA, "stream_k1_kernel cannot be resident");
    int dev = 0, nsm = 148;
    SCK(cudaGetDevice(&dev));
    SCK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    SArgs<T> a{D.bytes, D.coff, D.ic0, D.p1, (int32_t)D.n1, (int32_t)D.n2, static_cast<T*>(XT),
               static_cast<T*>(Y), D.pscr, D.pcnt, D.ctr};
    SCK(cudaMemsetAsync(D.ctr, 0, 16, st));
    void* args[] = {&a};
    SCK(cudaLaunchCooperativeKernel((const void*)fn, dim3(nsm), dim3(kNW * 32), args, smem, st));
    *grid_out = nsm;
    return VF_OK;
}

int matvec_k1(const DevLayout& D, int dtype, void* XT, void* Y, cudaStream_t st, int* grid_out) {
    if (!D.ok) return set_error(VF_EUNSUPPORTED, "no stream layout");
    return dtype == VF_F64 ? launch_t<double>(D, XT, Y, st, grid_out) : launch_t<float>(D, XT, Y, st, grid_out);
}

}  // namespace stream
}  // namespace vf
