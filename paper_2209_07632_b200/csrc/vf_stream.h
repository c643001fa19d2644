// vf_stream.h -- the chunk-stream layout of F-hat for the nrhs = 1 apply
// (SURVEY §8(a) a2 + a3; Alg. 5, "U(Sigma(V^T x))", the
// per-time-step MVP).  Internal to libvf; see DESIGN.md §6 / §7.
//
// Every work item -- a phase-1 (SVD row group, part of its V rows) item or a
// phase-2 output row -- is ONE contiguous run of self-describing chunks of at
// most kSlot bytes in a single global byte stream.  A warp of the streaming
// kernel copies an item's chunks into its private shared-memory ring with
// cp.async.bulk (the Blackwell bulk-copy engine, SASS UBLKCP) and consumes
// them from there, so the F-hat stream never passes through L1 or registers
// and the L1 serves only the x gathers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace vf {

namespace stream {

constexpr int kSlot = 4608;      // max chunk bytes (= one ring slot)
constexpr int kMaxPieces = 32;   // phase-2 pieces per chunk (one descriptor per lane)
constexpr int kMaxTerms = 576;   // phase-2 terms per chunk (the consumer's per-warp XT-row buffer)
constexpr int kP1J = 32;         // phase-1 chunks carry a multiple of 32 V rows (one per lane)
constexpr int kP1Part = 2048;    // V rows per phase-1 item (long blocks split over warps)

// chunk header, 16 B
struct Hdr {
    int32_t item;      // phase 1: item id (p1 table); phase 2: output tree row
    int16_t n;         // phase 1: G (T rows of the group); phase 2: pieces
    int16_t flags;     // bit 0: last chunk of its item; bit 1: phase-1 chunk
    int32_t nterm;     // phase 1: V rows j in this chunk; phase 2: terms
    int32_t src;       // phase 1: first X row of a contiguous V-row run, -1: int32 row list follows
};
// phase-2 piece descriptor, 8 B
struct Piece {
    int32_t src;       // first XT row (kind 0) or base XT row of the run (kind 1)
    uint16_t len;      // terms
    uint8_t kind;      // 0: XT rows src .. src+len (dense-leaf X rows or U_b's T rows); 1: src + u16 offset
    uint8_t pad;
};
// phase-1 item: T rows t0 .. t0+G (XT rows) of one SVD block, a part of its V rows
struct P1Item {
    int32_t t0;
    int16_t G;
    int16_t np;        // parts of the group (1: this item stores T directly)
    int32_t pidx;      // part index within the group
    int32_t group;     // group id (part counter of multi-part groups)
    int32_t sbase;     // first scratch row of the group's parts (multi-part groups)
    int32_t pad_;
};

// host-side result of the layout builder
struct HostLayout {
    std::vector<unsigned char> bytes;     // the chunk stream (16-B aligned chunks)
    std::vector<int64_t> coff;            // chunk c = bytes[coff[c], coff[c+1])
    std::vector<int32_t> ic0;             // item i = chunks [ic0[i], ic0[i+1]); phase-1 items first
    std::vector<P1Item> p1;               // phase-1 item table
    int64_t n1 = 0, n2 = 0, ngroups = 0;  // items of each phase, phase-1 groups
    int64_t nscratch = 0;                 // scratch rows of multi-part groups
    int64_t payload_bytes = 0;            // values + indices (algorithmic)
    int64_t meta_bytes = 0;               // headers + descriptors + padding
};

// device copy + launch (vf_stream.cu)
struct DevLayout {
    bool ok = false;
    unsigned char* bytes = nullptr;
    int64_t* coff = nullptr;
    int32_t* ic0 = nullptr;
    P1Item* p1 = nullptr;
    double* pscr = nullptr;
    int32_t* pcnt = nullptr;
    int32_t* ctr = nullptr;
    int64_t n1 = 0, n2 = 0, nchunks = 0;
    int w = 8;
    int64_t stream_bytes = 0, payload_bytes = 0, meta_bytes = 0, device_bytes = 0;
};
int upload(const HostLayout& L, int w, int64_t NT, DevLayout* D);
void free_dev(DevLayout* D);
// Y = F-hat X for one column.  XT: tree-order device vector [x (N) | T rows]
// (the XT buffer of vf_device.cu; T rows are written), Y: tree-order (N)
int matvec_k1(const DevLayout& D, int dtype, void* XT, void* Y, cudaStream_t st, int* grid);

}  // namespace stream
}  // namespace vf
