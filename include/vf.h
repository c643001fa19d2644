/*
 * vf.h -- C ABI of libvf, the B200 (sm_100a) compressed view-factor library.
 *
 * The operation (PAPER.md = "P:<line>", arXiv 2209.07632):
 *   F is the N x N view-factor matrix of a triangle mesh,
 *     F_ij = [n_i.(x_j - x_i)][n_j.(x_i - x_j)] V_ij A_j / (pi |x_i - x_j|^4),
 *   F_ii = 0                                   (eq. FF-def)
 *   with V_ij the culled, ray-cast visibility   (§3.2).
 *   F-hat is its hierarchical compression: a quadtree permutation (Alg. 2,
 *   P:198-213) and a dynamic-programming choice per block pair of
 *   Zero / CSR / dense / truncated-SVD U S V^T / subdivided (Alg. 3-4,
 *   P:219-256).  The hot path applies F-hat to many right-hand sides
 *   (Alg. 5) and iterates the Jacobi solves built on it
 *   (eq. radiosity-system).
 *
 * Conventions (all calls):
 *   - Every call returns an int status (vf_status); no exceptions cross the
 *     ABI.  vf_last_error() returns a thread-local message for the last
 *     failure on this thread.
 *   - Vectors are COLUMN-MAJOR N x nrhs with leading dimension N, in the
 *     caller's facet order (facet f = face f of the mesh).  Per-facet
 *     parameters (rho, albedo, emissivity) are length-N vectors shared by all
 *     columns.  Element type = the handle's dtype (VF_F64 -> double,
 *     VF_F32 -> float) unless stated otherwise.
 *   - Vector arguments may be DEVICE pointers (on the handle's device) or
 *     HOST pointers (pageable or pinned); the library detects which with
 *     cudaPointerGetAttributes and, for host pointers, stages through
 *     handle-owned device buffers inside the call.  The caller owns every
 *     vector; the library keeps no reference after the call returns.
 *   - Stream ordering: work is enqueued on the handle's stream
 *     (vf_set_stream; default: the legacy default stream).  vf_matvec with
 *     device pointers is asynchronous; solves synchronise the stream to test
 *     convergence and return when finished.
 *   - X must not alias Y.  B / T / Qvis / Qir are outputs only.
 *   - Scratch: the handle owns all device scratch, grown to the largest
 *     nrhs seen.  A handle is not thread-safe: one call at a time.
 *   - No CPU fallback: every apply/solve runs in the CUDA kernels of this
 *     library; without a usable sm_100 device those calls fail with
 *     VF_ENODEV.
 */
#ifndef VF_H_
#define VF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vf_handle_s* vf_handle;

typedef enum {
    VF_OK = 0,
    VF_EINVAL = -1,        /* bad argument (null pointer, size, dtype, ...)          */
    VF_ENOMEM = -2,        /* host or device allocation failed                        */
    VF_ECUDA = -3,         /* a CUDA runtime call or kernel failed                    */
    VF_ENOCONV = -4,       /* solve hit `iters` before `tol`; outputs hold last iterate */
    VF_EIO = -5,           /* file open/read/write failed or bad HVFM container       */
    VF_ENCCL = -6,         /* an NCCL call of the row-sharded mode failed             */
    VF_EUNSUPPORTED = -7,  /* valid request this build does not implement             */
    VF_ENODEV = -8         /* no usable CUDA device / handle has no device copy       */
} vf_status;

enum { VF_F64 = 1, VF_F32 = 2 };                 /* storage + arithmetic dtype     */
enum { VF_VIS_RAYCAST = 0, VF_VIS_CULL_ONLY = 1 };  /* V_ij: culling + ray cast, or
                                                      culling only (tests)  */

/* Triangle mesh, HOST arrays borrowed for the duration of the call.
 * V: nv x 3 row-major vertex coordinates (metres); F: nf x 3 row-major
 * 0-based vertex indices.  Facet data follows P:129: x_i = centroid,
 * A_i = area, n_i = unit normal (right-hand rule, flipped to n_z > 0 when
 * opts.orient_up, the height-field convention).  Zero-area faces -> VF_EINVAL. */
typedef struct {
    int64_t nv, nf;
    const double* V;
    const int32_t* F;
} vf_mesh;

typedef struct {
    int dtype;           /* VF_F64 (default) or VF_F32: factor/value + vector type  */
    int max_depth;       /* quadtree depth cap (Alg. 2 reading A3), default 16       */
    int min_leaf;        /* quadtree leaf size (A3), default 16                       */
    int64_t min_block;   /* |I||J| below which a block is CSR or dense (Alg. 4 step 2,
                            reading A4), default 16384                               */
    int k0;              /* initial rank guess of Alg. 3, default 8           */
    int visibility;      /* VF_VIS_RAYCAST (default) or VF_VIS_CULL_ONLY               */
    int orient_up;       /* 1 (default): n_z > 0; 0: keep right-hand-rule normals     */
    int device;          /* CUDA device to upload to; -1 = host-only handle (build,
                            save, info work; apply/solve return VF_ENODEV)            */
    int threads;         /* host threads for the build (0 = all cores)               */
    uint64_t seed;       /* seed of the randomized truncated SVD (default 0x5eed)      */
    int evaluator;       /* who evaluates F_ij and V_ij for Alg. 1:
                            VF_EVAL_AUTO (default): the device when device >= 0,
                            else the host; VF_EVAL_HOST; VF_EVAL_DEVICE.  Both take
                            bit-identical decisions and values (reading R-VIS)     */
    int tree;            /* spatial tree of the permutation: VF_TREE_QUAD
                            (default; centroids' x, y -- height fields) or
                            VF_TREE_OCT (x, y, z: closed bodies, overhangs; 64
                            first-level block pairs)                         */
} vf_build_opts;

enum { VF_EVAL_AUTO = 0, VF_EVAL_HOST = 1, VF_EVAL_DEVICE = 2 };
enum { VF_TREE_QUAD = 0, VF_TREE_OCT = 1 };

/* Fill *opts with the defaults above. */
void vf_default_opts(vf_build_opts* opts);

/* Assemble F-hat for a mesh with compression tolerance tol (eps of Alg. 3,
 * relative to each block's sigma_1).  Host-side, untimed: facet data,
 * BVH visibility (Alg. 1), quadtree (Alg. 2), rank estimation (Alg. 3) and
 * DP assembly (Alg. 4), then flattening and upload to opts->device.
 * opts may be NULL (defaults).  On success *out owns everything. */
int vf_build(const vf_mesh* mesh, double tol, const vf_build_opts* opts, vf_handle* out);

/* Same from explicit facet data (HOST, borrowed): x, n: N x 3 row-major
 * centroids and unit normals, A: N areas.  Visibility is culling only when
 * occluders == NULL or opts->visibility == VF_VIS_CULL_ONLY; otherwise the
 * occluder triangles are ray-cast (facet f is NOT excluded from its own ray
 * unless occluders->nf == N and face f is facet f).  Test hook for
 * sphere-exact facet data (pins P1/P4). */
int vf_build_facets(int64_t N, const double* x, const double* n, const double* A,
                    const vf_mesh* occluders, double tol, const vf_build_opts* opts,
                    vf_handle* out);

/* Load an HVFM container (format below) and upload it to `device` (-1: host
 * only).  Values are applied exactly as stored. */
int vf_load(const char* path, int device, vf_handle* out);

/* Write the handle's F-hat as an HVFM container. */
int vf_save(vf_handle h, const char* path);

/* Upload a host-only handle (device == -1 at build/load) to `device`. */
int vf_upload(vf_handle h, int device);

/* Release the handle, its host metadata and device memory.  NULL is OK. */
int vf_free(vf_handle h);

/* Order all subsequent work on `stream` (a cudaStream_t, e.g.
 * torch.cuda.current_stream().cuda_stream).  NULL = legacy default stream. */
int vf_set_stream(vf_handle h, void* stream);

/* Y = F-hat X (Alg. 5), overwrite, no clamping (reading A12).  X, Y: N x nrhs.
 * 2..8 columns on an F-hat whose device layout exceeds 256 MB are applied
 * column by column with the nrhs = 1 kernel (each column's result is bitwise
 * that of a separate nrhs = 1 call); env VF_MV_COLSPLIT=0/1 overrides.
 * More than 64 columns there run in 64-column chunks, the tail in 32/16-column
 * pieces, a 9..15-column rest batched, <= 8 columns one by one (env
 * VF_MV_CHUNK=c sets the chunk, 0 = one batch).  Not in ROWS mode. */
int vf_matvec(vf_handle h, const void* X, void* Y, int nrhs);

/* Jacobi solve of B = E + diag(rho) F-hat B (eq. radiosity-system):
 * B_0 = E; Q_k = F-hat B_k, clamped to >= 0 when clamp != 0;
 * B_{k+1} = E + rho * Q_k; per-column r_k = ||B_{k+1}-B_k||_2 / ||E||_2
 * (||E|| = 0 -> 0).  Stops when all columns have r_k <= tol, or after `iters`
 * iterations (-> VF_ENOCONV, B = last iterate).  E, B: N x nrhs; rho: N. */
int vf_solve_radiosity(vf_handle h, const void* E, const void* rho, void* B,
                       int nrhs, int iters, double tol, int clamp);

/* Equilibrium temperature (eq. 3d-equilbr):
 *   stage 1: the radiosity solve with rho = albedo, E = albedo * Qdir;
 *            Qrefl = the last clamped Q;  Qvis = Qdir + Qrefl;
 *   stage 2: rho = 1, E = (1 - albedo) * Qvis; Qir = the last clamped Q
 *            (eq. time-indep-system-2 with H = 0);
 *   T = (((1 - albedo) Qvis + emiss Qir) / (emiss sigma))^(1/4).
 * Qdir, T, Qvis, Qir: N x nrhs (Qvis/Qir may be NULL); albedo, emiss: N. */
int vf_solve_thermal(vf_handle h, const void* Qdir, const void* albedo, const void* emiss,
                     void* T, void* Qvis, void* Qir, int nrhs, int iters, double tol);

/* Iteration counts and max-over-columns final residuals of the last solve
 * (stage 2 values are 0 after a radiosity solve).  Any pointer may be NULL. */
int vf_last_solve_stats(vf_handle h, int* iters1, double* resid1, int* iters2, double* resid2);

/* Direct insolation (P:76-80 eq. insolation) with R_sun = 1 AU:
 * Q_if = S max(0, n_i.s_f) V_sun(x_i, s_f).  suns: k x 3 unit vectors (HOST);
 * Qdir: N x k column-major HOST double output.  Needs a mesh-built handle. */
int vf_insolation(vf_handle h, const double* suns, int k, double S, double* Qdir);

/* Finite solar disk as a sum over point sources: for each of the k
 * suns, Q_ic = sum_p w_p S max(0, n_i.d_{c,p}) V_sun(x_i, d_{c,p}) -- the
 * point-sun insolation above per source, weighted.  dirs: (k*P) x 3 unit
 * vectors, sun c's sources at rows c*P .. c*P+P-1 (HOST); w: P weights
 * (HOST); Qdir: N x k column-major HOST double output.  Sources are summed in
 * the order p = 0 .. P-1.  Needs a mesh-built handle. */
int vf_insolation_sum(vf_handle h, const double* dirs, const double* w, int k, int P, double S, double* Qdir);

/* Attach the mesh a loaded handle was built from (HOST arrays, copied) so
 * that vf_insolation works on it: facet f of the mesh is facet f of the
 * handle (nf must equal N); orient_up as in vf_build_opts. */
int vf_set_mesh(vf_handle h, const vf_mesh* mesh, int orient_up);

/*
 * Time-dependent thermal model (Alg. 6; NEXT-1): per step one
 * F-hat product of the 2 nscen columns [alpha (Q_dir^(n+1) + Q_refl^(n)) |
 * Q_rad^(n) + (1 - eps) Q_IR^(n)] (clamped >= 0, reading A12), Q_abs^(n+1) =
 * (1 - alpha)(Q_dir^(n+1) + Q_refl^(n+1)) + eps Q_IR^(n+1), then one
 * Crank-Nicolson step of every facet's subsurface column (reading
 * A27 in DESIGN.md: M layers, geometric thicknesses d_1 r^(j-1) to `depth`,
 * conductivity k_th, volumetric heat capacity rho_c, a capacity-free surface
 * node balanced at n+1 with eps sigma T^4 linearised about T_0^(n), bottom flux
 * H) and Q_rad = eps sigma T_0^4.  nscen independent scenarios (sites,
 * parameter sets) step together; steps are sequential.  The state lives on the
 * device, owned by the vf_tstate; vectors as for the solves (column-major
 * N x nscen, caller order, device or host, handle dtype).
 */
typedef struct vf_tstate_s* vf_tstate;
/* Initialise: Q_abs^(0) = (1 - alpha) Qdir0 + H, Q_refl = Q_IR = 0,
 * Q_rad^(0) = Q_abs^(0); every column starts uniform at T0 (N x nscen).
 * 1 <= M <= 128, depth > 0, ratio > 0, k_th > 0, rho_c > 0. */
int vf_ts_create(vf_handle h, int nscen, int M, double depth, double ratio, double k_th, double rho_c, double H,
                 const void* albedo, const void* emiss, const void* Qdir0, const void* T0, vf_tstate* out);
/* One step with the direct flux Q_dir^(n+1) (N x nscen) and time step dt (s);
 * Tsurf (N x nscen, nullable) receives the new surface temperature. */
int vf_ts_step(vf_tstate s, const void* Qdir, double dt, void* Tsurf);
/* Current Q_refl, Q_IR, Q_abs and surface T (each N x nscen, nullable). */
int vf_ts_get(vf_tstate s, void* Qrefl, void* Qir, void* Qabs, void* Tsurf);
int vf_ts_free(vf_tstate s);

/* TEST HOOK (not part of the apply/solve path): one ROWS-mode exchange with
 * world ranks emulated on the current device in sequence -- every rank's
 * pack (own rows [bounds[g], bounds[g+1]) of its new iterate + the sum over
 * its nblk CTA partials per column), the allgather as device copies of the
 * send slots, every rank's unpack and stop decision -- the kernels the
 * multi-GPU solve runs, exercised at world > 1 on one GPU.  HOST arrays:
 * xrank world x N x kp (rank g's iterate, row-major tree order), part
 * world x kp x nblk, enorm2 k; outputs xout world x N x kp, resid k, and per
 * rank the iteration count and stop flag after the decision. */
int vf_selftest_rows_exchange(int world, int kp, int k, int64_t N, const int64_t* bounds, const double* xrank,
                              const double* part, int nblk, const double* enorm2, double tol, int iters, int iter0,
                              double* xout, double* resid, int* iter_after, int* done_after);

typedef struct {
    int64_t N;             /* facets                                               */
    int dtype;             /* VF_F64 / VF_F32                                      */
    double tol;
    int64_t n_dense, n_csr, n_svd;        /* leaf counts by kind                    */
    int64_t bytes_dense, bytes_csr, bytes_svd;  /* A7/A8 accounting per kind          */
    int64_t nnz_csr;       /* stored CSR nonzeros                                  */
    int64_t sum_rank;      /* sum of q over SVD blocks                              */
    int64_t max_rank;
    int64_t active_rows;   /* rows of F-hat with any stored entry                    */
    int64_t device_bytes;  /* bytes of the device layout of F-hat (values, indices,
                              segment descriptors, permutation)                      */
    int64_t alg_bytes;     /* algorithmic bytes per apply, excluding X/Y traffic:
                              values + CSR column indices + SVD row indices          */
    int64_t alg_flops_per_col; /* 2 (sum q(mu+nv) + nnz + sum mn) + sum q            */
    int64_t visible_pairs; /* nonzeros of the exact F seen during the build (0 if loaded) */
    double build_seconds;
    int device;            /* -1 = host only                                       */
    /* device-layout accounting of the two apply phases (0 for host-only handles) */
    int64_t t_rows;        /* rank-1 terms = rows of T (sum of q)                   */
    int64_t p1_bytes;      /* phase 1 payload: V values + V row indices + S          */
    int64_t p2_bytes;      /* phase 2 payload: dense/U/CSR values + CSR indices      */
    int64_t p1_src_rows;   /* distinct X rows phase 1 reads                          */
    int64_t p2_src_rows;   /* distinct X/T rows phase 2 reads                        */
    int64_t p1_flops_per_col, p2_flops_per_col;
    int64_t groups1, groups2;  /* row groups of the batched layout (phase 1 / 2)      */
    int64_t resident;      /* 1: batched applies (nrhs >= 9) keep F-hat in shared
                              memory across iterations (res_kernel); 0: streamed    */
    /* chunk-stream layout of the nrhs = 1 apply (0 if absent): the F-hat bytes one
       apply streams = payload (values, 16-bit CSR column offsets, phase-1 row
       lists) + meta (chunk headers, piece descriptors, 16-B padding)            */
    int64_t stream_payload_bytes;
    int64_t stream_meta_bytes;
    int64_t stream_chunks;
    /* streamed-tile layout of wide batches (FP64, F-hat beyond the resident
       layout): tiles and sum over tiles of their K (16 K weights each)        */
    int64_t tiles;
    int64_t tile_sources;
    /* bytes one nrhs = 1 vf_matvec streams in the row layout of hot_kernel
       (values, S, V row indices, 16-bit CSR offsets; 0 if that layout is off) */
    int64_t k1_payload_bytes;
    /* which kernel runs an nrhs = 1 vf_matvec (fixed at upload; VF_K1_KERNEL env
       = rows | stream | pipe overrides the build default): 0 = hot_kernel<T,1,1>
       (row segments), 1 = stream_k1_kernel (chunk stream), 2 = k1p_kernel
       (pipelined per-warp cp.async rings)                                      */
    int64_t k1_kernel;
} vf_info_t;

int vf_info(vf_handle h, vf_info_t* out);

/* Per-launch timing of the dominant kernel of the last apply/solve, measured
 * with CUDA events on the handle's stream when enabled (0/1).  *ms is the
 * summed duration of the row-owner accumulate kernel (phase 2) over the last
 * call, *launches its launch count. */
int vf_enable_kernel_timing(vf_handle h, int on);
int vf_kernel_timing(vf_handle h, double* ms_phase2, int* launches_phase2,
                     double* ms_phase1, int* launches_phase1, int* launches_total);

/*
 * Block-row sharding (multi-GPU single-RHS solves; SURVEY §8(e) "ROWS",
 * §8(a) a6).  Alg. 5 sums Y_I = sum_J F_IJ X_J per block row, so
 * the operator splits by output rows: rank g of `world` owns the contiguous
 * tree-order rows [bounds[g], bounds[g+1]), cut so every rank streams about
 * the same F-hat bytes per apply (A7/A8 byte accounting).  A rank keeps the
 * leaf rows inside its range (SVD blocks: its rows of U; V and S duplicated)
 * and the full right-hand side; each Jacobi iteration ends with one
 * ncclAllGather of the ranks' new rows (and their residual partial sums).
 * One process per GPU; every rank makes the same calls with the same full
 * (caller-order, N x nrhs) inputs and receives the same full outputs.
 */

/* Cut points of the row partition for `world` ranks (bounds: world + 1
 * int64, HOST, caller-owned).  Does not modify the handle.  For a sharded
 * handle `world` must equal its world and its own cut points are returned. */
int vf_row_partition(vf_handle h, int world, int64_t* bounds);

/* Restrict the handle to rank `rank`'s rows of the partition above (host
 * metadata and, if uploaded, the device copy).  Irreversible; a handle can be
 * sharded once.  Without a communicator, vf_matvec on a sharded handle writes
 * this rank's rows of Y and zeros elsewhere, and the solves fail with
 * VF_EINVAL; after vf_comm_init every call returns full results. */
int vf_shard_rows(vf_handle h, int rank, int world);

/* This rank's tree-order row range [*lo, *hi) ([0, N) if not sharded). */
int vf_row_range(vf_handle h, int64_t* lo, int64_t* hi);

/* A fresh NCCL unique id (128 bytes written to id128, HOST).  Rank 0 creates
 * it and the caller broadcasts it (e.g. through a torch process group). */
int vf_get_nccl_id(void* id128);

/* Create the handle's NCCL communicator (rank, world as in vf_shard_rows; the
 * handle's device must be this process's GPU).  Collective over all ranks.
 * Failures -> VF_ENCCL.  Released by vf_free. */
int vf_comm_init(vf_handle h, int rank, int world, const void* id128);

const char* vf_last_error(void);

/*
 * HVFM v1 container (little-endian), written by vf_save and oracle/hmatrix.py:
 *   char  magic[4] = "HVFM"; u32 version = 1; u32 dtype (1 f64, 2 f32); u32 0;
 *   i64   N; f64 tol; i64 nleaves;
 *   i32   perm[N]              tree position r holds caller facet perm[r]
 *   then nleaves leaves in Alg. 5 order, each:
 *     i32 kind (1 dense, 2 csr, 3 svd); i32 level; i64 row0, m, col0, n
 *         (tree-order row range [row0, row0+m), column range [col0, col0+n))
 *     dense: val[m*n] row-major
 *     csr:   i64 nnz; i64 rowptr[m+1]; i32 col[nnz] (local to col0); val[nnz]
 *     svd:   i64 q, mu, nv; i32 urow[mu]; i32 vrow[nv] (local indices of the
 *            nonzero rows of U / V, reading A8); val S[q]; val U[mu*q] and
 *            val V[nv*q], both row-major (row r holds its q entries)
 *   val = double (dtype 1) or float (dtype 2).  The block contributes
 *   Y[row0+urow] += U diag(S) V^T X[col0+vrow] (svd) and the obvious
 *   products for dense / csr.  Zero blocks are not stored.
 */

#ifdef __cplusplus
}
#endif
#endif /* VF_H_ */
