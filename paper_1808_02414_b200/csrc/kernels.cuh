// Host-side launchers and device data descriptors of the sfmcov_b200 pipeline.
#pragma once

#include "common.cuh"

#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace sfm {

// Grow-only device allocation.
struct DBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            SFM_CUDA(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return p;
    }
    template <typename T>
    T* as(size_t count) { return static_cast<T*>(get(sizeof(T) * count)); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct Workspace {
    DBuf tmp;
    void* get_tmp(size_t bytes) { return tmp.get(bytes); }
};

// Scene pointers in device memory.
struct SceneDev {
    int n, m, t, P;
    const double* cams;
    const double* pts;
    const int* oc;
    const int* op;
    const double* u;
    const double* sigma;
    // host copy of u for the host API: u is only validated (finite), so it is
    // scanned on the host while the rest of the scene uploads, not copied
    const double* host_u = nullptr;
    // host API: the covariances upload on a side stream after the indices;
    // recorded when they have arrived (null: already on the library stream)
    cudaEvent_t sigma_ready = nullptr;
};

// CSR observation index (ascending observation ids per bucket) and the
// inverse permutation of the by-camera order.
struct IndexDev {
    int* off_cam;
    int* idx_cam;
    int* off_pt;
    int* idx_pt;
    int* pos_cam;
    int* key_scratch;
};

struct PairDev {
    DBuf buf_cnt, buf_off, buf_k0, buf_k1, buf_v0, buf_v1, buf_ukeys, buf_counts, buf_nruns, buf_seg, buf_chunk,
        buf_part, buf_segof;
    long long* cnt = nullptr;
    long long* off = nullptr;
    long long npairs = 0;
    unsigned int* keys = nullptr;
    unsigned long long* vals = nullptr;
    unsigned int* ukeys = nullptr;
    long long* seg_off = nullptr;
    int nseg = 0;
    int* chunk_off = nullptr;  // segment -> first chunk of <= chunk pairs (nseg + 1)
    int nchunks = 0, chunk = 0;
    int* seg_of = nullptr;     // chunk -> its segment (nchunks)
    double* part = nullptr;    // per-chunk partial blocks of multi-chunk segments
    void release() {
        buf_cnt.release(); buf_off.release(); buf_k0.release(); buf_k1.release(); buf_v0.release();
        buf_v1.release(); buf_ukeys.release(); buf_counts.release(); buf_nruns.release(); buf_seg.release();
        buf_chunk.release(); buf_part.release(); buf_segof.release();
    }
};

// Batched sub-scenes (one dense Z per scene, block-diagonal problem): camera
// c of the concatenated batch lives in scene scene_of_cam[c] at local index
// c - coff[scene], whose Z starts zstride doubles after the previous one.
struct ZMap {
    const int* scene_of_cam = nullptr;
    const int* coff = nullptr;
    long long zstride = 0;
};

// C = beta C + alpha A B^T with K = kNB (see dense.cu).
struct GemmArgs {
    double* C;
    long long ldc;
    const double* A;
    long long lda;
    const double* B;
    long long ldb;
    int tm, tn;
    int K;           // reduction length (multiple of 16)
    int tri;         // lower-triangular tile set (ti >= tj) of a tm x tm grid
    int alpha_neg;   // alpha = -1
    int beta;        // 1: accumulate into C
    int beta0_from;  // column tiles >= this use beta = 0 (-1: none)
    int b_kmajor;    // B stored K-contiguous
    int lower_only;  // skip tiles strictly above the matrix diagonal
    int row_off_tiles, col_off_tiles;  // C tile offsets relative to the diagonal
    int whole_tile;  // C aliases A (in-place trsm): one CTA per 128-wide tile
    int a_kmajor;    // A stored K-contiguous: (m, k) at A[m * lda + k]
    int k_from_row;  // K range of tile (ti, tj) starts at ti * 128 (X^T X of a lower-triangular X)
    int k_from_col;  // column tiles tj >= beta0_from: K starts at (tj - beta0_from) * 128 (B lower-triangular there)
    // Column-cyclic mode (cyc_R > 0, distributed sweep): C holds the local
    // columns of a rank owning panels rank, rank + R, ... of cyc_G tiles.
    // Grid tile (ti, tj) -> local column tile lt = tj + cyc_lt0, global
    // column tile gt of lt, global row tile gi = ti + cyc_row0; tiles with
    // gi < gt are skipped.  A rows / B rows are global tiles gi / gt,
    // relative to the panel buffer's first tile cyc_ab0.
    int cyc_R, cyc_rank, cyc_G, cyc_lt0, cyc_row0, cyc_ab0;
    // pad_skip: rows of C from real_rows on are identity padding whose A rows
    // are zero (beta = 1 updates only): their CTAs / warp tiles skip the
    // product and leave C unchanged, which is exact.  Batched (real_rows_b):
    // real_rows = real_rows_b[batch] - row_origin.
    int pad_skip, real_rows, row_origin;
    const int* real_rows_b;
    // batch > 1: grid.y = batch; operand b is offset by b * bs{A,B,C} doubles
    int batch;
    long long bsA, bsB, bsC;
    // col_step > 1: grid column tile tj addresses matrix column tile col_first + tj * col_step
    // (B rows, C columns, beta0_from / k_from_col): the inverse's column-interleaved halves
    int col_step, col_first;
};

// Several same-sized dense problems swept together (batched sub-scenes): Z,
// the Linv tiles, the panel ring and the pivots of problem b sit b * stride
// doubles after problem 0's; nreal_b[b] = its unpadded size.
struct SweepBatch {
    int B = 1;
    long long zs = 0, ls = 0, rs = 0, ps = 0;
    const int* nreal_b = nullptr;
};

// stage_a.cu
void launch_status_init(Status* st, cudaStream_t s);
void launch_validate(const SceneDev& sc, int check_sigma, Status* st, cudaStream_t s);
void launch_validate_values(const SceneDev& sc, Status* st, cudaStream_t s);
void launch_build_index(const SceneDev& sc, IndexDev& ix, Workspace& ws, cudaStream_t s);
void launch_structure_check(const SceneDev& sc, const IndexDev& ix, Status* st, cudaStream_t s);
void launch_jacobian(const SceneDev& sc, const int* idx_cam, double* R, double* rec, Status* st, cudaStream_t s);
void launch_weights(const SceneDev& sc, const int* idx_cam, double* rec, Status* st, cudaStream_t s);
void launch_depth_of(const SceneDev& sc, const double* R, int t, double* out, cudaStream_t s);
// raw != null (point-sharded stage A): the camera CTAs write their partial
// sums (n x (P^2 + 18)) there and stop; launch_camera_finish completes them.
void launch_reductions(const SceneDev& sc, const IndexDev& ix, const double* rec, double* D, double* Hr, double* A,
                       double* s_a, unsigned char* flags, Status* st, cudaStream_t s, cudaStream_t side,
                       cudaEvent_t fork, cudaEvent_t join, double* raw = nullptr);
void launch_camera_finish(int P, const double* raw, int n, double* D, double* Hr, double* s_a, unsigned char* flags,
                          Status* st, cudaStream_t s);
// sums of squares of the border columns over this scene's rows (cameras
// only when with_cams), and s_b from the summed squares
void launch_border_sums(const SceneDev& sc, const double* Hr, const double* s_a, int with_cams, double* partial,
                        double* sq, cudaStream_t s);
void launch_border_scale(const double* sq, double* s_b, cudaStream_t s);
void launch_border_scales(const SceneDev& sc, const double* Hr, const double* s_a, double* partial, double* s_b,
                          cudaStream_t s);
int border_partial_blocks(int n, int m);
void launch_write_h(const SceneDev& sc, const double* Hr, double* H, cudaStream_t s);

// schur.cu
int point_prep_blocks(int m);
// scene_of_pt (batched sub-scenes): s_b holds 7 scales per scene
void launch_point_prep(const SceneDev& sc, const IndexDev& ix, const double* rec, const double* A, const double* s_a,
                       const double* s_b, double* Lpt, double* Wb, double* V, double* Fpart, double* Pfirst,
                       double* Plast, double* Gsum, Status* st, cudaStream_t s, const int* scene_of_pt = nullptr);
// batch > 1: independent gauge blocks, each from nblocks partials (strided)
void launch_border_factor(const double* Fpart, int nblocks, double* LF, double* E, double* eigE, Status* st,
                          cudaStream_t s, int batch = 1);
// sums_out: write this rank's Σ W V per camera (n x P x 7) and stop;
// sums_in: use all-reduced sums instead of the warp partials
void launch_camera_border(const SceneDev& sc, const IndexDev& ix, const double* Pfirst, const double* Plast,
                          const double* Gsum, const double* Hr, const double* s_a, const double* s_b, const double* LF,
                          double* Gamma, double* G, cudaStream_t s, double* sums_out = nullptr,
                          const double* sums_in = nullptr, const int* scene_of_cam = nullptr);
void launch_fpart_sum(const double* Fpart, int nblocks, double* F28, cudaStream_t s);
void launch_fill(int P, double* Z, long long ld, int N, int Npad, const double* D, const double* s_a, const double* G,
                 int add_gg, cudaStream_t s);
void build_pairs(const SceneDev& sc, const IndexDev& ix, PairDev& pd, Workspace& ws, cudaStream_t s);
void launch_pair_reduce(int P, const PairDev& pd, const double* Wb, int n, double* Z, long long ld, cudaStream_t s,
                        int lo_min = 0, int lo_max = 1 << 30, ZMap zm = ZMap{});

// dense.cu
void dense_init_attributes();
void launch_gemm(const GemmArgs& g, cudaStream_t s);
GemmArgs gemm_args(double* C, long long ldc, const double* A, long long lda, const double* B, long long ldb, int tm,
                   int tn, int K);
void launch_potrf_diag(double* A, long long ld, double* Linv, double* pivots, int col0, Status* st, cudaStream_t s,
                       const SweepBatch* bt = nullptr);
// zm.scene_of_cam (batched sub-scenes): block i is camera i of the batch, in
// scene scene_of_cam[i]'s X (zstride apart), N from that scene's size
void launch_extract(int P, const double* X, long long ld, int N, int nblocks, const double* s_a, int scale, double* cov,
                    Status* st, int* psd_warn, cudaStream_t s, ZMap zm = ZMap{});
void launch_set_diag(double* Z, long long ld, int from, int to, cudaStream_t s);
void launch_minmax(const double* x, long long count, double* part, double* out, cudaStream_t s);
void launch_pivot_range(const double* piv, int N, double* out, cudaStream_t s);
// Extra inverse streams of the fused sweep: the columns of X are independent, so column
// tiles j with j % (n + 1) == q > 0 run on s[q - 1] (their ring-slot events eT[q - 1]).
struct InvSplit {
    int n;                 // extra streams (0..3)
    cudaStream_t s[3];
    cudaEvent_t* eT[3];    // per ring slot
};
int dense_sweep(double* Z, long long ld, int Npad, int G, double* Linv, double* pivots, Status* st, double* ring,
                int NB, cudaStream_t s, cudaStream_t s2, cudaStream_t s3, cudaEvent_t* eL, cudaEvent_t* eT,
                cudaEvent_t eR, cudaStream_t s4, cudaEvent_t eX, cudaEvent_t eN, cudaEvent_t eZ = nullptr,
                int nreal = 0, const SweepBatch* bt = nullptr, const InvSplit* isp = nullptr);
inline size_t sweep_ring_doubles(int Npad, int G, int NB) { return (size_t)NB * Npad * G * kNB; }

// ---- optional outputs (fullcov.cu) ------------------------------------------
struct FullCovArgs {
    int P, n, m, Npad;
    const double* X;         // L^-1 (lower, in Z after the sweep), ld = Npad
    double* Zi;              // Npad x Npad scratch -> Z_aug^-1 (full), then the camera matrix if cross
    const double* G;         // N x 7
    const double* LF;        // 7 x 7 lower, row-major
    const double *Lpt, *V, *Wb, *s_a;
    const int *off_pt, *idx_pt, *oc, *pos_cam;
    double *part, *Y, *gtt_part, *Eb;  // scratch
    double* point_cov;       // device m x 9, or null
    int cross;               // camera blocks from Zi + scaled camera matrix in Zi
    double* cam_cov;
    int* psd;
};
void full_covariance(const FullCovArgs& a, cudaStream_t s);
size_t full_cov_part_doubles(int N);

// ---- refinement against the exact bordered Fisher system (refine.cu) ------
struct RefineArgs {
    int P, n, m, t, Npad;
    long long ld;
    const double* X;  // L^-1 of Z_aug (lower, column-major, the Z buffer after the sweep)
    const double *rec, *D, *A, *Hr, *cams, *pts;
    const int *off_cam, *idx_cam, *off_pt, *idx_pt, *oc, *op, *pos_cam;
    const double *s_a, *s_b, *Lpt, *Wb, *V, *G, *LF;
    double* coupling;  // t x 27 scratch
    DBuf* scratch;
};
size_t refine_bytes(int N, int Npad, int m, int R);
void refine_camera_blocks(const RefineArgs& a, const std::vector<int>& sel, int iters, double* out_blocks,
                          double* history, cudaStream_t s);

// ---- stage functions on caller-supplied block systems (system.cu) ---------
void launch_nullspace_residual(int P, int t, int n, int m, const int* oc, const int* op, const int* pos_cam,
                               const double* rec, const double* H, int b, unsigned long long* mx, cudaStream_t s);
void launch_condition_columns(int P, int n, int m, int b, const double* D, const double* A, const double* border,
                              double* s_a, unsigned char* flags, double* part, double* s_b, cudaStream_t s);
size_t condition_part_doubles(int P, int n, int m, int b);
void launch_apply_conditioning(int P, int n, int m, int t, int b, double* D, double* A, double* Cp, const int* oc,
                               const int* op, double* border, const double* s_a, const double* s_b, cudaStream_t s);
struct SysSchurArgs {
    int P, n, m, t, b;
    const double *D, *A, *Cp, *border;  // device, the (conditioned or not) system
    const int* op;
    const IndexDev* ix;
    const PairDev* pairs;
    double *Lpt, *V, *Wb, *Z, *Gamma, *epart, *zp, *a_inv;  // scratch / outputs (a_inv may be null)
    Status* st;
};
void schur_system(const SysSchurArgs& a, cudaStream_t s);
size_t schur_system_epart_doubles(int m, int b);
void launch_extract_given(int P, int n, const double* Zi, long long ld, const double* s_a, double* cov, int* warn,
                          cudaStream_t s);
void launch_full_k(int P, int n, int m, int t, const double* D, const double* A, const double* rec, const int* oc,
                   const int* op, const int* pos_cam, const double* H, const double* s_a, const double* s_b, double* K,
                   long long ld, cudaStream_t s);
void launch_full_unscale(long long params, const double* S, long long lds, const double* s_a, double* sigma,
                         cudaStream_t s);

// ---- symmetric eigensolver (eigen.cu) ---------------------------------------
// src (n x n, col-major, ld lds, device) -> eigenvalues (host, unsorted) and
// eigenvectors V (device, n2 x n2 col-major, n2 = n rounded up to even, in
// dV); returns the number of Jacobi sweeps.
int sym_eigen(const double* src, long long lds, int n, DBuf& dA, DBuf& dV, DBuf& dwork, std::vector<double>& lam,
              double** V_out, int* ld_out, cudaStream_t s);
// S = V[:, keep] diag(w) V[:, keep]^T (n x n, device, ld = n rounded up to
// 128, symmetrised) through the DMMA GEMM.
void eig_reconstruct(const double* V, int ldv, int n, const std::vector<int>& keep, const std::vector<double>& wts,
                     DBuf& dL, DBuf& dR, DBuf& dS, DBuf& dkeep, double** S_out, long long* ld_out, cudaStream_t s);

// ---- dense pseudoinverse oracle (oraclegpu.cu) -----------------------------
void dense_pseudoinverse(const std::vector<double>& F, int N, DBuf& dA, DBuf& dW, DBuf& dwork, DBuf& dVs, DBuf& dVk,
                         DBuf& dS, DBuf& dkeep, std::vector<double>& lam, double** sigma, long long* ld_out,
                         cudaStream_t s);

// ---- column layouts and panel ownership (distributed path, dist.cu) ---------
// Camera-aligned layout (cpb > 0): cpb = floor(kNB / P) cameras per 128-block,
// the block's tail columns are identity padding, so no camera straddles a
// block (or a panel).  cpb = 0: natural layout, column = P cam + j.
struct ColMap {
    int P, cpb, n;
};
__host__ __device__ inline int cm_col(const ColMap& m, int cam, int j) {
    return m.cpb ? (cam / m.cpb) * kNB + (cam % m.cpb) * m.P + j : m.P * cam + j;
}
// layout column -> natural parameter index, or -1 for padding
__host__ __device__ inline int cm_nat(const ColMap& m, int col) {
    if (!m.cpb) return col < m.P * m.n ? col : -1;
    const int blk = col / kNB, w = col - blk * kNB;
    if (w >= m.cpb * m.P) return -1;
    const int cam = blk * m.cpb + w / m.P;
    return cam < m.n ? cam * m.P + (w - (w / m.P) * m.P) : -1;
}
inline int cm_npad(const ColMap& m) {
    return m.cpb ? ((m.n + m.cpb - 1) / m.cpb) * kNB : ((m.P * m.n + kNB - 1) / kNB) * kNB;
}
// 1D block-cyclic panels: panel q = 128-blocks [qG, qG + G), owner q % R;
// a rank stores its panels' columns contiguously (all Npad rows).
struct Ownership {
    int R, rank, G;
};
__host__ __device__ inline int own_lcol(const Ownership& o, int gcol) {
    const int blk = gcol / kNB, pan = blk / o.G;
    if (pan % o.R != o.rank) return -1;
    return ((pan / o.R) * o.G + (blk - pan * o.G)) * kNB + (gcol - blk * kNB);
}
__host__ __device__ inline int own_gcol(const Ownership& o, int lcol) {
    const int lblk = lcol / kNB, lpan = lblk / o.G;
    const int pan = lpan * o.R + o.rank;
    return (pan * o.G + (lblk - lpan * o.G)) * kNB + (lcol - lblk * kNB);
}
// number of local 128-blocks of a rank for K global blocks
inline int own_blocks(const Ownership& o, int K) {
    int b = 0;
    for (int q = o.rank; q * o.G < K; q += o.R) b += (K - q * o.G < o.G) ? K - q * o.G : o.G;
    return b;
}
// local blocks of the rank's panels with index <= q
inline int own_blocks_upto(const Ownership& o, int K, int q) {
    int b = 0;
    for (int p = o.rank; p <= q && p * o.G < K; p += o.R) b += (K - p * o.G < o.G) ? K - p * o.G : o.G;
    return b;
}

// ---- batched sub-scenes (batch.cu) ---------------------------------------------
// Device lists of a batch of B sub-scenes of one resident scene: per scene its
// sorted global camera ids cams[coff[s] .. coff[s+1]), point ids
// pts[poff[s] ..), and observation ids obs[toff[s] ..) (ascending).
struct BatchLists {
    int B = 0, nb = 0, mb = 0, tb = 0;
    const int *cams = nullptr, *coff = nullptr, *pts = nullptr, *poff = nullptr, *obs = nullptr, *toff = nullptr;
};
void launch_batch_scene_of(const int* off, int B, int count, int* out, cudaStream_t s);
void launch_batch_gather(const BatchLists& L, int P, const double* cams_full, const double* pts_full, const int* oc,
                         const int* op, const double* sigma, double* cams_b, double* pts_b, int* oc_b, int* op_b,
                         double* sigma_b, cudaStream_t s);
void launch_batch_border(int P, const BatchLists& L, const double* cams_b, const double* Hr, const double* pts_b,
                         const double* s_a, double* s_b, cudaStream_t s);
void launch_batch_F(const BatchLists& L, const double* V, double* F28, cudaStream_t s);
void launch_batch_wv(int P, int nb, const int* off_cam, const int* idx_cam, const int* op, const double* Wb,
                     const double* V, double* sums, cudaStream_t s);
void launch_batch_fill(int P, const BatchLists& L, double* Zb, int Npad, const double* D, const double* s_a,
                       const double* G, cudaStream_t s);
void launch_batch_ratio(const BatchLists& L, const double* piv, int Npad, int P, const double* eigE, int* bad,
                        cudaStream_t s);

// ---- point-sharded stage A (shard.cu) ---------------------------------------
// A rank's sub-scene: every camera, points [j0, j1), their observations in
// observation order (lt = their global observation ids).
struct ShardScene {
    SceneDev sc{};
    int j0 = 0, j1 = 0;
    const int* lt = nullptr;
    DBuf buf_flag, buf_iota, buf_lt, buf_cnt, buf_oc, buf_op, buf_sigma;
    Workspace ws;
    void release() {
        buf_flag.release(); buf_iota.release(); buf_lt.release(); buf_cnt.release(); buf_oc.release();
        buf_op.release(); buf_sigma.release(); ws.tmp.release();
    }
};
// point ranges of R ranks balanced by observation pairs (bounds: R + 1)
void shard_bounds(const long long* pair_off, int m, int R, int* d_bounds, std::vector<int>& bounds, cudaStream_t s);
int shard_extract(const SceneDev& g, int j0, int j1, ShardScene& out, cudaStream_t s);
void launch_seg_map(const unsigned int* ukeys_l, int nseg_l, const unsigned int* ukeys_g, int nseg_g,
                    const double* seg_l, double* seg_g, cudaStream_t s);
void launch_flags_or(const unsigned char* src, size_t count, unsigned char* dst, cudaStream_t s);

// dist.cu kernels
void launch_fill_local(const ColMap& cm, const Ownership& ow, double* Zl, long long ld, int Npad, int ncl,
                       const double* D, const double* s_a, const double* G, cudaStream_t s);
void launch_seg_scatter(const ColMap& cm, const Ownership& ow, const double* seg, const unsigned int* ukeys, int nseg,
                        double* Zl, long long ld, cudaStream_t s);
void launch_extract_local(const ColMap& cm, const Ownership& ow, const double* Zl, long long ld, int Npad,
                          const double* s_a, double* cov, Status* st, int* psd_warn, cudaStream_t s);
void launch_pivot_range_local(const ColMap& cm, const Ownership& ow, const double* piv, int Npad, double* out,
                              cudaStream_t s);
void launch_panel_take_at(double* Zc, long long ld, int row0, int W, int rows, double* Lb, cudaStream_t s);
void launch_add(double* y, const double* x, size_t count, cudaStream_t s);
void launch_range_combine(double* out, const double* in, int nranks, cudaStream_t s);
// pair reduction restricted to chunks [c_begin, c_end) into per-segment blocks
void launch_pair_reduce_segments(int P, const PairDev& pd, const double* Wb, int n, int c_begin, int c_end,
                                 double* seg_out, cudaStream_t s);

}  // namespace sfm
