// Host-side launchers and device data descriptors of the sfmcov_b200 pipeline.
#pragma once

#include "common.cuh"

#include <cuda_runtime.h>

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
        buf_part;
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
    double* part = nullptr;    // per-chunk partial blocks of multi-chunk segments
    void release() {
        buf_cnt.release(); buf_off.release(); buf_k0.release(); buf_k1.release(); buf_v0.release();
        buf_v1.release(); buf_ukeys.release(); buf_counts.release(); buf_nruns.release(); buf_seg.release();
        buf_chunk.release(); buf_part.release();
    }
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
};

// stage_a.cu
void launch_status_init(Status* st, cudaStream_t s);
void launch_validate(const SceneDev& sc, int check_sigma, Status* st, int* cam_cnt, int* pt_cnt, cudaStream_t s);
void launch_build_index(const SceneDev& sc, const int* cam_cnt, const int* pt_cnt, IndexDev& ix, Workspace& ws,
                        cudaStream_t s);
void launch_structure_check(const SceneDev& sc, const IndexDev& ix, Status* st, cudaStream_t s);
void launch_jacobian(const SceneDev& sc, double* R, double* rec, Status* st, cudaStream_t s);
void launch_depth_of(const SceneDev& sc, const double* R, int t, double* out, cudaStream_t s);
void launch_reductions(const SceneDev& sc, const IndexDev& ix, const double* rec, double* D, double* Hr, double* A,
                       double* s_a, unsigned char* flags, Status* st, cudaStream_t s);
void launch_border_scales(const SceneDev& sc, const double* Hr, const double* s_a, double* partial, double* s_b,
                          cudaStream_t s);
int border_partial_blocks(int n, int m);
void launch_write_h(const SceneDev& sc, const double* Hr, double* H, cudaStream_t s);

// schur.cu
int point_prep_blocks(int m);
void launch_point_prep(const SceneDev& sc, const IndexDev& ix, const double* rec, const double* A, const double* s_a,
                       const double* s_b, double* Lpt, double* Wb, double* V, double* Fpart, Status* st, cudaStream_t s);
void launch_border_factor(const double* Fpart, int nblocks, double* LF, double* E, double* eigE, Status* st,
                          cudaStream_t s);
void launch_camera_border(const SceneDev& sc, const IndexDev& ix, const double* Wb, const double* V, const double* Hr,
                          const double* s_a, const double* s_b, const double* LF, double* Gamma, double* G,
                          cudaStream_t s);
void launch_fill(int P, double* Z, long long ld, int N, int Npad, const double* D, const double* s_a, const double* G,
                 int add_gg, cudaStream_t s);
void build_pairs(const SceneDev& sc, const IndexDev& ix, PairDev& pd, Workspace& ws, cudaStream_t s);
void launch_pair_reduce(int P, const PairDev& pd, const double* Wb, int n, double* Z, long long ld, cudaStream_t s);

// dense.cu
void dense_init_attributes();
void launch_gemm(const GemmArgs& g, cudaStream_t s);
void launch_potrf_diag(double* A, long long ld, double* Linv, double* pivots, int col0, Status* st, cudaStream_t s);
void launch_copy_diag(double* X, long long ld, int k, const double* Linv, cudaStream_t s);
void launch_copy_panel(const double* X, long long ld, int k, int rows, double* Lp, cudaStream_t s);
void launch_copy_panel_w(const double* X, long long ld, int b0, int G, int rows, double* Lp, cudaStream_t s);
void launch_extract(int P, const double* X, long long ld, int N, int nblocks, const double* s_a, int scale, double* cov,
                    Status* st, int* psd_warn, cudaStream_t s);
void launch_set_diag(double* Z, long long ld, int from, int to, cudaStream_t s);
void launch_pivot_range(const double* piv, int N, double* out, cudaStream_t s);
int dense_cholesky(double* Z, long long ld, int Npad, int G, double* Linv, double* pivots, Status* st, cudaStream_t s,
                   cudaStream_t s2, cudaEvent_t e1, cudaEvent_t e2);
int dense_trtri(double* X, long long ld, int Npad, int G, const double* Linv, double* Lp, cudaStream_t s,
                cudaStream_t s2, cudaEvent_t e1, cudaEvent_t e2);
// Lp workspace (doubles) dense_trtri needs for panel width G.
int dense_sweep(double* Z, long long ld, int Npad, int G, double* Linv, double* pivots, Status* st, double* ring,
                int NB, cudaStream_t s, cudaStream_t s2, cudaStream_t s3, cudaEvent_t* eL, cudaEvent_t* eT,
                cudaEvent_t eR);
inline size_t sweep_ring_doubles(int Npad, int G, int NB) { return (size_t)NB * Npad * G * kNB; }
inline size_t trtri_lp_doubles(int Npad, int G) { return (size_t)Npad * kNB * G + (size_t)kNB * kNB * G; }

}  // namespace sfm
