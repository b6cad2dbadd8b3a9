// Point-sharded stage A of the multi-GPU pipeline (north_star: "the Schur
// assembly is partitioned by points"): the kernels that cut a rank's
// sub-scene out of the resident scene and that map its camera-pair blocks
// into the global block index the owners' reduce-scatter uses.
//
// A rank owns a contiguous range of points [j0, j1), balanced by their
// observation-pair counts Σ k(k+1)/2.  Its sub-scene keeps every camera, its
// points and exactly their observations (in observation order), so the
// single-GPU stage-A kernels run on it unchanged: every per-point quantity
// (A_j, the 3x3 factors, W_a, V_j) and every observation pair is local; the
// per-camera sums (D, the rotation normal equations, Σ W V) and the gauge
// terms (the border column norms, F = Σ V^T V) are partial and are
// all-reduced (capi.cu run_dist_sharded).  Reference: the stages it shards
// are src/projection.cpp:80-105, src/nullspace.cpp:33-62 and
// src/covariance.cpp:33-194.
#include "common.cuh"
#include "kernels.cuh"

#include <cub/cub.cuh>

#include <vector>

namespace sfm {

namespace {

// first point index j with pair_off[j] >= target (pair_off: m + 1 exclusive
// prefix of the per-point pair counts)
__global__ void k_shard_bounds(const long long* pair_off, int m, int R, int* bounds) {
    const int r = threadIdx.x;
    if (r > R) return;
    if (r == 0) { bounds[0] = 0; return; }
    if (r == R) { bounds[R] = m; return; }
    const long long total = pair_off[m];
    const long long target = total * r / R;
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pair_off[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    bounds[r] = lo;
}

__global__ void k_shard_flags(const int* op, int t, int j0, int j1, unsigned char* flag) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < t) flag[k] = (op[k] >= j0 && op[k] < j1) ? 1 : 0;
}

__global__ void k_shard_iota(int* v, int t) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < t) v[k] = k;
}

__global__ void k_shard_gather(const int* lt, int tr, const int* oc, const int* op, int j0, const double* sigma,
                               int* oc_r, int* op_r, double* sigma_r) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= tr) return;
    const int t = lt[k];
    oc_r[k] = oc[t];
    op_r[k] = op[t] - j0;
    if (sigma)
        for (int e = 0; e < 4; ++e) sigma_r[4 * (size_t)k + e] = sigma[4 * (size_t)t + e];
}

// local segment -> its global index (binary search of the key); the block is
// added into the rank's zeroed global-index buffer (one local segment per
// global index, so no two threads touch the same block)
__global__ void k_seg_map(const unsigned int* ukeys_l, int nseg_l, const unsigned int* ukeys_g, int nseg_g,
                          const double* seg_l, double* seg_g) {
    const int sgl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (sgl >= nseg_l) return;
    const unsigned int key = ukeys_l[sgl];
    int lo = 0, hi = nseg_g;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ukeys_g[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    for (int e = lane; e < 81; e += 32) seg_g[(size_t)lo * 81 + e] += seg_l[(size_t)sgl * 81 + e];
}

__global__ void k_flags_or(const unsigned char* src, size_t count, unsigned char* dst) {
    const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < count && src[k]) dst[k] = 1;
}

}  // namespace

void shard_bounds(const long long* pair_off, int m, int R, int* d_bounds, std::vector<int>& bounds, cudaStream_t s) {
    k_shard_bounds<<<1, 128, 0, s>>>(pair_off, m, R, d_bounds);
    SFM_LAUNCH_CHECK();
    bounds.resize(R + 1);
    SFM_CUDA(cudaMemcpyAsync(bounds.data(), d_bounds, sizeof(int) * (R + 1), cudaMemcpyDeviceToHost, s));
    SFM_CUDA(cudaStreamSynchronize(s));
}

int shard_extract(const SceneDev& g, int j0, int j1, ShardScene& out, cudaStream_t s) {
    const int t = g.t;
    unsigned char* flag = out.buf_flag.as<unsigned char>((size_t)t + 1);
    int* iota = out.buf_iota.as<int>((size_t)t + 1);
    int* lt = out.buf_lt.as<int>((size_t)t + 1);
    int* cnt = out.buf_cnt.as<int>(2);
    if (t) {
        k_shard_flags<<<cdiv(t, 256), 256, 0, s>>>(g.op, t, j0, j1, flag);
        SFM_LAUNCH_CHECK();
        k_shard_iota<<<cdiv(t, 256), 256, 0, s>>>(iota, t);
        SFM_LAUNCH_CHECK();
        size_t bytes = 0;
        cub::DeviceSelect::Flagged(nullptr, bytes, iota, flag, lt, cnt, t, s);
        SFM_CUDA(cub::DeviceSelect::Flagged(out.ws.get_tmp(bytes), bytes, iota, flag, lt, cnt, t, s));
    } else {
        SFM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), s));
    }
    int tr = 0;
    SFM_CUDA(cudaMemcpyAsync(&tr, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    SFM_CUDA(cudaStreamSynchronize(s));
    int* oc_r = out.buf_oc.as<int>((size_t)tr + 1);
    int* op_r = out.buf_op.as<int>((size_t)tr + 1);
    double* sig_r = g.sigma ? out.buf_sigma.as<double>(4 * (size_t)tr + 1) : nullptr;
    if (tr) {
        k_shard_gather<<<cdiv(tr, 256), 256, 0, s>>>(lt, tr, g.oc, g.op, j0, g.sigma, oc_r, op_r, sig_r);
        SFM_LAUNCH_CHECK();
    }
    SceneDev& l = out.sc;
    l = SceneDev{};
    l.n = g.n;
    l.m = j1 - j0;
    l.t = tr;
    l.P = g.P;
    l.cams = g.cams;
    l.pts = g.pts + 3 * (size_t)j0;
    l.oc = oc_r;
    l.op = op_r;
    l.u = nullptr;
    l.sigma = sig_r;
    out.lt = lt;
    out.j0 = j0;
    out.j1 = j1;
    return tr;
}

void launch_seg_map(const unsigned int* ukeys_l, int nseg_l, const unsigned int* ukeys_g, int nseg_g,
                    const double* seg_l, double* seg_g, cudaStream_t s) {
    if (!nseg_l) return;
    k_seg_map<<<cdiv(nseg_l, 8), 256, 0, s>>>(ukeys_l, nseg_l, ukeys_g, nseg_g, seg_l, seg_g);
    SFM_LAUNCH_CHECK();
}

void launch_flags_or(const unsigned char* src, size_t count, unsigned char* dst, cudaStream_t s) {
    if (!count) return;
    k_flags_or<<<cdiv((long long)count, 256), 256, 0, s>>>(src, count, dst);
    SFM_LAUNCH_CHECK();
}

}  // namespace sfm
