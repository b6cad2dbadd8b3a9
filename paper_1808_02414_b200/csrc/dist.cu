// Distributed (multi-GPU) tail of the pipeline: point-pair-sharded Schur
// assembly and the 1D block-cyclic fused Cholesky / triangular-inverse sweep.
//
// Layout.  The camera matrix uses the camera-aligned column layout (ColMap,
// kernels.cuh): floor(128/P) cameras per 128-block plus identity padding, so
// a camera's columns never straddle a panel.  Panels of G blocks are owned
// cyclically (panel q -> rank q % R); a rank stores the full Npad rows of its
// panels' columns contiguously (Ownership, kernels.cuh).
//
// Sweep step p (the single-GPU dense_sweep of dense.cu, distributed):
//   owner(p)   : u(p-1) on its panel p, potrf / trsm / inner updates, then
//                take(p): L[rows >= b0, panel] and the panel's Linv blocks
//                into ring slot p % NB; its W x W diagonal block := I.
//   all ranks  : broadcast of the slot from owner(p) (ncclBroadcast over
//                NVLink; an in-process copy when ranks are emulated);
//                rest(p): own panels beyond p (beyond p+1 on owner(p+1)) -=
//                L L^T (one column-cyclic GEMM launch); inverse step p on the
//                rank's own columns of panels <= p.
// Each rank then extracts the covariance blocks of the cameras it owns; the
// blocks, PSD warnings, pivot range and Cholesky status are combined with
// one all-reduce each.  Reference: the dense inversion it replaces is
// invert_schur (src/covariance.cpp:196-270).

#include "common.cuh"
#include "detmath.cuh"
#include "kernels.cuh"
#include "dist.h"

#include <cstdio>
#include <cstdlib>

#include <dlfcn.h>

#include <cub/cub.cuh>

#include <cstring>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <string>

namespace sfm {

// ---- kernels ----------------------------------------------------------------------

// Z_local(r, lc) for 64 x 64 tiles of (global row, local column) with the
// global row tile >= the global column tile:
//   [cam(r) == cam(c)] (s_a[r] D(r, c)) s_a[c] + Σ_l G(r, l) G(c, l)  (real r, c)
//   δ(r, c)                                                        (padding)
template <int P>
__global__ void k_fill_local(double* Zl, long long ld, int Npad, int nlt64, ColMap cm, Ownership ow, const double* D,
                             const double* s_a, const double* G) {
    __shared__ double gc[64][8];
    const int ti = blockIdx.x / nlt64, tj = blockIdx.x - ti * nlt64;  // row tile (global), local column tile
    const int lc0 = tj * 64;
    const int gc0 = own_gcol(ow, lc0);  // 64-tiles never straddle a 128-block
    if (ti * 64 + 63 < gc0) return;     // strictly upper tile
    const int tid = threadIdx.x;
    for (int e = tid; e < 64 * 7; e += blockDim.x) {
        const int cc = e / 7, l = e - 7 * (e / 7);
        const int nat = cm_nat(cm, gc0 + cc);
        gc[cc][l] = nat >= 0 ? G[(size_t)nat * 7 + l] : 0.0;
    }
    __syncthreads();
    const int rr = tid & 63;
    const int r = ti * 64 + rr;
    const int nr = cm_nat(cm, r);
    double g[7];
#pragma unroll
    for (int l = 0; l < 7; ++l) g[l] = nr >= 0 ? G[(size_t)nr * 7 + l] : 0.0;
    const double sr = nr >= 0 ? s_a[nr] : 0.0;
    for (int cc = tid >> 6; cc < 64; cc += blockDim.x >> 6) {
        const int c = gc0 + cc;
        const int nc = cm_nat(cm, c);
        double v;
        if (nr >= 0 && nc >= 0) {
            v = 0.0;
            const int ir = nr / P, ic = nc / P;
            if (ir == ic) v = (sr * D[(size_t)P * P * ir + P * (nr - P * ir) + (nc - P * ic)]) * s_a[nc];
            double gg = 0.0;
#pragma unroll
            for (int l = 0; l < 7; ++l) gg += g[l] * gc[cc][l];
            v += gg;
        } else {
            v = (r == c) ? 1.0 : 0.0;
        }
        Zl[(size_t)(lc0 + cc) * ld + r] = v;
    }
}

void launch_fill_local(const ColMap& cm, const Ownership& ow, double* Zl, long long ld, int Npad, int ncl,
                       const double* D, const double* s_a, const double* G, cudaStream_t s) {
    const int nrt = Npad / 64, nlt = ncl / 64;
    if (!nrt || !nlt) return;
    const unsigned blocks = (unsigned)nrt * (unsigned)nlt;
    if (cm.P == 8) k_fill_local<8><<<blocks, 256, 0, s>>>(Zl, ld, Npad, nlt, cm, ow, D, s_a, G);
    else k_fill_local<9><<<blocks, 256, 0, s>>>(Zl, ld, Npad, nlt, cm, ow, D, s_a, G);
    SFM_LAUNCH_CHECK();
}

// Z(cam hi row p, cam lo column q) -= seg(p, q) for the segments whose column
// camera this rank owns (diagonal blocks: lower part).
template <int P>
__global__ void __launch_bounds__(256) k_seg_scatter(const double* seg, const unsigned int* ukeys, int nseg, ColMap cm,
                                                     Ownership ow, double* Zl, long long ld) {
    const int sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (sg >= nseg) return;
    const unsigned int key = ukeys[sg];
    const int lo = (int)(key / (unsigned int)cm.n), hi = (int)(key - (unsigned int)lo * (unsigned int)cm.n);
    const int lc = own_lcol(ow, cm_col(cm, lo, 0));
    if (lc < 0) return;
    const int r0 = cm_col(cm, hi, 0);
    for (int en = lane; en < P * P; en += 32) {
        const int p = en / P, q = en - P * (en / P);
        if (lo == hi && p < q) continue;
        double* z = Zl + (size_t)(lc + q) * ld + r0 + p;
        *z = *z - seg[(size_t)sg * 81 + en];
    }
}

void launch_seg_scatter(const ColMap& cm, const Ownership& ow, const double* seg, const unsigned int* ukeys, int nseg,
                        double* Zl, long long ld, cudaStream_t s) {
    if (!nseg) return;
    if (cm.P == 8) k_seg_scatter<8><<<cdiv(nseg, 8), 256, 0, s>>>(seg, ukeys, nseg, cm, ow, Zl, ld);
    else k_seg_scatter<9><<<cdiv(nseg, 8), 256, 0, s>>>(seg, ukeys, nseg, cm, ow, Zl, ld);
    SFM_LAUNCH_CHECK();
}

// ---- pair blocks to their column owners (reduce-scatter) --------------------------
// owner rank of each segment's block column (the camera lo of key lo n + hi)
__global__ void k_seg_owner(const unsigned int* ukeys, int nseg, ColMap cm, Ownership ow, int* owner, int* cnt) {
    const int sg = blockIdx.x * blockDim.x + threadIdx.x;
    if (sg >= nseg) return;
    const int lo = (int)(ukeys[sg] / (unsigned int)cm.n);
    const int o = ((cm_col(cm, lo, 0) / kNB) / ow.G) % ow.R;
    owner[sg] = o;
    atomicAdd(&cnt[o], 1);  // integer counts: order independent
}
__global__ void k_iota_int(int* v, int count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) v[i] = i;
}
// send[g][k] = seg[perm[off_g + k]] (k < cnt_g), zero padding to Gmax blocks per group
__global__ void k_seg_pack(const double* seg, const int* perm, const int* off, const int* cnt, int R, int gmax,
                           double* send) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)R * gmax * 81) return;
    const long long blk = e / 81;
    const int en = (int)(e - blk * 81);
    const int g = (int)(blk / gmax), k = (int)(blk - (long long)g * gmax);
    send[e] = k < cnt[g] ? seg[(size_t)perm[off[g] + k] * 81 + en] : 0.0;
}
// Z(cam hi row p, cam lo column q) -= grp[k](p, q) for this rank's group
template <int P>
__global__ void __launch_bounds__(256) k_seg_scatter_group(const double* grp, const int* perm, int cnt,
                                                           const unsigned int* ukeys, ColMap cm, Ownership ow,
                                                           double* Zl, long long ld) {
    const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (k >= cnt) return;
    const unsigned int key = ukeys[perm[k]];
    const int lo = (int)(key / (unsigned int)cm.n), hi = (int)(key - (unsigned int)lo * (unsigned int)cm.n);
    const int lc = own_lcol(ow, cm_col(cm, lo, 0));
    if (lc < 0) return;  // (never: the group holds this rank's columns only)
    const int r0 = cm_col(cm, hi, 0);
    for (int en = lane; en < P * P; en += 32) {
        const int p = en / P, q = en - P * (en / P);
        if (lo == hi && p < q) continue;
        double* z = Zl + (size_t)(lc + q) * ld + r0 + p;
        *z = *z - grp[(size_t)k * 81 + en];
    }
}

void SegGroups::plan(const ColMap& cm, const Ownership& ow, const unsigned int* ukeys, int nseg, Workspace& ws,
                     cudaStream_t s) {
    R = ow.R;
    int* owner = buf_owner.as<int>((size_t)nseg + 1);
    int* owner2 = buf_owner2.as<int>((size_t)nseg + 1);
    int* ids = buf_ids.as<int>((size_t)nseg + 1);
    perm = buf_perm.as<int>((size_t)nseg + 1);
    int* dcnt = buf_cnt.as<int>(2 * (size_t)R + 2);
    SFM_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(int) * (size_t)R, s));
    if (nseg) {
        k_seg_owner<<<cdiv(nseg, 256), 256, 0, s>>>(ukeys, nseg, cm, ow, owner, dcnt);
        SFM_LAUNCH_CHECK();
        k_iota_int<<<cdiv(nseg, 256), 256, 0, s>>>(ids, nseg);
        SFM_LAUNCH_CHECK();
        int bits = 1;
        while ((1 << bits) < R) ++bits;
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, owner, owner2, ids, perm, nseg, 0, bits, s);
        SFM_CUDA(cub::DeviceRadixSort::SortPairs(ws.get_tmp(bytes), bytes, owner, owner2, ids, perm, nseg, 0, bits, s));
    }
    cnt.assign(R, 0);
    SFM_CUDA(cudaMemcpyAsync(cnt.data(), dcnt, sizeof(int) * (size_t)R, cudaMemcpyDeviceToHost, s));
    SFM_CUDA(cudaStreamSynchronize(s));
    off.assign(R + 1, 0);
    gmax = 0;
    for (int g = 0; g < R; ++g) {
        off[g + 1] = off[g] + cnt[g];
        gmax = std::max(gmax, cnt[g]);
    }
    gmax = std::max(gmax, 1);
    int* doff = dcnt + R;
    SFM_CUDA(cudaMemcpyAsync(doff, off.data(), sizeof(int) * (size_t)R, cudaMemcpyHostToDevice, s));
    d_off = doff;
    d_cnt = dcnt;
}

void SegGroups::pack(const double* seg, double* send, cudaStream_t s) const {
    const long long tot = (long long)R * gmax * 81;
    k_seg_pack<<<cdiv(tot, 256), 256, 0, s>>>(seg, perm, d_off, d_cnt, R, gmax, send);
    SFM_LAUNCH_CHECK();
}

void SegGroups::scatter(int g, const double* grp, const ColMap& cm, const Ownership& ow, const unsigned int* ukeys,
                        double* Zl, long long ld, cudaStream_t s) const {
    if (!cnt[g]) return;
    if (cm.P == 8)
        k_seg_scatter_group<8><<<cdiv(cnt[g], 8), 256, 0, s>>>(grp, perm + off[g], cnt[g], ukeys, cm, ow, Zl, ld);
    else
        k_seg_scatter_group<9><<<cdiv(cnt[g], 8), 256, 0, s>>>(grp, perm + off[g], cnt[g], ukeys, cm, ow, Zl, ld);
    SFM_LAUNCH_CHECK();
}

// Covariance blocks of the cameras whose columns this rank owns:
// cov_i = s_i (X_i^T X_i) s_i over the rows >= the camera's first column,
// plus the PSD test of k_extract (dense.cu).
template <int P>
__global__ void __launch_bounds__(256) k_extract_local(const double* Zl, long long ld, int Npad, ColMap cm, Ownership ow,
                                                       const double* s_a, double* cov, int* psd_warn) {
    constexpr int U = P * (P + 1) / 2;
    __shared__ double red[8][U];
    const int i = blockIdx.x;
    const int g0 = cm_col(cm, i, 0);
    const int lc = own_lcol(ow, g0);
    if (lc < 0) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.0;
    for (int r = g0 + threadIdx.x; r < Npad; r += 256) {
        double x[P];
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] = (r >= g0 + p) ? __ldcg(Zl + (size_t)(lc + p) * ld + r) : 0.0;
        int u = 0;
#pragma unroll
        for (int p = 0; p < P; ++p)
#pragma unroll
            for (int q = p; q < P; ++q, ++u) acc[u] += x[p] * x[q];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        double v = acc[u];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp][u] = v;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double b[P * P];
    int u = 0;
    for (int p = 0; p < P; ++p)
        for (int q = p; q < P; ++q, ++u) {
            double v = 0.0;
            for (int w = 0; w < 8; ++w) v += red[w][u];
            b[P * p + q] = v;
            b[P * q + p] = v;
        }
    double out[P * P];
    for (int p = 0; p < P; ++p)
        for (int q = 0; q < P; ++q) out[P * p + q] = (s_a[P * i + p] * b[P * p + q]) * s_a[P * i + q];
    double* o = cov + (size_t)P * P * i;
    for (int k = 0; k < P * P; ++k) o[k] = out[k];
    double tr = 0.0;
    for (int p = 0; p < P; ++p) tr += out[P * p + p];
    const double tau = kPsdTol * tr;
    double L[P * P];
    bool pd = true;
    for (int c = 0; c < P && pd; ++c) {
        double sdiag = out[P * c + c] + tau;
        for (int k = 0; k < c; ++k) sdiag -= L[P * c + k] * L[P * c + k];
        if (!(sdiag > 0.0)) { pd = false; break; }
        const double lcc = sqrt(sdiag);
        L[P * c + c] = lcc;
        for (int r = c + 1; r < P; ++r) {
            double x = out[P * r + c];
            for (int k = 0; k < c; ++k) x -= L[P * r + k] * L[P * c + k];
            L[P * r + c] = x / lcc;
        }
    }
    if (!pd) atomicAdd(psd_warn, 1);
}

void launch_extract_local(const ColMap& cm, const Ownership& ow, const double* Zl, long long ld, int Npad,
                          const double* s_a, double* cov, Status* st, int* psd_warn, cudaStream_t s) {
    (void)st;
    if (!cm.n) return;
    if (cm.P == 8) k_extract_local<8><<<cm.n, 256, 0, s>>>(Zl, ld, Npad, cm, ow, s_a, cov, psd_warn);
    else k_extract_local<9><<<cm.n, 256, 0, s>>>(Zl, ld, Npad, cm, ow, s_a, cov, psd_warn);
    SFM_LAUNCH_CHECK();
}

// Pivot range over this rank's real (non-padding) columns: out = {min, max}
// (+inf / 0 when it owns none).
__global__ void k_pivot_range_local(const double* piv, int Npad, ColMap cm, Ownership ow, double* out) {
    __shared__ double mn[256], mx[256];
    double a = INFINITY, b = 0.0;
    for (int i = threadIdx.x; i < Npad; i += 256)
        if (own_lcol(ow, i) >= 0 && cm_nat(cm, i) >= 0) {
            const double v = fabs(piv[i]);
            a = fmin(a, v);
            b = fmax(b, v);
        }
    mn[threadIdx.x] = a;
    mx[threadIdx.x] = b;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            mn[threadIdx.x] = fmin(mn[threadIdx.x], mn[threadIdx.x + w]);
            mx[threadIdx.x] = fmax(mx[threadIdx.x], mx[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) { out[0] = mn[0]; out[1] = mx[0]; }
}

void launch_pivot_range_local(const ColMap& cm, const Ownership& ow, const double* piv, int Npad, double* out,
                              cudaStream_t s) {
    k_pivot_range_local<<<1, 256, 0, s>>>(piv, Npad, cm, ow, out);
    SFM_LAUNCH_CHECK();
}

__global__ void k_range_combine(double* out, const double* in, int nranks) {
    if (threadIdx.x || blockIdx.x) return;
    double a = INFINITY, b = 0.0;
    for (int r = 0; r < nranks; ++r) { a = fmin(a, in[2 * r]); b = fmax(b, in[2 * r + 1]); }
    out[0] = a;
    out[1] = b;
}

void launch_range_combine(double* out, const double* in, int nranks, cudaStream_t s) {
    k_range_combine<<<1, 32, 0, s>>>(out, in, nranks);
    SFM_LAUNCH_CHECK();
}

__global__ void k_add(double* y, const double* x, size_t count) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) y[i] += x[i];
}

void launch_add(double* y, const double* x, size_t count, cudaStream_t s) {
    if (!count) return;
    k_add<<<cdiv((long long)count, 256), 256, 0, s>>>(y, x, count);
    SFM_LAUNCH_CHECK();
}

// Panel hand-over at an explicit column base: Lb(i, j) = Z(row0 + i, col j of
// the panel) for i < rows, and the panel's W x W diagonal block := I.
__global__ void k_panel_take_at(double* Zc, long long ld, int row0, int W, int rows, double* Lb) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int half = rows >> 1;
    if (e >= (long long)half * W) return;
    const int i = (int)(e % half) * 2, j = (int)(e / half);
    double2* zp = reinterpret_cast<double2*>(Zc + (size_t)j * ld + row0 + i);
    const double2 v = __ldcg(zp);
    *reinterpret_cast<double2*>(Lb + (size_t)j * rows + i) = v;
    if (i < W) {
        double2 x;
        x.x = (i == j) ? 1.0 : 0.0;
        x.y = (i + 1 == j) ? 1.0 : 0.0;
        *zp = x;
    }
}

void launch_panel_take_at(double* Zc, long long ld, int row0, int W, int rows, double* Lb, cudaStream_t s) {
    const long long total = (long long)(rows / 2) * W;
    if (!total) return;
    k_panel_take_at<<<cdiv(total, 256), 256, 0, s>>>(Zc, ld, row0, W, rows, Lb);
    SFM_LAUNCH_CHECK();
}

// ---- NCCL (loaded at run time; the library itself does not link it) ----------------
namespace {
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            a.why = "libnccl.so.2 not found";
            return a;
        }
        a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(lib, "ncclGetUniqueId");
        a.CommInitRank = (decltype(a.CommInitRank))dlsym(lib, "ncclCommInitRank");
        a.CommDestroy = (decltype(a.CommDestroy))dlsym(lib, "ncclCommDestroy");
        a.Broadcast = (decltype(a.Broadcast))dlsym(lib, "ncclBroadcast");
        a.AllReduce = (decltype(a.AllReduce))dlsym(lib, "ncclAllReduce");
        a.ReduceScatter = (decltype(a.ReduceScatter))dlsym(lib, "ncclReduceScatter");
        a.GetErrorString = (decltype(a.GetErrorString))dlsym(lib, "ncclGetErrorString");
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Broadcast && a.AllReduce && a.ReduceScatter && a.GetErrorString;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw CudaError(std::string("NCCL ") + what + ": " + nccl_api().GetErrorString(r));
}
}  // namespace

bool nccl_available(std::string* why) {
    NcclApi& a = nccl_api();
    if (!a.ok && why) *why = a.why;
    return a.ok;
}

void nccl_unique_id(void* out128) {
    NcclApi& a = nccl_api();
    if (!a.ok) throw CudaError("NCCL unavailable: " + a.why);
    ncclUniqueId id;
    nccl_check(a.GetUniqueId(&id), "GetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, 128);
}

void* nccl_comm_init(const void* id128, int nranks, int rank) {
    NcclApi& a = nccl_api();
    if (!a.ok) throw CudaError("NCCL unavailable: " + a.why);
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t comm = nullptr;
    nccl_check(a.CommInitRank(&comm, nranks, id, rank), "CommInitRank");
    return comm;
}

void nccl_comm_destroy(void* comm) {
    if (comm && nccl_api().ok) nccl_api().CommDestroy((ncclComm_t)comm);
}

// ---- per-rank state ------------------------------------------------------------------
void RankDense::init(int device) {
    (void)device;
    if (s) return;
    int lo = 0, hi = 0;
    SFM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SFM_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi));
    // the inverse chain (s3) above the trailing updates (s2), as in the
    // single-GPU sweep (capi.cu)
    SFM_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, lo));
    SFM_CUDA(cudaStreamCreateWithPriority(&s3, cudaStreamNonBlocking, (lo + hi) / 2));
    SFM_CUDA(cudaStreamCreateWithPriority(&sc, cudaStreamNonBlocking, hi));
    for (int i = 0; i < NB; ++i)
        for (cudaEvent_t* e : {&eL[i], &eB[i], &eRest[i], &eT[i], &eU[i]})
            SFM_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (cudaEvent_t* e : {&eX2, &eX3, &eXc, &eIn})
        SFM_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

void RankDense::release() {
    Z.release(); Linv.release(); piv.release(); ring.release(); range.release();
    if (!s) return;
    for (cudaStream_t q : {s, s2, s3, sc}) { cudaStreamSynchronize(q); cudaStreamDestroy(q); }
    for (int i = 0; i < NB; ++i)
        for (cudaEvent_t e : {eL[i], eB[i], eRest[i], eT[i], eU[i]}) cudaEventDestroy(e);
    for (cudaEvent_t e : {eX2, eX3, eXc, eIn}) cudaEventDestroy(e);
    s = s2 = s3 = sc = nullptr;
}

void RankDense::setup(const Ownership& o, int Npad_, long long ld_) {
    ow = o;
    Npad = Npad_;
    ld = ld_;
    K = Npad / kNB;
    ncl = own_blocks(ow, K) * kNB;
    zp = Z.as<double>((size_t)ld * (ncl > 0 ? ncl : 1));
    linv = Linv.as<double>((size_t)K * kNB * kNB);
    pv = piv.as<double>((size_t)Npad);
    ringp = ring.as<double>(slot_doubles() * NB);
    rangep = range.as<double>(2);
}

// ---- sweep --------------------------------------------------------------------------
namespace {
int owner_of(const Ownership& o, int p) { return p % o.R; }

void wait_slot_free(RankDense& r, cudaStream_t q, int slot) {
    SFM_CUDA(cudaStreamWaitEvent(q, r.eRest[slot], 0));
    SFM_CUDA(cudaStreamWaitEvent(q, r.eT[slot], 0));
    SFM_CUDA(cudaStreamWaitEvent(q, r.eU[slot], 0));
    SFM_CUDA(cudaStreamWaitEvent(q, r.eB[slot], 0));
}

// owner(p): u(p-1) on panel p, factorisation of panel p, hand-over to the slot
void owner_step(RankDense& r, int p, Status* st) {
    const int K = r.K, G = r.ow.G, R = r.ow.R;
    const long long ld = r.ld;
    const int b0 = p * G, g = std::min(G, K - b0), W = g * kNB;
    double* Zc = r.zp + (size_t)(p / R) * G * kNB * ld;  // first local column of panel p
    const int slot = p % RankDense::NB;
    if (p > 0) {
        const int ps = (p - 1) % RankDense::NB;
        const int pb0 = (p - 1) * G, pW = std::min(G, K - pb0) * kNB, prows = r.Npad - pb0 * kNB;
        const double* Lp = r.slot(p - 1);
        SFM_CUDA(cudaStreamWaitEvent(r.s, r.eB[ps], 0));
        if (p >= 2) SFM_CUDA(cudaStreamWaitEvent(r.s, r.eRest[(p - 2) % RankDense::NB], 0));
        GemmArgs u = gemm_args(Zc + (size_t)b0 * kNB, ld, Lp + pW, prows, Lp + pW, prows, K - b0, g, pW);
        u.alpha_neg = 1; u.beta = 1; u.lower_only = 1;
        launch_gemm(u, r.s);
        SFM_CUDA(cudaEventRecord(r.eU[ps], r.s));
    }
    for (int gg = 0; gg < g; ++gg) {
        const int c = b0 + gg;
        double* Acc = Zc + (size_t)gg * kNB * ld + (size_t)c * kNB;
        launch_potrf_diag(Acc, ld, r.linv + (size_t)c * kNB * kNB, r.pv, c * kNB, st, r.s);
        const int below = K - c - 1;
        if (below == 0) break;
        GemmArgs t = gemm_args(Acc + kNB, ld, Acc + kNB, ld, r.linv + (size_t)c * kNB * kNB, kNB, below, 1, kNB);
        t.whole_tile = 1;  // in place: every output column reads the whole row tile
        launch_gemm(t, r.s);
        const int inner = g - gg - 1;
        if (inner > 0) {
            GemmArgs u = gemm_args(Zc + (size_t)(gg + 1) * kNB * ld + (size_t)(c + 1) * kNB, ld, Acc + kNB, ld,
                                   Acc + kNB, ld, below, inner, kNB);
            u.alpha_neg = 1; u.beta = 1; u.lower_only = 1;
            launch_gemm(u, r.s);
        }
    }
    wait_slot_free(r, r.s, slot);
    const int rows = r.Npad - b0 * kNB;
    double* Lb = r.slot(p);
    launch_panel_take_at(Zc, ld, b0 * kNB, W, rows, Lb, r.s);
    SFM_CUDA(cudaMemcpyAsync(Lb + (size_t)rows * W, r.linv + (size_t)b0 * kNB * kNB, 8 * (size_t)W * kNB,
                             cudaMemcpyDeviceToDevice, r.s));
    SFM_CUDA(cudaEventRecord(r.eL[slot], r.s));
}

// rest(p) and inverse step p on every rank (what = 1: rest only, 2: the
// inverse step only, 3: both)
void update_step(RankDense& r, int p, int what = 3) {
    const int K = r.K, G = r.ow.G, R = r.ow.R, rank = r.ow.rank;
    const long long ld = r.ld;
    const int b0 = p * G, g = std::min(G, K - b0), W = g * kNB, nb0 = b0 + g, T2 = K - nb0;
    const int rows = r.Npad - b0 * kNB;
    const int slot = p % RankDense::NB;
    const double* Lb = r.slot(p);
    const int nlt = r.ncl / kNB;
    // ---- Cholesky trailing update of the rank's panels beyond p (beyond p+1 on owner(p+1))
    const int qmin = (T2 > 0 && owner_of(r.ow, p + 1) == rank) ? p + 2 : p + 1;
    const int lt0 = own_blocks_upto(r.ow, K, qmin - 1);
    if ((what & 1) && T2 > 0 && lt0 < nlt) {
        SFM_CUDA(cudaStreamWaitEvent(r.s2, r.eB[slot], 0));
        const int gt0 = own_gcol(r.ow, lt0 * kNB) / kNB;
        GemmArgs x = gemm_args(r.zp, ld, Lb, rows, Lb, rows, K - gt0, nlt - lt0, W);
        x.cyc_R = R; x.cyc_rank = rank; x.cyc_G = G; x.cyc_lt0 = lt0; x.cyc_row0 = gt0; x.cyc_ab0 = b0;
        x.alpha_neg = 1; x.beta = 1;
        launch_gemm(x, r.s2);
        SFM_CUDA(cudaEventRecord(r.eRest[slot], r.s2));
    }
    // ---- inverse step p on the rank's columns of panels <= p
    const bool own_p = owner_of(r.ow, p) == rank;
    const int before = own_blocks_upto(r.ow, K, p - 1);  // local tiles of own panels < p
    const int ntl = before + (own_p ? g : 0);
    if ((what & 2) && ntl > 0) {
        SFM_CUDA(cudaStreamWaitEvent(r.s3, r.eB[slot], 0));
        const double* Li = Lb + (size_t)rows * W;
        for (int gg = 0; gg < g; ++gg) {
            const int rb = b0 + gg;
            const int cnt = before + (own_p ? gg + 1 : 0);
            if (cnt == 0) continue;
            GemmArgs a = gemm_args(r.zp + (size_t)rb * kNB, ld, Li + (size_t)gg * kNB * kNB, kNB, r.zp + (size_t)rb * kNB,
                                   ld, 1, cnt, kNB);
            a.b_kmajor = 1;
            launch_gemm(a, r.s3);
            const int later = g - gg - 1;
            if (later > 0) {
                GemmArgs u = gemm_args(r.zp + (size_t)(rb + 1) * kNB, ld, Lb + (size_t)gg * kNB * rows + (size_t)(gg + 1) * kNB,
                                       rows, r.zp + (size_t)rb * kNB, ld, later, cnt, kNB);
                u.b_kmajor = 1; u.alpha_neg = 1; u.beta = 1;
                launch_gemm(u, r.s3);
            }
        }
        if (T2 > 0) {
            GemmArgs x = gemm_args(r.zp + (size_t)nb0 * kNB, ld, Lb + W, rows, r.zp + (size_t)b0 * kNB, ld, T2, ntl, W);
            x.b_kmajor = 1; x.alpha_neg = 1; x.beta = 1;
            x.beta0_from = own_p ? before : -1;
            x.k_from_col = own_p ? 1 : 0;  // the panel's own X block is lower triangular
            launch_gemm(x, r.s3);
        }
        SFM_CUDA(cudaEventRecord(r.eT[slot], r.s3));
    }
}

size_t slot_count(const RankDense& r, int p) {
    const int b0 = p * r.ow.G, W = std::min(r.ow.G, r.K - b0) * kNB;
    return (size_t)(r.Npad - b0 * kNB) * W + (size_t)W * kNB;
}
}  // namespace

// SFMCOV_DIST_TRACE=1 (emulated ranks only; diagnostics for the 1D-vs-2D
// model, tools/dist_schedule.py): every component of every step runs alone on
// the device -- the owner's panel factorisation (its columns' update by the
// previous panel, the tile chain, the hand-over), then each rank's trailing
// update and its inverse step -- and its device time is printed to stderr
// with the panel's broadcast bytes, so a schedule of R real GPUs can be
// replayed from measured per-rank work.
static bool dist_trace() {
    static bool v = [] { const char* e = std::getenv("SFMCOV_DIST_TRACE"); return e && e[0] == '1'; }();
    return v;
}
template <class F>
static float timed(cudaStream_t s, F&& launch) {
    cudaEvent_t a, b;
    SFM_CUDA(cudaDeviceSynchronize());
    SFM_CUDA(cudaEventCreate(&a));
    SFM_CUDA(cudaEventCreate(&b));
    SFM_CUDA(cudaEventRecord(a, s));
    launch();
    SFM_CUDA(cudaEventRecord(b, s));
    SFM_CUDA(cudaDeviceSynchronize());
    float ms = 0.f;
    SFM_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

void dist_sweep(DistGroup& grp, Status* const* st) {
    if (grp.ranks.empty()) return;
    const RankDense& r0 = *grp.ranks[0];
    const int K = r0.K, G = r0.ow.G, R = r0.ow.R;
    const int NP = (K + G - 1) / G;
    const bool trace = dist_trace() && !grp.nccl;
    if (trace) std::fprintf(stderr, "dtrace begin R %d K %d G %d NP %d Npad %d\n", R, K, G, NP, r0.Npad);
    for (int p = 0; p < NP; ++p) {
        const int o = p % R;
        const int slot = p % RankDense::NB;
        // (1) owner factorises and hands the panel over
        for (size_t i = 0; i < grp.ranks.size(); ++i)
            if (grp.ranks[i]->ow.rank == o) {
                if (trace) {
                    const float ms = timed(grp.ranks[i]->s, [&] { owner_step(*grp.ranks[i], p, st[i]); });
                    std::fprintf(stderr, "dtrace panel %d owner %d ms %.4f bytes %zu\n", p, o, ms,
                                 8 * slot_count(r0, p));
                } else {
                    owner_step(*grp.ranks[i], p, st[i]);
                }
            }
        // (2) broadcast of the slot from the owner
        const size_t count = slot_count(r0, p);
        if (grp.nccl) {
            RankDense& r = *grp.ranks[0];
            wait_slot_free(r, r.sc, slot);
            if (r.ow.rank == o) SFM_CUDA(cudaStreamWaitEvent(r.sc, r.eL[slot], 0));
            nccl_check(nccl_api().Broadcast(r.slot(p), r.slot(p), count, ncclDouble, o, (ncclComm_t)grp.nccl, r.sc),
                       "Broadcast");
            SFM_CUDA(cudaEventRecord(r.eB[slot], r.sc));
        } else {
            RankDense* root = nullptr;
            for (RankDense* r : grp.ranks)
                if (r->ow.rank == o) root = r;
            for (RankDense* r : grp.ranks) {
                if (r == root) continue;
                wait_slot_free(*r, r->sc, slot);
                SFM_CUDA(cudaStreamWaitEvent(r->sc, root->eL[slot], 0));
                SFM_CUDA(cudaMemcpyAsync(r->slot(p), root->slot(p), 8 * count, cudaMemcpyDeviceToDevice, r->sc));
                SFM_CUDA(cudaEventRecord(r->eB[slot], r->sc));
            }
            // the root's slot is busy until every copy has been taken
            SFM_CUDA(cudaStreamWaitEvent(root->sc, root->eL[slot], 0));
            for (RankDense* r : grp.ranks)
                if (r != root) SFM_CUDA(cudaStreamWaitEvent(root->sc, r->eB[slot], 0));
            SFM_CUDA(cudaEventRecord(root->eB[slot], root->sc));
        }
        // (3) trailing update and inverse step on every rank
        for (RankDense* r : grp.ranks) {
            if (trace) {
                const float u = timed(r->s2, [&] { update_step(*r, p, 1); });
                const float v = timed(r->s3, [&] { update_step(*r, p, 2); });
                std::fprintf(stderr, "dtrace update %d rank %d rest %.4f inv %.4f\n", p, r->ow.rank, u, v);
            } else {
                update_step(*r, p);
            }
        }
    }
    for (RankDense* r : grp.ranks) {
        SFM_CUDA(cudaEventRecord(r->eX2, r->s2));
        SFM_CUDA(cudaEventRecord(r->eX3, r->s3));
        SFM_CUDA(cudaEventRecord(r->eXc, r->sc));
        SFM_CUDA(cudaStreamWaitEvent(r->s, r->eX2, 0));
        SFM_CUDA(cudaStreamWaitEvent(r->s, r->eX3, 0));
        SFM_CUDA(cudaStreamWaitEvent(r->s, r->eXc, 0));
    }
}

void dist_allreduce(DistGroup& grp, double* buf, size_t count, int op, cudaStream_t s) {
    if (!grp.nccl || !count) return;
    const ncclRedOp_t o = op == 0 ? ncclSum : (op == 1 ? ncclMin : ncclMax);
    nccl_check(nccl_api().AllReduce(buf, buf, count, ncclDouble, o, (ncclComm_t)grp.nccl, s), "AllReduce");
}

void dist_reduce_scatter(DistGroup& grp, const double* send, double* recv, size_t count, cudaStream_t s) {
    if (!grp.nccl || !count) return;
    nccl_check(nccl_api().ReduceScatter(send, recv, count, ncclDouble, ncclSum, (ncclComm_t)grp.nccl, s),
               "ReduceScatter");
}

void dist_allreduce_ints(DistGroup& grp, int* buf, size_t count, int op, cudaStream_t s) {
    if (!grp.nccl || !count) return;
    const ncclRedOp_t o = op == 0 ? ncclSum : (op == 1 ? ncclMin : ncclMax);
    nccl_check(nccl_api().AllReduce(buf, buf, count, ncclInt32, o, (ncclComm_t)grp.nccl, s), "AllReduce");
}

void dist_allreduce_u8_max(DistGroup& grp, unsigned char* buf, size_t count, cudaStream_t s) {
    if (!grp.nccl || !count) return;
    nccl_check(nccl_api().AllReduce(buf, buf, count, ncclUint8, ncclMax, (ncclComm_t)grp.nccl, s), "AllReduce");
}

void dist_allreduce_int_min(DistGroup& grp, int* buf, cudaStream_t s) {
    if (!grp.nccl) return;
    nccl_check(nccl_api().AllReduce(buf, buf, 1, ncclInt32, ncclMin, (ncclComm_t)grp.nccl, s), "AllReduce");
}

void dist_allreduce_int_sum(DistGroup& grp, int* buf, cudaStream_t s) {
    if (!grp.nccl) return;
    nccl_check(nccl_api().AllReduce(buf, buf, 1, ncclInt32, ncclSum, (ncclComm_t)grp.nccl, s), "AllReduce");
}

}  // namespace sfm
