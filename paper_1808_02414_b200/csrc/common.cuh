// Shared host/device definitions for the sfmcov_b200 CUDA library.
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace sfm {

// Per-observation record (AoS, 288 B): [jc 2xP | jp 2x3 | W 2x2 | pad | tg 2x3 | pad],
// tg = the rotation-rhs factors -(d_C [C]x + d_X [X]x) (nullspace.cpp:40-50),
// stored at the observation's by-camera slot (pos_cam), so a camera's
// records are contiguous and the per-camera reductions stream them.
constexpr int kRec = 36;
template <int P> struct Layout {
    static constexpr int JC = 0;
    static constexpr int JP = 2 * P;
    static constexpr int WO = 2 * P + 6;
    static constexpr int TG = 28;
};
// Per-observation Schur factor W_a = C_s,a L_j^-T (P x 3 row-major), stride 28.
constexpr int kWStride = 28;

// Asynchronous 16-byte global -> shared copies (L2 only, no L1 allocation).
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Dense panel width of the blocked Cholesky / triangular inverse.
constexpr int kNB = 128;

// Device-side failure record; every field is "first offending index"
// (INT_MAX / LLONG_MAX = none) so reductions are order independent.
struct Status {
    int cam_bad;        // i*4 + code (1 non-finite, 2 focal <= 0)
    int pt_bad;         // j
    long long obs_bad;  // t*8 + code (1 cam range, 2 pt range, 3 non-finite, 4 asym, 5 not SPD)
    int dup;            // any duplicate (camera, point) pair (0/1)
    int cam_count_bad;  // i with < 4 observations
    int pt_count_bad;   // j with < 2 observations
    int jac_bad;        // t behind the camera
    int fisher_bad;     // t with non-SPD sigma (fisher stage)
    int rot_bad;        // camera with rank-deficient rotation system
    int pt_sing_bad;    // point with singular 3x3 block
    int border_bad;     // 1 if the 7x7 border block is not negative definite
    int chol_bad;       // first non-positive Cholesky pivot (global column)
    int nflag;          // flagged conditioning columns
    int pad;
};

inline Status status_init() {
    Status s;
    s.cam_bad = INT_MAX; s.pt_bad = INT_MAX; s.obs_bad = LLONG_MAX; s.dup = 0;
    s.cam_count_bad = INT_MAX; s.pt_count_bad = INT_MAX; s.jac_bad = INT_MAX; s.fisher_bad = INT_MAX;
    s.rot_bad = INT_MAX; s.pt_sing_bad = INT_MAX; s.border_bad = 0; s.chol_bad = INT_MAX; s.nflag = 0; s.pad = 0;
    return s;
}

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// A size limit of a device data structure (reported as SFMCOV_ERR_SIZE_GUARD).
struct SizeGuard : std::runtime_error {
    std::string stage;
    SizeGuard(std::string st, const std::string& what) : std::runtime_error(what), stage(std::move(st)) {}
};

#define SFM_CUDA(x)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            throw ::sfm::CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " + \
                                   __FILE__ + ":" + std::to_string(__LINE__));                   \
    } while (0)

// Every kernel launch of this library is followed by SFM_LAUNCH_CHECK(),
// which also counts it (sfmcov_cuda_last_counts reports the total).
extern thread_local long long g_kernel_launches;
#define SFM_LAUNCH_CHECK()                  \
    do {                                    \
        ++::sfm::g_kernel_launches;         \
        SFM_CUDA(cudaGetLastError());       \
    } while (0)

inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

}  // namespace sfm
