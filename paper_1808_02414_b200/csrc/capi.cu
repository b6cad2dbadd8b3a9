// C ABI and pipeline orchestration of the B200 covariance hot path.
//
// Pipeline (reference: compute_covariance, src/covariance.cpp:323-350):
//   validate + observation index          src/scene.cpp:19-90
//   Jacobian                              src/projection.cpp:80-105
//   gauge nullspace rotation blocks       src/nullspace.cpp:33-62
//   Fisher blocks + conditioning scales   src/covariance.cpp:33-135
//   point elimination (Schur) + border    src/covariance.cpp:137-194
//   gauge-fixed inversion + extraction    src/covariance.cpp:196-279
// Everything runs on the handle's device; the host only moves the scene in
// and the per-camera blocks out, and turns device status words into the
// reference's Error(kind, stage, message).
#include "sfmcov_b200.h"

#include "common.cuh"
#include "kernels.cuh"
#include "dist.h"

#include <algorithm>
#include <chrono>
#include <climits>
#include <limits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <future>
#include <thread>
#include <unistd.h>
#include <vector>

namespace sfm {
thread_local long long g_kernel_launches = 0;  // per calling thread: worker handles run concurrently
}

namespace {

using namespace sfm;

struct ApiError {
    int kind;
    std::string stage;
    std::string message;
};

enum Stage { ST_INDEX, ST_JACOBIAN, ST_REDUCE, ST_SCHUR_PREP, ST_PAIRS, ST_FILL, ST_PAIR_REDUCE, ST_CHOLESKY,
             ST_TRTRI, ST_EXTRACT, ST_COUNT };
const char* kStageNames[ST_COUNT] = {"validate_index", "jacobian", "camera_point_reduce", "schur_point_prep",
                                     "pair_sort", "dense_fill", "schur_pair_reduce", "cholesky", "trtri",
                                     "extract"};

enum Mode { M_INDEX, M_JACOBIAN, M_NULLSPACE, M_FISHER, M_SCHUR, M_FULL };

}  // namespace

// One rank's point-sharded stage A (run_dist_sharded): its sub-scene and
// the stage-A buffers over it.
struct RankA {
    sfm::ShardScene sh;
    sfm::DBuf off_cam, idx_cam, off_pt, idx_pt, pos_cam, key_scratch;
    sfm::DBuf R, rec, D, Hr, A, s_a, flags, raw, bpart, sq, Lpt, Wb, V, Fpart, Pfirst, Plast, Gsum, F28, S, seg_l, seg_g,
        status;
    sfm::Workspace ws, ws_pairs;
    sfm::PairDev pairs;
    sfm::IndexDev ix{};
    void release() {
        sh.release();
        for (sfm::DBuf* b : {&off_cam, &idx_cam, &off_pt, &idx_pt, &pos_cam, &key_scratch, &R, &rec, &D, &Hr, &A, &s_a,
                             &flags, &raw, &bpart, &sq, &Lpt, &Wb, &V, &Fpart, &Pfirst, &Plast, &Gsum, &F28, &S,
                             &seg_l, &seg_g, &status})
            b->release();
        ws.tmp.release();
        ws_pairs.tmp.release();
        pairs.release();
    }
};

struct sfmcov_handle {
    int device = 0;
    cudaStream_t s = nullptr, s2 = nullptr, s3 = nullptr, s4 = nullptr;
    cudaStream_t sx[3] = {nullptr, nullptr, nullptr};  // extra inverse streams (column-interleaved shares of X)
    cudaStream_t sp = nullptr;  // the pair-list build (high priority: ready before stage A ends)
    cudaEvent_t eX = nullptr, eN = nullptr;
    cudaEvent_t e_index = nullptr, e_pairs = nullptr;  // pair-list build on s2, overlapped with stage A
    cudaEvent_t e_ids = nullptr, e_sigma = nullptr;    // host API: σ uploads on s3 after the indices
    cudaEvent_t e_red_fork = nullptr, e_red_join = nullptr;  // point reduction on s4 beside the camera one
    cudaEvent_t e_fill = nullptr, e_zrest = nullptr;          // pair reduction of the later block columns on s2
    cudaEvent_t e_pr0 = nullptr, e_pr1 = nullptr;             // its duration (profiling)
    cudaEvent_t e1 = nullptr, e2 = nullptr;
    static constexpr int kRing = 4;  // panel ring buffers of the fused sweep
    cudaEvent_t eL[kRing], eT[kRing], eTx[3][kRing];
    cudaEvent_t ev[ST_COUNT + 1];
    bool profiling = false;
    // one caller at a time; recursive so that a multi-call session (the
    // sub-reconstruction pipeline, sfmcov_internal_session) can hold it
    // across its own calls while other threads wait
    std::recursive_mutex mu;
    Workspace ws, ws_pairs;
    // host-API staging of the scene
    DBuf h_cams, h_pts, h_oc, h_op, h_sigma;
    // index
    DBuf off_cam, idx_cam, off_pt, idx_pt, pos_cam, key_scratch;
    // stage buffers
    DBuf R, rec, D, Hr, A, s_a, flags, bpart, s_b, Lpt, Wb, V, Fpart, Pfirst, Plast, Gsum, LF, E, eigE, Gamma, G, Z, Linv, ring, piv, cov,
        psd, prange, status, depth, H;
    PairDev pairs;
    Status* st_host = nullptr;
    // distributed tail: 0 = single device, 1 = emulated ranks, 2 = NCCL rank
    int dist_mode = 0, dist_R = 1, dist_rank = 0, emu_R = 1;
    // Multi-GPU stage A: replicated on every rank (default: the single-GPU
    // summation order, so the sharded pipeline stays within the parity bar) or
    // point-sharded (sfmcov_cuda_set_sharded_stage_a / SFMCOV_SHARDED_STAGE_A=1)
    bool replicated_a = true;
    void* nccl = nullptr;
    std::vector<sfm::RankDense> ranks;
    std::vector<RankA> ranka;
    DBuf sh_bounds, sh_raw, sh_sq, sh_F, sh_S, sh_seg, sh_err;
    // batched sub-scenes (run_batch)
    DBuf bt_lists, bt_cams, bt_pts, bt_oc, bt_op, bt_sigma, bt_sofc, bt_sofp, bt_sb, bt_F, bt_LF, bt_E, bt_eigE, bt_Zb,
        bt_piv, bt_cov, bt_bad, bt_nreal, bt_linv, bt_ring;
    DBuf seg, seg_tmp, seg_send, seg_recv, prange_r, scale_mm;
    sfm::SegGroups seg_groups;
    DBuf zi, fc_part, fc_y, fc_gtt, fc_eb, fc_pc;
    DBuf or_a, or_w, or_work, or_vs, or_vk, or_s, or_keep;
    DBuf ref_c, ref_ws;  // refinement (verification) scratch
    DBuf sys[14];        // stage functions on caller-supplied systems (system.cu, eigen.cu)
    cudaEvent_t ev_ready = nullptr, ev_rank_done[64];
    bool ev_rank_init = false;
    // worker handles for batched independent problems (sub-reconstructions),
    // owned by this handle so their streams and workspaces persist
    std::vector<sfmcov_handle*> workers;
    // the batched sub-scene API in steps (begin, then chunks): the resident
    // full scene, and grow-only pinned host buffers for the chunks' id lists
    SceneDev bt_full{};
    bool bt_full_valid = false;
    // the host scene last copied into h_cams / h_pts / h_oc / h_op / h_sigma
    // (batch_begin reuses that copy when it is the same scene)
    sfmcov_scene last_up{};
    bool last_up_valid = false;
    void* pinned[2] = {nullptr, nullptr};
    size_t pinned_bytes[2] = {0, 0};
    double stage_ms[ST_COUNT] = {0};
    long long counts[10] = {0};
};

namespace {

void fill_error(sfmcov_error* e, const ApiError& x) {
    if (!e) return;
    e->kind = x.kind;
    std::snprintf(e->stage, sizeof e->stage, "%s", x.stage.c_str());
    std::snprintf(e->message, sizeof e->message, "%s: %s", x.stage.c_str(), x.message.c_str());
}

void clear_error(sfmcov_error* e) {
    if (!e) return;
    e->kind = 0;
    e->stage[0] = 0;
    e->message[0] = 0;
}

std::string fmt_f(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%f", v);
    return buf;
}

struct Outputs {
    // device
    double* d_cam_cov = nullptr;
    // host (stage APIs)
    double* jc = nullptr;
    double* jp = nullptr;
    double* H = nullptr;
    double* D = nullptr;
    double* A = nullptr;
    double* Cp = nullptr;
    double* s_a = nullptr;
    double* s_b = nullptr;
    double* z_p = nullptr;
    // optional outputs (host), CovarianceOptions::point_covariances / camera_cross_covariances
    double* h_point_cov = nullptr;
    double* h_camera_matrix = nullptr;
    int64_t* off_cam = nullptr;
    int32_t* idx_cam = nullptr;
    int64_t* off_pt = nullptr;
    int32_t* idx_pt = nullptr;
    sfmcov_diagnostics* diag = nullptr;
};

// Device -> host copy ordered after the handle's stream.  (A plain
// cudaMemcpy runs on the legacy default stream, which does not wait for the
// handle's non-blocking streams.)
void d2h(sfmcov_handle* h, void* dst, const void* src, size_t bytes) {
    SFM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->s));
    SFM_CUDA(cudaStreamSynchronize(h->s));
}

void sync_status(sfmcov_handle* h) {
    SFM_CUDA(cudaMemcpyAsync(h->st_host, h->status.p, sizeof(Status), cudaMemcpyDeviceToHost, h->s));
    SFM_CUDA(cudaStreamSynchronize(h->s));
}

void throw_validation(sfmcov_handle* h, const SceneDev& sc, bool full) {
    const Status& st = *h->st_host;
    if (full && st.cam_bad != INT_MAX) {
        const int i = st.cam_bad / 4, code = st.cam_bad % 4;
        throw ApiError{SFMCOV_ERR_INVARIANT, "validate",
                       "camera " + std::to_string(i) + (code == 1 ? " has non-finite parameters" : " has non-positive focal length")};
    }
    if (full && st.pt_bad != INT_MAX)
        throw ApiError{SFMCOV_ERR_INVARIANT, "validate", "point " + std::to_string(st.pt_bad) + " has non-finite coordinates"};
    if (st.obs_bad != LLONG_MAX) {
        const long long t = st.obs_bad / 8;
        const int code = (int)(st.obs_bad % 8);
        static const char* msg[] = {"", " camera index out of range", " point index out of range", " has non-finite values",
                                    " covariance not symmetric", " covariance not positive definite"};
        throw ApiError{SFMCOV_ERR_INVARIANT, "validate", "observation " + std::to_string(t) + msg[code]};
    }
    if (full && st.dup) throw ApiError{SFMCOV_ERR_INVARIANT, "validate", "duplicate (camera, point) observation pair"};
    (void)sc;
}

void throw_counts(sfmcov_handle* h) {
    const Status& st = *h->st_host;
    if (st.cam_count_bad != INT_MAX) {
        int c = 0;
        const int i = st.cam_count_bad;
        int o[2];
        d2h(h, o, (int*)h->off_cam.p + i, 2 * sizeof(int));
        c = o[1] - o[0];
        throw ApiError{SFMCOV_ERR_INVARIANT, "validate",
                       "camera " + std::to_string(i) + " observes " + std::to_string(c) + " points, need at least 4"};
    }
    if (st.pt_count_bad != INT_MAX) {
        const int j = st.pt_count_bad;
        int o[2];
        d2h(h, o, (int*)h->off_pt.p + j, 2 * sizeof(int));
        throw ApiError{SFMCOV_ERR_INVARIANT, "validate",
                       "point " + std::to_string(j) + " is observed by " + std::to_string(o[1] - o[0]) +
                           " cameras, need at least 2"};
    }
}

void throw_numeric(sfmcov_handle* h, const SceneDev& sc, Mode mode) {
    const Status& st = *h->st_host;
    if (st.jac_bad != INT_MAX) {
        double d = 0.0;
        launch_depth_of(sc, (const double*)h->R.p, st.jac_bad, (double*)h->depth.get(8), h->s);
        SFM_CUDA(cudaMemcpyAsync(&d, h->depth.p, 8, cudaMemcpyDeviceToHost, h->s));
        SFM_CUDA(cudaStreamSynchronize(h->s));
        throw ApiError{SFMCOV_ERR_DEGENERATE, "jacobian",
                       "observation " + std::to_string(st.jac_bad) + ": projection: point at camera-space depth " +
                           fmt_f(d) + " (behind camera or on the principal plane)"};
    }
    if (mode == M_JACOBIAN) return;
    if (st.rot_bad != INT_MAX)
        throw ApiError{SFMCOV_ERR_DEGENERATE, "nullspace",
                       "camera " + std::to_string(st.rot_bad) + " has a rank-deficient rotation system"};
    if (mode == M_NULLSPACE) return;
    if (st.fisher_bad != INT_MAX)
        throw ApiError{SFMCOV_ERR_DEGENERATE, "fisher",
                       "observation " + std::to_string(st.fisher_bad) + " covariance is not positive definite"};
    if (mode == M_FISHER) return;
    if (st.pt_sing_bad != INT_MAX)
        throw ApiError{SFMCOV_ERR_DEGENERATE, "schur", "point " + std::to_string(st.pt_sing_bad) + " has a singular 3x3 block"};
    if (mode == M_SCHUR) return;
    if (st.border_bad)
        throw ApiError{SFMCOV_ERR_DEGENERATE, "factorization",
                       "gauge border block is not negative definite; the scene is likely disconnected or its gauge degenerate"};
    if (st.chol_bad != INT_MAX)
        throw ApiError{SFMCOV_ERR_DEGENERATE, "factorization",
                       "non-positive pivot at index " + std::to_string(st.chol_bad) +
                           "; the scene is likely disconnected or its gauge degenerate"};
}

// Dense panel width in kNB blocks for K = Npad / kNB tiles over R ranks.
// Wider panels mean longer K in the trailing updates (better DMMA efficiency,
// fewer passes over the trailing matrix) but a longer per-panel critical
// chain; measured best (1 B200, round 1): K = 71 (config 3): 3 (4: +0.7 %);
// K = 211 (config 4): 8-12 (408 -> 397 ms vs 3); K = 704 (config 5): 16
// (14.83 -> 14.24 s vs 3).  Hence K / (24 R) clamped to [3, 16] on R > 1
// ranks (the distributed sweep keeps >= 24 panels per rank for its
// block-cyclic balance); one GPU: at least 4 from K = 60 on (below).
// SFMCOV_PANEL overrides.
int panel_blocks(int K, int R) {
    static int forced = [] {
        const char* e = std::getenv("SFMCOV_PANEL");
        const int v = e ? std::atoi(e) : 0;
        return (v >= 1 && v <= 16) ? v : 0;
    }();
    if (forced) return forced;
    // one GPU, with the tile kernel's early launch (round 2): the chain costs
    // less, so 4 blocks win at config 3 (K = 71: 16.75 -> 16.67 ms).  Config 4
    // (K = 211) would gain 0.3-0.5 % from 10-12 against 8, but the error of its
    // worst-conditioned camera against the exact inverse scatters with the
    // rounding order (widths 3 / 4 / 6 / 8 / 10 / 12 / 16: 6.8e-10, 9.6e-10,
    // 1.16e-9, 2.5e-10, 2.4e-10, 8.1e-10, 5.3e-10; median block 2-4e-12), so
    // the width that is verified on every camera (8, K / 24) stays.
    int g = K / (24 * (R > 0 ? R : 1));
    if (R <= 1 && K >= 60 && g < 4) g = 4;
    return g < 3 ? 3 : (g > 16 ? 16 : g);
}

// SFMCOV_SERIAL_DENSE=1 runs the lookahead updates on the main stream
// (debug aid: removes the two-stream overlap).
bool serial_dense() {
    static bool v = [] { const char* e = std::getenv("SFMCOV_SERIAL_DENSE"); return e && e[0] == '1'; }();
    return v;
}

// Cholesky + in-place triangular inverse of the padded matrix Z (lower
// triangle); serial = every launch on the main stream.
int run_dense(sfmcov_handle* h, double* Z, long long ld, int Npad, double* Linv, double* piv, Status* st, bool serial,
              bool mark_stages, cudaEvent_t eZ = nullptr, int nreal = 0);

void mark(sfmcov_handle* h, int i) {
    if (h->profiling) SFM_CUDA(cudaEventRecord(h->ev[i], h->s));
}

int run_dense(sfmcov_handle* h, double* Z, long long ld, int Npad, double* Linv, double* piv, Status* st, bool serial,
              bool mark_stages, cudaEvent_t eZ, int nreal) {
    cudaStream_t s = h->s;
    const int pw = panel_blocks(Npad / kNB, 1);
    double* ring = h->ring.as<double>(sweep_ring_doubles(Npad, pw, sfmcov_handle::kRing));
    const InvSplit isp{3, {h->sx[0], h->sx[1], h->sx[2]}, {h->eTx[0], h->eTx[1], h->eTx[2]}};
    const int launches = dense_sweep(Z, ld, Npad, pw, Linv, piv, st, ring, sfmcov_handle::kRing, s, serial ? s : h->s2,
                                     serial ? s : h->s3, h->eL, h->eT, h->e2, serial ? s : h->s4, h->eX, h->eN,
                                     serial ? nullptr : eZ, nreal, nullptr, serial ? nullptr : &isp);
    if (mark_stages) {
        mark(h, 8);
        mark(h, 9);
    }
    return launches;
}

// Diagnostics of a successful pipeline call (covariance.hpp:49-60).  The
// near-singular pivot test of invert_schur (covariance.cpp:236-240) runs on
// every call, whether or not the caller asked for the diagnostics.
void fill_diagnostics(sfmcov_handle* h, Outputs& out, const double* prange, const double* eigE, const int* psd,
                      const double* s_a, const unsigned char* flags, size_t ncols, int N, int64_t dense_bytes) {
    double pr[2], ee[8];
    int warn = 0;
    SFM_CUDA(cudaMemcpyAsync(pr, prange, 16, cudaMemcpyDeviceToHost, h->s));
    SFM_CUDA(cudaMemcpyAsync(ee, eigE, 56, cudaMemcpyDeviceToHost, h->s));
    if (out.diag) SFM_CUDA(cudaMemcpyAsync(&warn, psd, 4, cudaMemcpyDeviceToHost, h->s));
    SFM_CUDA(cudaStreamSynchronize(h->s));
    double mn = pr[0], mx = pr[1];
    for (int l = 0; l < 7; ++l) { mn = std::min(mn, std::fabs(ee[l])); mx = std::max(mx, std::fabs(ee[l])); }
    if (!(mn > 1e-12 * mx))
        throw ApiError{SFMCOV_ERR_DEGENERATE, "factorization",
                       "near-singular pivot (ratio " + fmt_f(mn / mx) +
                           "); the scene is likely disconnected or its gauge degenerate"};
    if (out.diag) {
        sfmcov_diagnostics* d = out.diag;
        d->min_pivot = mn;
        d->max_pivot = mx;
        d->inertia_positive = N;
        d->inertia_negative = 7;
        d->negative_eigenvalue_warnings = warn;
        d->largest_dense_dim = (int64_t)N + 7;
        d->peak_dense_bytes = dense_bytes;
        // scale range (device min/max) and flagged columns
        std::vector<unsigned char> f;
        double srange[2] = {1.0, 1.0};
        if (ncols) {
            double* mm = h->scale_mm.as<double>(2 * 296 + 2);
            launch_minmax(s_a, (long long)ncols, mm + 2, mm, h->s);
            d2h(h, srange, mm, 16);
        }
        if (h->st_host->nflag) {
            f.resize(ncols);
            d2h(h, f.data(), flags, ncols);
        }
        d->scale_min = srange[0];
        d->scale_max = srange[1];
        int64_t cnt = 0;
        if (h->st_host->nflag)
            for (size_t c = 0; c < ncols; ++c)
                if (f[c]) {
                    if (d->flagged && cnt < d->flagged_capacity) d->flagged[cnt] = (int64_t)c;
                    ++cnt;
                }
        d->n_flagged = (int32_t)cnt;
    }
}

void run_dist_tail(sfmcov_handle* h, const SceneDev& sc, Outputs& out, const double* D, const double* s_a,
                   const double* G, const double* Wb, Status* st, const unsigned char* flags, size_t ncols,
                   const double* eigE, const double* seg_in = nullptr);
void run_dist_sharded(sfmcov_handle* h, const SceneDev& sc, const IndexDev& ix, Outputs& out);

// First observation whose pixel u is not finite (LLONG_MAX if none); up to 8
// host threads for large scenes.
long long first_nonfinite_u(const double* u, long long t) {
    auto scan = [u](long long b, long long e) -> long long {
        for (long long k = b; k < e; ++k) {
            uint64_t x, y;
            std::memcpy(&x, u + 2 * k, 8);
            std::memcpy(&y, u + 2 * k + 1, 8);
            if (((x >> 52) & 0x7ff) == 0x7ff || ((y >> 52) & 0x7ff) == 0x7ff) return k;
        }
        return LLONG_MAX;
    };
    const long long kChunk = 1LL << 19;
    if (t <= kChunk) return scan(0, t);
    const int nt = (int)std::min<long long>(8, (t + kChunk - 1) / kChunk);
    std::vector<long long> r(nt, LLONG_MAX);
    std::vector<std::thread> th;
    for (int i = 1; i < nt; ++i) th.emplace_back([&, i] { r[i] = scan(t * i / nt, t * (i + 1) / nt); });
    r[0] = scan(0, t / nt);
    for (auto& x : th) x.join();
    return *std::min_element(r.begin(), r.end());
}

// The whole device pipeline.  `sc` points at device memory.
void run(sfmcov_handle* h, const SceneDev& sc, Mode mode, Outputs& out) {
    cudaStream_t s = h->s;
    const int n = sc.n, m = sc.m, t = sc.t, P = sc.P;
    if (P != 8 && P != 9) throw ApiError{SFMCOV_ERR_DIMENSION, "validate", "camera width must be 8 or 9"};
    if (n < 0 || m < 0 || t < 0) throw ApiError{SFMCOV_ERR_DIMENSION, "validate", "negative scene size"};
    if ((long long)n * n >= (1LL << 32)) throw ApiError{SFMCOV_ERR_SIZE_GUARD, "validate", "too many cameras for 32-bit pair keys"};
    const bool full = (mode == M_FULL || mode == M_SCHUR || mode == M_INDEX);
    // a host-API σ transfer still in flight is waited for on every exit, so
    // the caller's buffer is never read after the call returns
    struct SigmaWait {
        cudaEvent_t e;
        ~SigmaWait() { if (e) cudaEventSynchronize(e); }
    } sigma_wait{sc.sigma_ready};
    for (auto& v : h->stage_ms) v = 0.0;
    g_kernel_launches = 0;
    h->counts[9] = 0;
    Status* st = h->status.as<Status>(1);
    mark(h, 0);
    launch_status_init(st, s);
    launch_validate(sc, full ? 1 : 0, st, s);
    // host-API scenes: the finiteness of u is checked on host threads beside
    // the device work (an async task, joined at the last validation sync or
    // as soon as the device reports a failure, so it never sits on the
    // critical path of a valid scene) and merged as the reference's code-3
    // failure of that observation
    const bool split_values = full && sc.sigma_ready;  // σ checks after its upload
    std::future<long long> u_task;
    if (full && sc.host_u) u_task = std::async(std::launch::async, first_nonfinite_u, sc.host_u, (long long)t);
    long long u_bad = LLONG_MAX;
    auto sync_validation = [&](bool final_sync) {
        sync_status(h);
        const Status& q = *h->st_host;
        const bool failing = q.cam_bad != INT_MAX || q.pt_bad != INT_MAX || q.obs_bad != LLONG_MAX;
        if (u_task.valid() && (final_sync || failing)) u_bad = u_task.get();
        if (u_bad != LLONG_MAX) h->st_host->obs_bad = std::min(h->st_host->obs_bad, u_bad * 8 + 3);
    };
    sync_validation(!split_values);
    if (split_values) {
        const Status& q = *h->st_host;
        if (q.cam_bad != INT_MAX || q.pt_bad != INT_MAX || q.obs_bad != LLONG_MAX) {
            // failing scene: finish the value checks so the first failing
            // observation is reported, as the reference's single pass does
            SFM_CUDA(cudaStreamWaitEvent(s, sc.sigma_ready, 0));
            launch_validate_values(sc, st, s);
            sync_validation(true);
        }
    }
    throw_validation(h, sc, full);
    IndexDev ix;
    ix.off_cam = h->off_cam.as<int>(n + 1);
    ix.off_pt = h->off_pt.as<int>(m + 1);
    ix.idx_cam = h->idx_cam.as<int>(t);
    ix.idx_pt = h->idx_pt.as<int>(t);
    ix.pos_cam = h->pos_cam.as<int>(t);
    ix.key_scratch = h->key_scratch.as<int>(t);
    launch_build_index(sc, ix, h->ws, s);
    launch_structure_check(sc, ix, st, s);
    SFM_CUDA(cudaEventRecord(h->e_index, s));
    mark(h, 1);
    // ---- (a) Jacobian: the geometry needs no σ, so it runs while a host
    // scene's σ is still uploading (its errors are reported after validation's)
    double* R = nullptr;
    double* rec = nullptr;
    const bool sharded_a = h->dist_mode && mode == M_FULL && !h->replicated_a;
    if (mode != M_INDEX && !sharded_a) {
        R = h->R.as<double>(9 * (size_t)n);
        rec = h->rec.as<double>((size_t)kRec * t);
        launch_jacobian(sc, ix.idx_cam, R, rec, st, s);
        mark(h, 2);  // W = σ^-1 (k_weights) counts to the Fisher stage, as in the reference
    }
    if (sc.sigma_ready) SFM_CUDA(cudaStreamWaitEvent(s, sc.sigma_ready, 0));
    if (split_values) launch_validate_values(sc, st, s);
    if (full || mode == M_INDEX) {
        sync_validation(true);
        if (split_values) throw_validation(h, sc, full);
        if (h->st_host->dup) throw ApiError{SFMCOV_ERR_INVARIANT, "validate", "duplicate (camera, point) observation pair"};
        throw_counts(h);
    }
    if (sharded_a) {  // the multi-GPU path: point-sharded stage A (shard.cu)
        run_dist_sharded(h, sc, ix, out);
        return;
    }
    if (mode == M_INDEX) {
        std::vector<int> oc(n + 1), op(m + 1);
        d2h(h, oc.data(), ix.off_cam, 4 * (size_t)(n + 1));
        d2h(h, op.data(), ix.off_pt, 4 * (size_t)(m + 1));
        for (int i = 0; i <= n; ++i) out.off_cam[i] = oc[i];
        for (int j = 0; j <= m; ++j) out.off_pt[j] = op[j];
        d2h(h, out.idx_cam, ix.idx_cam, 4 * (size_t)t);
        d2h(h, out.idx_pt, ix.idx_pt, 4 * (size_t)t);
        return;
    }
    // The pair list depends only on the index: it is built on its own
    // high-priority stream by a host worker thread (its host reads of the
    // list sizes block that thread, not this one) while this thread queues
    // the numeric stage-A kernels on s.
    // W = σ^-1 first: the device restarts right after the validation sync,
    // before this thread spends time starting the pair-list worker
    launch_weights(sc, ix.idx_cam, rec, st, s);
    std::future<long long> pairs_task;
    if (mode == M_FULL || mode == M_SCHUR) {
        SFM_CUDA(cudaStreamWaitEvent(h->sp, h->e_index, 0));
        pairs_task = std::async(std::launch::async, [h, &sc, &ix] {
            SFM_CUDA(cudaSetDevice(h->device));
            g_kernel_launches = 0;
            build_pairs(sc, ix, h->pairs, h->ws_pairs, h->sp);
            SFM_CUDA(cudaEventRecord(h->e_pairs, h->sp));
            return g_kernel_launches;
        });
    }
    if (mode == M_JACOBIAN) {
        sync_status(h);
        throw_numeric(h, sc, mode);
        if (!out.jc) return;  // records stay on the device (nullspace_residual)
        std::vector<double> r((size_t)kRec * t);
        std::vector<int> pos(t);
        d2h(h, r.data(), rec, 8 * r.size());
        d2h(h, pos.data(), ix.pos_cam, 4 * (size_t)t);
        for (int k = 0; k < t; ++k) {  // records sit at by-camera slots
            std::memcpy(out.jc + (size_t)2 * P * k, &r[(size_t)kRec * pos[k]], 8 * 2 * P);
            std::memcpy(out.jp + (size_t)6 * k, &r[(size_t)kRec * pos[k] + 2 * P], 8 * 6);
        }
        return;
    }
    // ---- Fisher reductions, (c) rotation blocks, conditioning scales ------------
    const size_t ncols = (size_t)P * n + 3 * (size_t)m;
    double* D = h->D.as<double>((size_t)P * P * n);
    double* Hr = h->Hr.as<double>(9 * (size_t)n);
    double* A = h->A.as<double>(9 * (size_t)m);
    double* s_a = h->s_a.as<double>(ncols);
    unsigned char* flags = h->flags.as<unsigned char>(ncols);
    launch_reductions(sc, ix, rec, D, Hr, A, s_a, flags, st, s, h->s4, h->e_red_fork, h->e_red_join);
    double* bpart = h->bpart.as<double>(7 * (size_t)border_partial_blocks(n, m));
    double* s_b = h->s_b.as<double>(7);
    launch_border_scales(sc, Hr, s_a, bpart, s_b, s);
    mark(h, 3);
    if (mode == M_FISHER || mode == M_NULLSPACE) {
        sync_status(h);
        throw_numeric(h, sc, mode);
        if (out.H) {
            double* H = h->H.as<double>(ncols * 7);
            launch_write_h(sc, Hr, H, s);
            d2h(h, out.H, H, 8 * ncols * 7);
        }
        if (out.D) d2h(h, out.D, D, 8 * (size_t)P * P * n);
        if (out.A) d2h(h, out.A, A, 8 * 9 * (size_t)m);
        if (out.s_a) d2h(h, out.s_a, s_a, 8 * ncols);
        if (out.s_b) d2h(h, out.s_b, s_b, 8 * 7);
        if (out.Cp) {
            // couplings C_t = (J_c^T W) J_p from the records (host assembly of a test output)
            std::vector<double> r((size_t)kRec * t);
            std::vector<int> pos(t);
            d2h(h, r.data(), rec, 8 * r.size());
            d2h(h, pos.data(), ix.pos_cam, 4 * (size_t)t);
            for (int k = 0; k < t; ++k) {
                const double* jc = &r[(size_t)kRec * pos[k]];
                const double* jp = jc + 2 * P;
                const double* W = jp + 6;
                double* c = out.Cp + (size_t)P * 3 * k;
                for (int p = 0; p < P; ++p) {
                    const double t0 = jc[p] * W[0] + jc[P + p] * W[2];
                    const double t1 = jc[p] * W[1] + jc[P + p] * W[3];
                    for (int q = 0; q < 3; ++q) c[3 * p + q] = t0 * jp[q] + t1 * jp[3 + q];
                }
            }
        }
        if (out.diag) {
            std::vector<unsigned char> f(ncols);
            d2h(h, f.data(), flags, ncols);
            int64_t cnt = 0;
            for (size_t c = 0; c < ncols; ++c)
                if (f[c]) {
                    if (out.diag->flagged && cnt < out.diag->flagged_capacity) out.diag->flagged[cnt] = (int64_t)c;
                    ++cnt;
                }
            out.diag->n_flagged = (int32_t)cnt;
        }
        return;
    }
    // ---- (b) Schur: point preparation, border, pairs ----------------------------
    double* Wb = h->Wb.as<double>((size_t)kWStride * t);
    double* V = h->V.as<double>(21 * (size_t)m);
    const int ppb = point_prep_blocks(m);
    double* Fpart = h->Fpart.as<double>(28 * (size_t)ppb);
    double* Lpt = h->Lpt.as<double>(8 * (size_t)m);
    const size_t nwarps = ((size_t)t + 31) / 32;
    double* Pfirst = h->Pfirst.as<double>((size_t)P * 7 * nwarps);
    double* Plast = h->Plast.as<double>((size_t)P * 7 * nwarps);
    double* Gsum = h->Gsum.as<double>((size_t)P * 7 * n);
    launch_point_prep(sc, ix, rec, A, s_a, s_b, Lpt, Wb, V, Fpart, Pfirst, Plast, Gsum, st, s);
    double* LF = h->LF.as<double>(49);
    double* E = h->E.as<double>(49);
    double* eigE = h->eigE.as<double>(8);
    launch_border_factor(Fpart, ppb, LF, E, eigE, st, s);
    const int N = P * n;
    double* Gamma = h->Gamma.as<double>((size_t)N * 7);
    double* G = h->G.as<double>((size_t)N * 7);
    launch_camera_border(sc, ix, Pfirst, Plast, Gsum, Hr, s_a, s_b, LF, Gamma, G, s);
    mark(h, 4);
    g_kernel_launches += pairs_task.get();  // the pair list (started above on s2)
    SFM_CUDA(cudaStreamWaitEvent(s, h->e_pairs, 0));
    mark(h, 5);
    if (h->dist_mode && mode == M_FULL) {
        run_dist_tail(h, sc, out, D, s_a, G, Wb, st, flags, ncols, eigE);
        return;
    }
    const int Npad = ((N + kNB - 1) / kNB) * kNB;
    const long long ld = Npad;
    double* Z = h->Z.as<double>((size_t)Npad * Npad);
    launch_fill(P, Z, ld, N, Npad, D, s_a, G, mode == M_FULL ? 1 : 0, s);
    mark(h, 6);
    // The first panel of the sweep needs only its own block columns: those
    // are reduced here, the others on s2 beside its factorisation (the sweep
    // waits for them before its first next-panel update; disjoint blocks).
    const int pw0 = panel_blocks(Npad / kNB, 1);
    const int lo_split = std::min(n, (pw0 * kNB + P - 1) / P);  // cameras with a column in panel 0
    const bool split_pairs = mode == M_FULL && !serial_dense() && Npad / kNB > pw0 && lo_split < n;
    bool pr_timed = false;
    if (split_pairs) {
        SFM_CUDA(cudaEventRecord(h->e_fill, s));
        launch_pair_reduce(P, h->pairs, Wb, n, Z, ld, s, 0, lo_split);
        SFM_CUDA(cudaStreamWaitEvent(h->s2, h->e_fill, 0));
        if (h->profiling) SFM_CUDA(cudaEventRecord(h->e_pr0, h->s2));
        launch_pair_reduce(P, h->pairs, Wb, n, Z, ld, h->s2, lo_split, n);
        if (h->profiling) SFM_CUDA(cudaEventRecord(h->e_pr1, h->s2));
        SFM_CUDA(cudaEventRecord(h->e_zrest, h->s2));
        pr_timed = h->profiling;
    } else {
        launch_pair_reduce(P, h->pairs, Wb, n, Z, ld, s);
    }
    mark(h, 7);
    h->counts[0] = h->pairs.npairs;
    h->counts[1] = h->pairs.nseg;
    h->counts[2] = N;
    h->counts[3] = Npad;
    h->counts[4] = t;
    h->counts[5] = m;
    h->counts[6] = n;
    h->counts[7] = P;
    if (mode == M_SCHUR) {
        sync_status(h);
        throw_numeric(h, sc, mode);
        // bordered Z_p: [[Z, Γ], [Γ^T, E]] (host assembly of a test output)
        const size_t dim = (size_t)N + 7;
        std::vector<double> z((size_t)Npad * Npad), gm((size_t)N * 7), e(49);
        d2h(h, z.data(), Z, 8 * z.size());
        d2h(h, gm.data(), Gamma, 8 * gm.size());
        d2h(h, e.data(), E, 8 * 49);
        for (size_t c = 0; c < dim; ++c)
            for (size_t r = 0; r < dim; ++r) {
                double v;
                if (r < (size_t)N && c < (size_t)N) v = (r >= c) ? z[c * Npad + r] : z[r * Npad + c];
                else if (r < (size_t)N) v = gm[r * 7 + (c - N)];
                else if (c < (size_t)N) v = gm[c * 7 + (r - N)];
                else v = e[(r - N) * 7 + (c - N)];
                out.z_p[c * dim + r] = v;
            }
        return;
    }
    // ---- (d) dense gauge-fixed inversion ---------------------------------------
    const int K = Npad / kNB;
    double* Linv = h->Linv.as<double>((size_t)K * kNB * kNB);
    double* piv = h->piv.as<double>((size_t)Npad);
    const bool serial = serial_dense();
    run_dense(h, Z, ld, Npad, Linv, piv, st, serial, true, split_pairs ? h->e_zrest : nullptr, N);
    int* psd = h->psd.as<int>(1);
    SFM_CUDA(cudaMemsetAsync(psd, 0, sizeof(int), s));
    const bool cross = out.h_camera_matrix != nullptr;
    if (!cross) launch_extract(P, Z, ld, N, n, s_a, 1, out.d_cam_cov, st, psd, s);
    double* prange = h->prange.as<double>(2);
    launch_pivot_range(piv, N, prange, s);
    if (out.h_point_cov || cross) {
        // optional outputs: Z_aug^-1 = X^T X and the bordered-inverse blocks (fullcov.cu)
        FullCovArgs a{};
        a.P = P; a.n = n; a.m = m; a.Npad = Npad;
        a.X = Z;
        a.Zi = h->zi.as<double>((size_t)Npad * Npad);
        a.G = G; a.LF = LF; a.Lpt = Lpt; a.V = V; a.Wb = Wb; a.s_a = s_a;
        a.off_pt = ix.off_pt; a.idx_pt = ix.idx_pt; a.oc = sc.oc; a.pos_cam = ix.pos_cam;
        a.part = h->fc_part.as<double>(full_cov_part_doubles(N));
        a.Y = h->fc_y.as<double>((size_t)N * 7 + 7);
        a.gtt_part = h->fc_gtt.as<double>(49 * ((size_t)N / 64 + 2));
        a.Eb = h->fc_eb.as<double>(49);
        a.point_cov = out.h_point_cov ? h->fc_pc.as<double>(9 * (size_t)m + 9) : nullptr;
        a.cross = cross ? 1 : 0;
        a.cam_cov = out.d_cam_cov;
        a.psd = psd;
        full_covariance(a, s);
        if (out.h_point_cov && m) d2h(h, out.h_point_cov, a.point_cov, 8 * 9 * (size_t)m);
        if (cross && N)
            SFM_CUDA(cudaMemcpy2DAsync(out.h_camera_matrix, 8 * (size_t)N, a.Zi, 8 * ld, 8 * (size_t)N, N,
                                       cudaMemcpyDeviceToHost, s));
    }
    mark(h, 10);
    sync_status(h);
    h->counts[8] = g_kernel_launches;
    throw_numeric(h, sc, mode);
    if (h->profiling) {
        for (int i = 0; i < ST_COUNT; ++i) {
            float ms = 0.f;
            SFM_CUDA(cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]));
            h->stage_ms[i] = ms;
        }
        if (pr_timed) {
            // the later block columns' pair reduction ran on s2 beside the
            // first panel (its time also lies inside the cholesky stage)
            float ms = 0.f;
            SFM_CUDA(cudaEventElapsedTime(&ms, h->e_pr0, h->e_pr1));
            h->stage_ms[6] += ms;
        }
    }
    fill_diagnostics(h, out, prange, eigE, psd, s_a, flags, ncols, N, (int64_t)8 * Npad * (int64_t)Npad);
}

// Distributed tail (camera-aligned layout, 1D block-cyclic panels): the pair
// reduction over this rank's chunk range, all-reduce of the camera-pair
// blocks, local fill, the distributed sweep (dist.cu), local extraction and
// the all-reduces of the outputs.  Emulated ranks (dist_mode 1) run every
// rank of the group on this device and combine in rank order.
void run_dist_tail(sfmcov_handle* h, const SceneDev& sc, Outputs& out, const double* D, const double* s_a,
                   const double* G, const double* Wb, Status* st, const unsigned char* flags, size_t ncols,
                   const double* eigE, const double* seg_in) {
    cudaStream_t s = h->s;
    const int n = sc.n, P = sc.P, N = P * n;
    const ColMap cm{P, kNB / P, n};
    const int Npad = cm_npad(cm);
    const long long ld = Npad;
    const int R = h->dist_mode == 1 ? h->emu_R : h->dist_R;
    const int nloc = h->dist_mode == 1 ? R : 1;
    if (nloc > 64) throw ApiError{SFMCOV_ERR_DIMENSION, "options", "at most 64 emulated ranks"};
    const int Gp = panel_blocks(Npad / kNB, R);
    if ((int)h->ranks.size() < nloc) h->ranks.resize(nloc);
    if (!h->ev_rank_init) {
        SFM_CUDA(cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming));
        for (auto& e : h->ev_rank_done) SFM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->ev_rank_init = true;
    }
    DistGroup grp;
    grp.nccl = h->dist_mode == 2 ? h->nccl : nullptr;
    std::vector<Status*> sts(nloc, st);
    for (int i = 0; i < nloc; ++i) {
        const int gr = h->dist_mode == 1 ? i : h->dist_rank;
        h->ranks[i].init(h->device);
        h->ranks[i].setup(Ownership{R, gr, Gp}, Npad, ld);
        grp.ranks.push_back(&h->ranks[i]);
    }
    // ---- sharded Schur: this rank's chunks of the sorted pair list --------------
    // Each rank reduces its chunk range into per-segment blocks; the blocks
    // are grouped by the rank owning their block column and one
    // reduce-scatter hands every rank the sums of exactly its blocks
    // (nnz x 81 doubles in total instead of an all-reduce of all of them).
    const PairDev& pd = h->pairs;
    const size_t segd = (size_t)pd.nseg * 81;
    double* seg = seg_in ? const_cast<double*>(seg_in) : h->seg.as<double>(segd + 1);
    auto chunk_range = [&](int gr, int* cb, int* ce) {
        *cb = (int)((long long)pd.nchunks * gr / R);
        *ce = (int)((long long)pd.nchunks * (gr + 1) / R);
    };
    SegGroups& sgp = h->seg_groups;
    sgp.plan(cm, Ownership{R, 0, Gp}, pd.ukeys, pd.nseg, h->ws, s);
    const size_t gdoubles = (size_t)sgp.gmax * 81;
    double* send = h->seg_send.as<double>((size_t)R * gdoubles + 1);
    double* recv = nullptr;
    if (h->dist_mode == 1) {
        if (!seg_in) {
            double* tmp = h->seg_tmp.as<double>(segd + 1);
            for (int gr = 0; gr < R; ++gr) {
                int cb, ce;
                chunk_range(gr, &cb, &ce);
                launch_pair_reduce_segments(P, pd, Wb, n, cb, ce, gr == 0 ? seg : tmp, s);
                if (gr) launch_add(seg, tmp, segd, s);
            }
        }
        sgp.pack(seg, send, s);  // emulated ranks: the sum, grouped; rank g reads its slice
    } else {
        if (!seg_in) {
            int cb, ce;
            chunk_range(h->dist_rank, &cb, &ce);
            launch_pair_reduce_segments(P, pd, Wb, n, cb, ce, seg, s);
        }
        sgp.pack(seg, send, s);
        recv = h->seg_recv.as<double>(gdoubles + 1);
        dist_reduce_scatter(grp, send, recv, gdoubles, s);
    }
    mark(h, 6);
    int* psd = h->psd.as<int>(1);
    double* prange = h->prange.as<double>(2);
    double* pr_r = h->prange_r.as<double>(2 * (size_t)nloc);
    SFM_CUDA(cudaMemsetAsync(psd, 0, sizeof(int), s));
    SFM_CUDA(cudaMemsetAsync(out.d_cam_cov, 0, 8 * (size_t)P * P * n, s));
    SFM_CUDA(cudaEventRecord(h->ev_ready, s));
    for (int i = 0; i < nloc; ++i) {
        RankDense& r = h->ranks[i];
        SFM_CUDA(cudaStreamWaitEvent(r.s, h->ev_ready, 0));
        // NCCL operations of one communicator must not overlap: the panel
        // broadcasts (stream sc) start after the block all-reduce (stream s)
        SFM_CUDA(cudaStreamWaitEvent(r.sc, h->ev_ready, 0));
        launch_fill_local(cm, r.ow, r.zp, ld, Npad, r.ncl, D, s_a, G, r.s);
        const int g = r.ow.rank;
        sgp.scatter(g, recv ? recv : send + (size_t)g * gdoubles, cm, r.ow, pd.ukeys, r.zp, ld, r.s);
    }
    mark(h, 7);
    dist_sweep(grp, sts.data());
    for (int i = 0; i < nloc; ++i) {
        RankDense& r = h->ranks[i];
        launch_extract_local(cm, r.ow, r.zp, ld, Npad, s_a, out.d_cam_cov, st, psd, r.s);
        launch_pivot_range_local(cm, r.ow, r.pv, Npad, pr_r + 2 * i, r.s);
        SFM_CUDA(cudaEventRecord(h->ev_rank_done[i], r.s));
        SFM_CUDA(cudaStreamWaitEvent(s, h->ev_rank_done[i], 0));
    }
    mark(h, 8);
    mark(h, 9);
    launch_range_combine(prange, pr_r, nloc, s);
    if (grp.nccl) {
        dist_allreduce(grp, out.d_cam_cov, (size_t)P * P * n, 0, s);
        dist_allreduce(grp, prange, 1, 1, s);
        dist_allreduce(grp, prange + 1, 1, 2, s);
        dist_allreduce_int_sum(grp, psd, s);
        dist_allreduce_int_min(grp, &st->chol_bad, s);
    }
    mark(h, 10);
    h->counts[0] = pd.npairs;
    h->counts[1] = pd.nseg;
    h->counts[2] = N;
    h->counts[3] = Npad;
    h->counts[4] = sc.t;
    h->counts[5] = sc.m;
    h->counts[6] = n;
    h->counts[7] = P;
    h->counts[8] = g_kernel_launches;
    sync_status(h);
    throw_numeric(h, sc, M_FULL);
    if (h->profiling) {
        for (int i = 0; i < ST_COUNT; ++i) {
            float ms = 0.f;
            SFM_CUDA(cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]));
            h->stage_ms[i] = ms;
        }
    }
    int64_t local_bytes = 0;
    for (int i = 0; i < nloc; ++i) local_bytes = std::max<int64_t>(local_bytes, (int64_t)8 * ld * h->ranks[i].ncl);
    fill_diagnostics(h, out, prange, eigE, psd, s_a, flags, ncols, N, local_bytes);
}

// Point-sharded stage A of the multi-GPU path (shard.cu).  Every rank has
// validated and indexed the whole scene; rank r then takes the points
// [j0, j1) (balanced by observation pairs) with their observations and runs
// stage A on that sub-scene.  Per-camera sums and gauge terms are partial and
// summed across ranks (all-reduce; emulated ranks: in rank order):
//   D, rotation normal / rhs        n (P^2 + 18)   -> D, s_a, H_r (every rank)
//   border column squares           7              -> s_b
//   F = Σ V^T V                     28             -> L_F, E
//   Σ_a W_a V_j per camera          n P 7          -> Γ, G
// and each rank reduces only its points' observation pairs into the global
// camera-pair block index (every rank builds the same sorted key list), which
// run_dist_tail hands to the column owners with one reduce-scatter.
void run_dist_sharded(sfmcov_handle* h, const SceneDev& sc, const IndexDev& gix, Outputs& out) {
    cudaStream_t s = h->s;
    const int n = sc.n, m = sc.m, P = sc.P, N = P * n;
    const int R = h->dist_mode == 1 ? h->emu_R : h->dist_R;
    const int nloc = h->dist_mode == 1 ? R : 1;
    if (nloc > 64) throw ApiError{SFMCOV_ERR_DIMENSION, "options", "at most 64 emulated ranks"};
    DistGroup grp;
    grp.nccl = h->dist_mode == 2 ? h->nccl : nullptr;
    auto grank = [&](int i) { return h->dist_mode == 1 ? i : h->dist_rank; };
    Status* st = h->status.as<Status>(1);
    // the global camera-pair key list (identical on every rank) and the point ranges
    build_pairs(sc, gix, h->pairs, h->ws_pairs, s);
    std::vector<int> bounds;
    shard_bounds(h->pairs.off, m, R, h->sh_bounds.as<int>((size_t)R + 2), bounds, s);
    if ((int)h->ranka.size() < nloc) h->ranka.resize(nloc);
    const int NE = P * P + 18, NB = P * 7;
    double* raw = h->sh_raw.as<double>((size_t)NE * n + 1);
    double* sq = h->sh_sq.as<double>(8);
    double* F = h->sh_F.as<double>(32);
    double* Ssum = h->sh_S.as<double>((size_t)NB * n + 1);
    // summed partials: emulated ranks add in rank order, NCCL all-reduces
    auto combine = [&](double* total, size_t count, auto part_of) {
        for (int i = 0; i < nloc; ++i) {
            if (i == 0) SFM_CUDA(cudaMemcpyAsync(total, part_of(0), 8 * count, cudaMemcpyDeviceToDevice, s));
            else launch_add(total, part_of(i), count, s);
        }
        dist_allreduce(grp, total, count, 0, s);
    };
    // first failing index over the ranks, in the reference's (global) numbering
    int* err = h->sh_err.as<int>(8);
    auto rank_errors = [&](int field) {  // 0 jacobian obs, 1 fisher obs, 2 singular point
        std::vector<int> best(1, INT_MAX);
        for (int i = 0; i < nloc; ++i) {
            RankA& a = h->ranka[i];
            Status q;
            SFM_CUDA(cudaMemcpyAsync(&q, a.status.p, sizeof(Status), cudaMemcpyDeviceToHost, s));
            SFM_CUDA(cudaStreamSynchronize(s));
            const int v = field == 0 ? q.jac_bad : (field == 1 ? q.fisher_bad : q.pt_sing_bad);
            if (v == INT_MAX) continue;
            int g = v;
            if (field < 2) d2h(h, &g, a.sh.lt + v, sizeof(int));  // local observation -> global id
            else g = v + a.sh.j0;                                 // local point -> global id
            best[0] = std::min(best[0], g);
        }
        SFM_CUDA(cudaMemcpyAsync(err, best.data(), sizeof(int), cudaMemcpyHostToDevice, s));
        dist_allreduce_ints(grp, err, 1, 1, s);
        int g = INT_MAX;
        d2h(h, &g, err, sizeof(int));
        return g;
    };
    // ---- phase 1: sub-scenes, Jacobians, per-point blocks, camera partials -------
    for (int i = 0; i < nloc; ++i) {
        RankA& a = h->ranka[i];
        const int gr = grank(i);
        shard_extract(sc, bounds[gr], bounds[gr + 1], a.sh, s);
        const SceneDev& l = a.sh.sc;
        IndexDev& ix = a.ix;
        ix.off_cam = a.off_cam.as<int>((size_t)n + 1);
        ix.off_pt = a.off_pt.as<int>((size_t)l.m + 1);
        ix.idx_cam = a.idx_cam.as<int>((size_t)l.t + 1);
        ix.idx_pt = a.idx_pt.as<int>((size_t)l.t + 1);
        ix.pos_cam = a.pos_cam.as<int>((size_t)l.t + 1);
        ix.key_scratch = a.key_scratch.as<int>((size_t)l.t + 1);
        Status* lst = a.status.as<Status>(1);
        launch_status_init(lst, s);
        launch_build_index(l, ix, a.ws, s);
        double* Rr = a.R.as<double>(9 * (size_t)n + 1);
        double* rec = a.rec.as<double>((size_t)kRec * l.t + 1);
        if (l.t) launch_jacobian(l, ix.idx_cam, Rr, rec, lst, s);
        launch_weights(l, ix.idx_cam, rec, lst, s);
        const size_t ncl = (size_t)N + 3 * (size_t)l.m;
        launch_reductions(l, ix, rec, a.D.as<double>((size_t)P * P * n + 1), a.Hr.as<double>(9 * (size_t)n + 1),
                          a.A.as<double>(9 * (size_t)l.m + 1), a.s_a.as<double>(ncl + 1),
                          a.flags.as<unsigned char>(ncl + 1), lst, s, h->s4, h->e_red_fork, h->e_red_join,
                          a.raw.as<double>((size_t)NE * n + 1));
    }
    mark(h, 2);
    if (int g = rank_errors(0); g != INT_MAX) {
        double* Rg = h->R.as<double>(9 * (size_t)n + 1);
        SFM_CUDA(cudaMemcpyAsync(Rg, h->ranka[0].R.p, 72 * (size_t)n, cudaMemcpyDeviceToDevice, s));
        double d = 0.0;
        launch_depth_of(sc, Rg, g, (double*)h->depth.get(8), s);
        d2h(h, &d, h->depth.p, 8);
        throw ApiError{SFMCOV_ERR_DEGENERATE, "jacobian",
                       "observation " + std::to_string(g) + ": projection: point at camera-space depth " + fmt_f(d) +
                           " (behind camera or on the principal plane)"};
    }
    combine(raw, (size_t)NE * n, [&](int i) { return (const double*)h->ranka[i].raw.p; });
    // ---- phase 2: camera blocks, scales, rotation blocks; border scales ----------
    const size_t ncols = (size_t)N + 3 * (size_t)m;
    double* D = h->D.as<double>((size_t)P * P * n + 1);
    double* Hr = h->Hr.as<double>(9 * (size_t)n + 1);
    double* s_a = h->s_a.as<double>(ncols + 1);
    unsigned char* flags = h->flags.as<unsigned char>(ncols + 1);
    SFM_CUDA(cudaMemsetAsync(flags, 0, ncols, s));
    launch_camera_finish(P, raw, n, D, Hr, s_a, flags, st, s);
    sync_status(h);
    if (h->st_host->rot_bad != INT_MAX) throw_numeric(h, sc, M_NULLSPACE);
    if (int g = rank_errors(1); g != INT_MAX)
        throw ApiError{SFMCOV_ERR_DEGENERATE, "fisher", "observation " + std::to_string(g) + " covariance is not positive definite"};
    int nflag = h->st_host->nflag;  // camera columns
    std::vector<int> lflag(1, 0);
    for (int i = 0; i < nloc; ++i) {
        RankA& a = h->ranka[i];
        const SceneDev& l = a.sh.sc;
        // the camera scales into the rank's column layout; its point scales and
        // flags into the global one (disjoint ranges: summed / or-ed below)
        SFM_CUDA(cudaMemcpyAsync(a.s_a.p, s_a, 8 * (size_t)N, cudaMemcpyDeviceToDevice, s));
        if (i == 0) SFM_CUDA(cudaMemsetAsync(s_a + N, 0, 8 * 3 * (size_t)m, s));
        if (l.m)
            SFM_CUDA(cudaMemcpyAsync(s_a + N + 3 * (size_t)a.sh.j0, (const double*)a.s_a.p + N, 24 * (size_t)l.m,
                                     cudaMemcpyDeviceToDevice, s));
        launch_flags_or((const unsigned char*)a.flags.p + N, 3 * (size_t)l.m, flags + N + 3 * (size_t)a.sh.j0, s);
        Status q;
        SFM_CUDA(cudaMemcpyAsync(&q, a.status.p, sizeof(Status), cudaMemcpyDeviceToHost, s));
        SFM_CUDA(cudaStreamSynchronize(s));
        lflag[0] += q.nflag;
        launch_border_sums(l, Hr, (const double*)a.s_a.p, grank(i) == 0 ? 1 : 0,
                           a.bpart.as<double>(7 * (size_t)border_partial_blocks(n, l.m) + 7), a.sq.as<double>(8), s);
    }
    {  // flagged columns: the union over ranks; the count summed
        int* cnt = h->sh_err.as<int>(8) + 4;
        SFM_CUDA(cudaMemcpyAsync(cnt, lflag.data(), sizeof(int), cudaMemcpyHostToDevice, s));
        dist_allreduce_ints(grp, cnt, 1, 0, s);
        dist_allreduce_u8_max(grp, flags + N, 3 * (size_t)m, s);
        dist_allreduce(grp, s_a + N, 3 * (size_t)m, 0, s);  // each point's scales come from one rank
        int tot = 0;
        d2h(h, &tot, cnt, sizeof(int));
        h->st_host->nflag = nflag + tot;
        SFM_CUDA(cudaMemcpyAsync(&st->nflag, &h->st_host->nflag, sizeof(int), cudaMemcpyHostToDevice, s));
        SFM_CUDA(cudaStreamSynchronize(s));
    }
    combine(sq, 7, [&](int i) { return (const double*)h->ranka[i].sq.p; });
    double* s_b = h->s_b.as<double>(7);
    launch_border_scale(sq, s_b, s);
    mark(h, 3);
    // ---- phase 3: point factors, W, border partials ------------------------------
    for (int i = 0; i < nloc; ++i) {
        RankA& a = h->ranka[i];
        const SceneDev& l = a.sh.sc;
        const int ppb = point_prep_blocks(l.m);
        const size_t nwarps = ((size_t)l.t + 31) / 32;
        launch_point_prep(l, a.ix, (const double*)a.rec.p, (const double*)a.A.p, (const double*)a.s_a.p, s_b,
                          a.Lpt.as<double>(8 * (size_t)l.m + 8), a.Wb.as<double>((size_t)kWStride * l.t + 1),
                          a.V.as<double>(21 * (size_t)l.m + 21), a.Fpart.as<double>(28 * (size_t)ppb + 28),
                          a.Pfirst.as<double>((size_t)NB * nwarps + 1), a.Plast.as<double>((size_t)NB * nwarps + 1),
                          a.Gsum.as<double>((size_t)NB * n + 1), (Status*)a.status.p, s);
        launch_fpart_sum((const double*)a.Fpart.p, ppb, a.F28.as<double>(32), s);
        launch_camera_border(l, a.ix, (const double*)a.Pfirst.p, (const double*)a.Plast.p, (const double*)a.Gsum.p,
                             Hr, s_a, s_b, nullptr, nullptr, nullptr, s, a.S.as<double>((size_t)NB * n + 1), nullptr);
    }
    if (int g = rank_errors(2); g != INT_MAX)
        throw ApiError{SFMCOV_ERR_DEGENERATE, "schur", "point " + std::to_string(g) + " has a singular 3x3 block"};
    combine(F, 28, [&](int i) { return (const double*)h->ranka[i].F28.p; });
    combine(Ssum, (size_t)NB * n, [&](int i) { return (const double*)h->ranka[i].S.p; });
    // ---- phase 4: the gauge block and the border rows -------------------------------
    double* LF = h->LF.as<double>(49);
    double* E = h->E.as<double>(49);
    double* eigE = h->eigE.as<double>(8);
    launch_border_factor(F, 1, LF, E, eigE, st, s);
    double* Gamma = h->Gamma.as<double>((size_t)N * 7 + 1);
    double* G = h->G.as<double>((size_t)N * 7 + 1);
    launch_camera_border(sc, gix, nullptr, nullptr, nullptr, Hr, s_a, s_b, LF, Gamma, G, s, nullptr, Ssum);
    mark(h, 4);
    // ---- phase 5: each rank's observation pairs into the global block index ---------
    const PairDev& pg = h->pairs;
    const size_t segd = (size_t)pg.nseg * 81;
    double* seg = h->sh_seg.as<double>(segd + 1);
    for (int i = 0; i < nloc; ++i) {
        RankA& a = h->ranka[i];
        const SceneDev& l = a.sh.sc;
        build_pairs(l, a.ix, a.pairs, a.ws_pairs, s);
        double* seg_l = a.seg_l.as<double>((size_t)a.pairs.nseg * 81 + 1);
        launch_pair_reduce_segments(P, a.pairs, (const double*)a.Wb.p, n, 0, a.pairs.nchunks, seg_l, s);
        double* seg_g = nloc == 1 ? seg : a.seg_g.as<double>(segd + 1);
        SFM_CUDA(cudaMemsetAsync(seg_g, 0, 8 * segd, s));
        launch_seg_map(a.pairs.ukeys, a.pairs.nseg, pg.ukeys, pg.nseg, seg_l, seg_g, s);
    }
    if (nloc > 1)
        for (int i = 0; i < nloc; ++i) {
            if (i == 0) SFM_CUDA(cudaMemcpyAsync(seg, h->ranka[0].seg_g.p, 8 * segd, cudaMemcpyDeviceToDevice, s));
            else launch_add(seg, (const double*)h->ranka[i].seg_g.p, segd, s);
        }
    mark(h, 5);
    run_dist_tail(h, sc, out, D, s_a, G, nullptr, st, flags, ncols, eigE, seg);
}

// ---- batched sub-scenes ------------------------------------------------------------
// Thrown when a batch hits any failure: the caller then reruns the sub-scenes
// one by one, which reports the exact per-sub-scene error.
struct BatchFallback {};

sfmcov_handle* worker_of(sfmcov_handle* h, int i) {  // (h->mu is held by the caller)
    while ((int)h->workers.size() <= i) {
        sfmcov_error e{};
        sfmcov_handle* w = sfmcov_cuda_create(h->device, &e);
        if (!w) throw ApiError{SFMCOV_ERR_DEVICE, "device", e.message};
        h->workers.push_back(w);
    }
    return h->workers[i];
}

// One chunk of sub-scenes [s0, s1) of the batch, through one pipeline run
// (batch.cu): gather, stage A + Schur on the concatenation, per-scene gauge,
// one batched dense sweep over all the chunk's scenes (every launch covers the
// B problems over grid.y), extraction into cov (the chunk's cameras, in scene
// order).
void run_batch_chunk(sfmcov_handle* h, const SceneDev& full, int s0, int s1, const int32_t* cams, const int64_t* coff,
                     const int32_t* pts, const int64_t* poff, const int32_t* obs, const int64_t* toff, double* cov) {
    cudaStream_t s = h->s;
    // SFMCOV_SUBREC_TIMING=1: synchronised phase times of the chunk on stderr
    static const bool timing = [] { const char* e = std::getenv("SFMCOV_SUBREC_TIMING"); return e && e[0] == '1'; }();
    auto t_last = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
        if (!timing) return;
        SFM_CUDA(cudaStreamSynchronize(s));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  batch %-10s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    const int P = full.P, B = s1 - s0;
    const int nb = (int)(coff[s1] - coff[s0]), mb = (int)(poff[s1] - poff[s0]), tb = (int)(toff[s1] - toff[s0]);
    // device lists: cams | coff | pts | poff | obs | toff (offsets rebased to
    // the chunk), copied straight from the caller's concatenated arrays
    int* dl = h->bt_lists.as<int>((size_t)nb + mb + tb + 3 * ((size_t)B + 1) + 1);
    std::vector<int> offs(3 * ((size_t)B + 1));
    for (int k = 0; k <= B; ++k) {
        offs[k] = (int)(coff[s0 + k] - coff[s0]);
        offs[B + 1 + k] = (int)(poff[s0 + k] - poff[s0]);
        offs[2 * (B + 1) + k] = (int)(toff[s0 + k] - toff[s0]);
    }
    int* d_cams = dl;
    int* d_coff = d_cams + nb;
    int* d_pts = d_coff + B + 1;
    int* d_poff = d_pts + mb;
    int* d_obs = d_poff + B + 1;
    int* d_toff = d_obs + tb;
    SFM_CUDA(cudaMemcpyAsync(d_cams, cams + coff[s0], 4 * (size_t)nb, cudaMemcpyHostToDevice, s));
    SFM_CUDA(cudaMemcpyAsync(d_pts, pts + poff[s0], 4 * (size_t)mb, cudaMemcpyHostToDevice, s));
    SFM_CUDA(cudaMemcpyAsync(d_obs, obs + toff[s0], 4 * (size_t)tb, cudaMemcpyHostToDevice, s));
    SFM_CUDA(cudaMemcpyAsync(d_coff, offs.data(), 4 * ((size_t)B + 1), cudaMemcpyHostToDevice, s));
    SFM_CUDA(cudaMemcpyAsync(d_poff, offs.data() + B + 1, 4 * ((size_t)B + 1), cudaMemcpyHostToDevice, s));
    SFM_CUDA(cudaMemcpyAsync(d_toff, offs.data() + 2 * (B + 1), 4 * ((size_t)B + 1), cudaMemcpyHostToDevice, s));
    BatchLists L;
    L.B = B; L.nb = nb; L.mb = mb; L.tb = tb;
    L.cams = d_cams; L.coff = d_coff; L.pts = d_pts; L.poff = d_poff; L.obs = d_obs; L.toff = d_toff;
    SceneDev bsc{};
    bsc.n = nb; bsc.m = mb; bsc.t = tb; bsc.P = P;
    double* cams_b = h->bt_cams.as<double>((size_t)P * nb + 1);
    double* pts_b = h->bt_pts.as<double>(3 * (size_t)mb + 1);
    int* oc_b = h->bt_oc.as<int>((size_t)tb + 1);
    int* op_b = h->bt_op.as<int>((size_t)tb + 1);
    double* sig_b = full.sigma ? h->bt_sigma.as<double>(4 * (size_t)tb + 1) : nullptr;
    launch_batch_gather(L, P, full.cams, full.pts, full.oc, full.op, full.sigma, cams_b, pts_b, oc_b, op_b, sig_b, s);
    bsc.cams = cams_b; bsc.pts = pts_b; bsc.oc = oc_b; bsc.op = op_b; bsc.sigma = sig_b;
    phase("gather");
    // stage A and the Schur factors on the concatenation
    Status* st = h->status.as<Status>(1);
    launch_status_init(st, s);
    IndexDev ix;
    ix.off_cam = h->off_cam.as<int>((size_t)nb + 1);
    ix.off_pt = h->off_pt.as<int>((size_t)mb + 1);
    ix.idx_cam = h->idx_cam.as<int>((size_t)tb + 1);
    ix.idx_pt = h->idx_pt.as<int>((size_t)tb + 1);
    ix.pos_cam = h->pos_cam.as<int>((size_t)tb + 1);
    ix.key_scratch = h->key_scratch.as<int>((size_t)tb + 1);
    launch_build_index(bsc, ix, h->ws, s);
    launch_structure_check(bsc, ix, st, s);
    double* R = h->R.as<double>(9 * (size_t)nb + 1);
    double* rec = h->rec.as<double>((size_t)kRec * tb + 1);
    launch_jacobian(bsc, ix.idx_cam, R, rec, st, s);
    launch_weights(bsc, ix.idx_cam, rec, st, s);
    const size_t ncols = (size_t)P * nb + 3 * (size_t)mb;
    double* D = h->D.as<double>((size_t)P * P * nb + 1);
    double* Hr = h->Hr.as<double>(9 * (size_t)nb + 1);
    double* A = h->A.as<double>(9 * (size_t)mb + 1);
    double* s_a = h->s_a.as<double>(ncols + 1);
    unsigned char* flags = h->flags.as<unsigned char>(ncols + 1);
    launch_reductions(bsc, ix, rec, D, Hr, A, s_a, flags, st, s, h->s4, h->e_red_fork, h->e_red_join);
    phase("stage_a");
    double* s_b = h->bt_sb.as<double>(7 * (size_t)B + 7);
    launch_batch_border(P, L, cams_b, Hr, pts_b, s_a, s_b, s);
    int* sofc = h->bt_sofc.as<int>((size_t)nb + 1);
    int* sofp = h->bt_sofp.as<int>((size_t)mb + 1);
    launch_batch_scene_of(L.coff, B, nb, sofc, s);
    launch_batch_scene_of(L.poff, B, mb, sofp, s);
    const int ppb = point_prep_blocks(mb);
    const size_t nwarps = ((size_t)tb + 31) / 32;
    double* Lpt = h->Lpt.as<double>(8 * (size_t)mb + 8);
    double* Wb = h->Wb.as<double>((size_t)kWStride * tb + 1);
    double* V = h->V.as<double>(21 * (size_t)mb + 21);
    launch_point_prep(bsc, ix, rec, A, s_a, s_b, Lpt, Wb, V, h->Fpart.as<double>(28 * (size_t)ppb + 28),
                      h->Pfirst.as<double>((size_t)P * 7 * nwarps + 1), h->Plast.as<double>((size_t)P * 7 * nwarps + 1),
                      h->Gsum.as<double>((size_t)P * 7 * nb + 1), st, s, sofp);
    double* F28 = h->bt_F.as<double>(28 * (size_t)B + 28);
    double* LF = h->bt_LF.as<double>(49 * (size_t)B + 49);
    double* E = h->bt_E.as<double>(49 * (size_t)B + 49);
    double* eigE = h->bt_eigE.as<double>(8 * (size_t)B + 8);
    launch_batch_F(L, V, F28, s);
    launch_border_factor(F28, 1, LF, E, eigE, st, s, B);
    const int N = P * nb;
    double* Gamma = h->Gamma.as<double>((size_t)N * 7 + 1);
    double* G = h->G.as<double>((size_t)N * 7 + 1);
    double* wv = h->sh_S.as<double>((size_t)P * 7 * nb + 1);
    launch_batch_wv(P, nb, ix.off_cam, ix.idx_cam, bsc.op, Wb, V, wv, s);
    launch_camera_border(bsc, ix, nullptr, nullptr, nullptr, Hr, s_a, s_b, LF, Gamma, G, s, nullptr, wv, sofc);
    phase("schur_prep");
    build_pairs(bsc, ix, h->pairs, h->ws_pairs, s);
    phase("pairs");
    // one identity-padded Z per scene, the pair blocks routed there
    int maxn = 0;
    for (int k = s0; k < s1; ++k) maxn = std::max<int>(maxn, (int)(coff[k + 1] - coff[k]));
    const int Npad = std::max(kNB, ((P * maxn + kNB - 1) / kNB) * kNB);
    const long long zs = (long long)Npad * Npad;
    double* Zb = h->bt_Zb.as<double>((size_t)zs * B + 1);
    launch_batch_fill(P, L, Zb, Npad, D, s_a, G, s);
    launch_pair_reduce(P, h->pairs, Wb, nb, Zb, Npad, s, 0, 1 << 30, ZMap{sofc, L.coff, zs});
    double* piv = h->bt_piv.as<double>((size_t)Npad * B + 1);
    double* dcov = h->bt_cov.as<double>((size_t)P * P * nb + 1);
    int* psd = h->psd.as<int>(1);
    SFM_CUDA(cudaMemsetAsync(psd, 0, sizeof(int), s));
    phase("fill_reduce");
    // the dense stage: every scene's fused sweep in one batched sweep (each
    // launch covers all B problems over grid.y), then one extraction launch
    // over the batch's cameras
    const int K = Npad / kNB;
    const int pw = std::min(panel_blocks(K, 1), K);
    const int nslots = std::min(sfmcov_handle::kRing, (K + pw - 1) / pw);  // ring slots the sweep can use
    SweepBatch bt;
    bt.B = B;
    bt.zs = zs;
    bt.ls = (long long)K * kNB * kNB;
    bt.rs = (long long)sweep_ring_doubles(Npad, pw, nslots);
    bt.ps = Npad;
    std::vector<int> nreal(B);
    for (int k = 0; k < B; ++k) nreal[k] = P * (int)(coff[s0 + k + 1] - coff[s0 + k]);
    int* d_nreal = h->bt_nreal.as<int>((size_t)B);
    SFM_CUDA(cudaMemcpyAsync(d_nreal, nreal.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, s));
    bt.nreal_b = d_nreal;
    double* Linv = h->bt_linv.as<double>((size_t)bt.ls * B);
    double* ring = h->bt_ring.as<double>((size_t)bt.rs * B);
    dense_sweep(Zb, Npad, Npad, pw, Linv, piv, st, ring, nslots, s, h->s2, h->s3, h->eL, h->eT, h->e2,
                h->s4, h->eX, h->eN, nullptr, 0, &bt);
    launch_extract(P, Zb, Npad, 0, nb, s_a, 1, dcov, st, psd, s, ZMap{sofc, L.coff, zs});
    phase("dense");
    int* bad = h->bt_bad.as<int>((size_t)B + 1);
    launch_batch_ratio(L, piv, Npad, P, eigE, bad, s);
    std::vector<int> hb(B);
    d2h(h, hb.data(), bad, 4 * (size_t)B);
    sync_status(h);
    const Status& q = *h->st_host;
    const bool failed = q.cam_count_bad != INT_MAX || q.pt_count_bad != INT_MAX || q.jac_bad != INT_MAX ||
                        q.rot_bad != INT_MAX || q.fisher_bad != INT_MAX || q.pt_sing_bad != INT_MAX || q.border_bad ||
                        q.chol_bad != INT_MAX || std::find(hb.begin(), hb.end(), 1) != hb.end();
    if (failed) throw BatchFallback{};
    d2h(h, cov, dcov, 8 * (size_t)P * P * nb);
    phase("finish");
    if (timing) std::fprintf(stderr, "  batch chunk: %d scenes, %d cameras, %d points, %d observations, %lld pairs, Npad %d\n", B, nb, mb, tb, h->pairs.npairs, Npad);
}

// Copies a host scene into the handle's staging buffers.
SceneDev upload(sfmcov_handle* h, const sfmcov_scene* s) {
    SceneDev d;
    d.n = s->n_cams; d.m = s->n_pts; d.t = s->n_obs; d.P = s->cam_params;
    if (d.P != 8 && d.P != 9) throw ApiError{SFMCOV_ERR_DIMENSION, "validate", "camera width must be 8 or 9"};
    if (d.n < 0 || d.m < 0 || d.t < 0) throw ApiError{SFMCOV_ERR_DIMENSION, "validate", "negative scene size"};
    h->last_up = *s;
    h->last_up_valid = true;
    auto put = [&](DBuf& b, const void* src, size_t bytes) -> void* {
        void* p = b.get(bytes);
        if (bytes && src) SFM_CUDA(cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, h->s));
        return p;
    };
    d.cams = (const double*)put(h->h_cams, s->cams, 8 * (size_t)d.P * d.n);
    d.pts = (const double*)put(h->h_pts, s->pts, 24 * (size_t)d.m);
    d.oc = (const int*)put(h->h_oc, s->obs_cam, 4 * (size_t)d.t);
    d.op = (const int*)put(h->h_op, s->obs_pt, 4 * (size_t)d.t);
    d.u = nullptr;  // validated on the host (run()), never read on the device
    d.host_u = s->obs_u;
    // σ (the largest array) follows the indices on s3, so validation of the
    // indices and the index build on s overlap its transfer
    d.sigma = nullptr;
    if (s->obs_sigma) {
        void* p = h->h_sigma.get(32 * (size_t)d.t);
        d.sigma = (const double*)p;
        if (d.t) {
            SFM_CUDA(cudaEventRecord(h->e_ids, h->s));
            SFM_CUDA(cudaStreamWaitEvent(h->s3, h->e_ids, 0));
            SFM_CUDA(cudaMemcpyAsync(p, s->obs_sigma, 32 * (size_t)d.t, cudaMemcpyHostToDevice, h->s3));
            SFM_CUDA(cudaEventRecord(h->e_sigma, h->s3));
            d.sigma_ready = h->e_sigma;
        }
    }
    return d;
}

SceneDev as_device(const sfmcov_scene* s) {
    SceneDev d;
    d.n = s->n_cams; d.m = s->n_pts; d.t = s->n_obs; d.P = s->cam_params;
    d.cams = s->cams; d.pts = s->pts; d.oc = s->obs_cam; d.op = s->obs_pt; d.u = s->obs_u; d.sigma = s->obs_sigma;
    return d;
}

template <typename F>
int32_t guarded(sfmcov_handle* h, sfmcov_error* err, F&& body) {
    if (!h) {
        fill_error(err, ApiError{SFMCOV_ERR_DEVICE, "device", "null handle"});
        return SFMCOV_ERR_DEVICE;
    }
    std::lock_guard<std::recursive_mutex> lock(h->mu);
    try {
        SFM_CUDA(cudaSetDevice(h->device));
        body();
        clear_error(err);
        return SFMCOV_OK;
    } catch (const ApiError& e) {
        cudaStreamSynchronize(h->s);
        fill_error(err, e);
        return e.kind;
    } catch (const SizeGuard& e) {
        cudaStreamSynchronize(h->s);
        fill_error(err, ApiError{SFMCOV_ERR_SIZE_GUARD, e.stage, e.what()});
        return SFMCOV_ERR_SIZE_GUARD;
    } catch (const std::exception& e) {
        fill_error(err, ApiError{SFMCOV_ERR_DEVICE, "device", e.what()});
        return SFMCOV_ERR_DEVICE;
    }
}

// compute_covariance (camera blocks only) refuses the optional outputs: they
// need the output buffers of sfmcov_cuda_compute_covariance_full.
void check_options(const sfmcov_options* o) {
    if (o && (o->point_covariances || o->camera_cross_covariances))
        throw ApiError{SFMCOV_ERR_DIMENSION, "options",
                       "point / cross covariances need sfmcov_cuda_compute_covariance_full (output buffers)"};
}

}  // namespace

extern "C" {

sfmcov_handle* sfmcov_cuda_create(int32_t device, sfmcov_error* err) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count <= device || device < 0) {
        fill_error(err, ApiError{SFMCOV_ERR_DEVICE, "device",
                                 std::string("no usable CUDA device (") + cudaGetErrorString(e) + "); this library has no CPU path"});
        return nullptr;
    }
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    if (prop.major < 10) {
        fill_error(err, ApiError{SFMCOV_ERR_DEVICE, "device", std::string("device ") + prop.name + " is not sm_100"});
        return nullptr;
    }
    auto* h = new sfmcov_handle();
    try {
        h->device = device;
        {
            const char* e = std::getenv("SFMCOV_SHARDED_STAGE_A");
            h->replicated_a = !(e && e[0] == '1');
        }
        SFM_CUDA(cudaSetDevice(device));
        // critical path (panel factorisations) at high priority, bulk trailing updates low
        int lo = 0, hi = 0;
        SFM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        SFM_CUDA(cudaStreamCreateWithPriority(&h->s, cudaStreamNonBlocking, hi));
        // sweep streams: the inverse chain (s3) above the Cholesky trailing
        // updates (s2).  Both have slack, but the inverse's narrow row-panel
        // launches must not pile up behind the wide updates into a tail where
        // they underfill the GPU: config 3 sweep 17.57 -> 16.9 ms (the
        // inverse now ends 0.1 ms after the Cholesky instead of 3.7 ms).
        SFM_CUDA(cudaStreamCreateWithPriority(&h->s2, cudaStreamNonBlocking, lo));
        SFM_CUDA(cudaStreamCreateWithPriority(&h->s3, cudaStreamNonBlocking, (lo + hi) / 2));
        for (auto& x : h->sx) SFM_CUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, (lo + hi) / 2));
        SFM_CUDA(cudaStreamCreateWithPriority(&h->s4, cudaStreamNonBlocking, hi));
        SFM_CUDA(cudaStreamCreateWithPriority(&h->sp, cudaStreamNonBlocking, hi));
        SFM_CUDA(cudaEventCreateWithFlags(&h->eX, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->eN, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->e_index, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->e_pairs, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->e_ids, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->e_sigma, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->e_red_fork, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->e_red_join, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->e_fill, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->e_zrest, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreate(&h->e_pr0));
        SFM_CUDA(cudaEventCreate(&h->e_pr1));
        for (int i = 0; i < sfmcov_handle::kRing; ++i) {
            SFM_CUDA(cudaEventCreateWithFlags(&h->eL[i], cudaEventDisableTiming));
            SFM_CUDA(cudaEventCreateWithFlags(&h->eT[i], cudaEventDisableTiming));
            for (int q = 0; q < 3; ++q) SFM_CUDA(cudaEventCreateWithFlags(&h->eTx[q][i], cudaEventDisableTiming));
        }
        SFM_CUDA(cudaEventCreateWithFlags(&h->e1, cudaEventDisableTiming));
        SFM_CUDA(cudaEventCreateWithFlags(&h->e2, cudaEventDisableTiming));
        for (auto& ev : h->ev) SFM_CUDA(cudaEventCreate(&ev));
        SFM_CUDA(cudaMallocHost(&h->st_host, sizeof(Status)));
        dense_init_attributes();
    } catch (const std::exception& x) {
        fill_error(err, ApiError{SFMCOV_ERR_DEVICE, "device", x.what()});
        delete h;
        return nullptr;
    }
    clear_error(err);
    return h;
}

void sfmcov_cuda_destroy(sfmcov_handle* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->s);
    cudaStreamSynchronize(h->s2);
    cudaStreamSynchronize(h->s3);
    for (auto x : h->sx) cudaStreamSynchronize(x);
    cudaStreamSynchronize(h->s4);
    cudaStreamSynchronize(h->sp);
    DBuf* bufs[] = {&h->ws.tmp, &h->ws_pairs.tmp, &h->h_cams, &h->h_pts, &h->h_oc, &h->h_op, &h->h_sigma,
                    &h->off_cam, &h->idx_cam, &h->off_pt, &h->idx_pt, &h->pos_cam, &h->key_scratch,
                    &h->R, &h->rec, &h->D, &h->Hr, &h->A, &h->s_a, &h->flags, &h->bpart, &h->s_b, &h->Lpt, &h->Wb, &h->V,
                    &h->Fpart, &h->Pfirst, &h->Plast, &h->Gsum, &h->LF, &h->E, &h->eigE, &h->Gamma, &h->G, &h->Z, &h->Linv, &h->ring, &h->piv,
                    &h->cov, &h->psd, &h->prange, &h->status, &h->depth, &h->H};
    for (DBuf* b : bufs) b->release();
    h->pairs.release();
    for (auto& r : h->ranks) r.release();
    h->seg.release();
    h->seg_tmp.release();
    h->seg_send.release();
    h->seg_recv.release();
    h->seg_groups.release();
    for (auto& a : h->ranka) a.release();
    for (DBuf* b : {&h->sh_bounds, &h->sh_raw, &h->sh_sq, &h->sh_F, &h->sh_S, &h->sh_seg, &h->sh_err, &h->bt_lists,
                    &h->bt_cams, &h->bt_pts, &h->bt_oc, &h->bt_op, &h->bt_sigma, &h->bt_sofc, &h->bt_sofp, &h->bt_sb,
                    &h->bt_F, &h->bt_LF, &h->bt_E, &h->bt_eigE, &h->bt_Zb, &h->bt_piv, &h->bt_cov, &h->bt_bad,
                    &h->bt_nreal, &h->bt_linv, &h->bt_ring})
        b->release();
    h->prange_r.release();
    h->scale_mm.release();
    for (DBuf* b : {&h->zi, &h->fc_part, &h->fc_y, &h->fc_gtt, &h->fc_eb, &h->fc_pc, &h->or_a, &h->or_w, &h->or_work,
                    &h->or_vs, &h->or_vk, &h->or_s, &h->or_keep, &h->ref_c, &h->ref_ws})
        b->release();
    for (DBuf& b : h->sys) b.release();
    if (h->ev_rank_init) {
        cudaEventDestroy(h->ev_ready);
        for (auto& e : h->ev_rank_done) cudaEventDestroy(e);
    }
    if (h->nccl) sfm::nccl_comm_destroy(h->nccl);
    for (sfmcov_handle* w : h->workers) sfmcov_cuda_destroy(w);
    if (h->st_host) cudaFreeHost(h->st_host);
    for (void* p : h->pinned)
        if (p) cudaFreeHost(p);
    cudaEventDestroy(h->e1);
    cudaEventDestroy(h->e2);
    for (auto& ev : h->ev) cudaEventDestroy(ev);
    cudaStreamDestroy(h->s);
    cudaStreamDestroy(h->s2);
    cudaStreamDestroy(h->s3);
    cudaStreamDestroy(h->s4);
    for (auto x : h->sx) cudaStreamDestroy(x);
    cudaStreamDestroy(h->sp);
    cudaEventDestroy(h->eX);
    cudaEventDestroy(h->eN);
    cudaEventDestroy(h->e_index);
    cudaEventDestroy(h->e_pairs);
    cudaEventDestroy(h->e_ids);
    cudaEventDestroy(h->e_sigma);
    cudaEventDestroy(h->e_red_fork);
    cudaEventDestroy(h->e_red_join);
    cudaEventDestroy(h->e_fill);
    cudaEventDestroy(h->e_zrest);
    cudaEventDestroy(h->e_pr0);
    cudaEventDestroy(h->e_pr1);
    for (int i = 0; i < sfmcov_handle::kRing; ++i) {
        cudaEventDestroy(h->eL[i]);
        cudaEventDestroy(h->eT[i]);
        for (int q = 0; q < 3; ++q) cudaEventDestroy(h->eTx[q][i]);
    }
    delete h;
}

void* sfmcov_cuda_stream(sfmcov_handle* h) { return h ? (void*)h->s : nullptr; }

int32_t sfmcov_cuda_device(sfmcov_handle* h) { return h ? h->device : -1; }

sfmcov_handle* sfmcov_cuda_worker(sfmcov_handle* h, int32_t i, sfmcov_error* err) {
    if (!h || i < 0) return nullptr;
    std::lock_guard<std::recursive_mutex> lock(h->mu);
    while ((int32_t)h->workers.size() <= i) {
        sfmcov_handle* w = sfmcov_cuda_create(h->device, err);
        if (!w) return nullptr;
        h->workers.push_back(w);
    }
    return h->workers[i];
}

void sfmcov_cuda_set_sharded_stage_a(sfmcov_handle* h, int32_t on) {
    if (h) h->replicated_a = on == 0;
}

void sfmcov_cuda_set_profiling(sfmcov_handle* h, int32_t on) {
    if (h) h->profiling = on != 0;
}

int32_t sfmcov_cuda_compute_covariance(sfmcov_handle* h, const sfmcov_scene* scene, const sfmcov_options* opts,
                                       double* cam_cov, sfmcov_diagnostics* diag, sfmcov_error* err) {
    return guarded(h, err, [&] {
        check_options(opts);
        const SceneDev sc = upload(h, scene);
        const int P = sc.P;
        double* dcov = h->cov.as<double>((size_t)P * P * sc.n);
        Outputs out;
        out.d_cam_cov = dcov;
        out.diag = diag;
        run(h, sc, M_FULL, out);
        if (sc.n) SFM_CUDA(cudaMemcpyAsync(cam_cov, dcov, 8 * (size_t)P * P * sc.n, cudaMemcpyDeviceToHost, h->s));
        SFM_CUDA(cudaStreamSynchronize(h->s));
    });
}

int32_t sfmcov_cuda_compute_covariance_full(sfmcov_handle* h, const sfmcov_scene* scene, const sfmcov_options* opts,
                                            double* cam_cov, double* point_cov, double* camera_matrix,
                                            sfmcov_diagnostics* diag, sfmcov_error* err) {
    return guarded(h, err, [&] {
        const bool want_pc = opts && opts->point_covariances, want_cm = opts && opts->camera_cross_covariances;
        if ((want_pc && !point_cov) || (want_cm && !camera_matrix))
            throw ApiError{SFMCOV_ERR_DIMENSION, "options", "requested output buffer is null"};
        const SceneDev sc = upload(h, scene);
        const int P = sc.P;
        double* dcov = h->cov.as<double>((size_t)P * P * sc.n);
        Outputs out;
        out.d_cam_cov = dcov;
        out.diag = diag;
        out.h_point_cov = want_pc ? point_cov : nullptr;
        out.h_camera_matrix = want_cm ? camera_matrix : nullptr;
        run(h, sc, M_FULL, out);
        if (sc.n) SFM_CUDA(cudaMemcpyAsync(cam_cov, dcov, 8 * (size_t)P * P * sc.n, cudaMemcpyDeviceToHost, h->s));
        SFM_CUDA(cudaStreamSynchronize(h->s));
    });
}

int32_t sfmcov_cuda_compute_covariance_device(sfmcov_handle* h, const sfmcov_scene* d_scene, const sfmcov_options* opts,
                                              double* d_cam_cov, sfmcov_diagnostics* diag, sfmcov_error* err) {
    return guarded(h, err, [&] {
        check_options(opts);
        Outputs out;
        out.d_cam_cov = d_cam_cov;
        out.diag = diag;
        run(h, as_device(d_scene), M_FULL, out);
        SFM_CUDA(cudaStreamSynchronize(h->s));
    });
}

// ---- distributed entry points -------------------------------------------------
namespace {
// Runs the host pipeline with the distributed tail configured by (mode, R).
void run_dist_host(sfmcov_handle* h, const sfmcov_scene* scene, const sfmcov_options* opts, double* cam_cov,
                   sfmcov_diagnostics* diag, int mode, int R) {
    check_options(opts);
    struct Restore {
        sfmcov_handle* h;
        ~Restore() { h->dist_mode = 0; }
    } restore{h};
    h->dist_mode = mode;
    if (mode == 1) h->emu_R = R;
    const SceneDev sc = upload(h, scene);
    const int P = sc.P;
    double* dcov = h->cov.as<double>((size_t)P * P * sc.n);
    Outputs out;
    out.d_cam_cov = dcov;
    out.diag = diag;
    run(h, sc, M_FULL, out);
    if (sc.n) SFM_CUDA(cudaMemcpyAsync(cam_cov, dcov, 8 * (size_t)P * P * sc.n, cudaMemcpyDeviceToHost, h->s));
    SFM_CUDA(cudaStreamSynchronize(h->s));
}
}  // namespace

int32_t sfmcov_cuda_compute_covariance_emulated(sfmcov_handle* h, const sfmcov_scene* scene, const sfmcov_options* opts,
                                                int32_t ranks, double* cam_cov, sfmcov_diagnostics* diag,
                                                sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (ranks < 1 || ranks > 64) throw ApiError{SFMCOV_ERR_DIMENSION, "options", "ranks must be in [1, 64]"};
        run_dist_host(h, scene, opts, cam_cov, diag, 1, ranks);
    });
}

int32_t sfmcov_nccl_unique_id(char* id128, sfmcov_error* err) {
    try {
        sfm::nccl_unique_id(id128);
        clear_error(err);
        return SFMCOV_OK;
    } catch (const std::exception& x) {
        fill_error(err, ApiError{SFMCOV_ERR_DEVICE, "comm", x.what()});
        return SFMCOV_ERR_DEVICE;
    }
}

int32_t sfmcov_cuda_comm_init(sfmcov_handle* h, const char* id128, int32_t nranks, int32_t rank, sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (nranks < 1 || rank < 0 || rank >= nranks)
            throw ApiError{SFMCOV_ERR_DIMENSION, "comm", "rank must be in [0, nranks)"};
        if (h->nccl) sfm::nccl_comm_destroy(h->nccl);
        h->nccl = nullptr;
        h->dist_R = nranks;
        h->dist_rank = rank;
        if (nranks > 1) {
            try {
                h->nccl = sfm::nccl_comm_init(id128, nranks, rank);
            } catch (const std::exception& x) {
                throw ApiError{SFMCOV_ERR_DEVICE, "comm", x.what()};
            }
        }
    });
}

int32_t sfmcov_cuda_compute_covariance_sharded(sfmcov_handle* h, const sfmcov_scene* scene, const sfmcov_options* opts,
                                               double* cam_cov, sfmcov_diagnostics* diag, sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (h->dist_R > 1 && !h->nccl) throw ApiError{SFMCOV_ERR_DEVICE, "comm", "sfmcov_cuda_comm_init was not called"};
        if (h->dist_R <= 1) run_dist_host(h, scene, opts, cam_cov, diag, 1, 1);
        else run_dist_host(h, scene, opts, cam_cov, diag, 2, h->dist_R);
    });
}

int32_t sfmcov_cuda_compute_covariance_sharded_device(sfmcov_handle* h, const sfmcov_scene* d_scene,
                                                      const sfmcov_options* opts, double* d_cam_cov,
                                                      sfmcov_diagnostics* diag, sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (h->dist_R > 1 && !h->nccl) throw ApiError{SFMCOV_ERR_DEVICE, "comm", "sfmcov_cuda_comm_init was not called"};
        check_options(opts);
        struct Restore {
            sfmcov_handle* h;
            ~Restore() { h->dist_mode = 0; }
        } restore{h};
        h->dist_mode = h->dist_R > 1 ? 2 : 1;
        if (h->dist_mode == 1) h->emu_R = 1;
        Outputs out;
        out.d_cam_cov = d_cam_cov;
        out.diag = diag;
        run(h, as_device(d_scene), M_FULL, out);
        SFM_CUDA(cudaStreamSynchronize(h->s));
    });
}

int32_t sfmcov_cuda_pseudoinverse_covariance(sfmcov_handle* h, const sfmcov_scene* scene, int64_t max_params,
                                             double* cam_cov, double* sigma_full, double* singular_values,
                                             double* gauge_gap, sfmcov_error* err) {
    return guarded(h, err, [&] {
        const int P = scene->cam_params, n = scene->n_cams, m = scene->n_pts, t = scene->n_obs;
        const int64_t params = (int64_t)P * n + 3 * (int64_t)m;
        if (params > max_params)
            throw ApiError{SFMCOV_ERR_SIZE_GUARD, "oracle",
                           "scene has " + std::to_string(params) + " parameters, guard is " + std::to_string(max_params)};
        const SceneDev sc = upload(h, scene);
        {  // rec.validate()
            std::vector<int64_t> oc(n + 1), op(m + 1);
            std::vector<int32_t> ic(t > 0 ? t : 1), ip(t > 0 ? t : 1);
            Outputs o;
            o.off_cam = oc.data(); o.idx_cam = ic.data(); o.off_pt = op.data(); o.idx_pt = ip.data();
            run(h, sc, M_INDEX, o);
        }
        std::vector<double> D((size_t)P * P * n), A(9 * (size_t)m), Cp((size_t)P * 3 * t);
        Outputs o;
        o.D = D.data(); o.A = A.data(); o.Cp = Cp.data();
        run(h, sc, M_FISHER, o);
        const int N = (int)params;
        std::vector<double> F((size_t)N * N, 0.0);
        auto f = [&](int r, int c) -> double& { return F[(size_t)c * N + r]; };
        for (int i = 0; i < n; ++i)
            for (int p = 0; p < P; ++p)
                for (int q = 0; q < P; ++q) f(P * i + p, P * i + q) = D[(size_t)P * P * i + P * p + q];
        for (int j = 0; j < m; ++j)
            for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) f(P * n + 3 * j + p, P * n + 3 * j + q) = A[9 * (size_t)j + 3 * p + q];
        std::vector<int32_t> oc(t), op(t);
        std::memcpy(oc.data(), scene->obs_cam, 4 * (size_t)t);
        std::memcpy(op.data(), scene->obs_pt, 4 * (size_t)t);
        for (int k = 0; k < t; ++k)
            for (int p = 0; p < P; ++p)
                for (int q = 0; q < 3; ++q) {
                    const double v = Cp[(size_t)P * 3 * k + 3 * p + q];
                    f(P * oc[k] + p, P * n + 3 * op[k] + q) = v;
                    f(P * n + 3 * op[k] + q, P * oc[k] + p) = v;
                }
        std::vector<double> lam;
        double* S = nullptr;
        long long ld = 0;
        try {
            dense_pseudoinverse(F, N, h->or_a, h->or_w, h->or_work, h->or_vs, h->or_vk, h->or_s, h->or_keep, lam, &S,
                                &ld, h->s);
        } catch (const CudaError& x) {
            throw ApiError{SFMCOV_ERR_DEGENERATE, "oracle", x.what()};
        }
        for (int i = 0; i < n; ++i)
            SFM_CUDA(cudaMemcpy2DAsync(cam_cov + (size_t)P * P * i, 8 * (size_t)P, S + (size_t)P * i * ld + (size_t)P * i,
                                       8 * ld, 8 * (size_t)P, P, cudaMemcpyDeviceToHost, h->s));
        if (sigma_full)
            SFM_CUDA(cudaMemcpy2DAsync(sigma_full, 8 * (size_t)N, S, 8 * ld, 8 * (size_t)N, N, cudaMemcpyDeviceToHost,
                                       h->s));
        SFM_CUDA(cudaStreamSynchronize(h->s));
        // the blocks were copied column by column into row-major slots: transpose
        // each (Σ is symmetric, the copy gives Σ(q, p) at [p][q] before the swap)
        for (int i = 0; i < n; ++i) {
            double* b = cam_cov + (size_t)P * P * i;
            for (int p = 0; p < P; ++p)
                for (int q = p + 1; q < P; ++q) std::swap(b[P * p + q], b[P * q + p]);
        }
        std::vector<double> sv(N);
        for (int i = 0; i < N; ++i) sv[i] = std::fabs(lam[i]);
        std::sort(sv.begin(), sv.end(), std::greater<double>());
        if (singular_values) std::memcpy(singular_values, sv.data(), 8 * (size_t)N);
        if (gauge_gap) *gauge_gap = N >= 8 ? sv[N - 8] / sv[N - 7] : 0.0;
    });
}

int32_t sfmcov_plan_dense(int32_t n_cams, int32_t cam_params, int32_t nranks, int32_t rank, int32_t panel_blocks,
                          int64_t* npad, int64_t* local_cols, int32_t* cam_owned) {
    if (n_cams < 0 || (cam_params != 8 && cam_params != 9) || nranks < 1 || rank < 0 || rank >= nranks ||
        panel_blocks < 1)
        return SFMCOV_ERR_DIMENSION;
    const sfm::ColMap cm{cam_params, sfm::kNB / cam_params, n_cams};
    const sfm::Ownership ow{nranks, rank, panel_blocks};
    const int Np = sfm::cm_npad(cm);
    if (npad) *npad = Np;
    if (local_cols) *local_cols = (int64_t)sfm::own_blocks(ow, Np / sfm::kNB) * sfm::kNB;
    if (cam_owned)
        for (int i = 0; i < n_cams; ++i) cam_owned[i] = sfm::own_lcol(ow, sfm::cm_col(cm, i, 0)) >= 0 ? 1 : 0;
    return SFMCOV_OK;
}

int32_t sfmcov_plan_chunks(int64_t nchunks, int32_t nranks, int32_t rank, int64_t* begin, int64_t* end) {
    if (nchunks < 0 || nranks < 1 || rank < 0 || rank >= nranks) return SFMCOV_ERR_DIMENSION;
    *begin = nchunks * rank / nranks;
    *end = nchunks * (rank + 1) / nranks;
    return SFMCOV_OK;
}

int32_t sfmcov_cuda_observation_index(sfmcov_handle* h, const sfmcov_scene* scene, int64_t* off_cam, int32_t* idx_cam,
                                      int64_t* off_pt, int32_t* idx_pt, sfmcov_error* err) {
    return guarded(h, err, [&] {
        const SceneDev sc = upload(h, scene);
        Outputs out;
        out.off_cam = off_cam; out.idx_cam = idx_cam; out.off_pt = off_pt; out.idx_pt = idx_pt;
        run(h, sc, M_INDEX, out);
    });
}

int32_t sfmcov_cuda_jacobian(sfmcov_handle* h, const sfmcov_scene* scene, double* cam_blocks, double* point_blocks,
                             sfmcov_error* err) {
    return guarded(h, err, [&] {
        const SceneDev sc = upload(h, scene);
        Outputs out;
        out.jc = cam_blocks; out.jp = point_blocks;
        run(h, sc, M_JACOBIAN, out);
    });
}

int32_t sfmcov_cuda_nullspace(sfmcov_handle* h, const sfmcov_scene* scene, double* H, sfmcov_error* err) {
    return guarded(h, err, [&] {
        const SceneDev sc = upload(h, scene);
        Outputs out;
        out.H = H;
        run(h, sc, M_NULLSPACE, out);
    });
}

int32_t sfmcov_cuda_fisher(sfmcov_handle* h, const sfmcov_scene* scene, double* D, double* A, double* couplings,
                           double* s_a, double* s_b, sfmcov_diagnostics* diag, sfmcov_error* err) {
    return guarded(h, err, [&] {
        const SceneDev sc = upload(h, scene);
        Outputs out;
        out.D = D; out.A = A; out.Cp = couplings; out.s_a = s_a; out.s_b = s_b; out.diag = diag;
        run(h, sc, M_FISHER, out);
    });
}

int32_t sfmcov_cuda_schur(sfmcov_handle* h, const sfmcov_scene* scene, double* z_p, sfmcov_error* err) {
    return guarded(h, err, [&] {
        const SceneDev sc = upload(h, scene);
        Outputs out;
        out.z_p = z_p;
        run(h, sc, M_SCHUR, out);
    });
}

int32_t sfmcov_cuda_spd_inverse_blocks(sfmcov_handle* h, const double* a, int64_t n, int32_t block, double* blocks,
                                       double* min_pivot, double* max_pivot, sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (n <= 0 || block <= 0 || n % block) throw ApiError{SFMCOV_ERR_DIMENSION, "factorization", "n must be a positive multiple of block"};
        if (block != 8 && block != 9) throw ApiError{SFMCOV_ERR_DIMENSION, "factorization", "block must be 8 or 9"};
        cudaStream_t s = h->s;
        const int N = (int)n;
        const int Npad = ((N + kNB - 1) / kNB) * kNB;
        const long long ld = Npad;
        double* Z = h->Z.as<double>((size_t)Npad * Npad);
        // identity padding, then the user matrix (column by column)
        SFM_CUDA(cudaMemsetAsync(Z, 0, 8 * (size_t)Npad * Npad, s));
        launch_set_diag(Z, ld, N, Npad, s);
        SFM_CUDA(cudaMemcpy2DAsync(Z, 8 * ld, a, 8 * (size_t)N, 8 * (size_t)N, N, cudaMemcpyHostToDevice, s));
        Status* st = h->status.as<Status>(1);
        launch_status_init(st, s);
        const int K = Npad / kNB;
        double* Linv = h->Linv.as<double>((size_t)K * kNB * kNB);
        double* piv = h->piv.as<double>((size_t)Npad);
        run_dense(h, Z, ld, Npad, Linv, piv, st, serial_dense(), false);
        const int nb = N / block;
        double* dcov = h->cov.as<double>((size_t)block * block * nb);
        int* psd = h->psd.as<int>(1);
        SFM_CUDA(cudaMemsetAsync(psd, 0, sizeof(int), s));
        launch_extract(block, Z, ld, N, nb, nullptr, 0, dcov, st, psd, s);
        double* prange = h->prange.as<double>(2);
        launch_pivot_range(piv, N, prange, s);
        sync_status(h);
        if (h->st_host->chol_bad != INT_MAX)
            throw ApiError{SFMCOV_ERR_DEGENERATE, "factorization",
                           "non-positive pivot at index " + std::to_string(h->st_host->chol_bad) + "; matrix is not positive definite"};
        d2h(h, blocks, dcov, 8 * (size_t)block * block * nb);
        double pr[2];
        d2h(h, pr, prange, 16);
        if (min_pivot) *min_pivot = pr[0];
        if (max_pivot) *max_pivot = pr[1];
    });
}

int32_t sfmcov_cuda_refine_covariance(sfmcov_handle* h, const sfmcov_scene* scene, const int32_t* cams,
                                      int32_t n_sel, int32_t iters, double* refined, double* base, double* history,
                                      sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (n_sel < 0 || iters < 1 || iters > 16)
            throw ApiError{SFMCOV_ERR_DIMENSION, "refine", "need n_sel >= 0 and 1 <= iters <= 16"};
        for (int c = 0; c < n_sel; ++c)
            if (cams[c] < 0 || cams[c] >= scene->n_cams)
                throw ApiError{SFMCOV_ERR_DIMENSION, "refine", "camera id out of range"};
        // the product pipeline first (its blocks are the "base" answer, and
        // its factors are the approximate solver of the refinement)
        const SceneDev sc = upload(h, scene);
        const int P = sc.P, n = sc.n, m = sc.m, t = sc.t, N = P * n;
        double* dcov = h->cov.as<double>((size_t)P * P * n);
        Outputs out;
        out.d_cam_cov = dcov;
        run(h, sc, M_FULL, out);
        if (base && n_sel) {
            std::vector<double> all((size_t)P * P * n);
            d2h(h, all.data(), dcov, 8 * all.size());
            for (int c = 0; c < n_sel; ++c)
                std::memcpy(base + (size_t)P * P * c, &all[(size_t)P * P * cams[c]], 8 * (size_t)P * P);
        }
        const int Npad = ((N + kNB - 1) / kNB) * kNB;
        RefineArgs a{};
        a.P = P; a.n = n; a.m = m; a.t = t; a.Npad = Npad; a.ld = Npad;
        a.X = (const double*)h->Z.p;
        a.rec = (const double*)h->rec.p; a.D = (const double*)h->D.p; a.A = (const double*)h->A.p;
        a.Hr = (const double*)h->Hr.p; a.cams = sc.cams; a.pts = sc.pts;
        a.off_cam = (const int*)h->off_cam.p; a.idx_cam = (const int*)h->idx_cam.p;
        a.off_pt = (const int*)h->off_pt.p; a.idx_pt = (const int*)h->idx_pt.p;
        a.oc = sc.oc; a.op = sc.op; a.pos_cam = (const int*)h->pos_cam.p;
        a.s_a = (const double*)h->s_a.p; a.s_b = (const double*)h->s_b.p; a.Lpt = (const double*)h->Lpt.p;
        a.Wb = (const double*)h->Wb.p; a.V = (const double*)h->V.p; a.G = (const double*)h->G.p;
        a.LF = (const double*)h->LF.p;
        a.coupling = h->ref_c.as<double>((size_t)27 * (t > 0 ? t : 1));
        a.scratch = &h->ref_ws;
        // cameras per batch: as many as ~60 % of the free device memory holds
        size_t fr = 0, tot = 0;
        SFM_CUDA(cudaMemGetInfo(&fr, &tot));
        const size_t budget = (size_t)(0.6 * (double)(fr + h->ref_ws.cap));
        int per = 1;
        while (per < std::max(n_sel, 1) && per < 256 &&
               refine_bytes(N, Npad, m, ((P * 2 * per + 31) / 32) * 32) < budget)
            per *= 2;
        if (refine_bytes(N, Npad, m, ((P * per + 31) / 32) * 32) > budget && per > 1) per /= 2;
        std::vector<double> hist(iters, 0.0), hb(iters);
        for (int c0 = 0; c0 < n_sel; c0 += per) {
            const int c1 = std::min(n_sel, c0 + per);
            std::vector<int> sel(cams + c0, cams + c1);
            refine_camera_blocks(a, sel, iters, refined + (size_t)P * P * c0, hb.data(), h->s);
            for (int k = 0; k < iters; ++k) hist[k] = std::max(hist[k], hb[k]);
        }
        if (history) std::copy(hist.begin(), hist.end(), history);
    });
}

// ---- stage functions on caller-supplied systems (system.cu, eigen.cu) ---------
}  // extern "C"
namespace {
template <typename T>
T* up(sfmcov_handle* h, DBuf& b, const T* src, size_t count) {
    T* d = b.as<T>(count + 1);
    if (count && src) SFM_CUDA(cudaMemcpyAsync(d, src, sizeof(T) * count, cudaMemcpyHostToDevice, h->s));
    return d;
}
void check_system(int32_t n, int32_t m, int32_t t, int32_t P, int32_t b, const char* stage) {
    if (n < 0 || m < 0 || t < 0 || (P != 8 && P != 9) || b < 0 || b > 32)
        throw ApiError{SFMCOV_ERR_DIMENSION, stage, "bad system dimensions"};
}
}  // namespace
extern "C" {

int32_t sfmcov_cuda_nullspace_residual(sfmcov_handle* h, const sfmcov_scene* scene, const double* H, int32_t b,
                                       double* residual, sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (b < 1 || !H) throw ApiError{SFMCOV_ERR_DIMENSION, "nullspace", "nullspace shape does not match Jacobian"};
        const SceneDev sc = upload(h, scene);
        Outputs out;
        run(h, sc, M_JACOBIAN, out);
        const size_t rows = (size_t)sc.P * sc.n + 3 * (size_t)sc.m;
        const double* dH = up(h, h->sys[0], H, rows * b);
        auto* mx = h->sys[1].as<unsigned long long>(4);
        launch_nullspace_residual(sc.P, sc.t, sc.n, sc.m, sc.oc, sc.op, (const int*)h->pos_cam.p,
                                  (const double*)h->rec.p, dH, b, mx, h->s);
        unsigned long long v[3];
        d2h(h, v, mx, sizeof v);
        double d[3];
        std::memcpy(d, v, sizeof d);
        const double denom = d[1] * d[2];
        *residual = denom > 0.0 ? d[0] / denom : 0.0;
    });
}

int32_t sfmcov_cuda_condition_columns(sfmcov_handle* h, int32_t n, int32_t m, int32_t P, int32_t b, const double* D,
                                      const double* A, const double* border, double* s_a, double* s_b,
                                      int64_t* flagged, int64_t flagged_capacity, int64_t* n_flagged,
                                      sfmcov_error* err) {
    return guarded(h, err, [&] {
        check_system(n, m, 0, P, b, "conditioning");
        const size_t rows = (size_t)P * n + 3 * (size_t)m;
        const double* dD = up(h, h->sys[0], D, (size_t)P * P * n);
        const double* dA = up(h, h->sys[1], A, 9 * (size_t)m);
        const double* dB = up(h, h->sys[2], border, rows * b);
        double* dsa = h->sys[3].as<double>(rows + 1);
        unsigned char* fl = h->sys[4].as<unsigned char>(rows + 1);
        double* part = h->sys[5].as<double>(condition_part_doubles(P, n, m, b));
        double* dsb = h->sys[6].as<double>((size_t)b + 1);
        launch_condition_columns(P, n, m, b, dD, dA, dB, dsa, fl, part, dsb, h->s);
        if (rows) d2h(h, s_a, dsa, 8 * rows);
        if (b) d2h(h, s_b, dsb, 8 * (size_t)b);
        std::vector<unsigned char> f(rows);
        if (rows) d2h(h, f.data(), fl, rows);
        int64_t k = 0;
        for (size_t c = 0; c < rows; ++c)
            if (f[c]) {
                if (flagged && k < flagged_capacity) flagged[k] = (int64_t)c;
                ++k;
            }
        if (n_flagged) *n_flagged = k;
    });
}

int32_t sfmcov_cuda_apply_conditioning(sfmcov_handle* h, int32_t n, int32_t m, int32_t t, int32_t P, int32_t b,
                                       double* D, double* A, double* couplings, const int32_t* obs_cam,
                                       const int32_t* obs_pt, double* border, const double* s_a, const double* s_b,
                                       sfmcov_error* err) {
    return guarded(h, err, [&] {
        check_system(n, m, t, P, b, "conditioning");
        const size_t rows = (size_t)P * n + 3 * (size_t)m;
        for (int32_t k = 0; k < t; ++k)
            if (obs_cam[k] < 0 || obs_cam[k] >= n || obs_pt[k] < 0 || obs_pt[k] >= m)
                throw ApiError{SFMCOV_ERR_DIMENSION, "conditioning", "coupling index out of range"};
        double* dD = up(h, h->sys[0], (const double*)D, (size_t)P * P * n);
        double* dA = up(h, h->sys[1], (const double*)A, 9 * (size_t)m);
        double* dC = up(h, h->sys[2], (const double*)couplings, (size_t)P * 3 * t);
        const int* doc = up(h, h->sys[3], obs_cam, (size_t)t);
        const int* dop = up(h, h->sys[4], obs_pt, (size_t)t);
        double* dB = up(h, h->sys[5], (const double*)border, rows * b);
        const double* dsa = up(h, h->sys[6], s_a, rows);
        const double* dsb = up(h, h->sys[7], s_b, (size_t)b);
        launch_apply_conditioning(P, n, m, t, b, dD, dA, dC, doc, dop, dB, dsa, dsb, h->s);
        if (n) d2h(h, D, dD, 8 * (size_t)P * P * n);
        if (m) d2h(h, A, dA, 8 * 9 * (size_t)m);
        if (t) d2h(h, couplings, dC, 8 * (size_t)P * 3 * t);
        if (rows * b) d2h(h, border, dB, 8 * rows * b);
    });
}

int32_t sfmcov_cuda_schur_system(sfmcov_handle* h, int32_t n, int32_t m, int32_t t, int32_t P, int32_t b,
                                 const double* D, const double* A, const double* couplings, const int32_t* obs_cam,
                                 const int32_t* obs_pt, const double* border, double* z_p, double* a_inv,
                                 sfmcov_error* err) {
    return guarded(h, err, [&] {
        check_system(n, m, t, P, b, "schur");
        if ((long long)n * n >= (1LL << 32)) throw ApiError{SFMCOV_ERR_SIZE_GUARD, "schur", "too many cameras"};
        for (int32_t k = 0; k < t; ++k)
            if (obs_cam[k] < 0 || obs_cam[k] >= n || obs_pt[k] < 0 || obs_pt[k] >= m)
                throw ApiError{SFMCOV_ERR_DIMENSION, "schur", "coupling index out of range"};
        cudaStream_t s = h->s;
        const size_t rows = (size_t)P * n + 3 * (size_t)m;
        const int N = P * n;
        SysSchurArgs a{};
        a.P = P; a.n = n; a.m = m; a.t = t; a.b = b;
        a.D = up(h, h->sys[0], D, (size_t)P * P * n);
        a.A = up(h, h->sys[1], A, 9 * (size_t)m);
        a.Cp = up(h, h->sys[2], couplings, (size_t)P * 3 * t);
        const int* doc = up(h, h->sys[3], obs_cam, (size_t)t);
        a.op = up(h, h->sys[4], obs_pt, (size_t)t);
        a.border = up(h, h->sys[5], border, rows * b);
        // observation index and the camera-pair list of the system's couplings
        SceneDev sc{};
        sc.n = n; sc.m = m; sc.t = t; sc.P = P; sc.oc = doc; sc.op = a.op;
        IndexDev ix;
        ix.off_cam = h->off_cam.as<int>(n + 1);
        ix.off_pt = h->off_pt.as<int>(m + 1);
        ix.idx_cam = h->idx_cam.as<int>(t);
        ix.idx_pt = h->idx_pt.as<int>(t);
        ix.pos_cam = h->pos_cam.as<int>(t);
        ix.key_scratch = h->key_scratch.as<int>(t);
        launch_build_index(sc, ix, h->ws, s);
        build_pairs(sc, ix, h->pairs, h->ws_pairs, s);
        a.ix = &ix;
        a.pairs = &h->pairs;
        a.Lpt = h->sys[6].as<double>(8 * (size_t)m + 1);
        a.V = h->sys[7].as<double>(3 * (size_t)m * b + 1);
        a.Wb = h->sys[8].as<double>((size_t)kWStride * t + 1);
        a.Z = h->sys[9].as<double>((size_t)N * N + 1);
        a.Gamma = h->sys[10].as<double>((size_t)N * b + 1);
        a.epart = h->sys[11].as<double>(schur_system_epart_doubles(m, b));
        a.zp = h->sys[12].as<double>(((size_t)N + b) * ((size_t)N + b) + 1);
        a.a_inv = a_inv ? h->sys[13].as<double>(9 * (size_t)m + 1) : nullptr;
        Status* st = h->status.as<Status>(1);
        a.st = st;
        launch_status_init(st, s);
        schur_system(a, s);
        sync_status(h);
        if (h->st_host->pt_sing_bad != INT_MAX)
            throw ApiError{SFMCOV_ERR_DEGENERATE, "schur",
                           "point " + std::to_string(h->st_host->pt_sing_bad) + " has a singular 3x3 block"};
        const size_t dim = (size_t)N + b;
        if (dim) d2h(h, z_p, a.zp, 8 * dim * dim);
        if (a_inv && m) d2h(h, a_inv, a.a_inv, 8 * 9 * (size_t)m);
    });
}

int32_t sfmcov_cuda_invert_symmetric(sfmcov_handle* h, const double* z, int64_t dim, double* z_inv,
                                     double* min_pivot, double* max_pivot, int32_t* inertia_positive,
                                     int32_t* inertia_negative, sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (dim < 1) throw ApiError{SFMCOV_ERR_DIMENSION, "factorization", "matrix must be square"};
        if (dim > 46340) throw ApiError{SFMCOV_ERR_SIZE_GUARD, "factorization", "dense symmetric solve too large"};
        const int n = (int)dim;
        const double* dz = up(h, h->sys[0], z, (size_t)n * n);
        std::vector<double> lam;
        double* V = nullptr;
        int ldv = 0;
        sym_eigen(dz, n, n, h->sys[1], h->sys[2], h->sys[3], lam, &V, &ldv, h->s);
        double mn = std::numeric_limits<double>::infinity(), mx = 0.0;
        int pos = 0, neg = 0;
        for (double l : lam) {
            mn = std::min(mn, std::fabs(l));
            mx = std::max(mx, std::fabs(l));
            (l >= 0.0 ? pos : neg)++;
        }
        if (min_pivot) *min_pivot = mn;
        if (max_pivot) *max_pivot = mx;
        if (inertia_positive) *inertia_positive = pos;
        if (inertia_negative) *inertia_negative = neg;
        if (!(mn > 1e-12 * mx))
            throw ApiError{SFMCOV_ERR_DEGENERATE, "factorization",
                           "near-singular pivot (ratio " + fmt_f(mn / mx) +
                               "); the scene is likely disconnected or its gauge degenerate"};
        std::vector<int> keep(n);
        std::vector<double> w(n);
        for (int i = 0; i < n; ++i) { keep[i] = i; w[i] = 1.0 / lam[i]; }
        double* S = nullptr;
        long long lds = 0;
        eig_reconstruct(V, ldv, n, keep, w, h->sys[4], h->sys[5], h->sys[6], h->sys[7], &S, &lds, h->s);
        SFM_CUDA(cudaMemcpy2DAsync(z_inv, 8 * (size_t)n, S, 8 * lds, 8 * (size_t)n, n, cudaMemcpyDeviceToHost, h->s));
        SFM_CUDA(cudaStreamSynchronize(h->s));
    });
}

int32_t sfmcov_cuda_extract_camera_blocks(sfmcov_handle* h, const double* z_inv, int64_t dim, int32_t n, int32_t P,
                                          const double* s_a, double* cam_cov, int32_t* warnings, sfmcov_error* err) {
    return guarded(h, err, [&] {
        if ((P != 8 && P != 9) || n < 0 || (int64_t)P * n > dim)
            throw ApiError{SFMCOV_ERR_DIMENSION, "extract", "camera blocks do not fit the matrix"};
        const double* dz = up(h, h->sys[0], z_inv, (size_t)dim * dim);
        const double* dsa = s_a ? up(h, h->sys[1], s_a, (size_t)P * n) : nullptr;
        double* dc = h->sys[2].as<double>((size_t)P * P * n + 1);
        int* warn = h->sys[3].as<int>(1);
        launch_extract_given(P, n, dz, dim, dsa, dc, warn, h->s);
        if (n) d2h(h, cam_cov, dc, 8 * (size_t)P * P * n);
        int wv = 0;
        d2h(h, &wv, warn, sizeof wv);
        if (warnings) *warnings = wv;
    });
}

int32_t sfmcov_cuda_full_covariance(sfmcov_handle* h, const sfmcov_scene* scene, int64_t max_params, double* sigma,
                                    sfmcov_error* err) {
    return guarded(h, err, [&] {
        const int P = scene->cam_params, n = scene->n_cams, m = scene->n_pts, t = scene->n_obs;
        const int64_t params = (int64_t)P * n + 3 * (int64_t)m;
        if (params > max_params)
            throw ApiError{SFMCOV_ERR_SIZE_GUARD, "full-covariance",
                           "scene has " + std::to_string(params) + " parameters, guard is " + std::to_string(max_params)};
        const SceneDev sc = upload(h, scene);
        {  // rec.validate()
            std::vector<int64_t> oc(n + 1), op(m + 1);
            std::vector<int32_t> ic(t > 0 ? t : 1), ip(t > 0 ? t : 1);
            Outputs o;
            o.off_cam = oc.data(); o.idx_cam = ic.data(); o.off_pt = op.data(); o.idx_pt = ip.data();
            run(h, sc, M_INDEX, o);
        }
        Outputs o;
        run(h, sc, M_FISHER, o);
        cudaStream_t s = h->s;
        double* H = h->H.as<double>((size_t)params * 7 + 1);
        launch_write_h(sc, (const double*)h->Hr.p, H, s);
        const long long dimK = params + 7;
        double* K = h->sys[0].as<double>((size_t)dimK * dimK + 1);
        launch_full_k(P, n, m, t, (const double*)h->D.p, (const double*)h->A.p, (const double*)h->rec.p, sc.oc, sc.op,
                      (const int*)h->pos_cam.p, H, (const double*)h->s_a.p, (const double*)h->s_b.p, K, dimK, s);
        std::vector<double> lam;
        double* V = nullptr;
        int ldv = 0;
        sym_eigen(K, dimK, (int)dimK, h->sys[1], h->sys[2], h->sys[3], lam, &V, &ldv, s);
        double mn = std::numeric_limits<double>::infinity(), mx = 0.0;
        int neg = 0;
        for (double l : lam) {
            mn = std::min(mn, std::fabs(l));
            mx = std::max(mx, std::fabs(l));
            neg += l < 0.0;
        }
        if (!(mn > 1e-12 * mx) || neg != 7)
            throw ApiError{SFMCOV_ERR_DEGENERATE, "factorization",
                           "near-singular pivot (ratio " + fmt_f(mn / mx) +
                               "); the scene is likely disconnected or its gauge degenerate"};
        std::vector<int> keep((size_t)dimK);
        std::vector<double> w((size_t)dimK);
        for (long long i = 0; i < dimK; ++i) { keep[i] = (int)i; w[i] = 1.0 / lam[i]; }
        double* S = nullptr;
        long long lds = 0;
        eig_reconstruct(V, ldv, (int)dimK, keep, w, h->sys[4], h->sys[5], h->sys[6], h->sys[7], &S, &lds, s);
        double* out = h->sys[8].as<double>((size_t)params * params + 1);
        launch_full_unscale(params, S, lds, (const double*)h->s_a.p, out, s);
        if (params) d2h(h, sigma, out, 8 * (size_t)params * params);
    });
}

// The batched sub-scene path in steps, for a caller that forms the chunks
// itself (subrec.cpp pipelines planning, inducing and the device chunks):
// begin uploads the full scene once; every chunk call runs one pipeline
// chunk on it (<= 60000 cameras, <= 12M observations; arrays local to the
// chunk) and returns SFMCOV_ERR_DEGENERATE (stage "batch") if any of its
// sub-scenes fails; host_buffer hands out grow-only pinned staging (two
// slots) so the chunks' id lists go to the device at full PCIe rate.
int32_t sfmcov_internal_batch_begin(sfmcov_handle* h, const sfmcov_scene* full, sfmcov_error* err) {
    return guarded(h, err, [&] {
        h->bt_full_valid = false;
        const sfmcov_scene& l = h->last_up;
        const bool same = h->last_up_valid && l.n_cams == full->n_cams && l.n_pts == full->n_pts &&
                          l.n_obs == full->n_obs && l.cam_params == full->cam_params && l.cams == full->cams &&
                          l.pts == full->pts && l.obs_cam == full->obs_cam && l.obs_pt == full->obs_pt &&
                          l.obs_sigma == full->obs_sigma;
        if (same) {  // this call's validation has just copied it: the device copy is current
            SFM_CUDA(cudaStreamSynchronize(h->s3));  // (σ travels on s3)
            SceneDev& d = h->bt_full;
            d = SceneDev{};
            d.n = full->n_cams; d.m = full->n_pts; d.t = full->n_obs; d.P = full->cam_params;
            d.cams = (const double*)h->h_cams.p;
            d.pts = (const double*)h->h_pts.p;
            d.oc = (const int*)h->h_oc.p;
            d.op = (const int*)h->h_op.p;
            d.sigma = full->obs_sigma ? (const double*)h->h_sigma.p : nullptr;
        } else {
            h->bt_full = upload(h, full);
        }
        if (h->bt_full.sigma_ready) SFM_CUDA(cudaStreamWaitEvent(h->s, h->bt_full.sigma_ready, 0));
        h->bt_full.sigma_ready = nullptr;
        h->bt_full.host_u = nullptr;
        h->bt_full_valid = true;
    });
}

int32_t sfmcov_internal_batch_chunk(sfmcov_handle* h, int32_t nscenes, const int32_t* cams, const int64_t* coff,
                                    const int32_t* pts, const int64_t* poff, const int32_t* obs, const int64_t* toff,
                                    double* cov, sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (!h->bt_full_valid) throw ApiError{SFMCOV_ERR_INVARIANT, "batch", "no resident scene (batch_begin)"};
        if (nscenes < 1 || coff[nscenes] > 60000 || toff[nscenes] > 12000000)
            throw ApiError{SFMCOV_ERR_SIZE_GUARD, "batch", "chunk beyond 60000 cameras / 12M observations"};
        try {
            run_batch_chunk(h, h->bt_full, 0, nscenes, cams, coff, pts, poff, obs, toff, cov);
        } catch (const BatchFallback&) {
            throw ApiError{SFMCOV_ERR_DEGENERATE, "batch", "a sub-scene failed; rerun them one by one"};
        }
    });
}

// The observation index that sfmcov_internal_covis built last (by-camera and
// by-point CSR of observation ids, ascending within each camera / point), to
// the host: the sub-reconstruction planner's ByCam without a host sort.
int32_t sfmcov_internal_last_index(sfmcov_handle* h, int32_t n, int32_t m, int32_t t, int32_t* off_cam,
                                   int32_t* idx_cam, int32_t* off_pt, int32_t* idx_pt, sfmcov_error* err) {
    return guarded(h, err, [&] {
        if (!h->off_cam.p || !h->idx_cam.p || !h->off_pt.p || !h->idx_pt.p)
            throw ApiError{SFMCOV_ERR_INVARIANT, "batch", "no device index"};
        d2h(h, off_cam, h->off_cam.p, 4 * ((size_t)n + 1));
        d2h(h, off_pt, h->off_pt.p, 4 * ((size_t)m + 1));
        if (t) {
            d2h(h, idx_cam, h->idx_cam.p, 4 * (size_t)t);
            d2h(h, idx_pt, h->idx_pt.p, 4 * (size_t)t);
        }
    });
}

// Holds (lock = 1) or releases (0) the handle for a sequence of calls made
// by this thread -- the resident scene and staging of the batched
// sub-scene path must not be replaced by another thread's call in between.
void sfmcov_internal_session(sfmcov_handle* h, int32_t lock) {
    if (!h) return;
    if (lock) h->mu.lock();
    else h->mu.unlock();
}

void* sfmcov_internal_host_buffer(sfmcov_handle* h, int32_t slot, size_t bytes) {
    if (!h || slot < 0 || slot > 1) return nullptr;
    if (h->pinned_bytes[slot] < bytes) {
        if (h->pinned[slot]) cudaFreeHost(h->pinned[slot]);
        h->pinned[slot] = nullptr;
        h->pinned_bytes[slot] = 0;
        const size_t want = bytes + bytes / 4;  // headroom: chunks vary
        if (cudaSetDevice(h->device) != cudaSuccess || cudaHostAlloc(&h->pinned[slot], want, cudaHostAllocDefault) != cudaSuccess) {
            h->pinned[slot] = nullptr;
            return nullptr;
        }
        h->pinned_bytes[slot] = want;
    }
    return h->pinned[slot];
}

// The sub-reconstruction planner's view graph from the device pair list
// (subrec.cpp view_graph): the camera-pair blocks' observation-pair counts
// ARE the co-visibility counts (a camera observes a point at most once), so
// the index + pair-key sort that the covariance pipeline builds gives every
// edge weight in ~1 ms.  out: std::vector<int32_t>* of (a, b, w) triples,
// a < b, w >= min_covis, in (a, b) order.  The scene must be validated.
int32_t sfmcov_internal_covis(sfmcov_handle* h, const sfmcov_scene* full, int32_t min_covis, void* out,
                              sfmcov_error* err) {
    return guarded(h, err, [&] {
        auto& edges = *static_cast<std::vector<int32_t>*>(out);
        edges.clear();
        SceneDev sc;
        sc.n = full->n_cams; sc.m = full->n_pts; sc.t = full->n_obs; sc.P = full->cam_params;
        if ((long long)sc.n * sc.n >= (1LL << 32)) throw SizeGuard("subrec", "too many cameras for 32-bit pair keys");
        if (!sc.t) return;
        const sfmcov_scene& l = h->last_up;
        if (!(h->last_up_valid && l.obs_cam == full->obs_cam && l.obs_pt == full->obs_pt && l.n_obs == full->n_obs))
            h->last_up_valid = false;  // h_oc / h_op no longer hold the last uploaded scene's
        int* oc = (int*)h->h_oc.get(4 * (size_t)sc.t);
        int* op = (int*)h->h_op.get(4 * (size_t)sc.t);
        SFM_CUDA(cudaMemcpyAsync(oc, full->obs_cam, 4 * (size_t)sc.t, cudaMemcpyHostToDevice, h->s));
        SFM_CUDA(cudaMemcpyAsync(op, full->obs_pt, 4 * (size_t)sc.t, cudaMemcpyHostToDevice, h->s));
        sc.oc = oc;
        sc.op = op;
        IndexDev ix;
        ix.off_cam = h->off_cam.as<int>(sc.n + 1);
        ix.off_pt = h->off_pt.as<int>(sc.m + 1);
        ix.idx_cam = h->idx_cam.as<int>(sc.t);
        ix.idx_pt = h->idx_pt.as<int>(sc.t);
        ix.pos_cam = h->pos_cam.as<int>(sc.t);
        ix.key_scratch = h->key_scratch.as<int>(sc.t);
        launch_build_index(sc, ix, h->ws, h->s);
        build_pairs(sc, ix, h->pairs, h->ws_pairs, h->s);
        const PairDev& pd = h->pairs;
        std::vector<unsigned int> keys(pd.nseg);
        std::vector<long long> so((size_t)pd.nseg + 1);
        d2h(h, keys.data(), pd.ukeys, 4 * (size_t)pd.nseg);
        d2h(h, so.data(), pd.seg_off, 8 * ((size_t)pd.nseg + 1));
        const unsigned n = (unsigned)sc.n;
        for (int g = 0; g < pd.nseg; ++g) {
            const int a = (int)(keys[g] / n), b = (int)(keys[g] - (unsigned)a * n);
            const long long w = so[g + 1] - so[g];
            if (a != b && w >= min_covis) {
                edges.push_back(a);
                edges.push_back(b);
                edges.push_back((int32_t)w);
            }
        }
    });
}

// Internal (csrc/subrec.cpp; not in include/sfmcov_b200.h): the covariances
// of many sub-scenes of `full`, each given by its sorted camera ids, sorted
// point ids and ascending observation ids (the sub-scene induce_scene
// builds), in chunks of one pipeline run each.  Returns SFMCOV_OK with every
// sub-scene's blocks in cov (concatenated in scene and camera order), or
// SFMCOV_ERR_DEGENERATE with stage "batch" when any sub-scene fails anywhere:
// the caller then runs them one by one for the exact error.
int32_t sfmcov_internal_batch_covariance(sfmcov_handle* h, const sfmcov_scene* full, int32_t nscenes,
                                         const int32_t* cams, const int64_t* coff, const int32_t* pts,
                                         const int64_t* poff, const int32_t* obs, const int64_t* toff, double* cov,
                                         sfmcov_error* err) {
    return guarded(h, err, [&] {
        const auto t0 = std::chrono::steady_clock::now();
        const SceneDev sc = upload(h, full);
        if (sc.sigma_ready) SFM_CUDA(cudaStreamWaitEvent(h->s, sc.sigma_ready, 0));
        {
            static const bool timing = [] { const char* e = std::getenv("SFMCOV_SUBREC_TIMING"); return e && e[0] == '1'; }();
            if (timing) {
                SFM_CUDA(cudaStreamSynchronize(h->s));
                std::fprintf(stderr, "  batch upload     %8.3f ms\n",
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
            }
        }
        const int P = sc.P;
        int s0 = 0;
        while (s0 < nscenes) {  // chunks: <= 60000 cameras (32-bit pair keys), <= 12M observations
            int s1 = s0 + 1;
            while (s1 < nscenes && coff[s1 + 1] - coff[s0] <= 60000 && toff[s1 + 1] - toff[s0] <= 12000000) ++s1;
            try {
                run_batch_chunk(h, sc, s0, s1, cams, coff, pts, poff, obs, toff, cov + (size_t)P * P * coff[s0]);
            } catch (const BatchFallback&) {
                throw ApiError{SFMCOV_ERR_DEGENERATE, "batch", "a sub-scene failed; rerun them one by one"};
            }
            s0 = s1;
        }
    });
}

int32_t sfmcov_cuda_last_stage_times(sfmcov_handle* h, double* ms, int32_t capacity) {
    if (!h) return 0;
    const int k = std::min<int>(capacity, ST_COUNT);
    for (int i = 0; i < k; ++i) ms[i] = h->stage_ms[i];
    return k;
}

const char* sfmcov_cuda_stage_name(int32_t i) { return (i >= 0 && i < ST_COUNT) ? kStageNames[i] : ""; }

int32_t sfmcov_cuda_last_counts(sfmcov_handle* h, int64_t* counts, int32_t capacity) {
    if (!h) return 0;
    const int k = std::min(capacity, 10);
    for (int i = 0; i < k; ++i) counts[i] = h->counts[i];
    return k;
}

}  // extern "C"
