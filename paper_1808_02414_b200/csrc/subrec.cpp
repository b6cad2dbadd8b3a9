// Sub-reconstruction covariances (reference include/sfmcov/subrec.hpp,
// src/subrec.cpp): view graph, greedy neighborhoods, seeded coverings, and
// the per-camera aggregation over many independent sub-scene covariances.
//
// The planner is host logic (same algorithm, same std::mt19937_64 /
// uniform_int_distribution draws as the reference, so plans are identical).
// The B200 part is the batch: every sub-scene is an independent
// compute_covariance; a pool of worker threads, each with its own CUDA handle
// (stream, workspace), keeps several of them in flight on the device, and the
// results are aggregated in subset order afterwards (deterministic:
// smallest trace wins, earliest subset on ties, as in the reference).

#include "sfmcov_b200.h"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <climits>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

// capi.cu: all sub-scenes through one batched pipeline run per chunk
extern "C" int32_t sfmcov_internal_covis(sfmcov_handle* h, const sfmcov_scene* full, int32_t min_covis, void* out,
                                         sfmcov_error* err);
extern "C" int32_t sfmcov_internal_batch_begin(sfmcov_handle* h, const sfmcov_scene* full, sfmcov_error* err);
extern "C" int32_t sfmcov_internal_batch_chunk(sfmcov_handle* h, int32_t nscenes, const int32_t* cams,
                                               const int64_t* coff, const int32_t* pts, const int64_t* poff,
                                               const int32_t* obs, const int64_t* toff, double* cov,
                                               sfmcov_error* err);
extern "C" void* sfmcov_internal_host_buffer(sfmcov_handle* h, int32_t slot, size_t bytes);
extern "C" void sfmcov_internal_session(sfmcov_handle* h, int32_t lock);
extern "C" int32_t sfmcov_internal_last_index(sfmcov_handle* h, int32_t n, int32_t m, int32_t t, int32_t* off_cam,
                                              int32_t* idx_cam, int32_t* off_pt, int32_t* idx_pt, sfmcov_error* err);
extern "C" int32_t sfmcov_internal_batch_covariance(sfmcov_handle* h, const sfmcov_scene* full, int32_t nscenes,
                                                    const int32_t* cams, const int64_t* coff, const int32_t* pts,
                                                    const int64_t* poff, const int32_t* obs, const int64_t* toff,
                                                    double* cov, sfmcov_error* err);

namespace {

struct SubError {
    int32_t kind;
    std::string stage, message;  // message without the "stage: " prefix
};

void set_error(sfmcov_error* e, const SubError& x) {
    if (!e) return;
    e->kind = x.kind;
    std::snprintf(e->stage, sizeof e->stage, "%s", x.stage.c_str());
    std::snprintf(e->message, sizeof e->message, "%s: %s", x.stage.c_str(), x.message.c_str());
}

void clear(sfmcov_error* e) {
    if (!e) return;
    e->kind = 0;
    e->stage[0] = 0;
    e->message[0] = 0;
}

// Host copy of a scene (SoA, the C ABI layout).
struct HostScene {
    int32_t n = 0, m = 0, t = 0, P = 8;
    std::vector<double> cams, pts, u, sigma;
    std::vector<int32_t> oc, op;
    bool has_u = false, has_sigma = false;
    sfmcov_scene view() const {
        return sfmcov_scene{n, m, t, P, cams.data(), pts.data(), oc.data(), op.data(),
                            has_u ? u.data() : nullptr, has_sigma ? sigma.data() : nullptr};
    }
};

struct Graph {
    int64_t n = 0;
    std::vector<std::vector<std::pair<int32_t, int32_t>>> edges;  // (neighbor, weight), sorted
};

// build_view_graph (src/subrec.cpp:90-116): points' observers sorted, every
// pair counted; edges below min_covis dropped.
Graph view_graph(const sfmcov_scene& s, int min_covis) {
    std::vector<int64_t> off(s.n_pts + 1, 0);
    for (int32_t k = 0; k < s.n_obs; ++k) ++off[s.obs_pt[k] + 1];
    for (int32_t j = 0; j < s.n_pts; ++j) off[j + 1] += off[j];
    std::vector<int32_t> by_pt(s.n_obs), fill(off.begin(), off.end() - 1);
    for (int32_t k = 0; k < s.n_obs; ++k) by_pt[fill[s.obs_pt[k]]++] = k;
    Graph g;
    g.n = s.n_cams;
    g.edges.resize(s.n_cams);
    std::vector<int32_t> obs;
    auto for_pairs = [&](auto&& f) {
        for (int32_t j = 0; j < s.n_pts; ++j) {
            obs.clear();
            for (int64_t k = off[j]; k < off[j + 1]; ++k) obs.push_back(s.obs_cam[by_pt[k]]);
            std::sort(obs.begin(), obs.end());
            for (size_t a = 0; a < obs.size(); ++a)
                for (size_t b = a + 1; b < obs.size(); ++b) f(obs[a], obs[b]);
        }
    };
    const int64_t n = s.n_cams;
    if (n <= 8192) {  // dense pair counts (at most 256 MiB)
        std::vector<int32_t> cnt((size_t)n * n, 0);
        for_pairs([&](int32_t a, int32_t b) { ++cnt[(size_t)a * n + b]; });
        for (int64_t a = 0; a < n; ++a)
            for (int64_t b = a + 1; b < n; ++b) {
                const int32_t w = cnt[(size_t)a * n + b];
                if (w > 0 && w >= min_covis) {
                    g.edges[a].emplace_back((int32_t)b, w);
                    g.edges[b].emplace_back((int32_t)a, w);
                }
            }
    } else {  // sorted pair keys, run-length counted
        std::vector<uint64_t> keys;
        for_pairs([&](int32_t a, int32_t b) { keys.push_back((uint64_t(uint32_t(a)) << 32) | uint32_t(b)); });
        std::sort(keys.begin(), keys.end());
        for (size_t i = 0; i < keys.size();) {
            size_t e = i;
            while (e < keys.size() && keys[e] == keys[i]) ++e;
            const int32_t w = (int32_t)(e - i);
            if (w >= min_covis) {
                const int32_t a = int32_t(keys[i] >> 32), b = int32_t(keys[i] & 0xffffffffu);
                g.edges[a].emplace_back(b, w);
                g.edges[b].emplace_back(a, w);
            }
            i = e;
        }
    }
    for (auto& adj : g.edges) std::sort(adj.begin(), adj.end());
    return g;
}

// The same graph from the device pair list (capi.cu sfmcov_internal_covis:
// the co-visibility counts are the camera-pair blocks' observation-pair
// counts), for callers that hold a CUDA handle; the scene is validated.
Graph view_graph_device(sfmcov_handle* h, const sfmcov_scene& s, int min_covis) {
    std::vector<int32_t> e;
    sfmcov_error err{};
    if (const int32_t code = sfmcov_internal_covis(h, &s, min_covis, &e, &err)) {
        const std::string msg = err.message, st = err.stage;  // message is "stage: text"
        throw SubError{code, st, msg.rfind(st + ": ", 0) == 0 ? msg.substr(st.size() + 2) : msg};
    }
    Graph g;
    g.n = s.n_cams;
    g.edges.resize(s.n_cams);
    for (size_t k = 0; k + 2 < e.size(); k += 3) {
        g.edges[e[k]].emplace_back(e[k + 1], e[k + 2]);
        g.edges[e[k + 1]].emplace_back(e[k], e[k + 2]);
    }
    for (auto& adj : g.edges) std::sort(adj.begin(), adj.end());
    return g;
}

struct Sub {
    std::vector<int32_t> cams, pts, obs;  // sorted camera / point ids, ascending observation ids
    HostScene scene;                      // the induced scene's arrays (empty when built lists-only)
    bool truncated = false, has_scene = false;
};

// Observations by camera (ascending observation ids), built once per call so
// an induced scene only visits its own cameras' observations; the point id of
// each by-camera slot is stored beside it, so the filter below streams
// contiguous ranges instead of gathering obs_pt[t].
// Also each point's observing cameras (pt_off / pt_cam), for the filter's
// incremental removals.
struct ByCam {
    std::vector<int64_t> off, pt_off;
    std::vector<int32_t> idx, pt, pt_cam;
    // from the device's observation index (ascending observation ids within a
    // camera / point, as the host build below): two parallel gathers
    ByCam(const sfmcov_scene& s, const std::vector<int32_t>& off_cam, std::vector<int32_t>&& idx_cam,
          const std::vector<int32_t>& off_pt, const std::vector<int32_t>& idx_pt)
        : off(off_cam.begin(), off_cam.end()), pt_off(off_pt.begin(), off_pt.end()), idx(std::move(idx_cam)),
          pt(s.n_obs), pt_cam(s.n_obs) {
        const int64_t t = s.n_obs;
        const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(8, t / 65536));
        std::vector<std::thread> th;
        auto job = [&](int w) {
            for (int64_t k = t * w / nt; k < t * (w + 1) / nt; ++k) {
                pt[k] = s.obs_pt[idx[k]];
                pt_cam[k] = s.obs_cam[idx_pt[k]];
            }
        };
        for (int w = 1; w < nt; ++w) th.emplace_back(job, w);
        job(0);
        for (auto& x : th) x.join();
    }
    explicit ByCam(const sfmcov_scene& s)
        : off(s.n_cams + 1, 0), pt_off(s.n_pts + 1, 0), idx(s.n_obs), pt(s.n_obs), pt_cam(s.n_obs) {
        for (int32_t t = 0; t < s.n_obs; ++t) ++off[s.obs_cam[t] + 1];
        for (int32_t i = 0; i < s.n_cams; ++i) off[i + 1] += off[i];
        std::vector<int64_t> f(off.begin(), off.end() - 1);
        for (int32_t t = 0; t < s.n_obs; ++t) {
            const int64_t k = f[s.obs_cam[t]]++;
            idx[k] = t;
            pt[k] = s.obs_pt[t];
        }
        for (int32_t t = 0; t < s.n_obs; ++t) ++pt_off[s.obs_pt[t] + 1];
        for (int32_t j = 0; j < s.n_pts; ++j) pt_off[j + 1] += pt_off[j];
        std::vector<int64_t> g(pt_off.begin(), pt_off.end() - 1);
        for (int32_t t = 0; t < s.n_obs; ++t) pt_cam[g[s.obs_pt[t]]++] = s.obs_cam[t];
    }
};

// ByCam from the device index that view_graph_device just built (falls back to
// the host build if the index cannot be read)
ByCam bycam_device(sfmcov_handle* h, const sfmcov_scene& s) {
    if (s.n_obs == 0) return ByCam(s);  // (the device index is built only for observations)
    std::vector<int32_t> oc(s.n_cams + 1), ic(s.n_obs), op(s.n_pts + 1), ip(s.n_obs);
    sfmcov_error e{};
    if (sfmcov_internal_last_index(h, s.n_cams, s.n_pts, s.n_obs, oc.data(), ic.data(), op.data(), ip.data(), &e))
        return ByCam(s);
    return ByCam(s, oc, std::move(ic), op, ip);
}

// Scratch arrays of one planner thread, reset only where touched.
struct Scratch {
    std::vector<char> cam_in;
    std::vector<int32_t> pc, cc, cl, pl, queue;
    std::vector<uint64_t> obs_bits, pt_bits;
    void size(int64_t n, int64_t m, int64_t t) {
        if ((int64_t)cam_in.size() != n) { cam_in.assign(n, 0); cc.assign(n, 0); cl.assign(n, -1); }
        if ((int64_t)pc.size() != m) { pc.assign(m, 0); pl.assign(m, -1); pt_bits.assign((m + 63) / 64, 0); }
        if ((int64_t)obs_bits.size() != (t + 63) / 64) obs_bits.assign((t + 63) / 64, 0);
    }
};

// induced_scene's filter (src/subrec.cpp:24-86): points seen by >= 2 subset
// cameras, cameras with >= 4 surviving observations, to a fixpoint.  Leaves
// cam_in set for the surviving cameras and pc[j] = the point's surviving
// observer count; the caller resets them (reset_filter).
//
// The surviving set is the largest subset in which every camera keeps >= 4
// points seen twice (the property is closed under union), so removing failing
// cameras one at a time reaches the same fixpoint as the reference's rounds
// of simultaneous removals: one counting pass, then each removal updates the
// counts it changes (a point dropping to one observer costs its last
// surviving observer a good point) instead of recounting every camera.
void filter_fixpoint(const ByCam& bc, const std::vector<int32_t>& cams, Scratch& w) {
    for (int32_t c : cams) w.cam_in[c] = 1;
    for (int32_t c : cams)
        for (int64_t k = bc.off[c]; k < bc.off[c + 1]; ++k) ++w.pc[bc.pt[k]];
    std::vector<int32_t>& q = w.queue;
    q.clear();
    for (int32_t c : cams) {
        int32_t cnt = 0;
        for (int64_t k = bc.off[c]; k < bc.off[c + 1]; ++k) cnt += w.pc[bc.pt[k]] >= 2;
        w.cc[c] = cnt;
        if (cnt < 4) {
            w.cam_in[c] = 0;
            q.push_back(c);
        }
    }
    while (!q.empty()) {
        const int32_t c = q.back();
        q.pop_back();
        for (int64_t k = bc.off[c]; k < bc.off[c + 1]; ++k) {
            const int32_t j = bc.pt[k];
            if (--w.pc[j] != 1) continue;
            for (int64_t u = bc.pt_off[j]; u < bc.pt_off[j + 1]; ++u) {
                const int32_t c2 = bc.pt_cam[u];
                if (c2 != c && w.cam_in[c2]) {  // the point's one remaining counted observer, if still in
                    if (--w.cc[c2] < 4) {
                        w.cam_in[c2] = 0;
                        q.push_back(c2);
                    }
                    break;
                }
            }
        }
    }
}
void reset_filter(const ByCam& bc, const std::vector<int32_t>& cams, Scratch& w) {
    for (int32_t c : cams) {
        w.cam_in[c] = 0;
        w.cc[c] = 0;
        w.cl[c] = -1;
        for (int64_t k = bc.off[c]; k < bc.off[c + 1]; ++k) {
            w.pc[bc.pt[k]] = 0;
            w.pl[bc.pt[k]] = -1;
        }
    }
}

// The cameras that survive the induced filter (its fixpoint), ascending: the
// part of induced_scene the covering loop needs before its next draw.
std::vector<int32_t> induced_cams(const sfmcov_scene& s, const ByCam& bc, const std::vector<int32_t>& cams) {
    thread_local Scratch w;
    w.size(s.n_cams, s.n_pts, s.n_obs);
    filter_fixpoint(bc, cams, w);
    std::vector<int32_t> out;
    for (int32_t c : cams)
        if (w.cam_in[c]) out.push_back(c);
    std::sort(out.begin(), out.end());
    reset_filter(bc, cams, w);
    return out;
}

Sub induced(const sfmcov_scene& s, const ByCam& bc, const std::vector<int32_t>& cams, bool truncated,
            bool lists_only = false) {
    thread_local Scratch w;
    w.size(s.n_cams, s.n_pts, s.n_obs);
    filter_fixpoint(bc, cams, w);
    struct Reset {  // leave the scratch clean for the next call
        const ByCam& bc;
        const std::vector<int32_t>& cams;
        Scratch& w;
        ~Reset() { reset_filter(bc, cams, w); }
    } reset{bc, cams, w};
    // kept observations and points as bitmaps: scanning them gives ascending
    // observation ids (the reference's candidate order) and point ids
    int64_t t_lo = INT64_MAX, t_hi = -1, j_lo = INT64_MAX, j_hi = -1, nkept = 0;
    for (int32_t c : cams) {
        if (!w.cam_in[c]) continue;
        for (int64_t k = bc.off[c]; k < bc.off[c + 1]; ++k) {
            const int32_t j = bc.pt[k];
            if (w.pc[j] < 2) continue;
            const int64_t t = bc.idx[k];
            w.obs_bits[t >> 6] |= 1ULL << (t & 63);
            w.pt_bits[j >> 6] |= 1ULL << (j & 63);
            t_lo = std::min(t_lo, t); t_hi = std::max(t_hi, t);
            j_lo = std::min<int64_t>(j_lo, j); j_hi = std::max<int64_t>(j_hi, j);
            ++nkept;
        }
    }
    Sub sub;
    sub.truncated = truncated;
    const int P = s.cam_params;
    HostScene& h = sub.scene;
    h.P = P;
    h.has_u = s.obs_u != nullptr;
    h.has_sigma = s.obs_sigma != nullptr;
    {
        std::vector<int32_t> sorted_cams(cams.begin(), cams.end());
        std::sort(sorted_cams.begin(), sorted_cams.end());
        for (int32_t i : sorted_cams)
            if (w.cam_in[i]) {
                w.cl[i] = (int32_t)sub.cams.size();
                sub.cams.push_back(i);
            }
        h.cams.resize((size_t)P * sub.cams.size());
        for (size_t l = 0; l < sub.cams.size(); ++l)
            std::memcpy(&h.cams[(size_t)P * l], s.cams + (size_t)P * sub.cams[l], 8 * (size_t)P);
    }
    if (sub.cams.empty()) {
        for (int64_t t = t_lo; t <= t_hi; t += 64) w.obs_bits[t >> 6] = 0;
        throw SubError{SFMCOV_ERR_DEGENERATE, "subrec", "induced sub-reconstruction is empty"};
    }
    if (j_hi >= 0)
        for (int64_t wd = j_lo >> 6; wd <= (j_hi >> 6); ++wd)
            for (uint64_t bits = w.pt_bits[wd]; bits; bits &= bits - 1) {
                const int32_t j = (int32_t)(wd * 64 + __builtin_ctzll(bits));
                w.pl[j] = (int32_t)sub.pts.size();
                sub.pts.push_back(j);
            }
    if (lists_only) {  // ids only: the batched GPU path gathers the data from the resident scene
        sub.obs.reserve(nkept);
        if (t_hi >= 0)
            for (int64_t wd = t_lo >> 6; wd <= (t_hi >> 6); ++wd) {
                for (uint64_t bits = w.obs_bits[wd]; bits; bits &= bits - 1)
                    sub.obs.push_back((int32_t)(wd * 64 + __builtin_ctzll(bits)));
                w.obs_bits[wd] = 0;
            }
        if (j_hi >= 0)
            for (int64_t wd = j_lo >> 6; wd <= (j_hi >> 6); ++wd) w.pt_bits[wd] = 0;
        return sub;
    }
    sub.has_scene = true;
    h.pts.resize(3 * sub.pts.size());
    for (size_t l = 0; l < sub.pts.size(); ++l) std::memcpy(&h.pts[3 * l], s.pts + 3 * (size_t)sub.pts[l], 24);
    sub.obs.resize(nkept);
    h.oc.resize(nkept);
    h.op.resize(nkept);
    if (h.has_u) h.u.resize(2 * (size_t)nkept);
    if (h.has_sigma) h.sigma.resize(4 * (size_t)nkept);
    int64_t o = 0;
    if (t_hi >= 0)
        for (int64_t wd = t_lo >> 6; wd <= (t_hi >> 6); ++wd) {
            for (uint64_t bits = w.obs_bits[wd]; bits; bits &= bits - 1) {
                const int64_t t = wd * 64 + __builtin_ctzll(bits);
                sub.obs[o] = (int32_t)t;
                h.oc[o] = w.cl[s.obs_cam[t]];
                h.op[o] = w.pl[s.obs_pt[t]];
                if (h.has_u) std::memcpy(&h.u[2 * (size_t)o], s.obs_u + 2 * (size_t)t, 16);
                if (h.has_sigma) std::memcpy(&h.sigma[4 * (size_t)o], s.obs_sigma + 4 * (size_t)t, 32);
                ++o;
            }
            w.obs_bits[wd] = 0;
        }
    if (j_hi >= 0)
        for (int64_t wd = j_lo >> 6; wd <= (j_hi >> 6); ++wd) w.pt_bits[wd] = 0;
    h.n = (int32_t)sub.cams.size();
    h.m = (int32_t)sub.pts.size();
    h.t = (int32_t)h.oc.size();
    return sub;
}

// extract_neighborhood (src/subrec.cpp:118-152)
Sub neighborhood(const sfmcov_scene& s, const ByCam& bc, const Graph& g, int64_t center, int k_bar,
                 bool build = true) {
    const int64_t n = s.n_cams;
    if (k_bar < 2) throw SubError{SFMCOV_ERR_INVARIANT, "subrec", "subset size must be at least 2"};
    if (center < 0 || center >= n || g.n != n)
        throw SubError{SFMCOV_ERR_INVARIANT, "subrec", "center camera or view graph out of range"};
    std::vector<char> in(n, 0);
    std::vector<int64_t> weight(n, 0);
    std::vector<int32_t> chosen{(int32_t)center};
    in[center] = 1;
    for (const auto& [nb, w] : g.edges[center]) weight[nb] += w;
    bool truncated = false;
    while ((int)chosen.size() < k_bar) {
        int64_t best = -1, best_w = 0;
        for (int64_t i = 0; i < n; ++i)
            if (!in[i] && weight[i] > best_w) {
                best_w = weight[i];
                best = i;
            }
        if (best < 0) {
            truncated = true;
            break;
        }
        chosen.push_back((int32_t)best);
        in[best] = 1;
        for (const auto& [nb, w] : g.edges[best])
            if (!in[nb]) weight[nb] += w;
    }
    std::sort(chosen.begin(), chosen.end());
    if (build) return induced(s, bc, chosen, truncated);
    Sub sub;  // cameras only; the scene is built later
    sub.cams = induced_cams(s, bc, chosen);
    sub.truncated = truncated;
    if (sub.cams.empty()) throw SubError{SFMCOV_ERR_DEGENERATE, "subrec", "induced sub-reconstruction is empty"};
    return sub;
}

// plan_coverage (src/subrec.cpp:154-181); emit(sub) receives the subsets in
// the reference's order as they are drawn
template <class Emit>
void coverage_emit(const sfmcov_scene& s, const ByCam& bc, const Graph& g, int k_bar, uint64_t seed, bool build,
                   Emit&& emit) {
    const int64_t n = s.n_cams;
    std::mt19937_64 rng(seed);
    std::vector<char> covered(n, 0);
    int64_t remaining = n;
    std::vector<int64_t> pool;
    while (remaining > 0) {
        pool.clear();
        for (int64_t i = 0; i < n; ++i)
            if (!covered[i]) pool.push_back(i);
        const int64_t center = pool[std::uniform_int_distribution<std::size_t>(0, pool.size() - 1)(rng)];
        Sub sub = neighborhood(s, bc, g, center, k_bar, build);
        if (!std::binary_search(sub.cams.begin(), sub.cams.end(), (int32_t)center))
            throw SubError{SFMCOV_ERR_DEGENERATE, "subrec",
                           "camera " + std::to_string(center) + " cannot anchor a sub-reconstruction of size " +
                               std::to_string(k_bar)};
        for (int32_t c : sub.cams)
            if (!covered[c]) {
                covered[c] = 1;
                --remaining;
            }
        emit(std::move(sub));
    }
}

std::vector<Sub> coverage(const sfmcov_scene& s, const ByCam& bc, const Graph& g, int k_bar, uint64_t seed,
                          bool build = true) {
    std::vector<Sub> plan;
    coverage_emit(s, bc, g, k_bar, seed, build, [&](Sub&& sub) { plan.push_back(std::move(sub)); });
    return plan;
}

void check_scene(const sfmcov_scene* s) {
    if (!s || s->n_cams < 0 || s->n_pts < 0 || s->n_obs < 0 || (s->cam_params != 8 && s->cam_params != 9))
        throw SubError{SFMCOV_ERR_DIMENSION, "subrec", "bad scene"};
    for (int32_t k = 0; k < s->n_obs; ++k)
        if (s->obs_cam[k] < 0 || s->obs_cam[k] >= s->n_cams || s->obs_pt[k] < 0 || s->obs_pt[k] >= s->n_pts)
            throw SubError{SFMCOV_ERR_INVARIANT, "validate",
                           "observation " + std::to_string(k) + " index out of range"};
}

// SFMCOV_SUBREC_TIMING=1: wall time of each phase of a call on stderr.
struct PhaseClock {
    bool on = [] { const char* e = std::getenv("SFMCOV_SUBREC_TIMING"); return e && e[0] == '1'; }();
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "subrec %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// The covariance of every sub-scene, on `workers` handles of `device`.
struct SubResult {
    std::vector<double> cov;
    int32_t code = 0;
    sfmcov_error err{};
};

// One sub-scene at a time on `workers` handles (the fallback, and
// SFMCOV_SUBREC_BATCH=0): every Sub must have its scene built.
std::vector<SubResult> per_scene_covariances(sfmcov_handle* h0, const std::vector<const Sub*>& subs, int workers) {
    std::vector<SubResult> res(subs.size());
    // largest sub-scenes first: a worker's grow-only device buffers are then
    // sized by its first job, so later (smaller) ones never reallocate --
    // a cudaFree synchronises the whole device and stalls every worker
    std::vector<size_t> order(subs.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        const auto& x = subs[a]->scene;
        const auto& y = subs[b]->scene;
        return x.n != y.n ? x.n > y.n : x.t > y.t;
    });
    std::atomic<size_t> next{0};
    auto work = [&](sfmcov_handle* h) {
        for (size_t k = next++; k < subs.size(); k = next++) {
            const size_t i = order[k];
            const Sub& sb = *subs[i];
            const sfmcov_scene v = sb.scene.view();
            res[i].cov.resize((size_t)v.n_cams * v.cam_params * v.cam_params);
            sfmcov_options o{0, 0, 0, 0};
            res[i].code = sfmcov_cuda_compute_covariance(h, &v, &o, res[i].cov.data(), nullptr, &res[i].err);
        }
    };
    workers = std::max(1, std::min<int>(workers, (int)subs.size()));
    std::vector<sfmcov_handle*> hs;
    for (int w = 0; w < workers; ++w) {
        sfmcov_error e{};
        sfmcov_handle* h = sfmcov_cuda_worker(h0, w, &e);
        if (!h) break;
        hs.push_back(h);
    }
    if (hs.empty()) hs.push_back(h0);
    std::vector<std::thread> th;
    for (size_t w = 1; w < hs.size(); ++w) th.emplace_back(work, hs[w]);
    work(hs[0]);
    for (auto& t : th) t.join();
    return res;
}

bool subrec_batch_enabled() {
    static bool on = [] { const char* e = std::getenv("SFMCOV_SUBREC_BATCH"); return !(e && e[0] == '0'); }();
    return on;
}

// The covariance of every sub-scene: all of them through one batched
// pipeline run per chunk (capi.cu run_batch: one launch per stage over the
// concatenated sub-scenes, one dense sweep per sub-scene on worker streams);
// if any sub-scene fails anywhere, they are rerun one by one so the error is
// the reference's for the first failing subset.
std::vector<SubResult> batch_covariances(sfmcov_handle* h0, const sfmcov_scene& full, const ByCam& bc,
                                         const std::vector<Sub*>& subs, int workers) {
    const int P = full.cam_params;
    // (one sub-scene: nothing to batch -- and the single-scene pipeline keeps
    // a full-size window bitwise equal to compute_covariance, test_subrec.cpp:171-184)
    if (subrec_batch_enabled() && subs.size() > 1) {
        const size_t B = subs.size();
        std::vector<int64_t> coff(B + 1, 0), poff(B + 1, 0), toff(B + 1, 0);
        for (size_t i = 0; i < B; ++i) {
            coff[i + 1] = coff[i] + (int64_t)subs[i]->cams.size();
            poff[i + 1] = poff[i] + (int64_t)subs[i]->pts.size();
            toff[i + 1] = toff[i] + (int64_t)subs[i]->obs.size();
        }
        // uninitialised: the parallel copy below is the first touch of every page
        std::unique_ptr<int32_t[]> cams(new int32_t[coff[B] + 1]), pts(new int32_t[poff[B] + 1]),
            obs(new int32_t[toff[B] + 1]);
        {  // concatenated id lists, filled in parallel
            std::atomic<size_t> next{0};
            auto job = [&] {
                for (size_t i = next++; i < B; i = next++) {
                    std::copy(subs[i]->cams.begin(), subs[i]->cams.end(), cams.get() + coff[i]);
                    std::copy(subs[i]->pts.begin(), subs[i]->pts.end(), pts.get() + poff[i]);
                    std::copy(subs[i]->obs.begin(), subs[i]->obs.end(), obs.get() + toff[i]);
                }
            };
            const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), 16));
            std::vector<std::thread> th;
            for (int i = 1; i < nt; ++i) th.emplace_back(job);
            job();
            for (auto& t : th) t.join();
        }
        PhaseClock lc;
        std::vector<double> cov((size_t)P * P * coff[B] + 1);
        sfmcov_error e{};
        const int32_t code = sfmcov_internal_batch_covariance(h0, &full, (int32_t)subs.size(), cams.get(), coff.data(),
                                                              pts.get(), poff.data(), obs.get(), toff.data(),
                                                              cov.data(), &e);
        lc.mark("batched_gpu");
        if (code != SFMCOV_OK && PhaseClock{}.on) std::fprintf(stderr, "subrec batch fallback: %s\n", e.message);
        if (code == SFMCOV_OK) {
            std::vector<SubResult> res(subs.size());
            for (size_t i = 0; i < subs.size(); ++i)
                res[i].cov.assign(cov.begin() + (size_t)P * P * coff[i], cov.begin() + (size_t)P * P * coff[i + 1]);
            return res;
        }
    }
    {  // the per-sub-scene path needs the induced scenes' arrays
        std::atomic<size_t> next{0};
        auto job = [&] {
            for (size_t i = next++; i < subs.size(); i = next++)
                if (!subs[i]->has_scene) {
                    Sub built = induced(full, bc, subs[i]->cams, subs[i]->truncated);
                    subs[i]->scene = std::move(built.scene);
                    subs[i]->has_scene = true;
                }
        };
        const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), 32));
        std::vector<std::thread> th;
        for (int i = 1; i < nt; ++i) th.emplace_back(job);
        job();
        for (auto& t : th) t.join();
    }
    std::vector<const Sub*> cs(subs.begin(), subs.end());
    return per_scene_covariances(h0, cs, workers);
}

double trace_of(const double* c, int P) {
    double tr = 0.0;
    for (int p = 0; p < P; ++p) tr += c[P * p + p];
    return tr;
}

template <class F>
int32_t guarded(sfmcov_error* err, F&& body) {
    try {
        body();
        clear(err);
        return SFMCOV_OK;
    } catch (const SubError& x) {
        set_error(err, x);
        return x.kind;
    } catch (const std::exception& x) {
        set_error(err, SubError{SFMCOV_ERR_DEVICE, "subrec", x.what()});
        return SFMCOV_ERR_DEVICE;
    }
}

// "stage: message" -> message
std::string strip_stage(const sfmcov_error& e) {
    const std::string full = e.message;
    const std::string pre = std::string(e.stage) + ": ";
    return full.compare(0, pre.size(), pre) == 0 ? full.substr(pre.size()) : full;
}

// approximate_covariances' planning, inducing and device work as one
// pipeline: a planner thread per covering emits its subsets in the
// reference's order as they are drawn, a pool induces them (id lists), and
// this thread packs induced subsets into device chunks (<= 60000 cameras,
// <= 12M observations) in pinned staging and runs them while the planners
// and inducers keep going.  Results are kept per subset, so the aggregation
// (in covering-major subset order afterwards) is independent of the chunking;
// errors keep the sequential path's precedence (planning, then inducing in
// subset order, then the covariances).  A chunk with a failing sub-scene is
// rerun one sub-scene at a time; a single subset in total takes the
// single-scene path.  Outputs flat / deco / res in covering-major order.
// SFMCOV_SUBREC_MIN_CHUNK: sub-scenes that make a device chunk worth starting
// while the planners are still drawing (default 24)
int pipe_min_chunk() {
    static int v = [] {
        const char* e = std::getenv("SFMCOV_SUBREC_MIN_CHUNK");
        const int x = e ? std::atoi(e) : 24;
        return x >= 1 ? x : 24;
    }();
    return v;
}

// The first failure in the reference's order (src/subrec.cpp:202-222):
// covering d is drawn (neighborhoods and induced scenes, subset by subset)
// before any of its subsets is computed, and the coverings run in turn.
// key = d 2^33 + (0 drawing | 1 computing) 2^32 + the subset's index in d;
// a sharded call reports its own first key and the merge keeps the smallest.
struct FirstFailure {
    int64_t key = INT64_MAX;
    SubError err;
    static int64_t at(int d, int phase, size_t i) {
        return ((int64_t)d << 33) | ((int64_t)phase << 32) | (int64_t)i;
    }
    void note(int64_t k, const SubError& e) {
        if (k < key) {
            key = k;
            err = e;
        }
    }
    bool any() const { return key != INT64_MAX; }
};

struct PipeItem {
    Sub sub;
    int deco = 0;
    size_t idx = 0;  // index within its covering
    bool skip = false;  // another rank's subset (sharded call): planned, not computed
    bool ind_fail = false, done = false;
    SubError ind_err;
    SubResult res;
};

void pipelined_covariances(sfmcov_handle* h, const sfmcov_scene& scene, const ByCam& bc, const Graph& g, int k_bar,
                           int n_dec, uint64_t seed, int workers, std::vector<std::deque<PipeItem>>& plans,
                           std::vector<const Sub*>& flat, std::vector<int>& deco, std::vector<SubResult>& res,
                           FirstFailure& ff, std::vector<char>* mine = nullptr, int nranks = 1, int rank = 0) {
    const int P = scene.cam_params;
    plans.assign(n_dec, {});  // deque: stable addresses while planners append (the Subs outlive this call)
    std::mutex mu;
    std::condition_variable cv;
    std::deque<PipeItem*> to_induce, ready_q;
    int planners_left = n_dec, inducing = 0;
    size_t planned = 0;
    {
        sfmcov_error e{};
        if (const int32_t c = sfmcov_internal_batch_begin(h, &scene, &e)) throw SubError{c, e.stage, strip_stage(e)};
    }
    std::vector<std::thread> th;
    for (int d = 0; d < n_dec; ++d)
        th.emplace_back([&, d] {
            try {
                coverage_emit(scene, bc, g, k_bar, seed + uint64_t(d), false, [&](Sub&& sb) {
                    std::lock_guard<std::mutex> lk(mu);
                    const size_t i = plans[d].size();
                    plans[d].emplace_back();
                    PipeItem& it = plans[d].back();
                    it.sub = std::move(sb);
                    it.deco = d;
                    it.idx = i;
                    // sharded call: subset i of covering d belongs to rank (i n_dec + d) mod R
                    it.skip = nranks > 1 && (int)((i * (size_t)n_dec + (size_t)d) % (size_t)nranks) != rank;
                    if (!it.skip) to_induce.push_back(&it);
                    ++planned;  // all ranks' subsets: one in total takes the single-scene path
                    cv.notify_all();
                });
            } catch (const SubError& x) {  // drawing subset plans[d].size() of covering d failed
                std::lock_guard<std::mutex> lk(mu);
                ff.note(FirstFailure::at(d, 0, plans[d].size()), x);
            } catch (const std::exception& x) {
                std::lock_guard<std::mutex> lk(mu);
                ff.note(FirstFailure::at(d, 0, plans[d].size()), SubError{SFMCOV_ERR_DEVICE, "subrec", x.what()});
            }
            std::lock_guard<std::mutex> lk(mu);
            --planners_left;
            cv.notify_all();
        });
    const int n_ind = std::max(2, std::min<int>((int)std::thread::hardware_concurrency() - n_dec - 1, 32));
    for (int w = 0; w < n_ind; ++w)
        th.emplace_back([&] {
            for (;;) {
                PipeItem* it = nullptr;
                {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return !to_induce.empty() || planners_left == 0; });
                    if (to_induce.empty()) return;
                    it = to_induce.front();
                    to_induce.pop_front();
                    ++inducing;
                }
                try {
                    Sub full = induced(scene, bc, it->sub.cams, it->sub.truncated, true);
                    it->sub.pts = std::move(full.pts);
                    it->sub.obs = std::move(full.obs);
                } catch (const SubError& x) {
                    it->ind_err = x;
                    it->ind_fail = true;
                } catch (const std::exception& x) {
                    it->ind_err = SubError{SFMCOV_ERR_DEVICE, "subrec", x.what()};
                    it->ind_fail = true;
                }
                std::lock_guard<std::mutex> lk(mu);
                --inducing;
                if (!it->ind_fail) ready_q.push_back(it);
                cv.notify_all();
            }
        });
    // device chunks, packed in arrival order
    std::exception_ptr gpu_error;
    std::vector<PipeItem*> fallback;
    int slot = 0;
    for (;;) {
        std::vector<PipeItem*> chunk;
        int64_t nc = 0, nt = 0;
        bool finished = false;
        {
            std::unique_lock<std::mutex> lk(mu);
            for (;;) {
                const bool all_in = planners_left == 0 && to_induce.empty() && inducing == 0;
                while (!ready_q.empty()) {
                    PipeItem* it = ready_q.front();
                    const int64_t c = (int64_t)it->sub.cams.size(), t = (int64_t)it->sub.obs.size();
                    if (!chunk.empty() && (nc + c > 60000 || nt + t > 12000000)) break;
                    chunk.push_back(it);
                    ready_q.pop_front();
                    nc += c;
                    nt += t;
                }
                const bool full_chunk = !ready_q.empty();  // the next subset did not fit
                // the device is idle while this thread waits: go as soon as a
                // useful batch is ready instead of waiting for a full chunk
                const bool enough = (int)chunk.size() >= pipe_min_chunk();
                if (full_chunk || enough || (all_in && ready_q.empty())) {
                    finished = all_in && ready_q.empty();
                    break;
                }
                cv.wait(lk);
            }
            // a single subset in total, or one beyond a chunk's limits on its
            // own, takes the single-scene path (below)
            if ((finished && planned == 1) ||
                (chunk.size() == 1 && (nc > 60000 || nt > 12000000))) {
                for (PipeItem* it : chunk) fallback.push_back(it);
                chunk.clear();
            }
        }
        if (!chunk.empty() && !gpu_error) try {
            const size_t B = chunk.size();
            std::vector<int64_t> coff(B + 1, 0), poff(B + 1, 0), toff(B + 1, 0);
            for (size_t i = 0; i < B; ++i) {
                coff[i + 1] = coff[i] + (int64_t)chunk[i]->sub.cams.size();
                poff[i + 1] = poff[i] + (int64_t)chunk[i]->sub.pts.size();
                toff[i + 1] = toff[i] + (int64_t)chunk[i]->sub.obs.size();
            }
            const size_t ints = (size_t)(coff[B] + poff[B] + toff[B]) + 1;
            int32_t* buf = static_cast<int32_t*>(sfmcov_internal_host_buffer(h, slot, 4 * ints));
            std::vector<int32_t> heap;
            if (!buf) {  // no pinned memory: pageable staging
                heap.resize(ints);
                buf = heap.data();
            }
            slot ^= 1;
            int32_t* cams = buf;
            int32_t* pts = cams + coff[B];
            int32_t* obs = pts + poff[B];
            {  // concatenated id lists (tens of MB): filled by several threads
                std::atomic<size_t> next{0};
                auto job = [&] {
                    for (size_t i = next++; i < B; i = next++) {
                        const Sub& sb = chunk[i]->sub;
                        std::copy(sb.cams.begin(), sb.cams.end(), cams + coff[i]);
                        std::copy(sb.pts.begin(), sb.pts.end(), pts + poff[i]);
                        std::copy(sb.obs.begin(), sb.obs.end(), obs + toff[i]);
                    }
                };
                const int ncp = (int)std::min<size_t>(B, 8);
                std::vector<std::thread> cp;
                for (int i = 1; i < ncp; ++i) cp.emplace_back(job);
                job();
                for (auto& t : cp) t.join();
            }
            std::vector<double> cov((size_t)P * P * coff[B] + 1);
            sfmcov_error e{};
            const int32_t code = sfmcov_internal_batch_chunk(h, (int32_t)B, cams, coff.data(), pts, poff.data(), obs,
                                                             toff.data(), cov.data(), &e);
            if (code == SFMCOV_OK) {
                for (size_t i = 0; i < B; ++i) {
                    chunk[i]->res.cov.assign(cov.begin() + (size_t)P * P * coff[i],
                                             cov.begin() + (size_t)P * P * coff[i + 1]);
                    chunk[i]->done = true;
                }
            } else if (code == SFMCOV_ERR_DEGENERATE) {
                if (PhaseClock{}.on) std::fprintf(stderr, "subrec batch fallback: %s\n", e.message);
                for (PipeItem* it : chunk) fallback.push_back(it);
            } else {
                gpu_error = std::make_exception_ptr(SubError{code, e.stage, strip_stage(e)});
            }
        } catch (...) {  // the planners and inducers are still running: join them first
            gpu_error = std::current_exception();
        }
        if (finished) break;
    }
    for (auto& t : th) t.join();
    if (gpu_error) std::rethrow_exception(gpu_error);
    flat.clear();
    deco.clear();
    std::vector<PipeItem*> items;
    for (int d = 0; d < n_dec; ++d)
        for (PipeItem& it : plans[d]) items.push_back(&it);
    for (PipeItem* it : items)  // (only this rank's subsets are induced)
        if (it->ind_fail) ff.note(FirstFailure::at(it->deco, 0, it->idx), it->ind_err);
    if (!fallback.empty()) {  // one sub-scene at a time (the single-scene path; exact per-subset errors)
        std::vector<Sub*> subs;
        for (PipeItem* it : fallback) subs.push_back(&it->sub);
        std::vector<SubResult> r;
        if (subs.size() == 1) {
            r = batch_covariances(h, scene, bc, subs, workers);
        } else {
            std::atomic<size_t> next{0};
            auto job = [&] {
                for (size_t i = next++; i < subs.size(); i = next++) {
                    Sub built = induced(scene, bc, subs[i]->cams, subs[i]->truncated);
                    subs[i]->scene = std::move(built.scene);
                    subs[i]->has_scene = true;
                }
            };
            std::vector<std::thread> bt;
            const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), 32));
            for (int i = 1; i < nt; ++i) bt.emplace_back(job);
            job();
            for (auto& t : bt) t.join();
            std::vector<const Sub*> cs(subs.begin(), subs.end());
            r = per_scene_covariances(h, cs, workers);
        }
        for (size_t i = 0; i < fallback.size(); ++i) {
            fallback[i]->res = std::move(r[i]);
            fallback[i]->done = true;
        }
    }
    res.clear();
    if (mine) mine->clear();
    for (PipeItem* it : items) {
        flat.push_back(&it->sub);
        deco.push_back(it->deco);
        res.push_back(it->res);
        if (mine) mine->push_back(it->skip ? 0 : 1);
    }
}


// rec.validate() of the full scene on the device (the M_INDEX path of the
// CUDA library), its error passed through unchanged, as the reference's
// approximate_covariances / error_size_sweep do before planning
// (src/subrec.cpp:191, 262).
void validate_full(sfmcov_handle* h, const sfmcov_scene* s) {
    const size_t t = s->n_obs > 0 ? (size_t)s->n_obs : 1;
    std::vector<int64_t> oc((size_t)s->n_cams + 1), op((size_t)s->n_pts + 1);
    std::vector<int32_t> ic(t), ip(t);
    sfmcov_error e{};
    if (int32_t c = sfmcov_cuda_observation_index(h, s, oc.data(), ic.data(), op.data(), ip.data(), &e))
        throw SubError{c, e.stage, strip_stage(e)};
}

}  // namespace

extern "C" {

static void graph_csr(const Graph& g, int64_t* off, int32_t* nbr, int32_t* weight, int64_t capacity, int64_t* n_entries) {
    int64_t k = 0;
    off[0] = 0;
    for (int64_t i = 0; i < g.n; ++i) {
        for (const auto& [b, w] : g.edges[i]) {
            if (k < capacity) { nbr[k] = b; weight[k] = w; }
            ++k;
        }
        off[i + 1] = k;
    }
    *n_entries = k;
}

int32_t sfmcov_view_graph(const sfmcov_scene* scene, int32_t min_covis, int64_t* off, int32_t* nbr, int32_t* weight,
                          int64_t capacity, int64_t* n_entries, sfmcov_error* err) {
    return guarded(err, [&] {
        check_scene(scene);
        graph_csr(view_graph(*scene, min_covis), off, nbr, weight, capacity, n_entries);
    });
}

int32_t sfmcov_cuda_view_graph(sfmcov_handle* h, const sfmcov_scene* scene, int32_t min_covis, int64_t* off,
                               int32_t* nbr, int32_t* weight, int64_t capacity, int64_t* n_entries, sfmcov_error* err) {
    return guarded(err, [&] {
        if (!scene) throw SubError{SFMCOV_ERR_DIMENSION, "subrec", "bad scene"};
        validate_full(h, scene);
        check_scene(scene);
        graph_csr(view_graph_device(h, *scene, min_covis), off, nbr, weight, capacity, n_entries);
    });
}

int32_t sfmcov_extract_neighborhood(const sfmcov_scene* scene, int64_t center, int32_t k_bar, int32_t* cams,
                                    int64_t* n_cams, int32_t* pts, int64_t* n_pts, int32_t* truncated,
                                    sfmcov_error* err) {
    return guarded(err, [&] {
        check_scene(scene);
        const Graph g = view_graph(*scene, 1);
        const ByCam bc(*scene);
        const Sub sub = neighborhood(*scene, bc, g, center, k_bar);
        std::copy(sub.cams.begin(), sub.cams.end(), cams);
        std::copy(sub.pts.begin(), sub.pts.end(), pts);
        *n_cams = (int64_t)sub.cams.size();
        *n_pts = (int64_t)sub.pts.size();
        *truncated = sub.truncated ? 1 : 0;
    });
}

int32_t sfmcov_plan_coverage(const sfmcov_scene* scene, int32_t k_bar, uint64_t seed, int64_t* subset_off,
                             int64_t subset_capacity, int32_t* cams, int64_t cams_capacity, int64_t* n_subsets,
                             sfmcov_error* err) {
    return guarded(err, [&] {
        check_scene(scene);
        const Graph g = view_graph(*scene, 1);
        const ByCam bc(*scene);
        const std::vector<Sub> plan = coverage(*scene, bc, g, k_bar, seed, false);
        int64_t k = 0;
        subset_off[0] = 0;
        for (size_t i = 0; i < plan.size(); ++i) {
            for (int32_t c : plan[i].cams) {
                if (k < cams_capacity) cams[k] = c;
                ++k;
            }
            if ((int64_t)i + 1 < subset_capacity + 1) subset_off[i + 1] = k;
        }
        *n_subsets = (int64_t)plan.size();
    });
}

static int32_t approximate_impl(sfmcov_handle* h, const sfmcov_scene* scene, int32_t k_bar, int32_t n_decompositions,
                                uint64_t seed, int32_t workers, int32_t nranks, int32_t rank, double* cam_cov,
                                double* trace, int32_t* subset_id, int64_t* failed_key, sfmcov_error* err) {
    if (failed_key) *failed_key = -1;
    return guarded(err, [&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) throw SubError{SFMCOV_ERR_INVARIANT, "subrec", "bad rank / rank count"};
        if (k_bar < 2) throw SubError{SFMCOV_ERR_INVARIANT, "subrec", "subset size must be at least 2"};
        if (n_decompositions < 1) throw SubError{SFMCOV_ERR_INVARIANT, "subrec", "need at least one decomposition"};
        if (!scene) throw SubError{SFMCOV_ERR_DIMENSION, "subrec", "bad scene"};
        // the whole call is one session on the handle: the scene that
        // validation uploads is reused by the batched chunks
        struct Session {
            sfmcov_handle* h;
            explicit Session(sfmcov_handle* x) : h(x) { sfmcov_internal_session(h, 1); }
            ~Session() { sfmcov_internal_session(h, 0); }
        } session(h);
        PhaseClock clk;
        validate_full(h, scene);
        check_scene(scene);
        clk.mark("validate");
        const int P = scene->cam_params;
        const Graph g = view_graph_device(h, *scene, 1);
        const ByCam bc = bycam_device(h, *scene);
        std::vector<const Sub*> flat;
        std::vector<int> deco;
        std::vector<SubResult> res;
        std::vector<std::vector<Sub>> plans;
        std::vector<std::deque<PipeItem>> store;
        std::vector<char> mine;  // sharded call: this rank's subsets (empty: all)
        FirstFailure ff;
        if (subrec_batch_enabled()) {
            // planning, inducing and the device chunks overlapped (one pipeline)
            pipelined_covariances(h, *scene, bc, g, k_bar, n_decompositions, seed, std::max(1, (int)workers), store,
                                  flat, deco, res, ff, nranks > 1 ? &mine : nullptr, nranks, rank);
            clk.mark("pipeline");
        } else {
            // (one-by-one path: a sharded call computes every subset here;
            // the merge still equals the single call)
            // the coverings are independent (one seed each): drawn in parallel
            plans.resize(n_decompositions);
            {
                std::mutex fmu;
                std::vector<std::thread> th;
                for (int d = 0; d < n_decompositions; ++d)
                    th.emplace_back([&, d] {
                        try {
                            coverage_emit(*scene, bc, g, k_bar, seed + uint64_t(d), false,
                                          [&](Sub&& sb) { plans[d].push_back(std::move(sb)); });
                        } catch (const SubError& x) {
                            std::lock_guard<std::mutex> lk(fmu);
                            ff.note(FirstFailure::at(d, 0, plans[d].size()), x);
                        }
                    });
                for (auto& t : th) t.join();
            }
            clk.mark("plan");
            std::vector<size_t> idx;
            for (int d = 0; d < n_decompositions; ++d)
                for (size_t i = 0; i < plans[d].size(); ++i) {
                    flat.push_back(&plans[d][i]);
                    deco.push_back(d);
                    idx.push_back(i);
                }
            std::vector<char> bfail(flat.size(), 0);
            {  // induced scenes of every subset, in parallel (host)
                std::atomic<size_t> next{0};
                std::vector<SubError> berr(flat.size());
                auto job = [&] {
                    for (size_t i = next++; i < flat.size(); i = next++) {
                        Sub& sb = const_cast<Sub&>(*flat[i]);
                        try {
                            Sub full = induced(*scene, bc, sb.cams, sb.truncated, false);
                            sb.scene = std::move(full.scene);
                            sb.pts = std::move(full.pts);
                            sb.obs = std::move(full.obs);
                            sb.has_scene = full.has_scene;
                        } catch (const SubError& x) {
                            berr[i] = x;
                            bfail[i] = 1;
                        }
                    }
                };
                const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), 32));
                std::vector<std::thread> th;
                for (int i = 1; i < nt; ++i) th.emplace_back(job);
                job();
                for (auto& t : th) t.join();
                for (size_t i = 0; i < flat.size(); ++i)
                    if (bfail[i]) ff.note(FirstFailure::at(deco[i], 0, idx[i]), berr[i]);
            }
            clk.mark("induce");
            std::vector<Sub*> mflat;
            std::vector<size_t> at;
            for (size_t i = 0; i < flat.size(); ++i)
                if (!bfail[i]) {
                    mflat.push_back(const_cast<Sub*>(flat[i]));
                    at.push_back(i);
                }
            std::vector<SubResult> got = batch_covariances(h, *scene, bc, mflat, std::max(1, (int)workers));
            res.assign(flat.size(), SubResult{});
            for (size_t k = 0; k < at.size(); ++k) res[at[k]] = std::move(got[k]);
        }
        clk.mark("covariances");
        const int64_t n = scene->n_cams;
        std::vector<char> seen(n, 0);
        {  // the first failure in the reference's order (FirstFailure)
            std::vector<size_t> in_deco(n_decompositions, 0);
            for (size_t sid = 0; sid < flat.size(); ++sid) {
                const size_t i = in_deco[deco[sid]]++;
                if ((!mine.empty() && !mine[sid]) || !res[sid].code) continue;  // another rank's subset, or fine
                ff.note(FirstFailure::at(deco[sid], 1, i),
                        SubError{res[sid].code, "subrec",
                                 "subset " + std::to_string(sid) + " (decomposition " + std::to_string(deco[sid]) +
                                     "): " + std::string(res[sid].err.message)});
            }
            if (ff.any()) {
                if (failed_key) *failed_key = ff.key;
                throw ff.err;
            }
        }
        for (size_t sid = 0; sid < flat.size(); ++sid) {
            if (!mine.empty() && !mine[sid]) continue;  // another rank's subset
            const Sub& sb = *flat[sid];
            for (size_t l = 0; l < sb.cams.size(); ++l) {
                const int32_t gc = sb.cams[l];
                const double* c = &res[sid].cov[(size_t)P * P * l];
                const double tr = trace_of(c, P);
                if (!seen[gc] || tr < trace[gc]) {
                    seen[gc] = 1;
                    std::memcpy(cam_cov + (size_t)P * P * gc, c, 8 * (size_t)P * P);
                    trace[gc] = tr;
                    subset_id[gc] = (int32_t)sid;
                }
            }
        }
        for (int64_t i = 0; i < n; ++i)
            if (!seen[i]) {
                if (nranks > 1) {  // (covered by another rank's subsets, or checked after the merge)
                    trace[i] = INFINITY;
                    subset_id[i] = -1;
                    std::memset(cam_cov + (size_t)P * P * i, 0, 8 * (size_t)P * P);
                    continue;
                }
                throw SubError{SFMCOV_ERR_INVARIANT, "subrec", "camera " + std::to_string(i) + " was not covered by any subset"};
            }
        clk.mark("aggregate");
    });
}

int32_t sfmcov_cuda_approximate_covariances(sfmcov_handle* h, const sfmcov_scene* scene, int32_t k_bar,
                                            int32_t n_decompositions, uint64_t seed, int32_t workers,
                                            double* cam_cov, double* trace, int32_t* subset_id, sfmcov_error* err) {
    return approximate_impl(h, scene, k_bar, n_decompositions, seed, workers, 1, 0, cam_cov, trace, subset_id, nullptr,
                            err);
}

int32_t sfmcov_cuda_approximate_covariances_shard(sfmcov_handle* h, const sfmcov_scene* scene, int32_t k_bar,
                                                  int32_t n_decompositions, uint64_t seed, int32_t workers,
                                                  int32_t nranks, int32_t rank, double* cam_cov, double* trace,
                                                  int32_t* subset_id, int64_t* failed_key, sfmcov_error* err) {
    return approximate_impl(h, scene, k_bar, n_decompositions, seed, workers, nranks, rank, cam_cov, trace, subset_id,
                            failed_key, err);
}

int32_t sfmcov_cuda_monotonicity_check(sfmcov_handle* h, const sfmcov_scene* scene, const int32_t* small_cams,
                                       int64_t n_small, const int32_t* large_cams, int64_t n_large, double rel_tol,
                                       int32_t* violation_cams, double* trace_small, double* trace_large,
                                       int64_t* n_violations, int64_t* cameras_checked, sfmcov_error* err) {
    return guarded(err, [&] {
        check_scene(scene);
        std::vector<int32_t> sc(small_cams, small_cams + n_small), lc(large_cams, large_cams + n_large);
        for (int32_t c : sc) {
            if (c < 0 || c >= scene->n_cams) throw SubError{SFMCOV_ERR_INVARIANT, "subrec", "subset camera id out of range"};
            if (!std::binary_search(lc.begin(), lc.end(), c))
                throw SubError{SFMCOV_ERR_INVARIANT, "subrec",
                               "subsets are not nested: camera " + std::to_string(c) + " is missing from the larger subset"};
        }
        const ByCam bc(*scene);
        const Sub s_small = induced(*scene, bc, sc, false), s_large = induced(*scene, bc, lc, false);
        const int P = scene->cam_params;
        std::vector<double> cs((size_t)P * P * s_small.cams.size()), cl((size_t)P * P * s_large.cams.size());
        sfmcov_options o{0, 0, 0, 0};
        sfmcov_error e{};
        const sfmcov_scene vs = s_small.scene.view(), vl = s_large.scene.view();
        if (int32_t c = sfmcov_cuda_compute_covariance(h, &vs, &o, cs.data(), nullptr, &e))
            throw SubError{c, e.stage, strip_stage(e)};
        if (int32_t c = sfmcov_cuda_compute_covariance(h, &vl, &o, cl.data(), nullptr, &e))
            throw SubError{c, e.stage, strip_stage(e)};
        int64_t nv = 0, checked = 0;
        for (size_t l = 0; l < s_small.cams.size(); ++l) {
            const int32_t gcam = s_small.cams[l];
            const size_t pos = std::lower_bound(s_large.cams.begin(), s_large.cams.end(), gcam) - s_large.cams.begin();
            const double ts = trace_of(&cs[(size_t)P * P * l], P), tl = trace_of(&cl[(size_t)P * P * pos], P);
            ++checked;
            if (ts < tl - rel_tol * std::abs(tl)) {
                violation_cams[nv] = gcam;
                trace_small[nv] = ts;
                trace_large[nv] = tl;
                ++nv;
            }
        }
        *n_violations = nv;
        *cameras_checked = checked;
    });
}

// error_size_sweep (src/subrec.cpp:258-297): per window size, subsets_per_size
// centers drawn from a seeded shuffle; every subset camera's block compared
// with the full-scene block (Frobenius).  Rows: (k_bar, subset, camera,
// err_relative, err_absolute, trace) x capacity.
int32_t sfmcov_cuda_error_size_sweep(sfmcov_handle* h, const sfmcov_scene* scene, const int32_t* sizes, int32_t n_sizes,
                                     int32_t subsets_per_size, uint64_t seed, int32_t workers, int32_t* row_ints,
                                     double* row_vals, int64_t capacity, int64_t* n_rows, sfmcov_error* err) {
    return guarded(err, [&] {
        if (subsets_per_size < 1) throw SubError{SFMCOV_ERR_INVARIANT, "subrec", "need at least one subset per size"};
        if (!scene) throw SubError{SFMCOV_ERR_DIMENSION, "subrec", "bad scene"};
        validate_full(h, scene);
        check_scene(scene);
        const int P = scene->cam_params;
        const int64_t n = scene->n_cams;
        std::vector<double> full((size_t)P * P * n);
        {
            sfmcov_options o{0, 0, 0, 0};
            sfmcov_error e{};
            if (int32_t c = sfmcov_cuda_compute_covariance(h, scene, &o, full.data(), nullptr, &e))
                throw SubError{c, e.stage, strip_stage(e)};
        }
        const Graph g = view_graph_device(h, *scene, 1);
        const ByCam bc = bycam_device(h, *scene);
        std::mt19937_64 rng(seed);
        std::vector<int64_t> ids(n);
        std::vector<Sub> subs;
        std::vector<int> kbar, sidx;
        for (int si = 0; si < n_sizes; ++si) {
            const int k = sizes[si];
            std::iota(ids.begin(), ids.end(), int64_t{0});
            std::shuffle(ids.begin(), ids.end(), rng);
            for (int sub = 0; sub < subsets_per_size; ++sub) {
                const int64_t center = ids[(size_t)sub % ids.size()];
                subs.push_back(neighborhood(*scene, bc, g, center, k));
                kbar.push_back(k);
                sidx.push_back(sub);
            }
        }
        std::vector<Sub*> flat;
        for (Sub& sb : subs) flat.push_back(&sb);
        const std::vector<SubResult> res = batch_covariances(h, *scene, bc, flat, std::max(1, (int)workers));
        int64_t k = 0;
        for (size_t i = 0; i < subs.size(); ++i) {
            if (res[i].code)
                throw SubError{res[i].code, "subrec",
                               "sweep size " + std::to_string(kbar[i]) + " subset " + std::to_string(sidx[i]) + ": " +
                                   std::string(res[i].err.message)};
            for (size_t l = 0; l < subs[i].cams.size(); ++l, ++k) {
                if (k >= capacity) continue;
                const int32_t gc = subs[i].cams[l];
                const double* a = &res[i].cov[(size_t)P * P * l];
                const double* b = &full[(size_t)P * P * gc];
                double d2 = 0.0, r2 = 0.0;
                for (int e = 0; e < P * P; ++e) {
                    d2 += (a[e] - b[e]) * (a[e] - b[e]);
                    r2 += b[e] * b[e];
                }
                const double err_abs = std::sqrt(d2), ref = std::sqrt(r2);
                row_ints[3 * k] = kbar[i];
                row_ints[3 * k + 1] = sidx[i];
                row_ints[3 * k + 2] = gc;
                row_vals[3 * k] = ref > 0.0 ? err_abs / ref : err_abs;
                row_vals[3 * k + 1] = err_abs;
                row_vals[3 * k + 2] = trace_of(a, P);
            }
        }
        *n_rows = k;
    });
}

}  // extern "C"
