// Seeded synthetic scenes (host only; harness, not the hot path).
//
//  * generate_cube_scene / generate_random_scene / transform_scene restate the
//    reference generators (src/synthetic.cpp:52-194) with std::mt19937_64 and
//    libstdc++'s distributions.  Vector components are drawn in x, y, z order
//    (the reference leaves argument evaluation order to the compiler).
//  * generate_config(1..5) builds the BASELINE.json scenes (P = 9 cameras
//    (r, C, f, k1, k2), f = 1000, k1 = k2 = 0, unit observation covariance,
//    N(0, 1 px) pixel noise on u) — SURVEY.md §8(d).  The paper's datasets are
//    not available; these seeded scenes stand in for them.
//
// Exposed through a small C ABI (include/sfmcov_b200.h, "synthetic scenes").

#include "sfmcov_b200.h"
#include "scene_host.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;

struct V3 { double x, y, z; };
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }
inline V3 normalized(V3 a) { return (1.0 / norm(a)) * a; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

struct Rot { double m[3][3]; };

Rot rot_from_r(const double* r) {  // Rodrigues with libm (scene generation only)
    const double t2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
    double a, b;
    if (t2 < 1e-16) { a = 1.0 - t2 / 6.0; b = 0.5 - t2 / 24.0; }
    else { const double t = std::sqrt(t2); a = std::sin(t) / t; b = (1.0 - std::cos(t)) / t2; }
    const double K[3][3] = {{0, -r[2], r[1]}, {r[2], 0, -r[0]}, {-r[1], r[0], 0}};
    Rot R;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double k2 = 0;
            for (int k = 0; k < 3; ++k) k2 += K[i][k] * K[k][j];
            R.m[i][j] = (i == j ? 1.0 : 0.0) + a * K[i][j] + b * k2;
        }
    return R;
}

// rotation_log (src/rotation.cpp:30-68): quaternion extraction, largest pivot.
void rotation_log(const Rot& Rm, double* out) {
    const auto& R = Rm.m;
    double qw, qx, qy, qz;
    const double tr = R[0][0] + R[1][1] + R[2][2];
    if (tr > 0.0) {
        const double s = std::sqrt(tr + 1.0) * 2.0;
        qw = 0.25 * s; qx = (R[2][1] - R[1][2]) / s; qy = (R[0][2] - R[2][0]) / s; qz = (R[1][0] - R[0][1]) / s;
    } else if (R[0][0] >= R[1][1] && R[0][0] >= R[2][2]) {
        const double s = std::sqrt(std::max(0.0, 1.0 + R[0][0] - R[1][1] - R[2][2])) * 2.0;
        qw = (R[2][1] - R[1][2]) / s; qx = 0.25 * s; qy = (R[0][1] + R[1][0]) / s; qz = (R[0][2] + R[2][0]) / s;
    } else if (R[1][1] >= R[2][2]) {
        const double s = std::sqrt(std::max(0.0, 1.0 + R[1][1] - R[0][0] - R[2][2])) * 2.0;
        qw = (R[0][2] - R[2][0]) / s; qx = (R[0][1] + R[1][0]) / s; qy = 0.25 * s; qz = (R[1][2] + R[2][1]) / s;
    } else {
        const double s = std::sqrt(std::max(0.0, 1.0 + R[2][2] - R[0][0] - R[1][1])) * 2.0;
        qw = (R[1][0] - R[0][1]) / s; qx = (R[0][2] + R[2][0]) / s; qy = (R[1][2] + R[2][1]) / s; qz = 0.25 * s;
    }
    if (qw < 0.0) { qw = -qw; qx = -qx; qy = -qy; qz = -qz; }
    const double nv = std::sqrt(qx * qx + qy * qy + qz * qz);
    if (nv < 1e-12) { out[0] = 2 * qx; out[1] = 2 * qy; out[2] = 2 * qz; return; }
    const double f = 2.0 * std::atan2(nv, qw) / nv;
    out[0] = f * qx; out[1] = f * qy; out[2] = f * qz;
}

// look_at (src/synthetic.cpp:19-29): world-to-camera rotation, optical axis
// from C to target.
void look_at(V3 C, V3 target, double* r) {
    const V3 z = normalized(target - C);
    const V3 up = std::fabs(z.z) < 0.9 ? V3{0, 0, 1} : V3{0, 1, 0};
    const V3 x = normalized(cross(up, z));
    const V3 y = cross(z, x);
    Rot R;
    const V3 rows[3] = {x, y, z};
    for (int i = 0; i < 3; ++i) { R.m[i][0] = rows[i].x; R.m[i][1] = rows[i].y; R.m[i][2] = rows[i].z; }
    rotation_log(R, r);
}

using sfmhost::Scene;  // scene_host.hpp

// Camera-space point and projection u = f(1 + k1ρ + k2ρ²)u_n; false if depth <= eps.
bool project(const double* cam, int P, const double* X, double* u, double* vz = nullptr) {
    const Rot R = rot_from_r(cam);
    const double w[3] = {X[0] - cam[3], X[1] - cam[4], X[2] - cam[5]};
    double v[3];
    for (int i = 0; i < 3; ++i) v[i] = R.m[i][0] * w[0] + R.m[i][1] * w[1] + R.m[i][2] * w[2];
    if (vz) *vz = v[2];
    if (!(v[2] > 1e-9)) return false;
    const double un0 = v[0] / v[2], un1 = v[1] / v[2];
    const double rho = un0 * un0 + un1 * un1;
    double d = 1.0 + cam[7] * rho;
    if (P == 9) d += cam[8] * rho * rho;
    u[0] = cam[6] * d * un0;
    u[1] = cam[6] * d * un1;
    return true;
}

void add_obs(Scene& s, int32_t ci, int32_t pj, const Rot* R = nullptr) {
    double u[2] = {0, 0};
    if (R) {  // k1 = k2 = 0 configs with a precomputed camera rotation
        const double* c = &s.cams[size_t(s.P) * ci];
        const double* X = &s.pts[3 * size_t(pj)];
        const double w[3] = {X[0] - c[3], X[1] - c[4], X[2] - c[5]};
        double v[3];
        for (int a = 0; a < 3; ++a) v[a] = R->m[a][0] * w[0] + R->m[a][1] * w[1] + R->m[a][2] * w[2];
        u[0] = c[6] * (v[0] / v[2]);
        u[1] = c[6] * (v[1] / v[2]);
    } else {
        project(&s.cams[size_t(s.P) * ci], s.P, &s.pts[3 * size_t(pj)], u);
    }
    s.oc.push_back(ci);
    s.op.push_back(pj);
    s.u.push_back(u[0]);
    s.u.push_back(u[1]);
    const double I[4] = {1, 0, 0, 1};
    s.sigma.insert(s.sigma.end(), I, I + 4);
}

// add_noise (src/synthetic.cpp:31-42)
void add_noise(Scene& s, double noise_px, std::mt19937_64& rng) {
    if (noise_px > 0.0) {
        std::normal_distribution<double> gauss(0.0, noise_px);
        for (int64_t t = 0; t < s.t(); ++t) {
            s.u[2 * t] += gauss(rng);
            s.u[2 * t + 1] += gauss(rng);
            const double v = noise_px * noise_px;
            s.sigma[4 * t + 0] = v; s.sigma[4 * t + 1] = 0; s.sigma[4 * t + 2] = 0; s.sigma[4 * t + 3] = v;
        }
    }
}

void push_cam(Scene& s, V3 C, const double* r, double f, double k1, double k2) {
    s.cams.insert(s.cams.end(), {r[0], r[1], r[2], C.x, C.y, C.z, f, k1});
    if (s.P == 9) s.cams.push_back(k2);
}

// src/synthetic.cpp:52-84
Scene cube_scene(uint64_t seed, double noise_px, int P) {
    Scene s;
    s.P = P;
    const V3 dirs[6] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
    for (int i = 0; i < 6; ++i) {
        const V3 C = 10.0 * dirs[i];
        double r[3];
        look_at(C, {0, 0, 0}, r);
        push_cam(s, C, r, 100.0 + 5.0 * i, 0.01 * (i - 2.5) / 2.5, 0.0);
    }
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> coord(-5.0, 5.0);
    for (int j = 0; j < 15; ++j) {
        const double x = coord(rng), y = coord(rng), z = coord(rng);
        s.pts.insert(s.pts.end(), {x, y, z});
    }
    for (int i = 0; i < 6; ++i)
        for (int l = 0; l < 10; ++l) add_obs(s, i, (2 * i + l) % 15);
    add_noise(s, noise_px, rng);
    return s;
}

double angular_distance(double a, double b) {
    const double two_pi = 2.0 * kPi;
    const double d = std::fmod(std::fabs(a - b), two_pi);
    return std::min(d, two_pi - d);
}

// src/synthetic.cpp:86-183
Scene random_scene(int64_t n_cams, int64_t n_pts, double visibility, uint64_t seed, double noise_px, int P) {
    if (n_cams < 2) throw std::runtime_error("generate: need at least 2 cameras");
    if (n_pts < 8) throw std::runtime_error("generate: need at least 8 points");
    if (!(visibility > 0.0) || visibility > 1.0) throw std::runtime_error("generate: visibility must be in (0, 1]");
    const double two_pi = 2.0 * kPi, ring_radius = 10.0, point_radius = 6.0;
    Scene s;
    s.P = P;
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    for (int64_t i = 0; i < n_cams; ++i) {
        const double ang = two_pi * double(i) / double(n_cams);
        const V3 C{ring_radius * std::cos(ang), ring_radius * std::sin(ang), gauss(rng)};
        double r[3];
        look_at(C, {0, 0, 0}, r);
        const double c = 100.0 * (1.0 + 0.2 * unit(rng));
        const double k = 0.02 * gauss(rng);
        push_cam(s, C, r, c, k, 0.0);
    }
    std::uniform_real_distribution<double> coord(-point_radius, point_radius);
    for (int64_t j = 0; j < n_pts; ++j) {
        double x, y, z;
        do { x = coord(rng); y = coord(rng); z = coord(rng); } while (std::sqrt(x * x + y * y + z * z) > point_radius);
        s.pts.insert(s.pts.end(), {x, y, z});
    }
    const int views = (int)std::clamp<int64_t>(std::llround(visibility * double(n_cams)), 2, n_cams);
    const double step = two_pi / double(n_cams);
    std::vector<std::set<int32_t>> seen(n_cams);
    for (int64_t j = 0; j < n_pts; ++j) {
        const double ang = std::atan2(s.pts[3 * j + 1], s.pts[3 * j]);
        const int64_t center = std::llround(ang / step);
        std::vector<std::pair<double, int64_t>> cand;
        for (int64_t d = -views - 1; d <= views + 1; ++d) {
            const int64_t i = ((center + d) % n_cams + n_cams) % n_cams;
            cand.emplace_back(angular_distance(ang, step * double(i)), i);
        }
        std::sort(cand.begin(), cand.end());
        std::vector<int64_t> chosen;
        for (const auto& c : cand) {
            if (std::find(chosen.begin(), chosen.end(), c.second) == chosen.end()) chosen.push_back(c.second);
            if ((int)chosen.size() == views) break;
        }
        std::sort(chosen.begin(), chosen.end());
        for (int64_t i : chosen) { add_obs(s, (int32_t)i, (int32_t)j); seen[i].insert((int32_t)j); }
    }
    for (int64_t i = 0; i < n_cams; ++i) {
        if ((int64_t)seen[i].size() >= 4) continue;
        const double cam_ang = step * double(i);
        std::vector<std::pair<double, int64_t>> order;
        for (int64_t j = 0; j < n_pts; ++j)
            order.emplace_back(angular_distance(std::atan2(s.pts[3 * j + 1], s.pts[3 * j]), cam_ang), j);
        std::sort(order.begin(), order.end());
        for (const auto& o : order) {
            if ((int64_t)seen[i].size() >= 4) break;
            if (seen[i].count((int32_t)o.second)) continue;
            add_obs(s, (int32_t)i, (int32_t)o.second);
            seen[i].insert((int32_t)o.second);
        }
        if ((int64_t)seen[i].size() < 4)
            throw std::runtime_error("generate: visibility infeasible: camera " + std::to_string(i) + " cannot reach 4 observations");
    }
    add_noise(s, noise_px, rng);
    return s;
}

// src/synthetic.cpp:185-194: X' = sRX + t, r' = log(R(r) Rᵀ).
Scene transform(const Scene& in, const double* Rm, const double* t, double scale) {
    Scene s = in;
    Rot R;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) R.m[i][j] = Rm[3 * i + j];
    for (int64_t i = 0; i < s.n(); ++i) {
        double* c = &s.cams[size_t(s.P) * i];
        const Rot Rc = rot_from_r(c);
        Rot M;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double acc = 0;
                for (int k = 0; k < 3; ++k) acc += Rc.m[a][k] * R.m[b][k];
                M.m[a][b] = acc;
            }
        rotation_log(M, c);
        const double C[3] = {c[3], c[4], c[5]};
        for (int a = 0; a < 3; ++a) c[3 + a] = scale * (R.m[a][0] * C[0] + R.m[a][1] * C[1] + R.m[a][2] * C[2]) + t[a];
    }
    for (int64_t j = 0; j < s.m(); ++j) {
        double* X = &s.pts[3 * j];
        const double Y[3] = {X[0], X[1], X[2]};
        for (int a = 0; a < 3; ++a) X[a] = scale * (R.m[a][0] * Y[0] + R.m[a][1] * Y[1] + R.m[a][2] * Y[2]) + t[a];
    }
    return s;
}

// ---------------------------------------------------------------------------
// BASELINE.json configs.
// ---------------------------------------------------------------------------
struct ConfigSpec {
    int n_cams;
    int n_pts;
    int kmin, kmax;        // track length range
    int track;             // 0 uniform int, 1 clamp(2 + Geom(1/3), 2, 20)
    bool nearest;          // choose among angularly nearest visible cameras
    int pool_extra;        // nearest-candidate pool = k + pool_extra
    double jitter;         // relative radius / look-at jitter
    int blobs;             // 0 uniform cube, >0 Gaussian blobs (σ=1.5)
};

ConfigSpec spec(int idx) {
    switch (idx) {
        case 1: return {10, 1000, 2, 10, 0, false, 0, 0.0, 0};
        case 2: return {100, 20000, 2, 20, 1, true, 6, 0.10, 0};
        case 3: return {1000, 200000, 3, 12, 0, true, 10, 0.10, 0};
        case 4: return {3000, 1000000, 2, 10, 0, true, 10, 0.10, 8};
        case 5: return {10000, 4000000, 2, 8, 0, true, 8, 0.10, 0};
        default: throw std::runtime_error("generate: config index must be 1..5");
    }
}

// Fibonacci-sphere camera directions.
V3 fib_dir(int i, int n) {
    const double golden = kPi * (3.0 - std::sqrt(5.0));
    const double z = 1.0 - 2.0 * (i + 0.5) / n;
    const double rr = std::sqrt(std::max(0.0, 1.0 - z * z));
    const double th = golden * i;
    return {rr * std::cos(th), rr * std::sin(th), z};
}

// Uniform grid over camera unit directions for nearest-direction queries:
// cell size = the expected radius holding `want` cameras; a query gathers
// every camera within a ball of radius R (doubling R until it holds enough),
// so the result is the exact nearest set.
struct DirGrid {
    int g = 2;
    double cell = 1.0, r0 = 1.0;
    std::vector<std::vector<int32_t>> cells;
    std::vector<V3> dirs;
    int cell_of(double v) const { return std::min(g - 1, std::max(0, (int)((v + 1.0) / cell))); }
    int key(int a, int b, int c) const { return (a * g + b) * g + c; }
    void build(const std::vector<V3>& d, int n, int want) {
        dirs = d;
        const double spacing = std::sqrt(4.0 * kPi / std::max(1, n));
        r0 = 1.2 * spacing * std::sqrt((double)std::max(1, want));
        g = std::max(2, std::min(128, (int)std::ceil(2.0 / r0)));
        cell = 2.0 / g;
        cells.assign(size_t(g) * g * g, {});
        for (int i = 0; i < (int)d.size(); ++i) cells[key(cell_of(d[i].x), cell_of(d[i].y), cell_of(d[i].z))].push_back(i);
    }
    // cameras sorted by (squared) direction distance to q: all within R, R
    // grown until at least `want` are found (or all cameras are in)
    void nearest(V3 q, int want, std::vector<std::pair<double, int32_t>>& out) const {
        want = std::min<int>(want, (int)dirs.size());
        for (double R = r0;; R *= 2.0) {
            out.clear();
            const int ax = cell_of(q.x - R), bx = cell_of(q.x + R);
            const int ay = cell_of(q.y - R), by = cell_of(q.y + R);
            const int az = cell_of(q.z - R), bz = cell_of(q.z + R);
            const double R2 = R * R;
            for (int a = ax; a <= bx; ++a)
                for (int b = ay; b <= by; ++b)
                    for (int c = az; c <= bz; ++c)
                        for (int32_t i : cells[key(a, b, c)]) {
                            const V3 dd = dirs[i] - q;
                            const double d2 = dot(dd, dd);
                            if (d2 <= R2) out.emplace_back(d2, i);
                        }
            if ((int)out.size() >= want || R > 4.0) break;
        }
        std::sort(out.begin(), out.end());
    }
};

Scene config_scene(int idx, uint64_t seed) {
    const ConfigSpec c = spec(idx);
    Scene s;
    s.P = 9;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    std::uniform_real_distribution<double> sym(-1.0, 1.0);
    std::normal_distribution<double> gauss(0.0, 1.0);
    const double radius = 20.0, half = 5.0;
    std::vector<V3> cdir(c.n_cams);
    for (int i = 0; i < c.n_cams; ++i) {
        const V3 d = fib_dir(i, c.n_cams);
        const double rad = radius * (1.0 + c.jitter * sym(rng));
        const double tx = c.jitter * half * sym(rng), ty = c.jitter * half * sym(rng), tz = c.jitter * half * sym(rng);
        const V3 C = rad * d;
        double r[3];
        look_at(C, {tx, ty, tz}, r);
        push_cam(s, C, r, 1000.0, 0.0, 0.0);
        cdir[i] = d;
    }
    std::vector<V3> centers;
    for (int b = 0; b < c.blobs; ++b) {
        const double x = 3.5 * sym(rng), y = 3.5 * sym(rng), z = 3.5 * sym(rng);
        centers.push_back({x, y, z});
    }
    DirGrid grid;
    if (c.nearest) grid.build(cdir, c.n_cams, 2 * (c.kmax + c.pool_extra));
    std::vector<Rot> crot(c.n_cams);
    for (int i = 0; i < c.n_cams; ++i) crot[i] = rot_from_r(&s.cams[size_t(9) * i]);
    std::geometric_distribution<int> geo(1.0 / 3.0);
    std::uniform_int_distribution<int> kdist(c.kmin, c.kmax);
    std::vector<std::pair<double, int32_t>> cand;
    std::vector<int32_t> vis, chosen;
    const double fx = 1000.0, fy = 750.0;
    int64_t j = 0;
    while (j < c.n_pts) {
        double X[3];
        if (c.blobs > 0) {
            const V3 ctr = centers[std::uniform_int_distribution<int>(0, c.blobs - 1)(rng)];
            X[0] = std::clamp(ctr.x + 1.5 * gauss(rng), -half, half);
            X[1] = std::clamp(ctr.y + 1.5 * gauss(rng), -half, half);
            X[2] = std::clamp(ctr.z + 1.5 * gauss(rng), -half, half);
        } else {
            X[0] = half * sym(rng); X[1] = half * sym(rng); X[2] = half * sym(rng);
        }
        int k = c.track == 1 ? std::clamp(2 + geo(rng), c.kmin, c.kmax) : kdist(rng);
        // visible cameras: in front, inside the 2000 x 1500 image (centred)
        vis.clear();
        // k1 = k2 = 0 here, so u = f * (v_x / v_z, v_y / v_z)
        auto visible = [&](int32_t i) {
            const Rot& R = crot[i];
            const double* c = &s.cams[size_t(9) * i];
            const double w[3] = {X[0] - c[3], X[1] - c[4], X[2] - c[5]};
            double v[3];
            for (int a = 0; a < 3; ++a) v[a] = R.m[a][0] * w[0] + R.m[a][1] * w[1] + R.m[a][2] * w[2];
            if (!(v[2] > 1e-9)) return false;
            return std::fabs(c[6] * v[0] / v[2]) <= fx && std::fabs(c[6] * v[1] / v[2]) <= fy;
        };
        if (!c.nearest) {
            for (int32_t i = 0; i < c.n_cams; ++i) if (visible(i)) vis.push_back(i);
        } else {
            V3 q{X[0], X[1], X[2]};
            const double nq = norm(q);
            q = nq > 1e-9 ? (1.0 / nq) * q : V3{0, 0, 1};
            const int pool = std::min(c.n_cams, k + c.pool_extra);
            grid.nearest(q, std::min(c.n_cams, pool * 2), cand);
            for (const auto& pr : cand) {
                if ((int)vis.size() >= pool) break;
                if (visible(pr.second)) vis.push_back(pr.second);
            }
        }
        if ((int)vis.size() < 2) continue;  // redraw the point
        k = std::min<int>(k, (int)vis.size());
        // partial Fisher–Yates: k distinct cameras from the pool
        for (int a = 0; a < k; ++a) {
            std::uniform_int_distribution<int> pick(a, (int)vis.size() - 1);
            std::swap(vis[a], vis[pick(rng)]);
        }
        chosen.assign(vis.begin(), vis.begin() + k);
        std::sort(chosen.begin(), chosen.end());
        s.pts.insert(s.pts.end(), X, X + 3);
        for (int32_t i : chosen) add_obs(s, i, (int32_t)j, &crot[i]);
        ++j;
    }
    add_noise(s, 1.0, rng);
    // unit observation covariance (σ = 1 px)
    return s;
}

thread_local std::string g_last_error;

}  // namespace


extern "C" {

const char* sfmcov_synth_last_error(void) { return g_last_error.c_str(); }

sfmcov_synth_scene* sfmcov_synth_cube(uint64_t seed, double noise_px, int32_t cam_params) {
    try { return new sfmcov_synth_scene{cube_scene(seed, noise_px, cam_params)}; }
    catch (const std::exception& e) { g_last_error = e.what(); return nullptr; }
}

sfmcov_synth_scene* sfmcov_synth_random(int64_t n_cams, int64_t n_pts, double visibility, uint64_t seed,
                                        double noise_px, int32_t cam_params) {
    try { return new sfmcov_synth_scene{random_scene(n_cams, n_pts, visibility, seed, noise_px, cam_params)}; }
    catch (const std::exception& e) { g_last_error = e.what(); return nullptr; }
}

sfmcov_synth_scene* sfmcov_synth_config(int32_t config_index, uint64_t seed) {
    try { return new sfmcov_synth_scene{config_scene(config_index, seed)}; }
    catch (const std::exception& e) { g_last_error = e.what(); return nullptr; }
}

sfmcov_synth_scene* sfmcov_synth_transform(const sfmcov_synth_scene* in, const double* R, const double* t, double scale) {
    try { return new sfmcov_synth_scene{transform(in->s, R, t, scale)}; }
    catch (const std::exception& e) { g_last_error = e.what(); return nullptr; }
}

void sfmcov_synth_sizes(const sfmcov_synth_scene* h, int64_t* n, int64_t* m, int64_t* t, int32_t* P) {
    *n = h->s.n(); *m = h->s.m(); *t = h->s.t(); *P = h->s.P;
}

void sfmcov_synth_export(const sfmcov_synth_scene* h, double* cams, double* pts, int32_t* obs_cam, int32_t* obs_pt,
                         double* obs_u, double* obs_sigma) {
    const Scene& s = h->s;
    std::memcpy(cams, s.cams.data(), 8 * s.cams.size());
    std::memcpy(pts, s.pts.data(), 8 * s.pts.size());
    std::memcpy(obs_cam, s.oc.data(), 4 * s.oc.size());
    std::memcpy(obs_pt, s.op.data(), 4 * s.op.size());
    if (obs_u) std::memcpy(obs_u, s.u.data(), 8 * s.u.size());
    if (obs_sigma) std::memcpy(obs_sigma, s.sigma.data(), 8 * s.sigma.size());
}

void sfmcov_synth_free(sfmcov_synth_scene* h) { delete h; }

}  // extern "C"
