// Scene IO (reference include/sfmcov/scene_io.hpp, src/scene_io.cpp): the
// reference's JSON format and a binary format for large scenes.
//
// JSON: {"cameras": [{"C": [3], "c": f, "k": k1[, "k2": k2], "r": [3]}],
//        "observations": [{"cam": i, "pt": j, "u": [2][, "sigma": [s00, s01, s11]]}],
//        "points": [[3]]}
// written compact with sorted keys and shortest round-trip numbers (so the
// file round-trips bit-exactly and a second save reproduces the bytes), sigma
// omitted when it is the identity.  "k2" is this library's P = 9 extension.
// The loader streams the three top-level arrays (a 20M-observation scene is
// a multi-GB document) and reports errors with the reference's context
// ("camera 3: field 'r' must be an array of 3").  Validation of the loaded
// scene's invariants happens in the CUDA library (callers: the Python and
// C++ wrappers), as the reference's load ends with rec.validate().
//
// Binary: "SFMCOVB1", int32 n, m, t, P, has_sigma, then cams (n P), pts (3 m),
// obs_cam (t), obs_pt (t), u (2 t), sigma (4 t if has_sigma) little-endian.

#include "sfmcov_b200.h"
#include "scene_host.hpp"

#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

namespace {

struct IoError {
    int32_t kind;
    std::string stage, message;
};

thread_local IoError g_io_error{0, "", ""};

void set(sfmcov_error* e, const IoError& x) {
    g_io_error = x;
    if (!e) return;
    e->kind = x.kind;
    std::snprintf(e->stage, sizeof e->stage, "%s", x.stage.c_str());
    std::snprintf(e->message, sizeof e->message, "%s: %s", x.stage.c_str(), x.message.c_str());
}

[[noreturn]] void parse_fail(const std::string& msg) { throw IoError{SFMCOV_ERR_PARSE, "load", msg}; }

// ---- a small streaming JSON reader over a memory buffer -------------------------
struct Value {  // generic value (array elements: small)
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    double num = 0.0;
    bool is_int = false;
    std::string str;
    std::vector<Value> items;
    std::vector<std::pair<std::string, Value>> fields;
    const Value* find(const char* key) const {
        for (const auto& f : fields)
            if (f.first == key) return &f.second;
        return nullptr;
    }
};

struct Reader {
    const char* p;
    const char* end;
    const char* begin;
    void ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    [[noreturn]] void fail(const char* what) {
        parse_fail("[json.exception.parse_error] syntax error at byte " + std::to_string(p - begin) + ": " + what);
    }
    bool eat(char c) {
        ws();
        if (p < end && *p == c) {
            ++p;
            return true;
        }
        return false;
    }
    void expect(char c) {
        if (!eat(c)) fail((std::string("expected '") + c + "'").c_str());
    }
    std::string string() {
        ws();
        if (p >= end || *p != '"') fail("expected a string");
        ++p;
        std::string s;
        while (p < end && *p != '"') {
            if (*p == '\\') {
                ++p;
                if (p >= end) fail("bad escape");
                const char c = *p++;
                switch (c) {
                    case 'n': s += '\n'; break;
                    case 't': s += '\t'; break;
                    case 'r': s += '\r'; break;
                    case 'b': s += '\b'; break;
                    case 'f': s += '\f'; break;
                    case 'u': p += 4; s += '?'; break;  // (keys of this format are ASCII)
                    default: s += c;
                }
            } else {
                s += *p++;
            }
        }
        if (p >= end) fail("unterminated string");
        ++p;
        return s;
    }
    double number(bool* is_int) {
        ws();
        const char* q = p;
        bool integral = true;
        if (q < end && (*q == '-' || *q == '+')) ++q;
        while (q < end && ((*q >= '0' && *q <= '9') || *q == '.' || *q == 'e' || *q == 'E' || *q == '-' || *q == '+')) {
            if (*q == '.' || *q == 'e' || *q == 'E') integral = false;
            ++q;
        }
        double v = 0.0;
        const auto r = std::from_chars(p, q, v);
        if (r.ec != std::errc() || r.ptr != q) fail("invalid number");
        p = q;
        if (is_int) *is_int = integral;
        return v;
    }
    Value value() {
        ws();
        if (p >= end) fail("unexpected end of input");
        Value v;
        const char c = *p;
        if (c == '{') {
            ++p;
            v.kind = Value::Object;
            if (eat('}')) return v;
            do {
                std::string k = string();
                expect(':');
                v.fields.emplace_back(std::move(k), value());
            } while (eat(','));
            expect('}');
        } else if (c == '[') {
            ++p;
            v.kind = Value::Array;
            if (eat(']')) return v;
            do v.items.push_back(value());
            while (eat(','));
            expect(']');
        } else if (c == '"') {
            v.kind = Value::String;
            v.str = string();
        } else if (c == 't' && end - p >= 4 && !std::strncmp(p, "true", 4)) {
            p += 4;
            v.kind = Value::Bool;
            v.num = 1;
        } else if (c == 'f' && end - p >= 5 && !std::strncmp(p, "false", 5)) {
            p += 5;
            v.kind = Value::Bool;
        } else if (c == 'n' && end - p >= 4 && !std::strncmp(p, "null", 4)) {
            p += 4;
        } else if (c == '-' || (c >= '0' && c <= '9')) {
            v.kind = Value::Number;
            v.num = number(&v.is_int);
        } else {
            fail("invalid literal");
        }
        return v;
    }
};

double number_field(const Value& o, const char* key, const std::string& where) {
    const Value* v = o.find(key);
    if (!v) parse_fail(where + ": missing field '" + key + "'");
    if (v->kind != Value::Number) parse_fail(where + ": field '" + key + "' is not a number");
    return v->num;
}

void vector_field(const Value& o, const char* key, const std::string& where, int n, double* out) {
    const Value* v = o.find(key);
    if (!v) parse_fail(where + ": missing field '" + key + "'");
    if (v->kind != Value::Array || (int)v->items.size() != n)
        parse_fail(where + ": field '" + key + "' must be an array of " + std::to_string(n));
    for (int i = 0; i < n; ++i) {
        if (v->items[i].kind != Value::Number) parse_fail(where + ": field '" + key + "' has a non-number entry");
        out[i] = v->items[i].num;
    }
}

// Streams one top-level array, calling f(element, index).
template <class F>
void stream_array(Reader& r, F&& f) {
    r.ws();
    if (r.p >= r.end || *r.p != '[') parse_fail("top-level array expected");
    ++r.p;
    if (r.eat(']')) return;
    size_t i = 0;
    do f(r.value(), i++);
    while (r.eat(','));
    r.expect(']');
}

sfmhost::Scene load_json(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError{SFMCOV_ERR_IO, "load", "cannot open '" + path + "' for reading"};
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    Reader r{text.data(), text.data() + text.size(), text.data()};
    sfmhost::Scene s;
    bool have[3] = {false, false, false};
    std::vector<std::vector<double>> cam_rows;
    int P = 8;
    bool any_sigma = false;
    std::vector<double> sigma3;  // s00 s01 s11 per observation (identity when absent)
    r.ws();
    if (r.p >= r.end || *r.p != '{') {
        if (r.p < r.end && (*r.p == '[' || *r.p == '"' || *r.p == '-' || (*r.p >= '0' && *r.p <= '9'))) {
            r.value();
            r.ws();
            if (r.p == r.end) parse_fail("top level is not an object");
        }
        r.fail("invalid literal");
    }
    ++r.p;
    if (!r.eat('}')) {
        do {
            const std::string key = r.string();
            r.expect(':');
            r.ws();
            const bool is_array = r.p < r.end && *r.p == '[';
            if (key == "cameras" || key == "points" || key == "observations") {
                if (!is_array) {
                    r.value();
                    parse_fail("top-level '" + key + "' is not an array");
                }
                if (key == "cameras") {
                    have[0] = true;
                    stream_array(r, [&](const Value& v, size_t i) {
                        const std::string where = "camera " + std::to_string(i);
                        if (v.kind != Value::Object) parse_fail(where + ": not an object");
                        std::vector<double> c(9, 0.0);
                        vector_field(v, "r", where, 3, &c[0]);
                        vector_field(v, "C", where, 3, &c[3]);
                        c[6] = number_field(v, "c", where);
                        c[7] = number_field(v, "k", where);
                        if (v.find("k2")) {
                            c[8] = number_field(v, "k2", where);
                            P = 9;
                        }
                        cam_rows.push_back(std::move(c));
                    });
                } else if (key == "points") {
                    have[1] = true;
                    stream_array(r, [&](const Value& v, size_t j) {
                        const std::string where = "point " + std::to_string(j);
                        if (v.kind != Value::Array || v.items.size() != 3) parse_fail(where + ": must be an array of 3");
                        for (int a = 0; a < 3; ++a) {
                            if (v.items[a].kind != Value::Number) parse_fail(where + ": non-number coordinate");
                            s.pts.push_back(v.items[a].num);
                        }
                    });
                } else {
                    have[2] = true;
                    stream_array(r, [&](const Value& v, size_t t) {
                        const std::string where = "observation " + std::to_string(t);
                        if (v.kind != Value::Object) parse_fail(where + ": not an object");
                        s.oc.push_back((int32_t)number_field(v, "cam", where));
                        s.op.push_back((int32_t)number_field(v, "pt", where));
                        double u[2];
                        vector_field(v, "u", where, 2, u);
                        s.u.push_back(u[0]);
                        s.u.push_back(u[1]);
                        double sg[3] = {1.0, 0.0, 1.0};
                        if (v.find("sigma")) {
                            vector_field(v, "sigma", where, 3, sg);
                            any_sigma = true;
                        }
                        sigma3.insert(sigma3.end(), sg, sg + 3);
                    });
                }
            } else {
                r.value();  // unknown key: skipped
            }
        } while (r.eat(','));
        r.expect('}');
    }
    r.ws();
    if (r.p != r.end) r.fail("trailing characters");
    const char* names[3] = {"cameras", "points", "observations"};
    for (int k = 0; k < 3; ++k)
        if (!have[k]) parse_fail(std::string("missing top-level array '") + names[k] + "'");
    s.P = P;
    for (const auto& c : cam_rows) s.cams.insert(s.cams.end(), c.begin(), c.begin() + P);
    const size_t t = s.oc.size();
    s.sigma.resize(4 * t);
    for (size_t k = 0; k < t; ++k) {
        s.sigma[4 * k] = sigma3[3 * k];
        s.sigma[4 * k + 1] = sigma3[3 * k + 1];
        s.sigma[4 * k + 2] = sigma3[3 * k + 1];
        s.sigma[4 * k + 3] = sigma3[3 * k + 2];
    }
    (void)any_sigma;
    return s;
}

// shortest round-trip decimal, with ".0" for integral values (like the
// reference's JSON library)
void put_num(std::string& o, double v) {
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    o += s;
}

void save_json(const sfmcov_scene& sc, const std::string& path) {
    if (sc.n_cams <= 0) throw IoError{SFMCOV_ERR_INVARIANT, "save", "reconstruction has no cameras"};
    const int P = sc.cam_params;
    std::string o;
    o.reserve((size_t)sc.n_obs * 64 + (size_t)sc.n_pts * 64 + 1024);
    o += "{\"cameras\":[";
    for (int i = 0; i < sc.n_cams; ++i) {
        const double* c = sc.cams + (size_t)P * i;
        if (i) o += ',';
        o += "{\"C\":[";
        put_num(o, c[3]); o += ','; put_num(o, c[4]); o += ','; put_num(o, c[5]);
        o += "],\"c\":"; put_num(o, c[6]);
        o += ",\"k\":"; put_num(o, c[7]);
        if (P == 9) { o += ",\"k2\":"; put_num(o, c[8]); }
        o += ",\"r\":[";
        put_num(o, c[0]); o += ','; put_num(o, c[1]); o += ','; put_num(o, c[2]);
        o += "]}";
    }
    o += "],\"observations\":[";
    for (int t = 0; t < sc.n_obs; ++t) {
        if (t) o += ',';
        o += "{\"cam\":" + std::to_string(sc.obs_cam[t]) + ",\"pt\":" + std::to_string(sc.obs_pt[t]);
        if (sc.obs_sigma) {
            const double* g = sc.obs_sigma + 4 * (size_t)t;
            if (!(g[0] == 1.0 && g[1] == 0.0 && g[2] == 0.0 && g[3] == 1.0)) {
                o += ",\"sigma\":[";
                put_num(o, g[0]); o += ','; put_num(o, g[1]); o += ','; put_num(o, g[3]);
                o += ']';
            }
        }
        o += ",\"u\":[";
        const double u0 = sc.obs_u ? sc.obs_u[2 * (size_t)t] : 0.0, u1 = sc.obs_u ? sc.obs_u[2 * (size_t)t + 1] : 0.0;
        put_num(o, u0); o += ','; put_num(o, u1);
        o += "]}";
    }
    o += "],\"points\":[";
    for (int j = 0; j < sc.n_pts; ++j) {
        const double* x = sc.pts + 3 * (size_t)j;
        if (j) o += ',';
        o += '[';
        put_num(o, x[0]); o += ','; put_num(o, x[1]); o += ','; put_num(o, x[2]);
        o += ']';
    }
    o += "]}\n";
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError{SFMCOV_ERR_IO, "save", "cannot open '" + path + "' for writing"};
    out.write(o.data(), (std::streamsize)o.size());
    if (!out) throw IoError{SFMCOV_ERR_IO, "save", "write failed for '" + path + "'"};
}

const char kMagic[8] = {'S', 'F', 'M', 'C', 'O', 'V', 'B', '1'};

void save_binary(const sfmcov_scene& sc, const std::string& path) {
    if (sc.n_cams <= 0) throw IoError{SFMCOV_ERR_INVARIANT, "save", "reconstruction has no cameras"};
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError{SFMCOV_ERR_IO, "save", "cannot open '" + path + "' for writing"};
    const int32_t hdr[5] = {sc.n_cams, sc.n_pts, sc.n_obs, sc.cam_params, sc.obs_sigma ? 1 : 0};
    out.write(kMagic, 8);
    out.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
    auto w = [&](const void* p, size_t bytes) { out.write(reinterpret_cast<const char*>(p), (std::streamsize)bytes); };
    w(sc.cams, 8 * (size_t)sc.n_cams * sc.cam_params);
    w(sc.pts, 8 * 3 * (size_t)sc.n_pts);
    w(sc.obs_cam, 4 * (size_t)sc.n_obs);
    w(sc.obs_pt, 4 * (size_t)sc.n_obs);
    std::vector<double> zeros;
    if (sc.obs_u) w(sc.obs_u, 8 * 2 * (size_t)sc.n_obs);
    else { zeros.assign(2 * (size_t)sc.n_obs, 0.0); w(zeros.data(), 8 * zeros.size()); }
    if (sc.obs_sigma) w(sc.obs_sigma, 8 * 4 * (size_t)sc.n_obs);
    if (!out) throw IoError{SFMCOV_ERR_IO, "save", "write failed for '" + path + "'"};
}

sfmhost::Scene load_binary(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError{SFMCOV_ERR_IO, "load", "cannot open '" + path + "' for reading"};
    char magic[8];
    int32_t hdr[5];
    in.read(magic, 8);
    in.read(reinterpret_cast<char*>(hdr), sizeof hdr);
    if (!in || std::memcmp(magic, kMagic, 8)) parse_fail("not a binary scene file");
    const int32_t n = hdr[0], m = hdr[1], t = hdr[2], P = hdr[3];
    if (n < 0 || m < 0 || t < 0 || (P != 8 && P != 9)) parse_fail("bad binary scene header");
    sfmhost::Scene s;
    s.P = P;
    s.cams.resize((size_t)n * P);
    s.pts.resize(3 * (size_t)m);
    s.oc.resize(t);
    s.op.resize(t);
    s.u.resize(2 * (size_t)t);
    s.sigma.resize(4 * (size_t)t);
    auto r = [&](void* p, size_t bytes) { in.read(reinterpret_cast<char*>(p), (std::streamsize)bytes); };
    r(s.cams.data(), 8 * s.cams.size());
    r(s.pts.data(), 8 * s.pts.size());
    r(s.oc.data(), 4 * s.oc.size());
    r(s.op.data(), 4 * s.op.size());
    r(s.u.data(), 8 * s.u.size());
    if (hdr[4]) r(s.sigma.data(), 8 * s.sigma.size());
    else
        for (size_t k = 0; k < (size_t)t; ++k) {
            s.sigma[4 * k] = 1.0;
            s.sigma[4 * k + 3] = 1.0;
        }
    if (!in) parse_fail("truncated binary scene file");
    return s;
}

template <class F>
sfmcov_synth_scene* guard_load(sfmcov_error* err, F&& f) {
    try {
        auto* h = new sfmcov_synth_scene{f()};
        if (err) { err->kind = 0; err->stage[0] = 0; err->message[0] = 0; }
        return h;
    } catch (const IoError& x) {
        set(err, x);
        return nullptr;
    } catch (const std::exception& x) {
        set(err, IoError{SFMCOV_ERR_IO, "load", x.what()});
        return nullptr;
    }
}

template <class F>
int32_t guard_save(sfmcov_error* err, F&& f) {
    try {
        f();
        if (err) { err->kind = 0; err->stage[0] = 0; err->message[0] = 0; }
        return 0;
    } catch (const IoError& x) {
        set(err, x);
        return x.kind;
    } catch (const std::exception& x) {
        set(err, IoError{SFMCOV_ERR_IO, "save", x.what()});
        return SFMCOV_ERR_IO;
    }
}

// ---- covariance IO (reference src/covariance_io.cpp:17-122) ------------------
// The reference writes nlohmann::json's dump(): compact, object keys in sorted
// order, shortest round-trip doubles ("x.0" for integral ones), integers plain.
void put_int(std::string& o, long long v) { o += std::to_string(v); }

void pack_tri(const double* m, int P, double* tri) {
    int k = 0;
    for (int r = 0; r < P; ++r)
        for (int c = r; c < P; ++c) tri[k++] = m[P * r + c];
}
void unpack_tri(const double* tri, int P, double* m) {
    int k = 0;
    for (int r = 0; r < P; ++r)
        for (int c = r; c < P; ++c) {
            m[P * r + c] = tri[k];
            m[P * c + r] = tri[k];
            ++k;
        }
}

void write_file(const std::string& path, const std::string& text) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError{SFMCOV_ERR_IO, "save", "cannot open '" + path + "' for writing"};
    const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
    if (std::fclose(f) != 0 || !ok) throw IoError{SFMCOV_ERR_IO, "save", "failed writing '" + path + "'"};
}

void save_cov_json(const std::string& path, int64_t n, int P, const double* cov, const sfmcov_diagnostics& d) {
    std::string o;
    o.reserve((size_t)n * (P * (P + 1) / 2) * 24 + 512);
    o += "{\"cameras\":[";
    std::vector<double> tri(P * (P + 1) / 2);
    for (int64_t i = 0; i < n; ++i) {
        if (i) o += ',';
        o += "{\"cov\":[";
        pack_tri(cov + (size_t)P * P * i, P, tri.data());
        for (size_t k = 0; k < tri.size(); ++k) {
            if (k) o += ',';
            put_num(o, tri[k]);
        }
        o += "],\"id\":";
        put_int(o, i);
        o += '}';
    }
    o += "],\"diagnostics\":{\"flagged_columns\":[";
    const int64_t nf = d.flagged ? std::min<int64_t>(d.n_flagged, d.flagged_capacity) : 0;
    for (int64_t k = 0; k < nf; ++k) {
        if (k) o += ',';
        put_int(o, d.flagged[k]);
    }
    o += "],\"inertia_negative\":";
    put_int(o, d.inertia_negative);
    o += ",\"inertia_positive\":";
    put_int(o, d.inertia_positive);
    o += ",\"largest_dense_dim\":";
    put_int(o, d.largest_dense_dim);
    o += ",\"max_pivot\":";
    put_num(o, d.max_pivot);
    o += ",\"min_pivot\":";
    put_num(o, d.min_pivot);
    o += ",\"negative_eigenvalue_warnings\":";
    put_int(o, d.negative_eigenvalue_warnings);
    o += ",\"peak_dense_bytes\":";
    put_int(o, d.peak_dense_bytes);
    o += ",\"scale_max\":";
    put_num(o, d.scale_max);
    o += ",\"scale_min\":";
    put_num(o, d.scale_min);
    o += "}}\n";
    write_file(path, o);
}

std::string read_file(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoError{SFMCOV_ERR_IO, "load", "cannot open '" + path + "'"};
    std::string text;
    char buf[1 << 16];
    size_t k;
    while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) text.append(buf, k);
    std::fclose(f);
    return text;
}

int64_t load_cov_doc(const Value& doc, int P, int64_t capacity, double* cov, sfmcov_diagnostics* d);

// Parses the whole file; fills up to `capacity` blocks.
int64_t load_cov_json(const std::string& path, int P, int64_t capacity, double* cov, sfmcov_diagnostics* d) {
    const std::string text = read_file(path);
    Reader r{text.data(), text.data() + text.size(), text.data()};
    Value doc;
    try {
        doc = r.value();
        r.ws();
        if (r.p != r.end) r.fail("trailing characters");
    } catch (const IoError& x) {
        throw IoError{SFMCOV_ERR_PARSE, "load", "invalid JSON: " + x.message};
    }
    try {
        return load_cov_doc(doc, P, capacity, cov, d);
    } catch (const IoError& x) {
        if (x.kind != SFMCOV_ERR_PARSE) throw;
        throw IoError{SFMCOV_ERR_PARSE, "load", "bad covariance file: " + x.message};
    }
}

int64_t load_cov_doc(const Value& doc, int P, int64_t capacity, double* cov, sfmcov_diagnostics* d) {
    auto bad = [](const std::string& what) { parse_fail(what); };
    if (doc.kind != Value::Object) bad("document is not an object");
    const Value* cams = doc.find("cameras");
    if (!cams || cams->kind != Value::Array) bad("missing array 'cameras'");
    const int ntri = P * (P + 1) / 2;
    const int64_t n = (int64_t)cams->items.size();
    std::vector<double> tri(ntri);
    for (int64_t i = 0; i < n; ++i) {
        const Value& c = cams->items[i];
        if (c.kind != Value::Object) bad("camera entry is not an object");
        vector_field(c, "cov", "camera " + std::to_string(i), ntri, tri.data());
        if (i < capacity && cov) unpack_tri(tri.data(), P, cov + (size_t)P * P * i);
    }
    const Value* dg = doc.find("diagnostics");
    if (!dg || dg->kind != Value::Object) bad("missing object 'diagnostics'");
    if (d) {
        const std::string w = "diagnostics";
        d->scale_min = number_field(*dg, "scale_min", w);
        d->scale_max = number_field(*dg, "scale_max", w);
        d->min_pivot = number_field(*dg, "min_pivot", w);
        d->max_pivot = number_field(*dg, "max_pivot", w);
        d->inertia_positive = (int32_t)number_field(*dg, "inertia_positive", w);
        d->inertia_negative = (int32_t)number_field(*dg, "inertia_negative", w);
        d->negative_eigenvalue_warnings = (int32_t)number_field(*dg, "negative_eigenvalue_warnings", w);
        d->peak_dense_bytes = (int64_t)number_field(*dg, "peak_dense_bytes", w);
        d->largest_dense_dim = (int64_t)number_field(*dg, "largest_dense_dim", w);
        const Value* fl = dg->find("flagged_columns");
        if (!fl || fl->kind != Value::Array) bad("diagnostics: missing array 'flagged_columns'");
        d->n_flagged = (int32_t)fl->items.size();
        for (size_t k = 0; k < fl->items.size(); ++k) {
            if (fl->items[k].kind != Value::Number) bad("diagnostics: non-number flagged column");
            if (d->flagged && (int64_t)k < d->flagged_capacity) d->flagged[k] = (int64_t)fl->items[k].num;
        }
    }
    return n;
}

void save_cov_csv(const std::string& path, int64_t n, int P, const double* cov) {
    std::string o = "id";
    for (int r = 0; r < P; ++r)
        for (int c = r; c < P; ++c) o += ",cov_" + std::to_string(r) + "_" + std::to_string(c);
    o += '\n';
    std::vector<double> tri(P * (P + 1) / 2);
    char cell[40];
    for (int64_t i = 0; i < n; ++i) {
        o += std::to_string(i);
        pack_tri(cov + (size_t)P * P * i, P, tri.data());
        for (double v : tri) {
            std::snprintf(cell, sizeof cell, ",%.17g", v);
            o += cell;
        }
        o += '\n';
    }
    write_file(path, o);
}

}  // namespace

extern "C" {

sfmcov_synth_scene* sfmcov_scene_load(const char* path, sfmcov_error* err) {
    return guard_load(err, [&] { return load_json(path); });
}

int32_t sfmcov_scene_save(const sfmcov_scene* scene, const char* path, sfmcov_error* err) {
    return guard_save(err, [&] { save_json(*scene, path); });
}

sfmcov_synth_scene* sfmcov_scene_load_binary(const char* path, sfmcov_error* err) {
    return guard_load(err, [&] { return load_binary(path); });
}

int32_t sfmcov_scene_save_binary(const sfmcov_scene* scene, const char* path, sfmcov_error* err) {
    return guard_save(err, [&] { save_binary(*scene, path); });
}

void sfmcov_covio_pack_upper_triangle(const double* block, int32_t P, double* tri) { pack_tri(block, P, tri); }

void sfmcov_covio_unpack_upper_triangle(const double* tri, int32_t P, double* block) { unpack_tri(tri, P, block); }

int32_t sfmcov_covio_save_json(const char* path, int64_t n_cams, int32_t P, const double* cam_cov,
                                    const sfmcov_diagnostics* diag, sfmcov_error* err) {
    return guard_save(err, [&] {
        if (P != 8 && P != 9) throw IoError{SFMCOV_ERR_DIMENSION, "save", "camera width must be 8 or 9"};
        sfmcov_diagnostics d{};
        if (diag) d = *diag;
        save_cov_json(path, n_cams, P, cam_cov, d);
    });
}

int32_t sfmcov_covio_load_json(const char* path, int32_t P, int64_t capacity, double* cam_cov, int64_t* n_cams,
                                    sfmcov_diagnostics* diag, sfmcov_error* err) {
    try {
        if (P != 8 && P != 9) throw IoError{SFMCOV_ERR_DIMENSION, "load", "camera width must be 8 or 9"};
        const int64_t n = load_cov_json(path, P, capacity, cam_cov, diag);
        if (n_cams) *n_cams = n;
        if (err) { err->kind = 0; err->stage[0] = 0; err->message[0] = 0; }
        return 0;
    } catch (const IoError& x) {
        set(err, x);
        return x.kind;
    } catch (const std::exception& x) {
        set(err, IoError{SFMCOV_ERR_IO, "load", x.what()});
        return SFMCOV_ERR_IO;
    }
}

int32_t sfmcov_covio_save_csv(const char* path, int64_t n_cams, int32_t P, const double* cam_cov,
                                   sfmcov_error* err) {
    return guard_save(err, [&] {
        if (P != 8 && P != 9) throw IoError{SFMCOV_ERR_DIMENSION, "save", "camera width must be 8 or 9"};
        save_cov_csv(path, n_cams, P, cam_cov);
    });
}

}  // extern "C"
