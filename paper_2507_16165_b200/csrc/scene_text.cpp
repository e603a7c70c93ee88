// scene_text.cpp — scene text for the extended scene.
//
// The reference's key=value scene format (config.hpp: parse_kv, format_double,
// serialize_scene, parse_scene; config.cpp:27-132) carries only SceneConfig.
// This file reads and writes the same format for bhrt_scene: the fourteen
// reference keys (required, same order, same number syntax and error
// messages) plus optional extension keys for the north-star features. Absent
// extension keys keep bhrt_scene_defaults (= reference semantics), the
// reference's parse_scene ignores keys it does not know, and the formatter
// writes only extension keys that differ from the defaults — so a reference
// scene's text is byte-identical to the reference's serialize_scene output.
//
// Extension keys:
//   integrator      = reference | rk4 | rkf45 | table
//   step, max-step, chord-dphi, ambient, table-b-max, table-dpsi   (doubles)
//   table-entries, table-samples                                   (integers)
//   sky             = image | checker
//   checker         = nu,nv
//   checker-color-a, checker-color-b, disk-color-in, disk-color-out, light-dir  (x,y,z)
//   disk            = off | r_in,r_out          (enables the disk)
//   spheres         = count,seed[,shell_min,shell_max,radius_min,radius_max]
//                     (the seeded field of bhrt_make_spheres around `center`)
//   sphere.<i>      = cx,cy,cz,radius,r,g,b     (explicit, i = 0..n-1; wins over `spheres`)
#include <charconv>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <string_view>
#include <vector>

#include "bhrt_cuda.h"

namespace {

struct UsageFail {
    std::string msg;
};

using KvMap = std::map<std::string, std::string>;

std::string_view trim(std::string_view s) {  // config.cpp:11-17
    while (!s.empty() && (s.front() == ' ' || s.front() == '\t' || s.front() == '\r')) s.remove_prefix(1);
    while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
    return s;
}

KvMap parse_kv(std::string_view text) {  // config.cpp:27-44: '#' comments, later keys win
    KvMap out;
    std::size_t pos = 0;
    while (pos <= text.size()) {
        const std::size_t nl = text.find('\n', pos);
        const std::size_t eol = nl == std::string_view::npos ? text.size() : nl;
        const std::string_view line = trim(text.substr(pos, eol - pos));
        pos = eol + 1;
        if (line.empty() || line.front() == '#') continue;
        const std::size_t eq = line.find('=');
        if (eq == std::string_view::npos)
            throw UsageFail{"config: expected key=value, got '" + std::string(line) + "'"};
        const std::string_view key = trim(line.substr(0, eq));
        if (key.empty()) throw UsageFail{"config: empty key in '" + std::string(line) + "'"};
        out[std::string(key)] = std::string(trim(line.substr(eq + 1)));
    }
    return out;
}

const std::string& require(const KvMap& kv, const std::string& key) {
    const auto it = kv.find(key);
    if (it == kv.end()) throw UsageFail{"scene config: missing key '" + key + "'"};
    return it->second;
}

template <class T>
T parse_num(const std::string& v, const std::string& key, const char* what) {
    T out{};
    const char* b = v.c_str();
    const char* e = b + v.size();
    const auto r = std::from_chars(b, e, out);
    if (r.ec != std::errc() || r.ptr != e)
        throw UsageFail{"invalid " + key + ": '" + v + "' is not " + what};
    return out;
}
double pdouble(const std::string& v, const std::string& k) { return parse_num<double>(v, k, "a number"); }
int64_t pint(const std::string& v, const std::string& k) { return parse_num<int64_t>(v, k, "an integer"); }
uint64_t puint(const std::string& v, const std::string& k) {
    return parse_num<uint64_t>(v, k, "an unsigned integer");
}

std::vector<std::string> split(const std::string& v) {
    std::vector<std::string> parts;
    std::size_t pos = 0;
    for (;;) {
        const std::size_t c = v.find(',', pos);
        parts.push_back(v.substr(pos, c == std::string::npos ? std::string::npos : c - pos));
        if (c == std::string::npos) break;
        pos = c + 1;
    }
    return parts;
}

void pvec3(const std::string& v, const std::string& key, double out[3]) {  // config.cpp:86-94
    const std::size_t c1 = v.find(',');
    const std::size_t c2 = c1 == std::string::npos ? std::string::npos : v.find(',', c1 + 1);
    if (c2 == std::string::npos) throw UsageFail{"invalid " + key + ": expected 'x,y,z', got '" + v + "'"};
    out[0] = pdouble(v.substr(0, c1), key);
    out[1] = pdouble(v.substr(c1 + 1, c2 - c1 - 1), key);
    out[2] = pdouble(v.substr(c2 + 1), key);
}

std::string fmt(double v) {  // config.cpp:46-50: shortest round-trip decimal
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
}
std::string fmt3(const double* v) { return fmt(v[0]) + "," + fmt(v[1]) + "," + fmt(v[2]); }

const char* kIntegrators[] = {"reference", "rk4", "rkf45", "table"};

bool same3(const double* a, const double* b) { return std::memcmp(a, b, 3 * sizeof(double)) == 0; }
bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

}  // namespace

extern "C" int bhrt_scene_parse_text(const char* text, bhrt_scene* s, bhrt_sphere* spheres, int32_t cap,
                                     int32_t* n_spheres, bhrt_status_info* info) {
    auto fail = [&](int code, const std::string& m) {
        if (info) {
            info->code = code;
            info->px = info->py = -1;
            std::snprintf(info->message, sizeof info->message, "%s", m.c_str());
        }
        return code;
    };
    if (!text || !s) return fail(BHRT_INVALID_ARGUMENT, "scene text: NULL argument");
    if (n_spheres) *n_spheres = 0;
    try {
        const KvMap kv = parse_kv(text);
        bhrt_scene_defaults(s);
        // parse_scene, config.cpp:114-130 (same keys, order and syntax)
        s->mass = pdouble(require(kv, "mass"), "mass");
        pvec3(require(kv, "center"), "center", s->center);
        pvec3(require(kv, "cam-pos"), "cam-pos", s->cam_pos);
        pvec3(require(kv, "look-at"), "look-at", s->cam_look_at);
        s->vertical_fov = pdouble(require(kv, "fov-rad"), "fov-rad");
        s->width = static_cast<int32_t>(pint(require(kv, "width"), "width"));
        s->height = static_cast<int32_t>(pint(require(kv, "height"), "height"));
        s->spp = static_cast<int32_t>(pint(require(kv, "spp"), "spp"));
        s->seed = puint(require(kv, "seed"), "seed");
        s->epsilon = pdouble(require(kv, "epsilon"), "epsilon");
        s->escape_radius = pdouble(require(kv, "escape-radius"), "escape-radius");
        s->max_windings = static_cast<int32_t>(pint(require(kv, "max-windings"), "max-windings"));
        s->rel_tol = pdouble(require(kv, "rel-tol"), "rel-tol");
        s->abs_tol = pdouble(require(kv, "abs-tol"), "abs-tol");
        s->sky_rgb = nullptr;  // the background travels separately (parse_scene leaves it null)
        s->sky_width = s->sky_height = 0;

        auto opt = [&](const char* key) -> const std::string* {
            const auto it = kv.find(key);
            return it == kv.end() ? nullptr : &it->second;
        };
        if (const auto* v = opt("integrator")) {
            int found = -1;
            for (int i = 0; i < 4; ++i)
                if (*v == kIntegrators[i]) found = i;
            if (found < 0)
                throw UsageFail{"invalid integrator: '" + *v + "' (reference, rk4, rkf45 or table)"};
            s->integrator = found;
        }
        if (const auto* v = opt("step")) s->step = pdouble(*v, "step");
        if (const auto* v = opt("max-step")) s->max_step = pdouble(*v, "max-step");
        if (const auto* v = opt("chord-dphi")) s->chord_dphi = pdouble(*v, "chord-dphi");
        if (const auto* v = opt("ambient")) s->ambient = pdouble(*v, "ambient");
        if (const auto* v = opt("table-b-max")) s->table_b_max = pdouble(*v, "table-b-max");
        if (const auto* v = opt("table-dpsi")) s->table_dpsi = pdouble(*v, "table-dpsi");
        if (const auto* v = opt("table-entries"))
            s->table_entries = static_cast<int32_t>(pint(*v, "table-entries"));
        if (const auto* v = opt("table-samples"))
            s->table_samples = static_cast<int32_t>(pint(*v, "table-samples"));
        if (const auto* v = opt("sky")) {
            if (*v == "image")
                s->sky_kind = BHRT_SKY_IMAGE;
            else if (*v == "checker")
                s->sky_kind = BHRT_SKY_CHECKER;
            else
                throw UsageFail{"invalid sky: '" + *v + "' (image or checker)"};
        }
        if (const auto* v = opt("checker")) {
            const auto p = split(*v);
            if (p.size() != 2) throw UsageFail{"invalid checker: expected 'nu,nv', got '" + *v + "'"};
            s->checker_nu = static_cast<int32_t>(pint(p[0], "checker"));
            s->checker_nv = static_cast<int32_t>(pint(p[1], "checker"));
        }
        if (const auto* v = opt("checker-color-a")) pvec3(*v, "checker-color-a", s->checker_color_a);
        if (const auto* v = opt("checker-color-b")) pvec3(*v, "checker-color-b", s->checker_color_b);
        if (const auto* v = opt("disk-color-in")) pvec3(*v, "disk-color-in", s->disk_color_in);
        if (const auto* v = opt("disk-color-out")) pvec3(*v, "disk-color-out", s->disk_color_out);
        if (const auto* v = opt("light-dir")) pvec3(*v, "light-dir", s->light_dir);
        if (const auto* v = opt("disk")) {
            if (*v == "off") {
                s->disk_enabled = 0;
            } else {
                const auto p = split(*v);
                if (p.size() != 2) throw UsageFail{"invalid disk: expected 'r_in,r_out' or 'off', got '" + *v + "'"};
                s->disk_r_in = pdouble(p[0], "disk");
                s->disk_r_out = pdouble(p[1], "disk");
                s->disk_enabled = 1;
            }
        }
        // spheres: explicit sphere.<i> lines win over a generated field
        std::vector<bhrt_sphere> sph;
        int explicit_n = 0;
        while (kv.count("sphere." + std::to_string(explicit_n))) ++explicit_n;
        for (const auto& [k, v] : kv)
            if (k.rfind("sphere.", 0) == 0) {
                const std::string idx = k.substr(7);
                int64_t i = -1;
                const auto r = std::from_chars(idx.data(), idx.data() + idx.size(), i);
                if (r.ec != std::errc() || r.ptr != idx.data() + idx.size() || i < 0 || i >= explicit_n)
                    throw UsageFail{"invalid " + k + ": sphere keys must be sphere.0 .. sphere.<n-1>"};
            }
        if (explicit_n > 0) {
            for (int i = 0; i < explicit_n; ++i) {
                const std::string key = "sphere." + std::to_string(i);
                const auto p = split(kv.at(key));
                if (p.size() != 7)
                    throw UsageFail{"invalid " + key + ": expected 'cx,cy,cz,radius,r,g,b', got '" + kv.at(key) + "'"};
                bhrt_sphere b;
                for (int j = 0; j < 3; ++j) b.center[j] = pdouble(p[j], key);
                b.radius = pdouble(p[3], key);
                for (int j = 0; j < 3; ++j) b.albedo[j] = pdouble(p[4 + j], key);
                sph.push_back(b);
            }
        } else if (const auto* v = opt("spheres")) {
            const auto p = split(*v);
            if (p.size() != 2 && p.size() != 6)
                throw UsageFail{"invalid spheres: expected 'count,seed[,shell_min,shell_max,radius_min,radius_max]', got '" +
                                *v + "'"};
            const int64_t n = pint(p[0], "spheres");
            const uint64_t seed = puint(p[1], "spheres");
            double lim[4] = {8.0, 40.0, 0.5, 2.0};  // the BASELINE.json config-2 field
            if (p.size() == 6)
                for (int j = 0; j < 4; ++j) lim[j] = pdouble(p[2 + j], "spheres");
            if (n < 0 || n > 1 << 20) throw UsageFail{"invalid spheres: count out of range"};
            sph.resize(static_cast<size_t>(n));
            if (n > 0 && bhrt_make_spheres(seed, static_cast<int32_t>(n), s->center, lim[0], lim[1], lim[2],
                                           lim[3], sph.data()) != 0)
                throw UsageFail{"invalid spheres: bad shell or radius range"};
        }
        const int32_t need = static_cast<int32_t>(sph.size());
        if (n_spheres) *n_spheres = need;
        s->n_spheres = need;
        s->spheres = need ? spheres : nullptr;
        if (need > cap || (need > 0 && !spheres))
            return fail(BHRT_INVALID_ARGUMENT, "scene text: sphere buffer too small (need " +
                                                   std::to_string(need) + ")");
        if (need) std::memcpy(spheres, sph.data(), sizeof(bhrt_sphere) * sph.size());
    } catch (const UsageFail& e) {
        return fail(BHRT_USAGE, e.msg);
    }
    if (info) {
        info->code = 0;
        info->px = info->py = -1;
        info->message[0] = 0;
    }
    return 0;
}

extern "C" int bhrt_scene_format_text(const bhrt_scene* s, char* buf, size_t cap, size_t* len) {
    if (!s) return BHRT_INVALID_ARGUMENT;
    // serialize_scene, config.cpp:96-112 (same keys, order and number format)
    std::string o;
    o += "mass=" + fmt(s->mass) + "\n";
    o += "center=" + fmt3(s->center) + "\n";
    o += "cam-pos=" + fmt3(s->cam_pos) + "\n";
    o += "look-at=" + fmt3(s->cam_look_at) + "\n";
    o += "fov-rad=" + fmt(s->vertical_fov) + "\n";
    o += "width=" + std::to_string(s->width) + "\n";
    o += "height=" + std::to_string(s->height) + "\n";
    o += "spp=" + std::to_string(s->spp) + "\n";
    o += "seed=" + std::to_string(s->seed) + "\n";
    o += "epsilon=" + fmt(s->epsilon) + "\n";
    o += "escape-radius=" + fmt(s->escape_radius) + "\n";
    o += "max-windings=" + std::to_string(s->max_windings) + "\n";
    o += "rel-tol=" + fmt(s->rel_tol) + "\n";
    o += "abs-tol=" + fmt(s->abs_tol) + "\n";
    // extension keys that differ from bhrt_scene_defaults
    bhrt_scene d;
    bhrt_scene_defaults(&d);
    if (s->integrator != d.integrator && s->integrator >= 0 && s->integrator < 4)
        o += std::string("integrator=") + kIntegrators[s->integrator] + "\n";
    if (!same(s->step, d.step)) o += "step=" + fmt(s->step) + "\n";
    if (!same(s->max_step, d.max_step)) o += "max-step=" + fmt(s->max_step) + "\n";
    if (!same(s->chord_dphi, d.chord_dphi)) o += "chord-dphi=" + fmt(s->chord_dphi) + "\n";
    if (s->sky_kind != d.sky_kind) o += std::string("sky=") + (s->sky_kind == BHRT_SKY_CHECKER ? "checker" : "image") + "\n";
    if (s->checker_nu != d.checker_nu || s->checker_nv != d.checker_nv)
        o += "checker=" + std::to_string(s->checker_nu) + "," + std::to_string(s->checker_nv) + "\n";
    if (!same3(s->checker_color_a, d.checker_color_a)) o += "checker-color-a=" + fmt3(s->checker_color_a) + "\n";
    if (!same3(s->checker_color_b, d.checker_color_b)) o += "checker-color-b=" + fmt3(s->checker_color_b) + "\n";
    if (s->disk_enabled) o += "disk=" + fmt(s->disk_r_in) + "," + fmt(s->disk_r_out) + "\n";
    if (!same3(s->disk_color_in, d.disk_color_in)) o += "disk-color-in=" + fmt3(s->disk_color_in) + "\n";
    if (!same3(s->disk_color_out, d.disk_color_out)) o += "disk-color-out=" + fmt3(s->disk_color_out) + "\n";
    if (!same3(s->light_dir, d.light_dir)) o += "light-dir=" + fmt3(s->light_dir) + "\n";
    if (!same(s->ambient, d.ambient)) o += "ambient=" + fmt(s->ambient) + "\n";
    if (s->table_entries != d.table_entries) o += "table-entries=" + std::to_string(s->table_entries) + "\n";
    if (s->table_samples != d.table_samples) o += "table-samples=" + std::to_string(s->table_samples) + "\n";
    if (!same(s->table_b_max, d.table_b_max)) o += "table-b-max=" + fmt(s->table_b_max) + "\n";
    if (!same(s->table_dpsi, d.table_dpsi)) o += "table-dpsi=" + fmt(s->table_dpsi) + "\n";
    for (int i = 0; i < s->n_spheres && s->spheres; ++i) {
        const bhrt_sphere& b = s->spheres[i];
        o += "sphere." + std::to_string(i) + "=" + fmt3(b.center) + "," + fmt(b.radius) + "," + fmt3(b.albedo) + "\n";
    }
    if (len) *len = o.size();
    if (!buf || cap <= o.size()) return BHRT_INVALID_ARGUMENT;
    std::memcpy(buf, o.c_str(), o.size() + 1);
    return 0;
}
