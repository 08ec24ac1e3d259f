// cli.cpp -- `subsurf-b200`, a drop-in for the reference's `subsurf` CLI
// (cli.cpp:117-262) for the hot-path subcommands, running on the GPU:
//
//   subsurf-b200 segment --config FILE [--workers N] [--output PREFIX]
//   subsurf-b200 eoc [--max-n N] [--workers N] [--device D]
//   subsurf-b200 threshold-preview --config FILE [--output PREFIX]
//   subsurf-b200 track --config FILE [--output CSV]
//
// Config: `key = value` lines, `#` comments, later keys win (cli.cpp:193-215);
// the reference's keys and defaults (cli.cpp:73-107).  Extensions: `sor_rel_tol`
// (> 0: per-step tolerance rel * ||u^{n-1}||_2), `u0_header`/`u0_data` (an initial
// function instead of build_initial), `device`.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "subsurf_b200.h"
#include "subsurf_b200/io.hpp"
#include "subsurf_b200/subsurf.hpp"

using namespace subsurf;

namespace {

std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r");
    if (b == std::string::npos) return "";
    return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}

struct Config {
    std::map<std::string, std::string> kv;

    static Config load(const std::string& path) {
        std::ifstream in(path);
        if (!in) throw IoError("cannot open config file: " + path);
        Config c;
        std::string line;
        int lineno = 0;
        while (std::getline(in, line)) {
            ++lineno;
            line = trim(line.substr(0, line.find('#')));
            if (line.empty()) continue;
            const auto eq = line.find('=');
            if (eq == std::string::npos) throw FormatError(path + ":" + std::to_string(lineno) + ": expected key = value");
            const std::string key = trim(line.substr(0, eq));
            if (key.empty()) throw FormatError(path + ":" + std::to_string(lineno) + ": empty key");
            c.kv[key] = trim(line.substr(eq + 1));
        }
        return c;
    }
    bool has(const std::string& k) const { return kv.count(k) > 0; }
    std::string str(const std::string& k) const {
        auto it = kv.find(k);
        if (it == kv.end()) throw ValidationError("config: missing required key \"" + k + "\"");
        return it->second;
    }
    std::string str(const std::string& k, const std::string& dflt) const { return has(k) ? kv.at(k) : dflt; }
    double num(const std::string& k, double dflt) const {
        if (!has(k)) return dflt;
        try {
            return std::stod(kv.at(k));
        } catch (const std::exception&) {
            throw ValidationError("config: key \"" + k + "\" is not a number: " + kv.at(k));
        }
    }
    int integer(const std::string& k, int dflt) const {
        if (!has(k)) return dflt;
        try {
            return std::stoi(kv.at(k));
        } catch (const std::exception&) {
            throw ValidationError("config: key \"" + k + "\" is not an integer: " + kv.at(k));
        }
    }
    bool boolean(const std::string& k, bool dflt) const {
        if (!has(k)) return dflt;
        const std::string& v = kv.at(k);
        if (v == "1" || v == "true" || v == "yes" || v == "on") return true;
        if (v == "0" || v == "false" || v == "no" || v == "off") return false;
        throw ValidationError("config: key \"" + k + "\" is not a boolean: " + v);
    }
};

// cli.cpp:73-107 defaults, flattened into ss_seg_params
ss_seg_params params_of(const Config& c, const GridSpec& spec) {
    ss_seg_params p{};
    const double h = spec.common_h().value_or(spec.h1);
    p.tau = c.num("tau", 1.0);
    p.epsilon = c.num("epsilon", h * h);
    p.omega = c.num("omega", 1.85);
    p.sor_tol = c.num("sor_tol", 1e-8);
    p.sor_max_iter = c.integer("sor_max_iter", 10000);
    p.n_steps = c.integer("n_steps", 10);
    p.rescale_each_step = c.boolean("rescale_each_step", true) ? 1 : 0;
    p.sor_rel_tol = c.num("sor_rel_tol", 0.0);
    p.sigma = c.num("sigma", 0.0);
    p.smooth_steps = c.integer("smooth_steps", 1);
    p.smooth_tol = 1e-10;  // SmoothingParams defaults (not config keys in the reference)
    p.smooth_max_iter = 10000;
    p.smooth_omega = 1.85;
    p.lambda = c.num("lambda", 0.5);
    p.background = c.num("background", 0.0);
    p.K = c.num("K", 1.0);
    p.delta = c.num("delta", 1.0);
    p.vartheta = c.num("vartheta", 0.0);
    p.init_v = c.num("init_v", 1.0);
    p.init_R = c.num("init_R", 10.0);
    const std::string prof = c.str("init_profile", "peak");
    if (prof != "peak" && prof != "linear")
        throw ValidationError("config: init_profile must be peak or linear, got " + prof);
    p.init_profile = prof == "peak" ? 0 : 1;
    // set => explicit radius, even <= 0 (cli.cpp:104: the optional is engaged); unset =>
    // std::nullopt, NaN on the ABI (per-row radii)
    p.rescale_radius = c.has("rescale_radius") ? c.num("rescale_radius", 0.0) : std::nan("");
    return p;
}

void check(ss_status st) {
    if (st == SS_OK) return;
    const std::string m = ss_last_error();
    switch (st) {
        case SS_ERR_VALIDATION: throw ValidationError(m);
        case SS_ERR_NOCONVERGE: throw SolverError(m, 0.0, 0);
        case SS_ERR_NONFINITE: throw NumericalError(m);
        default: throw DeviceError(m);
    }
}

int cmd_segment(const std::string& config_path, int workers, const std::string& output_override) {
    const Config cfg = Config::load(config_path);
    const Field4D image = read_image4d(cfg.str("input_header"), cfg.str("input_data"));
    const GridSpec& spec = image.spec();
    const CentersTable centers = read_centers(cfg.str("centers"), spec);
    const int w = workers > 0 ? workers : cfg.integer("workers", 1);
    const int wc = Partition::clamp_workers(spec.n4, w);
    if (wc != w)  // cli.cpp:109-115 (the GPU path ignores the worker count otherwise)
        std::cerr << "note: " << w << " workers cannot tile " << spec.n4 << " time slices; using " << wc << "\n";
    const ss_seg_params p = params_of(cfg, spec);
    Field4D u0;
    if (cfg.has("u0_header")) u0 = read_image4d(cfg.str("u0_header"), cfg.str("u0_data"));
    const std::string output = output_override.empty() ? cfg.str("output") : output_override;

    std::vector<ss_center> cs;
    for (const CenterRow& r : centers.rows) cs.push_back(ss_center{r.frame, r.x, r.y, r.z, r.radius});
    const ss_grid g{spec.n1, spec.n2, spec.n3, spec.n4, spec.h1, spec.h2, spec.h3, spec.h4};
    Field4D u(spec);
    std::vector<ss_step_diag> d(p.n_steps);
    const ss_status st = ss_segment(&g, image.data(), cs.data(), (int)cs.size(), &p,
                                    u0.size() ? u0.data() : nullptr, u.data(), d.data());
    for (int s = 0; s < p.n_steps && d[s].iterations > 0 && d[s].tol >= 0.0; ++s)  // completed steps (solver.cpp:433-438)
        std::cerr << "step " << s + 1 << "/" << p.n_steps << " sor_iters=" << d[s].iterations
                  << " residual=" << d[s].residual << " min=" << d[s].umin << " max=" << d[s].umax << "\n";
    if (st == SS_ERR_NOCONVERGE)
        for (int s = 0; s < p.n_steps; ++s)
            if (d[s].tol < 0.0) throw SolverError(ss_last_error(), d[s].residual, d[s].iterations);
    check(st);
    write_image4d(u, output + ".json", output + ".raw");
    if (cfg.boolean("export_vtk", false))
        for (int l = 1; l <= spec.n4; ++l) export_frame_vtk(u, l, output + "_f" + std::to_string(l - 1) + ".vtk");
    return 0;
}

int cmd_threshold_preview(const std::string& config_path, const std::string& output_override) {
    const Config cfg = Config::load(config_path);
    const Field4D image = read_image4d(cfg.str("input_header"), cfg.str("input_data"));
    const CentersTable centers = read_centers(cfg.str("centers"), image.spec());
    ThresholdParams tp;
    tp.lambda = cfg.num("lambda", 0.5);
    tp.background = cfg.num("background", 0.0);
    const Field4D out = local_threshold(image, centers, tp);
    const std::string output = output_override.empty() ? cfg.str("output") : output_override;
    write_image4d(out, output + ".json", output + ".raw");
    return 0;
}

// cmd_track (cli.cpp:161-188): labelling, distance transform and predecessor
// candidates on the GPU, per-cell linking on the host
int cmd_track(const std::string& config_path, const std::string& output_override) {
    const Config cfg = Config::load(config_path);
    const Field4D u = read_image4d(cfg.str("input_header"), cfg.str("input_data"));
    TrackParams params;
    params.level = cfg.num("level", 0.5);
    params.window = cfg.integer("window", 3);
    params.radius = cfg.num("radius", 5.0);
    const std::string output = output_override.empty() ? cfg.str("output") : output_override;
    write_trajectories(track(u, params), output);
    if (cfg.has("vtk_prefix")) {
        const LabelField labels = label_components(extract_mask(u, params.level));
        const GridSpec& spec = u.spec();
        Field4D lf(spec, 0.0);
        for (int l = 1; l <= spec.n4; ++l)
            for (int k = 1; k <= spec.n3; ++k)
                for (int j = 1; j <= spec.n2; ++j)
                    for (int i = 1; i <= spec.n1; ++i)
                        lf.at(i, j, k, l) = double(labels.frames[l - 1][labels.voxel(i - 1, j - 1, k - 1)]);
        for (int l = 1; l <= spec.n4; ++l)
            export_frame_vtk(lf, l, cfg.str("vtk_prefix") + "_f" + std::to_string(l - 1) + ".vtk");
    }
    return 0;
}

// run_eoc + print_report (eoc.cpp:175-205) on the GPU
int cmd_eoc(int max_n, int device) {
    static const int sched[5] = {10, 20, 40, 80, 160};
    bool valid = false;
    for (int n : sched) valid = valid || n == max_n;
    if (!valid)
        throw ValidationError("EOC schedule has no row n=" + std::to_string(max_n) + " (valid: 10, 20, 40, 80, 160)");
    static const int steps[5] = {1, 4, 16, 64, 256};
    std::cout << "   n          h  final step         error        EOC\n";
    double prev = 0.0;
    for (int q = 0; q < 5 && sched[q] <= max_n; ++q) {
        const int n = sched[q];
        const double h = 2.5 / n;
        const ss_grid g{n, n, n, n, h, h, h, h};
        ss_session* s = nullptr;
        check(ss_session_create(&g, device, &s));
        double err = 0.0;
        long long sweeps = 0;
        const ss_status st = ss_session_eoc_row(s, n, 1.5, 1e-8, 10000, &err, &sweeps);
        ss_session_destroy(s);
        check(st);
        std::cout << std::setw(4) << n << "  " << std::setw(9) << h << "  " << std::setw(10) << steps[q] << "  "
                  << std::scientific << std::setprecision(6) << err << std::defaultfloat;
        if (q > 0) std::cout << "   " << std::fixed << std::setprecision(6) << std::log2(prev / err) << std::defaultfloat;
        std::cout << "\n";
        prev = err;
    }
    return 0;
}

void usage(std::ostream& o) {
    o << "subsurf-b200: 4D generalized subjective-surface segmentation on B200 (GPU)\n"
         "  segment --config FILE [--workers N] [--output PREFIX]\n"
         "  eoc [--max-n 10|20|40|80|160] [--workers N] [--device D]\n"
         "  threshold-preview --config FILE [--output PREFIX]\n"
         "  track --config FILE [--output CSV]\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
        usage(argc < 2 ? std::cerr : std::cout);
        return argc < 2 ? 2 : 0;
    }
    const std::string cmd = argv[1];
    std::string config_path, output;
    int workers = 0, max_n = 40, device = 0;
    for (int a = 2; a < argc; ++a) {
        const std::string opt = argv[a];
        auto value = [&](const char* name) -> std::string {
            if (a + 1 >= argc) {
                std::cerr << "error: " << name << " needs a value\n";
                std::exit(2);
            }
            return argv[++a];
        };
        try {
            if (opt == "--config") config_path = value("--config");
            else if (opt == "--output") output = value("--output");
            else if (opt == "--workers") workers = std::stoi(value("--workers"));
            else if (opt == "--max-n") max_n = std::stoi(value("--max-n"));
            else if (opt == "--device") device = std::stoi(value("--device"));
            else {
                std::cerr << "error: unknown option " << opt << "\n";
                usage(std::cerr);
                return 2;
            }
        } catch (const std::exception&) {
            std::cerr << "error: bad value for " << opt << "\n";
            return 2;
        }
    }
    try {
        if (cmd == "segment" || cmd == "threshold-preview" || cmd == "track") {
            if (config_path.empty()) {
                std::cerr << "error: --config is required\n";
                return 2;
            }
            if (cmd == "track") return cmd_track(config_path, output);
            return cmd == "segment" ? cmd_segment(config_path, workers, output)
                                    : cmd_threshold_preview(config_path, output);
        }
        if (cmd == "eoc") return cmd_eoc(max_n, device);
        std::cerr << "error: unknown subcommand " << cmd << "\n";
        usage(std::cerr);
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
