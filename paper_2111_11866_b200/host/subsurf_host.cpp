// subsurf_host.cpp -- the C++ drop-in (include/subsurf_b200/subsurf.hpp) over the
// C ABI.  Parameter validation mirrors the reference (messages included) so
// callers see the same exceptions; the compute goes to the CUDA library.
#include "subsurf_b200/subsurf.hpp"

#include <algorithm>
#include <cmath>
#include <ostream>

#include "subsurf_b200.h"
#include "subsurf_b200/track_link.hpp"

namespace subsurf {

namespace {

ss_grid grid_of(const GridSpec& s) { return ss_grid{s.n1, s.n2, s.n3, s.n4, s.h1, s.h2, s.h3, s.h4}; }

std::vector<ss_center> centers_of(const CentersTable& t) {
    std::vector<ss_center> v;
    v.reserve(t.rows.size());
    for (const CenterRow& r : t.rows) v.push_back(ss_center{r.frame, r.x, r.y, r.z, r.radius});
    return v;
}

// status -> the reference's exception types (errors.hpp:9-39)
void raise(ss_status st, int iterations = 0, double residual = 0.0) {
    if (st == SS_OK) return;
    const std::string msg = ss_last_error();
    switch (st) {
        case SS_ERR_VALIDATION: throw ValidationError(msg);
        case SS_ERR_NOCONVERGE: throw SolverError(msg, residual, iterations);
        case SS_ERR_NONFINITE: throw NumericalError(msg);
        default: throw DeviceError(msg);
    }
}

void require(bool ok, const char* msg) {
    if (!ok) throw ValidationError(msg);
}

}  // namespace

GridSpec::GridSpec(int a, int b, int c, int d, double e, double f, double g, double h)
    : n1(a), n2(b), n3(c), n4(d), h1(e), h2(f), h3(g), h4(h) {
    require(n1 >= 1 && n2 >= 1 && n3 >= 1 && n4 >= 1, "GridSpec: doxel counts must be >= 1");
    require(h1 > 0.0 && h2 > 0.0 && h3 > 0.0 && h4 > 0.0, "GridSpec: spacings must be > 0");
}

void apply_dirichlet(Field4D& f, double value) {
    const ss_grid g = grid_of(f.spec());
    raise(ss_apply_dirichlet(&g, f.data(), value));
}

void apply_mirror_ghosts(Field4D& f) {
    const ss_grid g = grid_of(f.spec());
    raise(ss_apply_mirror_ghosts(&g, f.data()));
}

std::pair<double, double> interior_minmax(const Field4D& f) {
    const ss_grid g = grid_of(f.spec());
    double lo = 0.0, hi = 0.0;
    raise(ss_interior_minmax(&g, f.data(), &lo, &hi));
    return {lo, hi};
}

std::vector<CenterRow> CentersTable::for_frame(int frame) const {
    std::vector<CenterRow> out;
    for (const CenterRow& r : rows)
        if (r.frame == frame) out.push_back(r);
    return out;
}

void validate_centers(const CentersTable& t, const GridSpec& s) {
    for (std::size_t n = 0; n < t.rows.size(); ++n) {
        const CenterRow& r = t.rows[n];
        const std::string where = "centers row " + std::to_string(n + 1);
        if (r.frame < 0 || r.frame >= s.n4)
            throw ValidationError(where + ": frame " + std::to_string(r.frame) + " out of range [0," +
                                  std::to_string(s.n4 - 1) + "]");
        if (!(r.radius > 0.0)) throw ValidationError(where + ": radius must be > 0");
        if (r.x < 0.0 || r.x > s.n1 - 1 || r.y < 0.0 || r.y > s.n2 - 1 || r.z < 0.0 || r.z > s.n3 - 1)
            throw ValidationError(where + ": center outside volume bounds");
    }
}

Partition Partition::create(int n4, int workers) {
    require(n4 >= 1, "Partition: n4 must be >= 1");
    require(workers >= 1, "Partition: worker count must be >= 1");
    Partition p;
    p.n4_ = n4;
    p.workers_ = workers;
    p.chunk_ = (n4 + workers - 1) / workers;
    p.last_ = n4 - (workers - 1) * p.chunk_;
    if (p.last_ < 1)
        throw ValidationError("Partition: " + std::to_string(workers) + " workers leave the last one with " +
                              std::to_string(p.last_) + " slices of " + std::to_string(n4));
    return p;
}

int Partition::clamp_workers(int n4, int requested) {
    for (int w = std::min(requested, n4); w > 1; --w)
        if (n4 - (w - 1) * ((n4 + w - 1) / w) >= 1) return w;
    return 1;
}

Partition::Range Partition::range(int worker) const {
    const int b = worker * chunk_ + 1;
    return Range{b, b + (worker == workers_ - 1 ? last_ : chunk_) - 1};
}

void EdgeParams::validate() const {
    require(!(K < 0.0), "EdgeParams: K must be >= 0");
    require(!(delta < 0.0 || delta > 1.0), "EdgeParams: delta must be in [0,1]");
    require(!(vartheta < 0.0 || vartheta > 1.0), "EdgeParams: vartheta must be in [0,1]");
}

void SmoothingParams::validate() const {
    require(!(sigma < 0.0), "SmoothingParams: sigma must be >= 0");
    require(steps >= 1, "SmoothingParams: steps must be >= 1");
    require(sor_tol > 0.0, "SmoothingParams: sor_tol must be > 0");
    require(sor_max_iter >= 1, "SmoothingParams: sor_max_iter must be >= 1");
    require(omega > 0.0 && omega < 2.0, "SmoothingParams: omega must lie in (0,2)");
}

void ThresholdParams::validate() const {
    require(!(lambda < 0.0 || lambda > 1.0), "ThresholdParams: lambda must be in [0,1]");
}

void InitParams::validate() const {
    require(v > 0.0, "InitParams: v must be > 0");
    require(R > 0.0, "InitParams: R must be > 0");
}

void SolverParams::validate() const {
    require(!(tau < 0.0), "SolverParams: tau must be >= 0");
    require(epsilon > 0.0, "SolverParams: epsilon must be > 0");
    require(omega > 0.0 && omega < 2.0, "SolverParams: omega must lie in (0,2)");
    require(sor_tol > 0.0, "SolverParams: sor_tol must be > 0");
    require(sor_max_iter >= 1, "SolverParams: sor_max_iter must be >= 1");
    require(n_steps >= 1, "SolverParams: n_steps must be >= 1");
}

FaceCoefficientField face_coefficients(const Field4D& I0s, const Field4D& ITs, const EdgeParams& p,
                                       const GridSpec& spec, int) {
    p.validate();
    if (I0s.spec() != spec || ITs.spec() != spec)
        throw ValidationError("face_coefficients: images must share the grid spec");
    FaceCoefficientField out(spec);
    const ss_grid g = grid_of(spec);
    raise(ss_face_coefficients(&g, I0s.data(), ITs.data(), p.K, p.delta, p.vartheta,
                               reinterpret_cast<double*>(out.data())));
    return out;
}

Field4D heat_smooth(const Field4D& image, const SmoothingParams& p, int) {
    p.validate();
    Field4D out(image.spec());
    const ss_grid g = grid_of(image.spec());
    raise(ss_heat_smooth(&g, image.data(), p.sigma, p.steps, p.omega, p.sor_tol, p.sor_max_iter, out.data()));
    return out;
}

Field4D local_threshold(const Field4D& image, const CentersTable& c, const ThresholdParams& p) {
    p.validate();
    validate_centers(c, image.spec());
    Field4D out(image.spec());
    const ss_grid g = grid_of(image.spec());
    const std::vector<ss_center> cs = centers_of(c);
    raise(ss_local_threshold(&g, image.data(), cs.data(), (int)cs.size(), p.lambda, p.background, out.data()));
    return out;
}

Field4D build_initial(const CentersTable& c, const InitParams& p, const GridSpec& spec) {
    p.validate();
    validate_centers(c, spec);
    Field4D u(spec);
    const ss_grid g = grid_of(spec);
    const std::vector<ss_center> cs = centers_of(c);
    raise(ss_build_initial(&g, cs.data(), (int)cs.size(), p.v, p.R, p.profile == InitProfile::peak ? 0 : 1,
                           u.data()));
    return u;
}

void local_rescale(Field4D& u, const CentersTable& c, std::optional<double> radius) {
    validate_centers(c, u.spec());
    const ss_grid g = grid_of(u.spec());
    const std::vector<ss_center> cs = centers_of(c);
    raise(ss_local_rescale(&g, u.data(), cs.data(), (int)cs.size(), radius.value_or(std::nan(""))));
}

StepCoefficients assemble_step(const Field4D& u_prev, const FaceCoefficientField* G, const SolverParams& p,
                               const GridSpec& spec, int) {
    p.validate();
    if (u_prev.spec() != spec) throw ValidationError("assemble_step: field/spec mismatch");
    if (G && G->spec() != spec) throw ValidationError("assemble_step: G/spec mismatch");
    StepCoefficients c;
    c.spec = spec;
    c.offdiag.resize(spec.padded_size());
    c.diag.resize(spec.padded_size());
    c.abar.resize(spec.padded_size());
    const ss_grid g = grid_of(spec);
    raise(ss_assemble_step(&g, u_prev.data(), G ? reinterpret_cast<const double*>(G->data()) : nullptr, p.tau,
                           p.epsilon, reinterpret_cast<double*>(c.offdiag.data()), c.diag.data(), c.abar.data()));
    return c;
}

StepCoefficients assemble_heat_step(const GridSpec& spec, double dt, int) {
    require(dt > 0.0, "assemble_heat_step: dt must be > 0");
    StepCoefficients c;
    c.spec = spec;
    c.offdiag.resize(spec.padded_size());
    c.diag.resize(spec.padded_size());
    c.abar.resize(spec.padded_size());
    const ss_grid g = grid_of(spec);
    raise(ss_assemble_heat_step(&g, dt, reinterpret_cast<double*>(c.offdiag.data()), c.diag.data(),
                                c.abar.data()));
    return c;
}

SorResult redblack_sor(const StepCoefficients& coeff, const Field4D& rhs, Field4D u_guess,
                       const SolverParams& p, const Partition& partition) {
    p.validate();
    const GridSpec& spec = u_guess.spec();
    if (coeff.spec != spec || rhs.spec() != spec)
        throw ValidationError("redblack_sor: grid mismatch between coefficients and fields");
    if (partition.n4() != spec.n4) throw ValidationError("redblack_sor: partition built for a different time axis");
    const ss_grid g = grid_of(spec);
    int it = 0;
    double res = 0.0;
    const ss_status st = ss_redblack_sor(&g, reinterpret_cast<const double*>(coeff.offdiag.data()), rhs.data(),
                                         u_guess.data(), p.omega, p.sor_tol, p.sor_max_iter,
                                         partition.worker_count(), &it, &res);
    raise(st, it, res);
    return SorResult{std::move(u_guess), it, res};
}

bool check_minmax(const Field4D& u_next, const Field4D& u_prev_rescaled, double slack) {
    const auto [nlo, nhi] = interior_minmax(u_next);
    const auto [plo, phi] = interior_minmax(u_prev_rescaled);
    return plo - slack <= nlo && nhi <= phi + slack;
}

Field4D segment(const Field4D& image, const CentersTable& centers, const SegmentationParams& sp,
                std::ostream* diagnostics) {
    sp.solver.validate();
    sp.smoothing.validate();
    sp.threshold.validate();
    sp.edge.validate();
    sp.init.validate();
    validate_centers(centers, image.spec());
    ss_seg_params p{};
    p.tau = sp.solver.tau;
    p.epsilon = sp.solver.epsilon;
    p.omega = sp.solver.omega;
    p.sor_tol = sp.solver.sor_tol;
    p.sor_max_iter = sp.solver.sor_max_iter;
    p.n_steps = sp.solver.n_steps;
    p.rescale_each_step = sp.solver.rescale_each_step ? 1 : 0;
    p.sor_rel_tol = 0.0;
    p.sigma = sp.smoothing.sigma;
    p.smooth_steps = sp.smoothing.steps;
    p.smooth_tol = sp.smoothing.sor_tol;
    p.smooth_max_iter = sp.smoothing.sor_max_iter;
    p.smooth_omega = sp.smoothing.omega;
    p.lambda = sp.threshold.lambda;
    p.background = sp.threshold.background;
    p.K = sp.edge.K;
    p.delta = sp.edge.delta;
    p.vartheta = sp.edge.vartheta;
    p.init_v = sp.init.v;
    p.init_R = sp.init.R;
    p.init_profile = sp.init.profile == InitProfile::peak ? 0 : 1;
    p.rescale_radius = sp.rescale_radius.value_or(std::nan(""));
    Field4D u(image.spec());
    std::vector<ss_step_diag> d(sp.solver.n_steps);
    const ss_grid g = grid_of(image.spec());
    const std::vector<ss_center> cs = centers_of(centers);
    const ss_status st = ss_segment(&g, image.data(), cs.data(), (int)cs.size(), &p, nullptr, u.data(), d.data());
    // steps that completed print their diagnostics line (solver.cpp:433-438); a SolverError
    // carries the failing step's iterations and last residual
    int done = sp.solver.n_steps, failed = -1;
    if (st == SS_ERR_NOCONVERGE)
        for (int s = 0; s < sp.solver.n_steps; ++s)
            if (d[s].tol < 0.0) {  // ss_segment marks the failing step
                failed = s;
                done = s;
                break;
            }
    if (st != SS_OK && failed < 0) done = 0;
    if (diagnostics)
        for (int s = 0; s < done; ++s)
            (*diagnostics) << "step " << s + 1 << "/" << sp.solver.n_steps << " sor_iters=" << d[s].iterations
                           << " residual=" << d[s].residual << " min=" << d[s].umin << " max=" << d[s].umax
                           << "\n";
    if (failed >= 0) raise(st, d[failed].iterations, d[failed].residual);
    raise(st);
    return u;
}

MaskFrames extract_mask(const Field4D& u, double level) {
    const GridSpec& s = u.spec();
    MaskFrames m;
    m.n1 = s.n1;
    m.n2 = s.n2;
    m.n3 = s.n3;
    std::vector<std::uint8_t> all(s.interior_size());
    const ss_grid g = grid_of(s);
    raise(ss_extract_mask(&g, u.data(), level, all.data()));
    m.frames.resize(s.n4);
    for (int l = 0; l < s.n4; ++l)
        m.frames[l].assign(all.begin() + std::size_t(l) * m.frame_size(),
                           all.begin() + std::size_t(l + 1) * m.frame_size());
    return m;
}

// ---------------------------------------------------------------- tracking
namespace {

ss_grid frames_grid(int n1, int n2, int n3, std::size_t frames) {
    return ss_grid{n1, n2, n3, int(frames), 1.0, 1.0, 1.0, 1.0};
}

std::vector<std::int32_t> flat_labels(const LabelField& L) {
    std::vector<std::int32_t> all;
    all.reserve(L.frame_size() * L.frames.size());
    for (const auto& f : L.frames) {
        if (f.size() != L.frame_size()) throw ValidationError("label frame size mismatch");
        all.insert(all.end(), f.begin(), f.end());
    }
    return all;
}

ssb_track::Cell cell_of(const CellRecord& r) {
    ssb_track::Cell c;
    c.frame = r.frame;
    c.label = r.label;
    c.cx = r.center[0];
    c.cy = r.center[1];
    c.cz = r.center[2];
    c.max_distance = r.max_distance;
    c.voxel_count = (long long)r.voxel_count;
    return c;
}

}  // namespace

MaskFrames mask_from_labels(const LabelField& labels) {  // tracking.cpp:55-67
    MaskFrames m;
    m.n1 = labels.n1;
    m.n2 = labels.n2;
    m.n3 = labels.n3;
    m.frames.resize(labels.frames.size());
    for (std::size_t f = 0; f < labels.frames.size(); ++f) {
        m.frames[f].resize(labels.frames[f].size());
        for (std::size_t v = 0; v < labels.frames[f].size(); ++v) m.frames[f][v] = labels.frames[f][v] > 0 ? 1 : 0;
    }
    return m;
}

LabelField label_components(const MaskFrames& mask) {
    LabelField L;
    L.n1 = mask.n1;
    L.n2 = mask.n2;
    L.n3 = mask.n3;
    const std::size_t F = mask.frames.size(), fs = mask.frame_size();
    L.frames.resize(F);
    L.labels_per_frame.assign(F, 0);
    if (F == 0 || fs == 0) return L;
    std::vector<std::uint8_t> all;
    all.reserve(fs * F);
    for (const auto& f : mask.frames) {
        if (f.size() != fs) throw ValidationError("mask frame size mismatch");
        all.insert(all.end(), f.begin(), f.end());
    }
    std::vector<std::int32_t> lab(fs * F);
    const ss_grid g = frames_grid(mask.n1, mask.n2, mask.n3, F);
    raise(ss_label_components(&g, all.data(), lab.data(), L.labels_per_frame.data()));
    for (std::size_t f = 0; f < F; ++f) L.frames[f].assign(lab.begin() + f * fs, lab.begin() + (f + 1) * fs);
    return L;
}

std::vector<CellRecord> distance_centers(const LabelField& labels) {
    const std::size_t F = labels.frames.size();
    std::vector<CellRecord> out;
    if (F == 0 || labels.frame_size() == 0) return out;
    const std::vector<std::int32_t> all = flat_labels(labels);
    int n = 0;
    for (int k : labels.labels_per_frame) n += k;
    std::vector<ss_cell_record> r(std::max(n, 1));
    const ss_grid g = frames_grid(labels.n1, labels.n2, labels.n3, F);
    int got = 0;
    raise(ss_distance_centers(&g, all.data(), labels.labels_per_frame.data(), r.data(), n, &got));
    out.resize(got);
    for (int i = 0; i < got; ++i) {
        out[i].frame = r[i].frame;
        out[i].label = r[i].label;
        out[i].center = {r[i].cx, r[i].cy, r[i].cz};
        out[i].max_distance = r[i].max_distance;
        out[i].voxel_count = std::size_t(r[i].voxel_count);
    }
    return out;
}

std::vector<Trajectory> backtrack_link(const std::vector<CellRecord>& records, const LabelField& labels) {
    const std::size_t F = labels.frames.size();
    std::vector<Trajectory> out;
    if (F == 0 || labels.frame_size() == 0) return out;
    const std::vector<std::int32_t> all = flat_labels(labels);
    std::vector<ss_cell_record> r(records.size());
    for (std::size_t i = 0; i < records.size(); ++i)
        r[i] = ss_cell_record{records[i].frame, records[i].label, records[i].center[0], records[i].center[1],
                              records[i].center[2], records[i].max_distance, (long long)records[i].voxel_count};
    std::vector<int> idx(std::max<std::size_t>(records.size(), 1)), starts(records.size() + 2);
    int nc = 0;
    const ss_grid g = frames_grid(labels.n1, labels.n2, labels.n3, F);
    raise(ss_backtrack_link(&g, all.data(), labels.labels_per_frame.data(), r.data(), int(records.size()),
                            idx.data(), starts.data(), &nc));
    out.resize(nc);
    for (int c = 0; c < nc; ++c) {
        out[c].id = c + 1;
        for (int k = starts[c]; k < starts[c + 1]; ++k) out[c].records.push_back(records[idx[k]]);
    }
    return out;
}

std::vector<Trajectory> prolong_and_merge(std::vector<Trajectory> partials, int window, double radius) {
    std::vector<ssb_track::Cell> cells;
    std::vector<CellRecord> recs;
    std::vector<ssb_track::Chain> parts(partials.size());
    for (std::size_t p = 0; p < partials.size(); ++p)
        for (const CellRecord& r : partials[p].records) {
            parts[p].push_back(int(cells.size()));
            cells.push_back(cell_of(r));
            recs.push_back(r);
        }
    const std::vector<ssb_track::Chain> merged = ssb_track::merge(cells, parts, window, radius);
    std::vector<Trajectory> out(merged.size());
    for (std::size_t t = 0; t < merged.size(); ++t) {
        out[t].id = int(t) + 1;
        for (int c : merged[t]) out[t].records.push_back(recs[c]);
    }
    return out;
}

std::vector<Trajectory> track_cells(const Field4D& u, const TrackParams& params) {
    const LabelField labels = label_components(extract_mask(u, params.level));
    const std::vector<CellRecord> records = distance_centers(labels);
    std::vector<Trajectory> merged =
        prolong_and_merge(backtrack_link(records, labels), params.window, params.radius);
    std::sort(merged.begin(), merged.end(), [&](const Trajectory& a, const Trajectory& b) {  // tracking.cpp:379-386
        const CellRecord& ra = a.records.front();
        const CellRecord& rb = b.records.front();
        if (ra.frame != rb.frame) return ra.frame < rb.frame;
        return labels.voxel(ra.center[0], ra.center[1], ra.center[2]) <
               labels.voxel(rb.center[0], rb.center[1], rb.center[2]);
    });
    for (std::size_t t = 0; t < merged.size(); ++t) merged[t].id = int(t) + 1;
    return merged;
}

TrajectoryFile track(const Field4D& u, const TrackParams& params) {
    const ss_grid g = grid_of(u.spec());
    std::vector<ss_track_point> pts(4096);
    int n = 0;
    ss_status st = ss_track(&g, u.data(), params.level, params.window, params.radius, pts.data(), int(pts.size()), &n);
    if (st != SS_OK && n > int(pts.size())) {
        pts.resize(n);
        st = ss_track(&g, u.data(), params.level, params.window, params.radius, pts.data(), n, &n);
    }
    raise(st);
    TrajectoryFile f;
    f.points.resize(n);
    for (int i = 0; i < n; ++i) f.points[i] = TrajectoryPoint{pts[i].trajectory_id, pts[i].frame, pts[i].x, pts[i].y, pts[i].z};
    return f;
}

}  // namespace subsurf
