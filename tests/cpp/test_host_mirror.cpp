// C++ drop-in test: the namespace-subsurf API (include/subsurf_b200/subsurf.hpp)
// against the oracle restatement (oracle/subsurf_oracle.c), bit for bit.
// Built and run by tests/test_gpu_host_cpp.py on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>

#include "subsurf_b200/subsurf.hpp"
#include "subsurf_oracle.h"

using namespace subsurf;

static int failures = 0;
#define CHECK(cond, what)                                         \
    do {                                                          \
        if (!(cond)) {                                            \
            std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
            ++failures;                                           \
        }                                                         \
    } while (0)

static bool same(const double* a, const double* b, std::size_t n) { return std::memcmp(a, b, n * 8) == 0; }

static Field4D random_field(const GridSpec& s, unsigned seed, double lo = 0.0, double hi = 1.0) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> d(lo, hi);
    Field4D f(s);
    for (std::size_t n = 0; n < f.size(); ++n) f.data()[n] = d(rng);
    return f;
}

int main() {
    const GridSpec spec(9, 7, 6, 5, 0.2, 0.25, 0.3, 0.5);
    const or_grid og{spec.n1, spec.n2, spec.n3, spec.n4, spec.h1, spec.h2, spec.h3, spec.h4};
    const std::size_t P = spec.padded_size();

    // assemble_step with G
    Field4D u = random_field(spec, 1);
    FaceCoefficientField G(spec);
    {
        std::mt19937_64 rng(2);
        std::uniform_real_distribution<double> d(0.05, 1.0);
        for (std::size_t n = 0; n < P; ++n)
            for (int f = 0; f < 8; ++f) G.data()[n][f] = d(rng);
    }
    SolverParams sp;
    sp.tau = 0.07;
    sp.epsilon = 2e-3;
    sp.omega = 1.3;
    sp.sor_tol = 1e-12;
    const StepCoefficients c = assemble_step(u, &G, sp, spec);
    std::vector<double> off(8 * P), dg(P), ab(P);
    or_assemble_step(&og, u.data(), reinterpret_cast<const double*>(G.data()), sp.tau, sp.epsilon, off.data(),
                     dg.data(), ab.data());
    CHECK(same(reinterpret_cast<const double*>(c.offdiag.data()), off.data(), 8 * P), "assemble offdiag");
    CHECK(same(c.diag.data(), dg.data(), P), "assemble diag");
    CHECK(same(c.abar.data(), ab.data(), P), "assemble abar");

    // redblack_sor
    const Field4D rhs = random_field(spec, 3);
    const SorResult r = redblack_sor(c, rhs, u, sp, Partition::create(spec.n4, 3));
    std::vector<double> uo(u.data(), u.data() + P);
    int it = 0;
    double res = 0.0;
    or_redblack_sor(&og, off.data(), rhs.data(), uo.data(), sp.omega, sp.sor_tol, sp.sor_max_iter, &it, &res);
    CHECK(r.iterations == it, "sor iterations");
    CHECK(same(r.u.data(), uo.data(), P), "sor u");
    CHECK(std::fabs(r.residual - res) <= 1e-12 * res, "sor residual");

    // SolverError carries iterations and residual
    {
        SolverParams bad = sp;
        bad.sor_tol = 1e-300;
        bad.sor_max_iter = 5;
        bool thrown = false;
        try {
            redblack_sor(c, rhs, u, bad, Partition::create(spec.n4, 1));
        } catch (const SolverError& e) {
            thrown = e.iterations == 5 && e.last_residual > 0.0;
        }
        CHECK(thrown, "SolverError");
    }
    {
        bool thrown = false;
        try {
            SolverParams bad = sp;
            bad.omega = 2.0;
            assemble_step(u, nullptr, bad, spec);
        } catch (const ValidationError&) {
            thrown = true;
        }
        CHECK(thrown, "ValidationError");
    }

    // preprocess + edge
    const Field4D img = random_field(spec, 4);
    SmoothingParams smp;
    smp.sigma = 0.3;
    smp.steps = 2;
    const Field4D I0s = heat_smooth(img, smp);
    std::vector<double> tmp(P);
    or_heat_smooth(&og, img.data(), smp.sigma, smp.steps, smp.omega, smp.sor_tol, smp.sor_max_iter, tmp.data());
    CHECK(same(I0s.data(), tmp.data(), P), "heat_smooth");

    CentersTable ct;
    ct.rows = {{0, 4.0, 3.0, 2.5, 2.0}, {0, 5.0, 3.5, 2.5, 1.5}, {3, 1.0, 1.0, 1.0, 2.5}, {4, 8.0, 6.0, 5.0, 3.0}};
    std::vector<or_center> oc;
    for (const CenterRow& rr : ct.rows) oc.push_back(or_center{rr.frame, rr.x, rr.y, rr.z, rr.radius});
    ThresholdParams tp;
    tp.lambda = 0.4;
    const Field4D th = local_threshold(img, ct, tp);
    or_local_threshold(&og, img.data(), oc.data(), (int)oc.size(), tp.lambda, tp.background, tmp.data());
    CHECK(same(th.data(), tmp.data(), P), "local_threshold");

    EdgeParams ep;
    ep.K = 30.0;
    ep.delta = 0.5;
    ep.vartheta = 0.5;
    const FaceCoefficientField Gf = face_coefficients(I0s, th, ep, spec);
    std::vector<double> gref(8 * P);
    or_face_coefficients(&og, I0s.data(), th.data(), ep.K, ep.delta, ep.vartheta, gref.data());
    CHECK(same(reinterpret_cast<const double*>(Gf.data()), gref.data(), 8 * P), "face_coefficients");

    // seedinit
    InitParams ip;
    ip.R = 3.0;
    const Field4D u0 = build_initial(ct, ip, spec);
    or_build_initial(&og, oc.data(), (int)oc.size(), ip.v, ip.R, 0, tmp.data());
    CHECK(same(u0.data(), tmp.data(), P), "build_initial");
    Field4D ur = img;
    local_rescale(ur, ct, 2.2);
    std::memcpy(tmp.data(), img.data(), P * 8);
    or_local_rescale(&og, tmp.data(), oc.data(), (int)oc.size(), 2.2);
    CHECK(same(ur.data(), tmp.data(), P), "local_rescale");

    // grid helpers
    Field4D mg = img;
    apply_mirror_ghosts(mg);
    std::memcpy(tmp.data(), img.data(), P * 8);
    or_apply_mirror_ghosts(&og, tmp.data());
    CHECK(same(mg.data(), tmp.data(), P), "apply_mirror_ghosts");
    const auto [lo, hi] = interior_minmax(img);
    double olo, ohi;
    or_interior_minmax(&og, img.data(), &olo, &ohi);
    CHECK(lo == olo && hi == ohi, "interior_minmax");

    // segment() end to end with diagnostics
    SegmentationParams seg;
    seg.solver.tau = 0.125;
    seg.solver.epsilon = 1e-3;
    seg.solver.omega = 1.4;
    seg.solver.sor_tol = 1e-9;
    seg.solver.n_steps = 2;
    seg.smoothing.sigma = 0.2;
    seg.edge = ep;
    seg.init.R = 3.0;
    seg.rescale_radius = 2.5;
    std::ostringstream diag;
    const Field4D us = segment(img, ct, seg, &diag);
    or_seg_params op{};
    op.tau = seg.solver.tau;
    op.epsilon = seg.solver.epsilon;
    op.omega = seg.solver.omega;
    op.sor_tol = seg.solver.sor_tol;
    op.sor_max_iter = seg.solver.sor_max_iter;
    op.n_steps = seg.solver.n_steps;
    op.rescale_each_step = 1;
    op.sigma = seg.smoothing.sigma;
    op.smooth_steps = 1;
    op.smooth_tol = 1e-10;
    op.smooth_max_iter = 10000;
    op.smooth_omega = 1.85;
    op.lambda = 0.5;
    op.K = ep.K;
    op.delta = ep.delta;
    op.vartheta = ep.vartheta;
    op.init_v = 1.0;
    op.init_R = 3.0;
    op.rescale_radius = 2.5;
    std::vector<or_step_diag> od(2);
    or_segment(&og, img.data(), oc.data(), (int)oc.size(), &op, nullptr, tmp.data(), od.data());
    CHECK(same(us.data(), tmp.data(), P), "segment");
    CHECK(diag.str().find("step 2/2 sor_iters=" + std::to_string(od[1].iterations)) != std::string::npos,
          "segment diagnostics line");

    // segment() with sor_max_iter too small for one of the steps: the completed steps'
    // diagnostics lines, then SolverError with the failing solve's iterations
    // (solver.cpp:391-395, :433-438)
    {
        SegmentationParams bad = seg;
        const int M = od[1].iterations > od[0].iterations ? od[0].iterations
                                                           : std::min(od[0].iterations, od[1].iterations) - 1;
        const int fail = od[1].iterations > od[0].iterations ? 2 : (od[0].iterations > M ? 1 : 2);
        bad.solver.sor_max_iter = M;
        std::ostringstream bd;
        bool thrown = false;
        try {
            segment(img, ct, bad, &bd);
        } catch (const SolverError& e) {
            thrown = e.iterations == M && e.last_residual > 0.0;
        }
        CHECK(thrown, "segment SolverError payload");
        CHECK((bd.str().find("step 1/2") != std::string::npos) == (fail == 2) &&
                  bd.str().find("step 2/2") == std::string::npos,
              "segment diagnostics before SolverError");
    }

    const MaskFrames m = extract_mask(us, 0.5);
    std::vector<unsigned char> om(spec.interior_size());
    or_extract_mask(&og, us.data(), 0.5, om.data());
    bool mok = (int)m.frames.size() == spec.n4;
    for (int l = 0; l < spec.n4 && mok; ++l)
        mok = std::memcmp(m.frames[l].data(), om.data() + l * m.frame_size(), m.frame_size()) == 0;
    CHECK(mok, "extract_mask");

    // tracking: the composed C++ pipeline (label_components -> distance_centers ->
    // backtrack_link -> prolong_and_merge -> order) == the one-call GPU track()
    {
        const GridSpec ts(20, 16, 8, 6, 1.0, 1.0, 1.0, 1.0);
        Field4D tu(ts, 0.0);
        for (int l = 1; l <= ts.n4; ++l)
            for (int c = 0; c < 3; ++c) {
                const double cx = 4.0 + 5.0 * c + 0.7 * l, cy = 5.0 + 2.0 * c + 0.4 * l, cz = 3.5;
                for (int k = 1; k <= ts.n3; ++k)
                    for (int j = 1; j <= ts.n2; ++j)
                        for (int i = 1; i <= ts.n1; ++i) {
                            const double d = (i - 1 - cx) * (i - 1 - cx) / 4.0 + (j - 1 - cy) * (j - 1 - cy) / 3.0 +
                                             (k - 1 - cz) * (k - 1 - cz) / 2.0;
                            if (d < 1.0 && !(c == 1 && l == 3)) tu.at(i, j, k, l) = 1.0 - 0.3 * d;
                        }
            }
        const std::vector<Trajectory> tc = track_cells(tu, TrackParams{});
        const TrajectoryFile tf = track(tu, TrackParams{});
        std::size_t q = 0;
        bool tok = true;
        for (const Trajectory& t : tc)
            for (const CellRecord& r : t.records) {
                tok = tok && q < tf.points.size() && tf.points[q].trajectory_id == t.id && tf.points[q].frame == r.frame &&
                      tf.points[q].x == r.center[0] && tf.points[q].y == r.center[1] && tf.points[q].z == r.center[2];
                ++q;
            }
        CHECK(tok && q == tf.points.size() && !tc.empty(), "track_cells == track");
        const MaskFrames tm = mask_from_labels(label_components(extract_mask(tu, 0.5)));
        CHECK(tm.frames == extract_mask(tu, 0.5).frames, "mask_from_labels(label_components(mask)) == mask");
    }

    std::printf(failures ? "FAILED %d\n" : "ALL OK\n", failures);
    return failures ? 1 : 0;
}
