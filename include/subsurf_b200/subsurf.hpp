// subsurf.hpp -- C++ drop-in for the reference's solver API (namespace subsurf),
// executed on B200 through the C ABI in include/subsurf_b200.h.
//
// A program written against /root/reference/proj/include/subsurf/{grid,edge,
// preprocess,seedinit,solver,errors}.hpp compiles against this header unchanged
// for the hot-path calls: the same type names, members and free-function
// signatures (file:line of each original is cited), the same exceptions.
// Link with -lsubsurf_b200_host -lsubsurf_b200.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace subsurf {

// ---------------------------------------------------------------- errors (errors.hpp:9-39)
struct FormatError : std::runtime_error {
    explicit FormatError(const std::string& w) : std::runtime_error(w) {}
};
struct ValidationError : std::runtime_error {
    explicit ValidationError(const std::string& w) : std::runtime_error(w) {}
};
struct IoError : std::runtime_error {
    explicit IoError(const std::string& w) : std::runtime_error(w) {}
};
struct SolverError : std::runtime_error {
    SolverError(const std::string& w, double last_residual_, int iterations_)
        : std::runtime_error(w), last_residual(last_residual_), iterations(iterations_) {}
    double last_residual;
    int iterations;
};
struct NumericalError : std::runtime_error {
    explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};
// CUDA / device failures (no reference counterpart: the reference has no device)
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

// ---------------------------------------------------------------- grid (grid.hpp:16-119)
struct GridSpec {
    int n1 = 0, n2 = 0, n3 = 0, n4 = 0;
    double h1 = 1.0, h2 = 1.0, h3 = 1.0, h4 = 1.0;

    GridSpec() = default;
    GridSpec(int n1_, int n2_, int n3_, int n4_, double h1_, double h2_, double h3_, double h4_);
    static GridSpec cubic(int n1, int n2, int n3, int n4, double h) {
        return GridSpec(n1, n2, n3, n4, h, h, h, h);
    }
    static GridSpec isotropic(int n, double h) { return cubic(n, n, n, n, h); }
    int count(int axis) const { return axis == 0 ? n1 : axis == 1 ? n2 : axis == 2 ? n3 : n4; }
    double spacing(int axis) const { return axis == 0 ? h1 : axis == 1 ? h2 : axis == 2 ? h3 : h4; }
    std::optional<double> common_h() const {
        if (h1 == h2 && h2 == h3 && h3 == h4) return h1;
        return std::nullopt;
    }
    int i_max() const { return n1 + 2; }
    int j_max() const { return n2 + 2; }
    int k_max() const { return n3 + 2; }
    int l_max() const { return n4 + 2; }
    std::size_t padded_size() const { return std::size_t(i_max()) * j_max() * k_max() * l_max(); }
    std::size_t interior_size() const { return std::size_t(n1) * n2 * n3 * n4; }
    std::size_t frame_interior_size() const { return std::size_t(n1) * n2 * n3; }
    bool operator==(const GridSpec&) const = default;
};

struct Index4 {
    int i = 0, j = 0, k = 0, l = 0;
    bool operator==(const Index4&) const = default;
};

class Field4D {
public:
    Field4D() = default;
    explicit Field4D(const GridSpec& spec, double fill = 0.0) : spec_(spec), v_(spec.padded_size(), fill) {}
    const GridSpec& spec() const { return spec_; }
    std::size_t offset(int i, int j, int k, int l) const {
        return ((std::size_t(l) * spec_.k_max() + k) * spec_.j_max() + j) * spec_.i_max() + i;
    }
    double& at(int i, int j, int k, int l) { return v_[offset(i, j, k, l)]; }
    double at(int i, int j, int k, int l) const { return v_[offset(i, j, k, l)]; }
    double& operator[](const Index4& x) { return at(x.i, x.j, x.k, x.l); }
    double operator[](const Index4& x) const { return at(x.i, x.j, x.k, x.l); }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    std::size_t size() const { return v_.size(); }

private:
    GridSpec spec_;
    std::vector<double> v_;
};

void apply_dirichlet(Field4D& field, double value);           // grid.cpp:126-136
void apply_mirror_ghosts(Field4D& field);                     // grid.cpp:138-156
std::pair<double, double> interior_minmax(const Field4D& f);  // grid.cpp:158-171

// ---------------------------------------------------------------- io types used by the path (io.hpp:23-34)
struct CenterRow {
    int frame = 0;
    double x = 0.0, y = 0.0, z = 0.0;
    double radius = 0.0;
};
struct CentersTable {
    std::vector<CenterRow> rows;
    bool empty() const { return rows.empty(); }
    std::vector<CenterRow> for_frame(int frame) const;
};
void validate_centers(const CentersTable& table, const GridSpec& spec);  // io.cpp:128-140

// ---------------------------------------------------------------- parallel (parallel.hpp:13-47)
class Partition {
public:
    struct Range {
        int l_begin, l_end;
        int count() const { return l_end - l_begin + 1; }
    };
    Partition() = default;
    static Partition create(int n4, int workers);
    static int clamp_workers(int n4, int requested);
    int worker_count() const { return workers_; }
    int n4() const { return n4_; }
    int chunk() const { return chunk_; }
    Range range(int worker) const;

private:
    int n4_ = 1, workers_ = 1, chunk_ = 1, last_ = 1;
};

// ---------------------------------------------------------------- edge (edge.hpp:12-97)
struct EdgeParams {
    double K = 1.0, delta = 1.0, vartheta = 0.0;
    void validate() const;
};
inline double perona_malik(double s, double K) { return 1.0 / (1.0 + K * s * s); }

class FaceCoefficientField {
public:
    FaceCoefficientField() = default;
    explicit FaceCoefficientField(const GridSpec& spec)
        : spec_(spec), v_(spec.padded_size(), {1, 1, 1, 1, 1, 1, 1, 1}) {}
    const GridSpec& spec() const { return spec_; }
    std::size_t flat(int i, int j, int k, int l) const {
        return ((std::size_t(l) * spec_.k_max() + k) * spec_.j_max() + j) * spec_.i_max() + i;
    }
    std::array<double, 8>& at(int i, int j, int k, int l) { return v_[flat(i, j, k, l)]; }
    const std::array<double, 8>& at(int i, int j, int k, int l) const { return v_[flat(i, j, k, l)]; }
    const std::array<double, 8>* data() const { return v_.data(); }
    std::array<double, 8>* data() { return v_.data(); }

private:
    GridSpec spec_;
    std::vector<std::array<double, 8>> v_;
};

FaceCoefficientField face_coefficients(const Field4D& smoothed_image, const Field4D& smoothed_threshold,
                                       const EdgeParams& params, const GridSpec& spec, int workers = 1);

// ---------------------------------------------------------------- preprocess (preprocess.hpp:10-37)
struct SmoothingParams {
    double sigma = 0.0;
    int steps = 1;
    double sor_tol = 1e-10;
    int sor_max_iter = 10000;
    double omega = 1.85;
    void validate() const;
};
Field4D heat_smooth(const Field4D& image, const SmoothingParams& params, int workers = 1);

struct ThresholdParams {
    double lambda = 0.5, background = 0.0;
    void validate() const;
};
Field4D local_threshold(const Field4D& image, const CentersTable& centers, const ThresholdParams& params);

// ---------------------------------------------------------------- seedinit (seedinit.hpp:10-33)
enum class InitProfile { peak, linear };
struct InitParams {
    double v = 1.0, R = 10.0;
    InitProfile profile = InitProfile::peak;
    void validate() const;
};
Field4D build_initial(const CentersTable& centers, const InitParams& params, const GridSpec& spec);
void local_rescale(Field4D& u, const CentersTable& centers, std::optional<double> radius = std::nullopt);

// ---------------------------------------------------------------- solver (solver.hpp:19-92)
struct SolverParams {
    double tau = 1.0, epsilon = 1e-4, omega = 1.85, sor_tol = 1e-8;
    int sor_max_iter = 10000, n_steps = 10;
    bool rescale_each_step = true;
    void validate() const;
};

struct StepCoefficients {
    GridSpec spec;
    std::vector<std::array<double, 8>> offdiag;
    std::vector<double> diag;
    std::vector<double> abar;
    std::size_t flat(int i, int j, int k, int l) const {
        return ((std::size_t(l) * spec.k_max() + k) * spec.j_max() + j) * spec.i_max() + i;
    }
};

StepCoefficients assemble_step(const Field4D& u_prev, const FaceCoefficientField* G,
                               const SolverParams& params, const GridSpec& spec, int workers = 1);
StepCoefficients assemble_heat_step(const GridSpec& spec, double dt, int workers = 1);

struct SorResult {
    Field4D u;
    int iterations = 0;
    double residual = 0.0;
};
SorResult redblack_sor(const StepCoefficients& coeff, const Field4D& rhs, Field4D u_guess,
                       const SolverParams& params, const Partition& partition);
bool check_minmax(const Field4D& u_next, const Field4D& u_prev_rescaled, double slack = 0.0);

struct SegmentationParams {
    SolverParams solver;
    SmoothingParams smoothing;
    ThresholdParams threshold;
    EdgeParams edge;
    InitParams init;
    std::optional<double> rescale_radius;
    int workers = 1;
};
Field4D segment(const Field4D& image, const CentersTable& centers, const SegmentationParams& params,
                std::ostream* diagnostics = nullptr);

// ---------------------------------------------------------------- tracking (tracking.hpp:13-82)
struct MaskFrames {
    int n1 = 0, n2 = 0, n3 = 0;
    std::vector<std::vector<std::uint8_t>> frames;
    std::size_t voxel(int x, int y, int z) const { return (std::size_t(z) * n2 + y) * n1 + x; }
    std::size_t frame_size() const { return std::size_t(n1) * n2 * n3; }
};
struct LabelField {  // tracking.hpp:23-34
    int n1 = 0, n2 = 0, n3 = 0;
    std::vector<std::vector<std::int32_t>> frames;
    std::vector<int> labels_per_frame;
    std::size_t voxel(int x, int y, int z) const { return (std::size_t(z) * n2 + y) * n1 + x; }
    std::size_t frame_size() const { return std::size_t(n1) * n2 * n3; }
};
struct CellRecord {  // tracking.hpp:36-42
    int frame = 0;
    int label = 0;
    std::array<int, 3> center{};
    int max_distance = 0;
    std::size_t voxel_count = 0;
};
struct Trajectory {  // tracking.hpp:44-47
    int id = 0;
    std::vector<CellRecord> records;
};
struct TrackParams {  // tracking.hpp:49-53
    double level = 0.5;
    int window = 3;
    double radius = 5.0;
};
struct TrajectoryPoint {  // io.hpp:36-40
    int trajectory_id = 0;
    int frame = 0;
    double x = 0.0, y = 0.0, z = 0.0;
};
struct TrajectoryFile {  // io.hpp:42-44
    std::vector<TrajectoryPoint> points;
};
MaskFrames extract_mask(const Field4D& u, double level = 0.5);  // GPU
MaskFrames mask_from_labels(const LabelField& labels);          // host
LabelField label_components(const MaskFrames& mask);            // GPU
std::vector<CellRecord> distance_centers(const LabelField& labels);  // GPU
// GPU predecessor candidates + host linking
std::vector<Trajectory> backtrack_link(const std::vector<CellRecord>& records, const LabelField& labels);
// host
std::vector<Trajectory> prolong_and_merge(std::vector<Trajectory> partials, int window, double radius);
// the whole pipeline: GPU per-voxel work, host per-cell linking
std::vector<Trajectory> track_cells(const Field4D& u, const TrackParams& params = {});
TrajectoryFile track(const Field4D& u, const TrackParams& params = {});

}  // namespace subsurf
