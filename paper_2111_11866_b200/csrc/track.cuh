// track.cuh -- GPU half of cell tracking (tracking.cpp): 26-connected
// component labelling, the chessboard distance transform, per-cell centres and
// the predecessor candidates used by backward linking.  See track.cu.
#pragma once

#include <vector>

#include "domain.cuh"
#include "subsurf_b200/track_link.hpp"

namespace ssb {

// F frames of n1*n2*n3 voxels (0-based x fastest, tracking.hpp:14-21).
class Tracker {
public:
    Tracker(int n1, int n2, int n3, int F, cudaStream_t s);

    uint8_t* mask() { return mask_.p; }   // fill before label() (device, frame-major)
    int* labels() { return lab_.p; }      // valid after label() / set_labels()
    long long frame_size() const { return fs_; }
    int n1() const { return n1_; }
    int n2() const { return n2_; }

    // label_components (tracking.cpp:69-127): final labels 1..k per frame by
    // decreasing size, ties by first voxel in scan order
    void label();
    // labels given by the caller (device or host array of F*fs int32)
    void set_labels(const int* labels, const std::vector<int>& labels_per_frame);
    const std::vector<int>& labels_per_frame() const { return lpf_; }

    // distance_centers (tracking.cpp:189-215): one cell per (frame, label)
    void centers();
    const std::vector<ssb_track::Cell>& cells() const { return cells_; }
    const std::vector<int>& first() const { return first_; }  // index of (f, label 1) in cells()
    // records given by the caller instead of centers() (ordered by frame, label)
    void set_cells(const std::vector<ssb_track::Cell>& cells);

    // backtrack_link's two predecessor candidates per cell (tracking.cpp:262-286):
    // label of frame f-1 under the centre, and at the distance centre of the
    // overlap with frame f-1's foreground (0 = none / frame 0)
    void targets(std::vector<int>& proj, std::vector<int>& overlap);

private:
    void distance(int mode);  // chessboard distance transform into dist_
    void cell_keys(int mode);  // per-cell argmax keys (+ voxel counts for mode 0)
    int n1_, n2_, n3_, F_;
    long long fs_, total_;
    cudaStream_t s_;
    Dev<uint8_t> mask_;
    Dev<int> parent_, lab_, dA_, dB_, aux_;
    Dev<unsigned long long> key_;
    Dev<int> count_, first_dev_;
    std::vector<int> lpf_, first_;
    std::vector<ssb_track::Cell> cells_;
};

// the whole pipeline (track_cells, tracking.cpp:374-391) on a filled mask:
// trajectories as (id, frame, x, y, z) rows in output order (tracking.cpp:393-401)
void track_points(Tracker& t, int window, double radius, std::vector<ss_track_point>& out);

}  // namespace ssb
