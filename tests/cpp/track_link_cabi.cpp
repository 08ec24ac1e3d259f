// C-ABI wrapper of the header-only host linking code (include/subsurf_b200/track_link.hpp)
// for the CPU test tests/test_track_link_cpu.py: prolong_and_merge on partials given as
// records (frame, x, y, z) concatenated + sizes.  Test infrastructure only.
#include "subsurf_b200/track_link.hpp"

extern "C" int tl_merge(int np, const int* sizes, const int* fxyz, int window, double radius, int* out_fxyz,
                        int* out_sizes) {
    std::vector<ssb_track::Cell> cells;
    std::vector<ssb_track::Chain> parts(np);
    int k = 0;
    for (int p = 0; p < np; ++p)
        for (int r = 0; r < sizes[p]; ++r, ++k) {
            ssb_track::Cell c;
            c.frame = fxyz[4 * k];
            c.cx = fxyz[4 * k + 1];
            c.cy = fxyz[4 * k + 2];
            c.cz = fxyz[4 * k + 3];
            parts[p].push_back((int)cells.size());
            cells.push_back(c);
        }
    const std::vector<ssb_track::Chain> m = ssb_track::merge(cells, parts, window, radius);
    int q = 0;
    for (size_t t = 0; t < m.size(); ++t) {
        out_sizes[t] = (int)m[t].size();
        for (int c : m[t]) {
            out_fxyz[4 * q] = cells[c].frame;
            out_fxyz[4 * q + 1] = cells[c].cx;
            out_fxyz[4 * q + 2] = cells[c].cy;
            out_fxyz[4 * q + 3] = cells[c].cz;
            ++q;
        }
    }
    return (int)m.size();
}
