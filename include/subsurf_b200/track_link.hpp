// track_link.hpp -- the host-side (sequential, per-cell) half of the tracking
// pipeline of tracking.cpp: backward-in-time linking (backtrack_link,
// tracking.cpp:220-296), tangent prolongation + greedy merge (prolong_and_merge,
// tracking.cpp:312-372) and the final (first frame, first centre) ordering
// (track_cells, tracking.cpp:374-391).
//
// The per-voxel half (26-connected labelling, the chessboard distance
// transform, per-cell centres, the two predecessor candidates of every cell)
// runs on the GPU (paper_2111_11866_b200/csrc/track.cu); what arrives here is
// one record per cell plus its two candidate predecessor labels, so this code
// touches O(cells) data only.  Header-only so the CUDA library (C ABI
// ss_track) and the C++ mirror (subsurf::backtrack_link / prolong_and_merge)
// share one implementation.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <vector>

namespace ssb_track {

struct Cell {  // one labelled component of one frame (CellRecord, tracking.hpp:36-42)
    int frame = 0, label = 0;
    int cx = 0, cy = 0, cz = 0;  // 0-based voxel centre
    int max_distance = 0;
    long long voxel_count = 0;
};

// A partial / merged trajectory: indices into the cell array, frames increasing.
using Chain = std::vector<int>;

// backtrack_link (tracking.cpp:220-296).  `first[f]` = index of the cell
// (f, label 1) in `cells` (cells of a frame are stored by label);
// `proj[c]` = label of frame f-1 under cell c's centre (0: background) and
// `overlap[c]` = label of frame f-1 at the distance centre of the overlap of c
// with frame f-1's foreground (0: no overlap) -- both computed on the GPU.
inline std::vector<Chain> backtrack(const std::vector<int>& labels_per_frame, const std::vector<int>& first,
                                    const std::vector<Cell>& cells, const std::vector<int>& proj,
                                    const std::vector<int>& overlap) {
    const int F = (int)labels_per_frame.size();
    std::vector<Chain> rev;   // chains in decreasing frame order while building
    std::vector<int> tails;   // chain ending at (frame f, label) or -1
    for (int f = F - 1; f >= 0; --f) {
        const int k = labels_per_frame[f];
        if (f == F - 1) tails.assign((size_t)k, -1);
        for (int lb = 1; lb <= k; ++lb) {  // cells nobody linked to start a partial
            if (tails[lb - 1] >= 0) continue;
            rev.push_back(Chain{first[f] + lb - 1});
            tails[lb - 1] = (int)rev.size() - 1;
        }
        if (f == 0) break;
        const int kp = labels_per_frame[f - 1];
        std::vector<int> next(kp, -1);
        std::vector<char> claimed(kp, 0);
        std::vector<int> order(k);
        std::iota(order.begin(), order.end(), 1);
        std::sort(order.begin(), order.end(), [&](int a, int b) {  // larger cells claim first
            const long long na = cells[first[f] + a - 1].voxel_count, nb = cells[first[f] + b - 1].voxel_count;
            return na != nb ? na > nb : a < b;
        });
        for (int lb : order) {
            const int c = first[f] + lb - 1;
            const int target = proj[c] > 0 ? proj[c] : overlap[c];
            if (target > 0 && !claimed[target - 1]) {
                claimed[target - 1] = 1;
                rev[tails[lb - 1]].push_back(first[f - 1] + target - 1);
                next[target - 1] = tails[lb - 1];
            }
        }
        tails.swap(next);
    }
    for (Chain& ch : rev) std::reverse(ch.begin(), ch.end());
    return rev;
}

// prolong_and_merge (tracking.cpp:312-372): same candidate set, tie order and
// greedy pass; expressions evaluated as the reference writes them.
inline std::vector<Chain> merge(const std::vector<Cell>& cells, const std::vector<Chain>& parts, int window,
                                double radius) {
    struct Cand {
        int gap;
        double dist;
        int a, b;
    };
    auto pt = [&](int c, double out[3]) {
        out[0] = (double)cells[c].cx;
        out[1] = (double)cells[c].cy;
        out[2] = (double)cells[c].cz;
    };
    auto d3 = [](const double p[3], const double q[3]) {
        const double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
        return std::sqrt(dx * dx + dy * dy + dz * dz);
    };
    const int np = (int)parts.size();
    std::vector<Cand> cand;
    for (int a = 0; a < np; ++a) {
        const Chain& A = parts[a];
        const int a_last = A.back();
        for (int b = 0; b < np; ++b) {
            if (a == b) continue;
            const Chain& B = parts[b];
            const int b_first = B.front();
            const int gap = cells[b_first].frame - cells[a_last].frame;
            if (gap < 1 || gap > window) continue;
            double best = std::numeric_limits<double>::infinity();
            if (A.size() >= 2) {  // A's end, prolonged forward by gap frames
                double p1[3], p2[3], q[3], pred[3];
                pt(A[A.size() - 2], p1);
                pt(a_last, p2);
                pt(b_first, q);
                for (int d = 0; d < 3; ++d) pred[d] = p2[d] + gap * (p2[d] - p1[d]);
                best = std::min(best, d3(pred, q));
            }
            if (B.size() >= 2) {  // B's start, prolonged backward
                double q1[3], q2[3], p[3], pred[3];
                pt(b_first, q1);
                pt(B[1], q2);
                pt(a_last, p);
                for (int d = 0; d < 3; ++d) pred[d] = q1[d] - gap * (q2[d] - q1[d]);
                best = std::min(best, d3(pred, p));
            }
            if (best <= radius) cand.push_back({gap, best, a, b});
        }
    }
    std::sort(cand.begin(), cand.end(), [](const Cand& x, const Cand& y) {
        if (x.gap != y.gap) return x.gap < y.gap;
        if (x.dist != y.dist) return x.dist < y.dist;
        if (x.a != y.a) return x.a < y.a;
        return x.b < y.b;
    });
    std::vector<int> next(np, -1);
    std::vector<char> end_used(np, 0), start_used(np, 0);
    for (const Cand& c : cand) {
        if (end_used[c.a] || start_used[c.b]) continue;
        end_used[c.a] = start_used[c.b] = 1;
        next[c.a] = c.b;
    }
    std::vector<Chain> out;
    for (int h = 0; h < np; ++h) {
        if (start_used[h]) continue;  // not the head of a merged chain
        Chain m;
        for (int c = h; c != -1; c = next[c]) m.insert(m.end(), parts[c].begin(), parts[c].end());
        out.push_back(std::move(m));
    }
    return out;
}

// track_cells' final order (tracking.cpp:379-388): first frame, then the
// linear voxel index of the first centre.
inline void order(const std::vector<Cell>& cells, std::vector<Chain>& chains, int n1, int n2) {
    auto key = [&](const Chain& ch) {
        const Cell& c = cells[ch.front()];
        return std::make_pair(c.frame, ((long long)c.cz * n2 + c.cy) * n1 + c.cx);
    };
    std::sort(chains.begin(), chains.end(), [&](const Chain& a, const Chain& b) { return key(a) < key(b); });
}

}  // namespace ssb_track
