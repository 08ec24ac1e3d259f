// track.cu -- the per-voxel half of cell tracking (tracking.cpp) on the GPU.
//
// label_components (tracking.cpp:69-127).  The reference flood-fills in scan
// order and then ranks components by (size desc, first voxel asc).  Here:
// lock-free union-find over the 13 backward 26-neighbours, always linking the
// larger root under the smaller (atomicMin), so every component's root is its
// smallest linear index = its first voxel in scan order, whatever order the
// unions ran in; sizes by atomics; the per-frame ranking sort runs on the host
// over the (few) roots; a scatter + gather writes the final labels.
//
// bfs_distance (tracking.cpp:131-176) is the 26-neighbourhood BFS distance
// from the boundary voxels (those with a background or out-of-volume
// neighbour, distance 1).  For any foreground set that equals the chessboard
// (L-infinity) distance to the nearest non-member voxel, outside counting as
// non-member: the voxels strictly closer than that are all members, so the
// straight chessboard path stays inside the set.  The chessboard distance
// transform is separable: 1D run lengths along x, then
// D(y) = min_b max(|y-b|, D1(b)) along y and the same along z, each scan
// stopping once |y-b| reaches the best value so far (cells are a few voxels
// thick).  With "member" meaning "same class", one pass serves both uses:
//   mode 0: class = foreground (distance_centers, tracking.cpp:189-215);
//   mode 1: class = label of the cell where frame f-1 is foreground, the
//           overlap regions of backtrack_link (tracking.cpp:268-284), all
//           cells of all frames at once.
// Cell centre = max distance, ties by smallest linear index: one 64-bit
// atomicMax per voxel on (distance << 32 | ~index).
#include <algorithm>
#include <cstring>

#include "track.cuh"

namespace ssb {

namespace {

constexpr int kTB = 256;

__device__ __forceinline__ int ld_vol(const int* p) { return *(volatile const int*)p; }

__device__ __forceinline__ int find_root(const int* base, int x) {
    int p = ld_vol(base + x);
    while (p != x) {
        x = p;
        p = ld_vol(base + x);
    }
    return x;
}

// link the two components; the root of the union is the smaller index
__device__ __forceinline__ void unite(int* base, int a, int b) {
    while (true) {
        a = find_root(base, a);
        b = find_root(base, b);
        if (a == b) return;
        if (a < b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicMin(base + a, b);
        if (old == a) return;
        a = old;  // a was linked elsewhere meanwhile: unite that tree with b
    }
}

struct Geo3 {
    int n1, n2, n3;
    long long fs;
};

__global__ void ccl_init(const uint8_t* __restrict__ mask, int* parent, long long total, long long fs) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
         v += (long long)gridDim.x * blockDim.x)
        parent[v] = mask[v] ? (int)(v % fs) : -1;
}

__global__ void ccl_merge(const uint8_t* __restrict__ mask, int* parent, Geo3 g, long long total) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
         v += (long long)gridDim.x * blockDim.x) {
        if (!mask[v]) continue;
        const long long f = v / g.fs;
        const int loc = (int)(v - f * g.fs);
        const int x = loc % g.n1, y = (loc / g.n1) % g.n2, z = loc / (g.n1 * g.n2);
        int* base = parent + f * g.fs;
        const uint8_t* mb = mask + f * g.fs;
        // the 13 neighbours that precede this voxel in scan order
#pragma unroll
        for (int q = 0; q < 13; ++q) {
            const int dz = q < 9 ? -1 : 0;
            const int r = q < 9 ? q : q - 9;  // dz = -1: 3x3 plane; dz = 0: (-1,-1) (0,-1) (1,-1) (-1,0)
            const int dy = dz < 0 ? r / 3 - 1 : (r < 3 ? -1 : 0);
            const int dx = dz < 0 ? r % 3 - 1 : (r < 3 ? r - 1 : -1);
            const int nx = x + dx, ny = y + dy, nz = z + dz;
            if (nx < 0 || nx >= g.n1 || ny < 0 || ny >= g.n2 || nz < 0) continue;
            const int nl = (nz * g.n2 + ny) * g.n1 + nx;
            if (mb[nl]) unite(base, loc, nl);
        }
    }
}

// flatten to roots; count each component at its root; count the roots
__global__ void ccl_flatten(int* parent, int* count, long long total, long long fs, unsigned long long* n_roots) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
         v += (long long)gridDim.x * blockDim.x) {
        if (parent[v] < 0) continue;
        const long long f = v / fs;
        const int loc = (int)(v - f * fs);
        const int r = find_root(parent + f * fs, loc);
        parent[v] = r;
        atomicAdd(count + f * fs + r, 1);
        if (r == loc) atomicAdd(n_roots, 1ull);
    }
}

__global__ void ccl_roots(const int* parent, const int* count, long long total, long long fs,
                          unsigned long long* slot, long long* roots, int* sizes) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
         v += (long long)gridDim.x * blockDim.x) {
        const long long f = v / fs;
        if (parent[v] != (int)(v - f * fs)) continue;
        const unsigned long long i = atomicAdd(slot, 1ull);
        roots[i] = v;
        sizes[i] = count[v];
    }
}

__global__ void scatter_rank(const long long* roots, const int* rank, long long n, int* at_root) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        at_root[roots[i]] = rank[i];
}

__global__ void apply_labels(const int* parent, const int* at_root, int* lab, long long total, long long fs) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
         v += (long long)gridDim.x * blockDim.x) {
        const int p = parent[v];
        lab[v] = p < 0 ? 0 : at_root[(v / fs) * fs + p];
    }
}

template <int MODE>
__device__ __forceinline__ int vclass(const int* __restrict__ lab, long long v, long long fs) {
    if (MODE == 0) return lab[v] > 0;
    return v >= fs && lab[v - fs] > 0 ? lab[v] : 0;  // frame 0 has no predecessor
}

// 1D run lengths along x: one thread per row
template <int MODE>
__global__ void dt_x(const int* __restrict__ lab, int* __restrict__ d, Geo3 g, long long rows) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
         r += (long long)gridDim.x * blockDim.x) {
        const long long b = r * g.n1;
        int run = 0, prev = 0;
        for (int x = 0; x < g.n1; ++x) {
            const int c = vclass<MODE>(lab, b + x, g.fs);
            run = c == 0 ? 0 : (x > 0 && c == prev ? run + 1 : 1);
            d[b + x] = run;
            prev = c;
        }
        run = 0;
        prev = 0;
        for (int x = g.n1 - 1; x >= 0; --x) {
            const int c = vclass<MODE>(lab, b + x, g.fs);
            run = c == 0 ? 0 : (x < g.n1 - 1 && c == prev ? run + 1 : 1);
            d[b + x] = min(d[b + x], run);
            prev = c;
        }
    }
}

// D_out(p) = min over b on the axis line of max(|p-b|, D_in(b)) (D_in(b) = 0
// for non-members and outside the volume)
template <int MODE>
__global__ void dt_axis(const int* __restrict__ lab, const int* __restrict__ din, int* __restrict__ dout, Geo3 g,
                        long long total, int axis) {
    const long long stride = axis == 1 ? g.n1 : (long long)g.n1 * g.n2;
    const int n = axis == 1 ? g.n2 : g.n3;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
         v += (long long)gridDim.x * blockDim.x) {
        const int c = vclass<MODE>(lab, v, g.fs);
        if (c == 0) {
            dout[v] = 0;
            continue;
        }
        const int loc = (int)(v % g.fs);
        const int pos = axis == 1 ? (loc / g.n1) % g.n2 : loc / (g.n1 * g.n2);
        int best = din[v];
        for (int r = 1; r < best; ++r) {
#pragma unroll
            for (int sgn = -1; sgn <= 1; sgn += 2) {
                const int q = pos + sgn * r;
                int cand;
                if (q < 0 || q >= n) {
                    cand = r;
                } else {
                    const long long w = v + sgn * r * stride;
                    cand = vclass<MODE>(lab, w, g.fs) != c ? r : max(r, din[w]);
                }
                best = min(best, cand);
            }
        }
        dout[v] = best;
    }
}

// per-cell argmax key (distance desc, linear index asc) and, in mode 0, size
template <int MODE>
__global__ void cell_argmax(const int* __restrict__ lab, const int* __restrict__ dist, const int* __restrict__ first,
                            long long total, long long fs, unsigned long long* key, int* count) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
         v += (long long)gridDim.x * blockDim.x) {
        if (vclass<MODE>(lab, v, fs) == 0) continue;
        const long long f = v / fs;
        const unsigned loc = (unsigned)(v - f * fs);
        const int c = first[f] + lab[v] - 1;
        atomicMax(key + c, ((unsigned long long)(unsigned)dist[v] << 32) | (0xffffffffu - loc));
        if (MODE == 0) atomicAdd(count + c, 1);
    }
}

__global__ void gather_labels(const int* lab, const long long* idx, int n, int* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = idx[i] < 0 ? 0 : lab[idx[i]];
}

int blocks_for(long long n) { return (int)std::min<long long>((n + kTB - 1) / kTB, 148LL * 16); }

}  // namespace

Tracker::Tracker(int n1, int n2, int n3, int F, cudaStream_t s)
    : n1_(n1), n2_(n2), n3_(n3), F_(F), fs_((long long)n1 * n2 * n3), total_(fs_ * F), s_(s) {
    if (fs_ > 0x7fffffffLL) throw Error(SS_ERR_VALIDATION, "track: frame larger than 2^31 voxels");
    mask_.alloc(total_);
    lab_.alloc(total_);
    first_dev_.alloc(std::max(1, F));
}

void Tracker::label() {
    parent_.alloc(total_);
    aux_.alloc(total_);
    const int B = blocks_for(total_);
    const Geo3 g{n1_, n2_, n3_, fs_};
    Dev<unsigned long long> ctr;
    ctr.alloc(2);
    SSB_CUDA(cudaMemsetAsync(ctr.p, 0, 2 * sizeof(unsigned long long), s_));
    SSB_CUDA(cudaMemsetAsync(aux_.p, 0, total_ * sizeof(int), s_));
    ccl_init<<<B, kTB, 0, s_>>>(mask_.p, parent_.p, total_, fs_);
    SSB_LAUNCHED();
    ccl_merge<<<B, kTB, 0, s_>>>(mask_.p, parent_.p, g, total_);
    SSB_LAUNCHED();
    ccl_flatten<<<B, kTB, 0, s_>>>(parent_.p, aux_.p, total_, fs_, ctr.p);
    SSB_LAUNCHED();
    unsigned long long nr = 0;
    SSB_CUDA(cudaMemcpyAsync(&nr, ctr.p, sizeof nr, cudaMemcpyDeviceToHost, s_));
    SSB_CUDA(cudaStreamSynchronize(s_));
    std::vector<long long> roots(nr);
    std::vector<int> sizes(nr), rank(nr);
    lpf_.assign(F_, 0);
    if (nr > 0) {
        Dev<long long> droots;
        Dev<int> dsizes;
        droots.alloc(nr);
        dsizes.alloc(nr);
        ccl_roots<<<B, kTB, 0, s_>>>(parent_.p, aux_.p, total_, fs_, ctr.p + 1, droots.p, dsizes.p);
        SSB_LAUNCHED();
        SSB_CUDA(cudaMemcpyAsync(roots.data(), droots.p, nr * sizeof(long long), cudaMemcpyDeviceToHost, s_));
        SSB_CUDA(cudaMemcpyAsync(sizes.data(), dsizes.p, nr * sizeof(int), cudaMemcpyDeviceToHost, s_));
        SSB_CUDA(cudaStreamSynchronize(s_));
        // rank per frame: size desc, first voxel (= root) asc (tracking.cpp:115-124)
        std::vector<long long> ord(nr);
        for (long long i = 0; i < (long long)nr; ++i) ord[i] = i;
        std::sort(ord.begin(), ord.end(), [&](long long a, long long b) {
            const long long fa = roots[a] / fs_, fb = roots[b] / fs_;
            if (fa != fb) return fa < fb;
            if (sizes[a] != sizes[b]) return sizes[a] > sizes[b];
            return roots[a] < roots[b];
        });
        for (long long i : ord) rank[i] = ++lpf_[roots[i] / fs_];
        Dev<int> drank;
        drank.alloc(nr);
        SSB_CUDA(cudaMemcpyAsync(drank.p, rank.data(), nr * sizeof(int), cudaMemcpyHostToDevice, s_));
        scatter_rank<<<blocks_for(nr), kTB, 0, s_>>>(droots.p, drank.p, (long long)nr, aux_.p);
        SSB_LAUNCHED();
        apply_labels<<<B, kTB, 0, s_>>>(parent_.p, aux_.p, lab_.p, total_, fs_);
        SSB_LAUNCHED();
        SSB_CUDA(cudaStreamSynchronize(s_));  // host buffers above go out of scope
    } else {
        SSB_CUDA(cudaMemsetAsync(lab_.p, 0, total_ * sizeof(int), s_));
    }
    parent_.reset();
    aux_.reset();
}

void Tracker::set_labels(const int* labels, const std::vector<int>& lpf) {
    require((int)lpf.size() == F_, "labels_per_frame size");
    SSB_CUDA(cudaMemcpyAsync(lab_.p, labels, total_ * sizeof(int), cudaMemcpyDefault, s_));
    lpf_ = lpf;
}

void Tracker::distance(int mode) {
    dA_.alloc(total_);
    dB_.alloc(total_);
    const Geo3 g{n1_, n2_, n3_, fs_};
    const long long rows = total_ / std::max(1, n1_);
    const int B = blocks_for(total_);
    if (mode == 0) {
        dt_x<0><<<blocks_for(rows), kTB, 0, s_>>>(lab_.p, dA_.p, g, rows);
        SSB_LAUNCHED();
        dt_axis<0><<<B, kTB, 0, s_>>>(lab_.p, dA_.p, dB_.p, g, total_, 1);
        SSB_LAUNCHED();
        dt_axis<0><<<B, kTB, 0, s_>>>(lab_.p, dB_.p, dA_.p, g, total_, 2);
        SSB_LAUNCHED();
    } else {
        dt_x<1><<<blocks_for(rows), kTB, 0, s_>>>(lab_.p, dA_.p, g, rows);
        SSB_LAUNCHED();
        dt_axis<1><<<B, kTB, 0, s_>>>(lab_.p, dA_.p, dB_.p, g, total_, 1);
        SSB_LAUNCHED();
        dt_axis<1><<<B, kTB, 0, s_>>>(lab_.p, dB_.p, dA_.p, g, total_, 2);
        SSB_LAUNCHED();
    }
}

void Tracker::cell_keys(int mode) {
    first_.assign(F_, 0);
    int nc = 0;
    for (int f = 0; f < F_; ++f) {
        first_[f] = nc;
        nc += lpf_[f];
    }
    key_.alloc(std::max(1, nc));
    count_.alloc(std::max(1, nc));
    SSB_CUDA(cudaMemcpyAsync(first_dev_.p, first_.data(), F_ * sizeof(int), cudaMemcpyHostToDevice, s_));
    SSB_CUDA(cudaMemsetAsync(key_.p, 0, std::max(1, nc) * sizeof(unsigned long long), s_));
    SSB_CUDA(cudaMemsetAsync(count_.p, 0, std::max(1, nc) * sizeof(int), s_));
    distance(mode);
    const int B = blocks_for(total_);
    if (mode == 0)
        cell_argmax<0><<<B, kTB, 0, s_>>>(lab_.p, dA_.p, first_dev_.p, total_, fs_, key_.p, count_.p);
    else
        cell_argmax<1><<<B, kTB, 0, s_>>>(lab_.p, dA_.p, first_dev_.p, total_, fs_, key_.p, count_.p);
    SSB_LAUNCHED();
}

void Tracker::centers() {
    cell_keys(0);
    const int nc = first_.empty() ? 0 : first_.back() + lpf_.back();
    std::vector<unsigned long long> key(nc);
    std::vector<int> cnt(nc);
    if (nc) {
        SSB_CUDA(cudaMemcpyAsync(key.data(), key_.p, nc * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s_));
        SSB_CUDA(cudaMemcpyAsync(cnt.data(), count_.p, nc * sizeof(int), cudaMemcpyDeviceToHost, s_));
    }
    SSB_CUDA(cudaStreamSynchronize(s_));
    cells_.assign(nc, ssb_track::Cell{});
    for (int f = 0; f < F_; ++f)
        for (int lb = 1; lb <= lpf_[f]; ++lb) {
            const int c = first_[f] + lb - 1;
            ssb_track::Cell& r = cells_[c];
            r.frame = f;
            r.label = lb;
            r.voxel_count = cnt[c];
            r.max_distance = (int)(key[c] >> 32);
            if (cnt[c] == 0) throw Error(SS_ERR_VALIDATION, "label field: label " + std::to_string(lb) +
                                                                " of frame " + std::to_string(f) + " has no voxel");
            const long long loc = 0xffffffffLL - (long long)(key[c] & 0xffffffffull);
            r.cx = (int)(loc % n1_);
            r.cy = (int)((loc / n1_) % n2_);
            r.cz = (int)(loc / ((long long)n1_ * n2_));
        }
}

void Tracker::targets(std::vector<int>& proj, std::vector<int>& overlap) {
    const int nc = (int)cells_.size();
    // overlap-region distance centres of every cell (mode 1), then one gather
    // of frame f-1's labels at both candidate voxels
    cell_keys(1);
    std::vector<unsigned long long> key(nc);
    if (nc) SSB_CUDA(cudaMemcpyAsync(key.data(), key_.p, nc * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s_));
    SSB_CUDA(cudaStreamSynchronize(s_));
    std::vector<long long> idx(2 * (size_t)nc, -1);
    for (int c = 0; c < nc; ++c) {
        const ssb_track::Cell& r = cells_[c];
        if (r.frame == 0) continue;
        const long long prev = (long long)(r.frame - 1) * fs_;
        idx[c] = prev + ((long long)r.cz * n2_ + r.cy) * n1_ + r.cx;
        if (key[c]) idx[nc + c] = prev + (0xffffffffLL - (long long)(key[c] & 0xffffffffull));
    }
    proj.assign(nc, 0);
    overlap.assign(nc, 0);
    if (!nc) return;
    Dev<long long> di;
    Dev<int> dout;
    di.alloc(2 * (size_t)nc);
    dout.alloc(2 * (size_t)nc);
    SSB_CUDA(cudaMemcpyAsync(di.p, idx.data(), idx.size() * sizeof(long long), cudaMemcpyHostToDevice, s_));
    gather_labels<<<blocks_for(2LL * nc), kTB, 0, s_>>>(lab_.p, di.p, 2 * nc, dout.p);
    SSB_LAUNCHED();
    std::vector<int> out(2 * (size_t)nc);
    SSB_CUDA(cudaMemcpyAsync(out.data(), dout.p, out.size() * sizeof(int), cudaMemcpyDeviceToHost, s_));
    SSB_CUDA(cudaStreamSynchronize(s_));
    std::copy(out.begin(), out.begin() + nc, proj.begin());
    std::copy(out.begin() + nc, out.end(), overlap.begin());
}

void Tracker::set_cells(const std::vector<ssb_track::Cell>& cells) {
    first_.assign(F_, 0);
    int nc = 0;
    for (int f = 0; f < F_; ++f) {
        first_[f] = nc;
        nc += lpf_[f];
    }
    require((int)cells.size() == nc, "records: expected one record per (frame, label)");
    for (int c = 0; c < nc; ++c) {
        const ssb_track::Cell& r = cells[c];
        require(r.frame >= 0 && r.frame < F_ && r.label >= 1 && r.label <= lpf_[r.frame] &&
                    first_[r.frame] + r.label - 1 == c,
                "records must be ordered by (frame, label)");
        require(r.cx >= 0 && r.cx < n1_ && r.cy >= 0 && r.cy < n2_ && r.cz >= 0 && r.cz < n3_,
                "record centre outside the frame");
    }
    cells_ = cells;
}

void track_points(Tracker& t, int window, double radius, std::vector<ss_track_point>& out) {
    t.label();
    t.centers();
    std::vector<int> proj, overlap;
    t.targets(proj, overlap);
    const std::vector<ssb_track::Cell>& cells = t.cells();
    const std::vector<ssb_track::Chain> parts =
        ssb_track::backtrack(t.labels_per_frame(), t.first(), cells, proj, overlap);
    std::vector<ssb_track::Chain> merged = ssb_track::merge(cells, parts, window, radius);
    ssb_track::order(cells, merged, t.n1(), t.n2());
    out.clear();
    for (size_t id = 0; id < merged.size(); ++id)  // track(), tracking.cpp:393-401
        for (int c : merged[id])
            out.push_back(ss_track_point{(int)id + 1, cells[c].frame, (double)cells[c].cx, (double)cells[c].cy,
                                         (double)cells[c].cz});
}

}  // namespace ssb
