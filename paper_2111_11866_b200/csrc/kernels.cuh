// kernels.cuh -- device data structures and host launchers of every kernel.
#pragma once

#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)

#include "common.cuh"

namespace ssb {

// ---------------------------------------------------------------- SOR solve
// Device-resident loop control of one redblack_sor call (solver.cpp:163-214).
// The red pass of iteration n reads n_red, the black pass n_black; the
// finalize kernel between them decides convergence of iteration n-1 and
// advances the counters, so every kernel has fixed launch arguments and the
// loop body can live in a CUDA-graph conditional WHILE node.
struct SorState {
    int n_red, n_black;
    int done, converged;
    int iterations, max_iter;
    int fixed;      // 0: to tolerance; 1: exactly max_iter sweeps, the last iteration's residual evaluated;
                    // 2: exactly max_iter sweeps and no residual at all (nobody asked for diagnostics)
    int nonfinite;  // assemble_step found a non-finite coefficient (solver.cpp:71-75): no solve
    unsigned int counter;
    unsigned int item_ctr[2];  // dynamic item counters of the TMA colour passes (zeroed by the other pass)
    int epoch_base;  // distinct per solve: completion flags of the wavefront kernel compare to epoch_base + n
    double tol, residual;
};

constexpr int kStateBuffers = 4;  // guess + 3 rotating outputs
__host__ __device__ __forceinline__ int out_buf(int n) { return 1 + (n - 1) % 3; }
__host__ __device__ __forceinline__ int in_buf(int n) { return n == 1 ? 0 : out_buf(n - 1); }

struct SorArgs {
    Layout L;
    // [buffer][colour].  Buffer 0 holds the initial guess and is never written;
    // iteration n writes buffer out(n) = 1 + (n-1) % 3 and reads in(n) = n == 1 ? 0
    // : out(n-1), so the rhs may alias buffer 0 and the iterate of a decided
    // iteration survives the up to two iterations computed after it (the
    // lagged residual of the two-pass loop, the two-iteration wavefront).
    double* U[kStateBuffers][2];
    const double* rhs[2];   // colour-packed rhs
    const float* coef[2];   // colour-packed fp32 off-diagonals, 8 per doxel (kFaceOffsets order)
    double* part[4][2];     // squared-residual partials, [iteration n & 3][red / black pass]
    double* slice_res;      // per-slice residual of the owned slices (solver.cpp:195-199)
    const double* all_slices;  // residuals of all n4g slices in global order (== slice_res on 1 slab)
    int inline_decide;      // single slab: finalize also decides
    int fuse_final;         // TMA single slab: the black pass sums slices and decides in its head
    // halo push (slab groups): the TMA pass stores the values it computes on its first /
    // last owned plane ALSO into the low / high neighbour's halo plane -- the exchange
    // happens inside the compute kernel.  [buffer][colour] neighbour arrays (null: none)
    // and the index offset from this slab's packed index to the neighbour's.
    double* push_lo[kStateBuffers][2];
    double* push_hi[kStateBuffers][2];
    long long push_lo_off, push_hi_off;
    // 2D-tiled TMA items (tile2d): rows x 32-slot segments loaded with tensor maps
    int tile2d;
    const struct TmaMaps* maps;  // device copy of the maps of U / rhs / coef (null: bulk copies)
    SorState* st;
    double omega, keep;
    double hc[4];           // heat stencil constants float(-dt/h_a^2) (solver.cpp:100-110)
    int bps;                // residual partials (tiles) per l-slice of one pass
    int tx, ty, tk;         // tile grid of one slice (pass_tiles)
    long long tiles;
    int tma;                // 1: TMA-fed pass kernel (sor_tma.cu), 0: LDG pass (sor.cu)
    int l_lo, l_hi;         // slices (local, 1-based) a pass launch covers (default 1 .. n4)
    int l_step;             // ... every l_step-th of them (TMA pass; 1: all, n4 - 1: the two end slices)
    int pdl_off;            // launch without programmatic dependent launch (side-stream launches)
    int grid_short;         // TMA pass: CTA slots this launch leaves free (0: the full persistent grid)
    int dyn;                // TMA pass: items from the colour's atomic counter (one such launch per pass)
    int wave;               // 1: two-iteration wavefront kernel per loop body, 2: one-sweep k-wavefront
    int kwj;                // one-sweep wavefront marches along j (1) or k (0)
    int* flags;             // wavefront item completion flags (epochs)
    int snake;              // TMA pass: black passes walk the items in reverse (L2 reuse at the turn)
    int order;              // TMA pass item order: 0 slice-major, 1 slice-fastest
    int l2hint;             // TMA pass L2 policies: bit0 coef/rhs evict_first, bit1 u loads evict_last,
                            // bit2 u stores evict_last
    int use_cond;
    cudaGraphConditionalHandle cond;
};

// Tensor maps of the 2D-tiled TMA pass (sor_tma.cu): 2D views [rows][slots] of the
// colour-packed arrays, boxes of kTileR rows x (kTileS + 2) slots (fp64) or kTileS
// slots x 8 faces (fp32 coefficients); the UK maps load kTileR + 2 rows.
constexpr int kTileR = 8, kTileS = 32;
struct TmaMaps {
    CUtensorMap u_main[kStateBuffers][2];
    CUtensorMap u_uk[kStateBuffers][2];
    CUtensorMap rhs[2];
    CUtensorMap coef[2];
};
// encode the maps of a's arrays into host memory (false: driver entry point unavailable)
bool encode_tma_maps(const SorArgs& a, TmaMaps& m);

constexpr int kPassBX = 32;  // doxels of one colour along a row
constexpr int kPassBY = 8;   // rows (j) per block
#ifndef SSB_PASS_KC
#define SSB_PASS_KC 4
#endif
#ifndef SSB_PASS_BATCH
#define SSB_PASS_BATCH 1
#endif
#ifndef SSB_PASS_MINB
#define SSB_PASS_MINB 4
#endif
constexpr int kPassKC = SSB_PASS_KC;        // planes (k) per tile
constexpr int kPassBatch = SSB_PASS_BATCH;  // doxels whose loads a thread issues together

void pass_tiles(const Layout& L, SorArgs& a);
// TMA-fed pass (sor_tma.cu)
bool tma_pass_supported(const Layout& L);
void tma_pass_tiles(const Layout& L, SorArgs& a);
size_t tma_partials(const Layout& L);
bool tma_fuse_ok(const Layout& L);  // single slab: the finalize can move into the black pass
double tma_lane_utilization(const Layout& L, bool tile2d);
void launch_sor_pass_tma(cudaStream_t s, const SorArgs& a, int colour, bool heat);
int pass_snake();   // SorArgs::snake default (env SSB_SNAKE)
int pass_l2hint();  // SorArgs::l2hint default (env SSB_L2HINT)
int pass_order();   // SorArgs::order default (env SSB_ORDER)
int pass_fuse_final();  // SorArgs::fuse_final allowed (env SSB_FUSE_FINAL)
int pass_pdl();         // programmatic dependent launch of the TMA passes (env SSB_PDL)
int pass_grid_short();  // CTA slots every TMA pass launch leaves free (env SSB_GRID_SHORT, default 0)
bool wave_supported(const Layout& L);
size_t wave_flags(const Layout& L);
// one-sweep k-wavefront (kernel 7, sor_tma.cu): support test, flag / partial sizes,
// partials per slice, launch (one iteration: red + black)
bool kwave_supported(const Layout& L);
int kwave_axis_j(const Layout& L);  // 1: the one-sweep wavefront marches along j
size_t kwave_flags(const Layout& L);
size_t kwave_partials(const Layout& L);
int kwave_bps(const Layout& L);
void launch_sor_kwave(cudaStream_t s, const SorArgs& a);
int wave_iters();  // SOR iterations per wavefront launch (SSB_WAVE_PHASES / 2)
void launch_sor_wave(cudaStream_t s, const SorArgs& a, bool heat);
dim3 pass_grid(const Layout& L);
// bad_local: this slab's assembly flag (int, non-zero = a non-finite diag), bad_all: the
// all-gathered flags of every slab (n_all doubles); either may be null.  A set flag makes the
// solve stop after its first decision with nonfinite = 1 -- the host reads it with the final
// state, so no host round trip sits between the assembly and the SOR loop.
void launch_sor_init(cudaStream_t s, SorState* st, double tol, const double* norm_slices,
                     int n_slices, double rel, int max_iter, int fixed, int epoch_base,
                     const int* bad_local = nullptr, const double* bad_all = nullptr, int n_all = 0);
// out[0] = flag[0] != 0 (the value a slab contributes to the flag all-gather)
void launch_flag_to_double(cudaStream_t s, const int* flag, double* out);
// single-slab loop body: red, finalize (inline decision), black
void launch_sor_body(cudaStream_t s, const SorArgs& a, bool heat, cudaEvent_t* ev /*4 or null*/);
// pieces for the multi-slab body (halo exchange / all-gather between them)
void launch_sor_pass(cudaStream_t s, const SorArgs& a, int colour, bool heat);
// the same pass restricted to slices [lo, hi] (boundary-first halo overlap)
void launch_sor_pass_range(cudaStream_t s, const SorArgs& a, int colour, bool heat, int lo, int hi,
                           bool dyn = false);
// the two end slices (1 and n4: the planes a t-slab exchanges) of a colour pass
void launch_sor_pass_ends(cudaStream_t s, const SorArgs& a, int colour, bool heat);
void launch_sor_finalize(cudaStream_t s, const SorArgs& a);
// whole solve in one cooperative launch (LDG tiles, state in L2); single slab
bool resident_supported(const Layout& L);
// false (nothing launched) when the grid cannot be co-resident: use the pass kernels
bool launch_sor_resident(cudaStream_t s, const SorArgs& a, bool heat);
size_t resident_partials(const Layout& L);  // partial slots per colour of the resident passes
void launch_sor_decide(cudaStream_t s, const SorArgs& a);

// ---------------------------------------------------------------- assembly
struct AsmArgs {
    Layout L;
    const double* u[2];     // colour-packed u_prev (ghosts = previous boundary data)
    const double* G[2];     // colour-packed 8 x fp64 per doxel, or null (G == 1)
    float* coef[2];         // output, colour-packed
    double t_h2[4];         // tau / h_a^2 (solver.cpp:36-38)
    double eps;
    double h[4];
    double hinv[4];         // 1/h (used only when every h is a power of two)
    int* bad;               // set when a diag is non-finite (solver.cpp:71-75)
    int* guard;             // device flag for the tile kernel's scaled gradients (null: exact path)
    // export (per-call API): padded outputs, may be null
    double* off_out;        // 8 per padded doxel
    double* diag_out;
    double* abar_out;
};
void launch_assemble(cudaStream_t s, const AsmArgs& a);

struct EdgeArgs {
    Layout L;
    const double* I0[2];
    const double* IT[2];
    double* G[2];           // colour-packed output
    double* G_out;          // padded export (8 per doxel), may be null
    double K, delta, vartheta;
    double h[4];
    double hinv[4];
    int* guard;             // 2 ints of scratch for the range guard of the scaled gradients (may be null)
};
void launch_face_coefficients(cudaStream_t s, const EdgeArgs& a);
// TMA-staged tile kernels (assemble_tile.cu); false = not launched (no tensor-map encoder)
bool assemble_tile_supported(const Layout& L);
double rsqrt_approx_bound();  // self-test: max relative error of rsqrt.approx.f64 (exhaustive)
void launch_assemble_guard(cudaStream_t s, const Layout& L, const double* u0, const double* u1, int* flag);
bool launch_assemble_tile(cudaStream_t s, const AsmArgs& a, bool pow2);
// the same restricted to slices [l_lo, l_hi] (the upload-overlapped assembly of step_host)
bool launch_assemble_tile_range(cudaStream_t s, const AsmArgs& a, int l_lo, int l_hi);
bool launch_edge_tile(cudaStream_t s, const EdgeArgs& a, bool pow2);

// padded fp64 off-diagonals (8 per doxel) -> colour-packed fp32 rows
// (pack_coefficients, solver.cpp:233-249)
void launch_pack_coef(cudaStream_t s, const Layout& L, const double* off, float* coef0,
                      float* coef1);
// colour-packed fp32 rows -> padded fp64 off-diagonals (the session's coefficients, for tests)
void launch_unpack_coef(cudaStream_t s, const Layout& L, const float* c0, const float* c1, double* off);
// padded 8-vector field -> colour-packed
void launch_pack8(cudaStream_t s, const Layout& L, const double* src, double* d0, double* d1);
// heat-step export (assemble_heat_step, solver.cpp:79-116)
void launch_heat_export(cudaStream_t s, const Layout& L, double dt_h2[4], double* off,
                        double* diag, double* abar);

// ---------------------------------------------------------------- fields
// src (padded) -> dst; ghost doxels are also written into the twins (null members skipped)
void launch_pack(cudaStream_t s, const Layout& L, const double* src, PField dst, PField twin0,
                 PField twin1, PField twin2);
void launch_fill_raw(cudaStream_t s, double* p, long long n, double v);
void launch_unpack(cudaStream_t s, const Layout& L, PField src, double* dst);
// compact interior arrays (n1*n2*n3*n4 doubles, i fastest, no ghosts): slices [l_lo, l_hi]
// of src (indexed from slice 1) into dst's interior / every interior doxel of src out
void launch_pack_interior(cudaStream_t s, const Layout& L, const double* src, PField dst, int l_lo, int l_hi);
void launch_unpack_interior(cudaStream_t s, const Layout& L, PField src, double* dst, int l_lo = 1,
                            int l_hi = -1);
void launch_fill(cudaStream_t s, const Layout& L, PField f, double v);
void launch_set_ghosts(cudaStream_t s, const Layout& L, PField f, double v);
// ghost doxels of src copied into dst
void launch_copy_ghosts(cudaStream_t s, const Layout& L, PField dst, PField src);
// grid.cpp:138-156 axes [a0, a1); axis 3 only at global boundaries
void launch_mirror_ghosts(cudaStream_t s, const Layout& L, PField f, int a0 = 0, int a1 = 4);
void launch_copy_field(cudaStream_t s, const Layout& L, PField dst, PField src);
// deterministic interior reductions; out[0] = sum of squares or (min,max)
void launch_norm_sq(cudaStream_t s, const Layout& L, PField f, double* scratch, double* out);
// per owned slice: sum of squares over the slice's interior (fixed order)
constexpr int kNormChunks = 64;  // row chunks per slice of launch_norm_slices
// scratch: n4 * kNormChunks doubles
void launch_norm_slices(cudaStream_t s, const Layout& L, PField f, double* scratch, double* out);
void launch_minmax(cudaStream_t s, const Layout& L, PField f, double* scratch, double* out2);
void launch_mask(cudaStream_t s, const Layout& L, PField f, double level, uint8_t* mask);
constexpr int kReduceBlocks = 592;  // 4 x 148 SMs; fixed => deterministic order

// ---------------------------------------------------------------- balls
struct Ball {
    int l, i0, i1, j0, j1, k0, k1, pad;
    double x, y, z, r, r_sq;
};
// threshold: per-ball alpha/beta over the raw image (preprocess.cpp:77-88)
void launch_ball_minmax(cudaStream_t s, const Layout& L, PField f, const Ball* balls, int n,
                        double* ab, int* empty_flag);
void launch_threshold_write(cudaStream_t s, const Layout& L, PField img, PField out,
                            const Ball* balls, int n, const double* ab, double lambda);
void launch_rescale(cudaStream_t s, const Layout& L, PField u, const Ball* balls, int n);
void launch_initial(cudaStream_t s, const Layout& L, PField u, const Ball* balls, int n,
                    double v, double R, int profile);

}  // namespace ssb
