// domain.cuh -- host-side runtime: slabs, transports and the device-resident
// segment() domain behind the C ABI.
//
// A Domain is the grid (or, under NCCL, one rank's share of it) split along the
// time axis l into slabs (Partition::create semantics, parallel.cpp:9-19).  Each
// Slab owns its device buffers and a local Layout whose colour parity uses the
// GLOBAL l; planes 0 and n4+1 of a slab are either global ghosts or halos that a
// Transport fills with the neighbours' boundary planes (solver.cpp:253-265).
//   NullTransport   one slab = the whole grid (single GPU; the default)
//   LocalTransport  several slabs on one device and one stream (tests the
//                   decomposition bit for bit on a single GPU)
//   NcclTransport   one slab per process/GPU, ncclSend/Recv of colour-packed
//                   half-planes and ncclAllGather of per-slice residuals
#pragma once

#include <array>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace ssb {

template <class T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    Dev() = default;
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    ~Dev() { reset(); }
    void alloc(size_t count) {
        if (count == n && p) return;
        reset();
        if (count == 0) return;
        SSB_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

struct DevField {
    Dev<double> c[2];
    void alloc(const Layout& L) {
        c[0].alloc(L.cs);
        c[1].alloc(L.cs);
    }
    PField pf() const {
        PField f;
        f.c[0] = c[0].p;
        f.c[1] = c[1].p;
        return f;
    }
};

// Balls grouped into waves preserving table order among overlapping balls.
struct BallSet {
    std::vector<Ball> host;     // wave-sorted
    std::vector<int> row;       // wave-sorted index -> centres-table row
    std::vector<int> wave_off;  // waves + 1 offsets into host
    Dev<Ball> dev;
    int count() const { return (int)host.size(); }
    int waves() const { return (int)wave_off.size() - 1; }
};
// rows whose frame lies in the slab [l0+1, l0+n4_local] only; ball.l is local
void build_balls(BallSet& bs, const ss_grid& g_local, int l0, const ss_center* c, int n,
                 double radius, bool fixed_radius);

void require(bool ok, const std::string& msg);
bool pass_tile2d();  // env SSB_TILE2D
bool halo_push();    // env SSB_PUSH
void validate_grid(const ss_grid* g);
void validate_solver(double tau, double eps, double omega, double tol, int max_iter, int n_steps);
void validate_smoothing(double sigma, int steps, double tol, int max_iter, double omega);
void validate_edge(double K, double delta, double vartheta);
void validate_centers(const ss_grid& g, const ss_center* c, int n);
void validate_seg_params(const ss_seg_params& p);

struct SolveOut {
    int iterations = 0;
    double residual = 0.0, tol = 0.0;
    bool converged = false;
    bool nonfinite = false;  // the assembly flagged a non-finite coefficient (no solve was made)
};

struct SolverErrT : Error {
    int iterations;
    double residual;
    explicit SolverErrT(const SolveOut& o);
};

// ------------------------------------------------------------------ slab
struct Slab {
    ss_grid gl{};   // local grid (n4 = owned slices)
    Layout L{};
    int index = 0;  // position of the slab along l (= rank for NCCL)
    cudaStream_t stream = nullptr;  // borrowed from the Domain

    DevField S[kStateBuffers];  // rotating state buffers (guess + 3 outputs)
    DevField rhs_sep;    // explicit rhs (per-call redblack_sor)
    Dev<float> coef[2];
    Dev<double> G[2];
    bool have_G = false;
    Dev<double> part[4][2];
    Dev<double> slice_res;   // chunk entries (zero padded)
    Dev<double> all_slices;  // world * chunk (gathered), unused when world == 1
    Dev<double> norm_loc, norm_all;
    Dev<double> norm_part;   // chunk * kNormChunks partials of launch_norm_slices
    Dev<double> gloc, gall;  // small host-driven gathers (k <= 8 values per slab)
    Dev<int> wflags;         // wavefront item completion flags
    Dev<SorState> st;
    Dev<double> scratch, scal;
    Dev<int> flags;
    Dev<double> bad_all;     // all-gathered assembly flags (world doubles; slab groups / ranks)
    Dev<double> stage, stage8;
    Dev<double> dstage;      // step_host_async: the download staging (the upload keeps `stage`)
    BallSet rescale_balls;

    Slab(const ss_grid& global, int l0, int n4_local, int index, int chunk, int world,
         cudaStream_t s);
    double* stage_p();
    double* dstage_p();
    double* stage8_p();
    void upload(const double* host_padded, PField dst, PField twin0 = PField(), PField twin1 = PField(),
                PField twin2 = PField());
    void upload_state(const double* host_padded, int role);
    void download(PField src, double* host_padded);
    void sync_ghosts_from(int role);
    void assemble(PField u, bool with_G, double tau, double eps, double* off_out, double* diag_out,
                  double* abar_out);
    AsmArgs asm_args(PField u, bool with_G, double tau, double eps) const;
    void face_coefficients(PField I0s, PField ITs, double K, double delta, double vartheta,
                           double* G_out);
    void rescale(int role);
    void threshold_minmax(PField img, const BallSet& bs, double* ab);
    void threshold_write(PField img, PField out, const BallSet& bs, const double* ab, double lambda);
    void initial(PField u, const ss_center* c, int n, double v, double R, int profile);
    SorArgs sor_args(const PField B[kStateBuffers], const PField& rhs, bool heat, double omega,
                     const double hc[4], int world, int kernel) const;
    // tensor maps of the 2D-tiled pass, device copies cached per pointer set
    struct MapEntry {
        const void* key[2 * kStateBuffers + 4];
        TmaMaps* dev = nullptr;
    };
    mutable std::vector<MapEntry> map_cache;
    const TmaMaps* maps_for(const SorArgs& a) const;
    ~Slab();
};

// ------------------------------------------------------------------ transports
struct Transport {
    virtual ~Transport() = default;
    // owned boundary planes of F[s] (colour mask: 1 red, 2 black) into the
    // l-neighbours' halo planes, issued on stream s
    virtual void exchange(std::vector<Slab*>& slabs, const std::vector<PField>& F, int colours,
                          cudaStream_t s) = 0;
    // every slab's local[s] (chunk doubles) -> all[s'][rank * chunk] for all s'
    // on stream st (nullptr: the slabs' own stream)
    virtual void allgather(std::vector<Slab*>& slabs, const std::vector<double*>& local,
                           const std::vector<double*>& all, int chunk, cudaStream_t st = nullptr) = 0;
};

struct NullTransport : Transport {
    void exchange(std::vector<Slab*>&, const std::vector<PField>&, int, cudaStream_t) override {}
    void allgather(std::vector<Slab*>&, const std::vector<double*>&, const std::vector<double*>&, int,
                   cudaStream_t) override {}
};

struct LocalTransport : Transport {
    void exchange(std::vector<Slab*>& slabs, const std::vector<PField>& F, int colours,
                  cudaStream_t s) override;
    void allgather(std::vector<Slab*>& slabs, const std::vector<double*>& local,
                   const std::vector<double*>& all, int chunk, cudaStream_t st = nullptr) override;
};

std::unique_ptr<Transport> make_nccl_transport(const unsigned char* uid, int rank, int world);
// host-staged exchanges / all-gathers through the caller's callbacks (transport_host.cu)
std::unique_ptr<Transport> make_host_transport(const ss_host_comm& c, int rank, int world);

// large host <-> device copies (hostio.cu): pinned host memory direct and async;
// pageable memory through pinned chunks filled / drained by host threads.  Both
// return with the host buffer reusable (d2h: data arrived).
void copy_h2d(void* dev, const void* host, size_t bytes, cudaStream_t s);
void copy_d2h(void* host, const void* dev, size_t bytes, cudaStream_t s);
bool host_pinned(const void* p);  // page-locked (or registered) host memory

// NVLink peer links of one rank (opt-in, SSB_P2P=1): the l-neighbours' state
// arrays and flag words mapped into this process with CUDA IPC, so the TMA pass
// pushes its boundary planes straight into the neighbours' halo planes over
// NVLink (no NCCL exchange), and per-pass completion counters order the passes.
struct PeerLinks {
    bool on = false;
    double* S[2][kStateBuffers][2] = {};    // [0 = low neighbour, 1 = high][buffer][colour]
    unsigned long long* peer_flag[2] = {};  // the word this rank writes in the low / high neighbour
    Dev<unsigned long long> my_flags;       // [0] written by the low neighbour, [1] by the high one
    unsigned long long count = 0;           // passes completed by this rank (identical on every rank)
    int n4[2] = {0, 0};                     // owned slices of the low / high neighbour
};
// exchanges IPC handles of the slab's state arrays over the transport's NCCL
// communicator and opens the neighbours' (transport_nccl.cu)
void setup_peer_links(Transport& tr, Slab& s, int rank, int world, int chunk, int n4_global, PeerLinks& pl);
void launch_p2p_wait(cudaStream_t st, const PeerLinks& pl, unsigned long long target);
void launch_p2p_signal(cudaStream_t st, const PeerLinks& pl, unsigned long long value);
void nccl_unique_id(unsigned char out[128]);

// ------------------------------------------------------------------ domain
struct Domain {
    ss_grid g{};        // global grid
    int world = 1;      // total slabs (ranks for NCCL)
    int chunk = 0;      // ceil(n4 / world)
    int device = 0;
    bool distributed = false;  // NCCL: slabs.size() == 1 < world
    PeerLinks peers;           // NVLink halo push between ranks (SSB_P2P=1)
    // fixed-sweep solves: 1 = the last iteration's residual is evaluated (diagnostics, ss_session_fixed_sweeps),
    // 2 = no residual (step_fixed / step_host* without a diag struct): SorState::fixed
    int fixed_mode = 1;
    bool want_residual = false;  // set around ss_session_fixed_sweeps
    int comm_reserve = 0;      // CTA slots a pass's interior launch leaves free for NCCL's send/recv kernels
    cudaStream_t stream = nullptr, cap_stream = nullptr;
    cudaStream_t comm = nullptr;  // halo exchanges (overlapped with interior slices)
    cudaStream_t bnd = nullptr;   // high priority: a colour pass's end slices, concurrent with its interior
    cudaEvent_t ev_pre = nullptr; // the pass's start on the main stream (the end-slice launch waits for it)
    cudaStream_t dec = nullptr;   // high priority: slab-group residual + decision, overlapped with the black pass
    cudaEvent_t ev_red = nullptr, ev_dec = nullptr;
    cudaEvent_t ev_bnd = nullptr, ev_xchg = nullptr;
    std::vector<std::unique_ptr<Slab>> slabs;
    std::vector<Slab*> sp;  // raw pointers, rank order
    std::unique_ptr<Transport> tr;
    int cur = 0;

    bool prepared = false;
    ss_seg_params prm{};

    int loop_mode = 1;
    int last_kernel = -1;  // kernel code the last non-heat solve ran (ss_session_sor_kernel)
    int kernel = 4;   // SOR: 4 = auto (default: resident when the working set fits L2, else TMA),
                      // 1 = TMA two-pass, 0 = LDG two-pass, 3 = resident (one cooperative launch
                      // per solve), 2 = TMA wavefront (experimental, slower; sor_tma.cu)
    int solve_count = 0;
    bool profiling = false;
    ss_profile prof{};
    SorState* st_host = nullptr;
    int* flag_host = nullptr;
    double* scal_host = nullptr;
    struct GraphEntry;
    std::vector<std::unique_ptr<GraphEntry>> graphs;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

    // world == 1 (single GPU) or a local group of n_slabs on one device
    Domain(const ss_grid& grid, int device, int n_slabs);
    // one rank of an NCCL job
    Domain(const ss_grid& grid, int device, int rank, int world, const unsigned char* uid);
    // one rank of a job whose exchanges go through the host (ss_host_comm callbacks)
    Domain(const ss_grid& grid, int device, int rank, int world, const ss_host_comm& comm);
    ~Domain();

    void sync();
    void clear_graphs();  // drop the captured SOR loops (after a kernel switch)
    int slabs_local() const { return (int)sp.size(); }
    bool single() const { return sp.size() == 1 && world == 1; }
    long long host_plane() const;  // padded doubles per l-plane of a host array
    const double* host_slab(const double* base, const Slab& s) const;
    double* host_slab(double* base, const Slab& s) const;

    std::vector<PField> role_fields(int role) const;
    void exchange_role(int role, int colours);
    void exchange(const std::vector<PField>& F, int colours);
    // k doubles from every local slab -> world*k doubles in rank order, identical on all ranks
    std::vector<double> gather_values(const std::vector<std::vector<double>>& per_slab, int k);

    using Triple = std::array<PField, kStateBuffers>;  // guess + the 3 rotating outputs
    std::vector<Triple> role_triples(const int roles[kStateBuffers]) const;
    // red-black SOR on every slab: guess B[s][0] (never written), rhs[s]; the
    // result lands in B[s][*result].  Non-convergence is reported, not thrown.
    SolveOut solve(const std::vector<Triple>& B, const std::vector<PField>& rhs, bool heat,
                   double omega, const double hc[4], double tol_abs, bool use_norm, double rel,
                   int max_iter, bool fixed, int* result, bool check_assembly = false);
    // heat_smooth over per-slab buffer triples; returns the index of the result
    int heat_smooth(const std::vector<Triple>& B, double sigma, int steps, double omega, double tol,
                    int max_iter);
    void mirror_all(const std::vector<PField>& F);

    void set_u(const double* host);
    void get_u(double* host);
    void get_mask(double level, uint8_t* mask);
    void prepare(const double* image, const ss_center* c, int n, const ss_seg_params& p,
                 const double* u0);
    // one time step (solver.cpp:428-438); fixed > 0: exactly `fixed` sweeps, no stopping
    // test (BASELINE config 4); rescale = false skips local_rescale (ss_session_fixed_sweeps)
    SolveOut step(ss_step_diag* diag, int fixed = 0, bool rescale = true);
    double fixed_sweeps(int n_sweeps);
    // step() with the step's input / result as compact host interiors (n1*n2*n3*n4 doubles of
    // this domain's owned slices, i fastest; ghosts stay the device's Dirichlet data); either
    // may be null.  Single slab + page-locked input: the upload streams in slice chunks on a
    // copy stream and the assembly of each chunk's slices starts as soon as their l+1
    // neighbours have arrived (ss_session_step_host)
    SolveOut step_host(const double* in, double* out, int fixed, ss_step_diag* diag);
    void set_u_interior(const double* host);
    void get_u_interior(double* host);
    // step_host with the result's download left in flight (one slab per process -- a single
    // domain or a rank of a distributed one -- and page-locked buffers; otherwise exactly
    // step_host): out is complete after wait_transfers(), and when the next
    // call's input is this call's output, each upload chunk waits on the device for its
    // download chunk, so the D2H of step n and the H2D of step n + 1 run concurrently on the
    // two copy directions (ss_session_step_host_async)
    SolveOut step_host_async(const double* in, double* out, int fixed, ss_step_diag* diag);
    void wait_transfers();
    // EOC verification row (eoc.cpp:83-137) on an n^4 session; returns the space-time L2 error
    double eoc_row(int n, double omega, double sor_tol, int max_iter, long long* total_sweeps);

private:
    cudaStream_t h2d = nullptr;        // step_host: chunked upload of the step's input
    std::vector<cudaEvent_t> up_ev;   // ... one event per chunk (+ the staging-free event)
    cudaStream_t d2h = nullptr;        // step_host_async: chunked download of the step's result
    std::vector<cudaEvent_t> dn_ev;   // ... per chunk: unpacked (C + q) / copied (q); [2C]: all copied
    const double* dn_host = nullptr;  // the host buffer the in-flight download writes (null: none)
    void download_async(double* host);
    SolveOut step_impl(ss_step_diag* diag, int fixed, bool rescale, const double* host_in);
    // chunked upload of a page-locked input (chained to an in-flight download of the same
    // buffer); assemble: each chunk's slices assembled as soon as their l+1 neighbour is in
    // (single domain), else the upload alone (a rank: its halos are exchanged after it)
    void upload_chunks(const double* host, bool assemble);
    void init_common();
    void init_rank(int rank);  // the rank's slab (distributed constructors)
    cudaEvent_t pool_event(size_t idx);
    cudaGraphExec_t graph_for(const SorArgs& a, bool heat);
    void body_single(const SorArgs& a, bool heat, cudaEvent_t* ev4);
    void body_multi(const std::vector<SorArgs>& a, const std::vector<Triple>& B, bool heat, int n,
                    cudaEvent_t* ev4, cudaEvent_t* xev6);
};

}  // namespace ssb
