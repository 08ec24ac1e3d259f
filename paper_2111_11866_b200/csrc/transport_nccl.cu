// transport_nccl.cu -- the multi-GPU transport: one slab per rank/GPU.
//
// Per colour pass the just-updated colour of the first and last owned planes
// (one contiguous colour-packed block each, Layout::plane() doubles) goes to
// the l-neighbours with grouped ncclSend/ncclRecv on the session stream
// (the paper's Isend/Irecv of overlap slices; the
// reference's pull_halos, solver.cpp:253-265).  Per-slice residual partials are
// all-gathered and summed in global l order by every rank, so the stopping
// decision -- and hence every iterate -- is independent of the GPU count.
//
// NCCL is loaded with dlopen("libnccl.so.2") on first use (torch's bundled
// copy when torch has loaded it, else the system library); nothing links
// against it, so single-GPU use never needs it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "domain.cuh"

namespace ssb {

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!a.h) {
            err = dlerror() ? dlerror() : "dlopen failed";
            return;
        }
#define SSB_SYM(name, field) a.field = reinterpret_cast<decltype(a.field)>(dlsym(a.h, name))
        SSB_SYM("ncclGetUniqueId", GetUniqueId);
        SSB_SYM("ncclCommInitRank", CommInitRank);
        SSB_SYM("ncclCommDestroy", CommDestroy);
        SSB_SYM("ncclCommSplit", CommSplit);
        SSB_SYM("ncclGroupStart", GroupStart);
        SSB_SYM("ncclGroupEnd", GroupEnd);
        SSB_SYM("ncclSend", Send);
        SSB_SYM("ncclRecv", Recv);
        SSB_SYM("ncclAllGather", AllGather);
        SSB_SYM("ncclGetErrorString", GetErrorString);
#undef SSB_SYM
    });
    if (!a.h || !a.AllGather || !a.Send || !a.CommInitRank || !a.CommSplit)
        throw Error(SS_ERR_NCCL, "NCCL unavailable: " + (err.empty() ? std::string("missing symbols") : err));
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(SS_ERR_NCCL, std::string(what) + ": " + (api().GetErrorString ? api().GetErrorString(r) : "?"));
}

// Two communicators: `halo` for the send/recv exchanges (always issued on the
// Domain's comm stream) and `comm` for the residual all-gathers (main stream),
// so each communicator's operations are issued from one stream in the same
// order on every rank.
struct NcclTransport : Transport {
    ncclComm_t comm = nullptr, halo = nullptr;
    int rank, world;
    NcclTransport(const unsigned char* uid, int r, int w) : rank(r), world(w) {
        ncclUniqueId id;
        std::memcpy(id.internal, uid, NCCL_UNIQUE_ID_BYTES);
        check(api().CommInitRank(&comm, w, id, r), "ncclCommInitRank");
        check(api().CommSplit(comm, 0, r, &halo, nullptr), "ncclCommSplit");
    }
    ~NcclTransport() override {
        if (halo) api().CommDestroy(halo);
        if (comm) api().CommDestroy(comm);
    }
    void exchange(std::vector<Slab*>& slabs, const std::vector<PField>& F, int colours, cudaStream_t st) override {
        Slab& s = *slabs[0];
        const size_t P1 = (size_t)s.L.plane();
        const int n4 = s.L.n4;
        NcclApi& a = api();
        check(a.GroupStart(), "ncclGroupStart");
        for (int c = 0; c < 2; ++c) {
            if (!(colours & (1 << c))) continue;
            double* f = F[0].c[c];
            if (rank > 0) {
                check(a.Send(f + P1, P1, ncclDouble, rank - 1, halo, st), "ncclSend");
                check(a.Recv(f, P1, ncclDouble, rank - 1, halo, st), "ncclRecv");
            }
            if (rank + 1 < world) {
                check(a.Send(f + (size_t)n4 * P1, P1, ncclDouble, rank + 1, halo, st), "ncclSend");
                check(a.Recv(f + (size_t)(n4 + 1) * P1, P1, ncclDouble, rank + 1, halo, st), "ncclRecv");
            }
        }
        check(a.GroupEnd(), "ncclGroupEnd");
    }
    void allgather(std::vector<Slab*>& slabs, const std::vector<double*>& local, const std::vector<double*>& all,
                   int chunk, cudaStream_t st) override {
        check(api().AllGather(local[0], all[0], (size_t)chunk, ncclDouble, comm, st ? st : slabs[0]->stream),
              "ncclAllGather");
    }
    void allgather_bytes(const void* d_local, void* d_all, size_t bytes, cudaStream_t st) {
        check(api().AllGather(d_local, d_all, bytes, ncclChar, comm, st), "ncclAllGather");
    }
};

__global__ void p2p_wait_kernel(const unsigned long long* f, int lo, int hi, unsigned long long target) {
    for (int i = 0; i < 2; ++i) {
        if (!(i == 0 ? lo : hi)) continue;
        while (true) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f + i) : "memory");
            if (v >= target) break;
            __nanosleep(200);
        }
    }
}

__global__ void p2p_signal_kernel(unsigned long long* lo, unsigned long long* hi, unsigned long long v) {
    __threadfence_system();  // the pass kernel's peer stores are ordered before the counter
    if (lo) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(lo), "l"(v) : "memory");
    if (hi) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(hi), "l"(v) : "memory");
}

}  // namespace

void launch_p2p_wait(cudaStream_t st, const PeerLinks& pl, unsigned long long target) {
    p2p_wait_kernel<<<1, 1, 0, st>>>(pl.my_flags.p, pl.S[0][0][0] != nullptr, pl.S[1][0][0] != nullptr, target);
    SSB_LAUNCHED();
}

void launch_p2p_signal(cudaStream_t st, const PeerLinks& pl, unsigned long long value) {
    p2p_signal_kernel<<<1, 1, 0, st>>>(pl.peer_flag[0], pl.peer_flag[1], value);
    SSB_LAUNCHED();
}

void setup_peer_links(Transport& t, Slab& s, int rank, int world, int chunk, int n4_global, PeerLinks& pl) {
    auto* tr = dynamic_cast<NcclTransport*>(&t);
    require(tr != nullptr, "peer links need the NCCL transport");
    constexpr int H = 2 * kStateBuffers + 1;  // state arrays + the flag words
    pl.my_flags.alloc(2);
    SSB_CUDA(cudaMemset(pl.my_flags.p, 0, 2 * sizeof(unsigned long long)));
    cudaIpcMemHandle_t mine[H];
    for (int b = 0; b < kStateBuffers; ++b)
        for (int c = 0; c < 2; ++c) SSB_CUDA(cudaIpcGetMemHandle(&mine[2 * b + c], s.S[b].c[c].p));
    SSB_CUDA(cudaIpcGetMemHandle(&mine[H - 1], pl.my_flags.p));
    Dev<unsigned char> dl, da;
    dl.alloc(sizeof mine);
    da.alloc(sizeof mine * world);
    SSB_CUDA(cudaMemcpy(dl.p, mine, sizeof mine, cudaMemcpyHostToDevice));
    tr->allgather_bytes(dl.p, da.p, sizeof mine, s.stream);
    std::vector<cudaIpcMemHandle_t> all((size_t)H * world);
    SSB_CUDA(cudaMemcpyAsync(all.data(), da.p, sizeof mine * world, cudaMemcpyDeviceToHost, s.stream));
    SSB_CUDA(cudaStreamSynchronize(s.stream));
    for (int side = 0; side < 2; ++side) {
        const int r = side == 0 ? rank - 1 : rank + 1;
        if (r < 0 || r >= world) continue;
        pl.n4[side] = r == world - 1 ? n4_global - (world - 1) * chunk : chunk;
        for (int b = 0; b < kStateBuffers; ++b)
            for (int c = 0; c < 2; ++c) {
                void* p = nullptr;
                SSB_CUDA(cudaIpcOpenMemHandle(&p, all[(size_t)r * H + 2 * b + c], cudaIpcMemLazyEnablePeerAccess));
                pl.S[side][b][c] = static_cast<double*>(p);
            }
        void* f = nullptr;
        SSB_CUDA(cudaIpcOpenMemHandle(&f, all[(size_t)r * H + H - 1], cudaIpcMemLazyEnablePeerAccess));
        // the low neighbour's word [1] is written by its high neighbour (this rank), and vice versa
        pl.peer_flag[side] = static_cast<unsigned long long*>(f) + (side == 0 ? 1 : 0);
    }
    pl.on = true;
}

std::unique_ptr<Transport> make_nccl_transport(const unsigned char* uid, int rank, int world) {
    return std::unique_ptr<Transport>(new NcclTransport(uid, rank, world));
}

void nccl_unique_id(unsigned char out[128]) {
    ncclUniqueId id;
    check(api().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
}

}  // namespace ssb
