// transport_host.cu -- a host-staged Transport over caller-provided callbacks.
//
// The product's distributed Domain (one t-slab per process) with its halo
// exchange and residual all-gathers routed through the host: the boundary
// planes are copied device -> pinned host, handed to the caller's sendrecv /
// allgather callbacks (e.g. torch.distributed over gloo), and the received
// planes copied back into the halo planes.  Same message pattern as the NCCL
// transport (transport_nccl.cu: plane 1 <-> rank-1's plane n4'+1, plane n4 <->
// rank+1's plane 0, per colour; per-slice partials all-gathered in rank order),
// so iterates and iteration counts equal the single domain's bit for bit.
//
// It exists to run the multi-process path where only one GPU is available
// (several processes on one device exchange through the host, never waiting on
// each other inside a kernel) and to test it; it is synchronous and slow by
// design and is not the multi-GPU data path (NCCL / NVLink push are).
#include <cstring>

#include "domain.cuh"

namespace ssb {

namespace {

struct HostBuf {
    void* p = nullptr;
    size_t n = 0;
    void need(size_t bytes) {
        if (bytes <= n) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        SSB_CUDA(cudaMallocHost(&p, bytes));
        n = bytes;
    }
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
};

struct HostTransport : Transport {
    ss_host_comm cb;
    int rank, world;
    HostBuf send, recv, loc, all;
    HostTransport(const ss_host_comm& c, int r, int w) : cb(c), rank(r), world(w) {}

    void call(int rc, const char* what) {
        if (rc != 0) throw Error(SS_ERR_NCCL, std::string("host transport: ") + what + " callback failed (" +
                                                  std::to_string(rc) + ")");
    }

    void exchange(std::vector<Slab*>& slabs, const std::vector<PField>& F, int colours, cudaStream_t st) override {
        Slab& s = *slabs[0];
        const size_t P1 = (size_t)s.L.plane();
        const size_t B = P1 * sizeof(double);
        const int n4 = s.L.n4;
        send.need(2 * B);
        recv.need(2 * B);
        for (int c = 0; c < 2; ++c) {
            if (!(colours & (1 << c))) continue;
            double* f = F[0].c[c];
            double* sb = static_cast<double*>(send.p);
            double* rb = static_cast<double*>(recv.p);
            if (rank > 0) SSB_CUDA(cudaMemcpyAsync(sb, f + P1, B, cudaMemcpyDeviceToHost, st));
            if (rank + 1 < world) SSB_CUDA(cudaMemcpyAsync(sb + P1, f + (size_t)n4 * P1, B, cudaMemcpyDeviceToHost, st));
            SSB_CUDA(cudaStreamSynchronize(st));
            // lower neighbour first: rank r's second call pairs with rank r+1's first
            if (rank > 0) call(cb.sendrecv(cb.ctx, rank - 1, sb, rb, B), "sendrecv");
            if (rank + 1 < world) call(cb.sendrecv(cb.ctx, rank + 1, sb + P1, rb + P1, B), "sendrecv");
            if (rank > 0) SSB_CUDA(cudaMemcpyAsync(f, rb, B, cudaMemcpyHostToDevice, st));
            if (rank + 1 < world) SSB_CUDA(cudaMemcpyAsync(f + (size_t)(n4 + 1) * P1, rb + P1, B, cudaMemcpyHostToDevice, st));
            SSB_CUDA(cudaStreamSynchronize(st));  // the staging buffers are reused next
        }
    }

    void allgather(std::vector<Slab*>& slabs, const std::vector<double*>& local, const std::vector<double*>& a,
                   int chunk, cudaStream_t st) override {
        cudaStream_t s = st ? st : slabs[0]->stream;
        const size_t B = (size_t)chunk * sizeof(double);
        loc.need(B);
        all.need(B * world);
        SSB_CUDA(cudaMemcpyAsync(loc.p, local[0], B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        call(cb.allgather(cb.ctx, loc.p, all.p, B), "allgather");
        SSB_CUDA(cudaMemcpyAsync(a[0], all.p, B * world, cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaStreamSynchronize(s));
    }
};

}  // namespace

std::unique_ptr<Transport> make_host_transport(const ss_host_comm& c, int rank, int world) {
    require(c.sendrecv != nullptr && c.allgather != nullptr, "host transport: null callback");
    return std::unique_ptr<Transport>(new HostTransport(c, rank, world));
}

}  // namespace ssb
