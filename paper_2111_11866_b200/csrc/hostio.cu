// hostio.cu -- large host <-> device copies.
//
// Pinned host memory (cudaHostAlloc / cudaHostRegister, e.g. torch pin_memory)
// goes straight to the copy engine, asynchronously.  Pageable memory (numpy
// arrays, std::vector) would take the driver's own staging path (~11 GB/s on
// the B200 boxes); instead it streams through two pinned 16 MB chunks that
// several host threads fill (H2D) or drain (D2H) while the copy engine moves
// the other chunk.  Both directions leave the host buffer free to reuse when
// they return, like the pageable cudaMemcpyAsync they replace.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "domain.cuh"

namespace ssb {

namespace {

constexpr size_t kChunk = 16u << 20;

struct Staging {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int device = -1;
};

std::mutex g_mu;

Staging& staging() {  // per device, allocated on first use (held under g_mu)
    static std::vector<Staging> per(64);
    int dev = 0;
    SSB_CUDA(cudaGetDevice(&dev));
    Staging& st = per[dev % 64];
    if (!st.buf[0]) {
        for (int b = 0; b < 2; ++b) {
            SSB_CUDA(cudaHostAlloc(&st.buf[b], kChunk, cudaHostAllocPortable));
            SSB_CUDA(cudaEventCreateWithFlags(&st.done[b], cudaEventDisableTiming));
        }
        st.device = dev;
    }
    return st;
}

bool pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t n) {
    static const unsigned T = std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2));
    if (n < (1u << 20) || T == 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const size_t part = (n + T - 1) / T;
    for (unsigned t = 0; t < T; ++t) {
        const size_t o = t * part;
        if (o >= n) break;
        const size_t m = std::min(part, n - o);
        th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, m); });
    }
    for (auto& x : th) x.join();
}

}  // namespace

bool host_pinned(const void* p) { return pinned(p); }

void copy_h2d(void* dev, const void* host, size_t bytes, cudaStream_t s) {
    if (bytes < (4u << 20) || pinned(host)) {
        SSB_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    Staging& st = staging();
    int b = 0;
    for (size_t off = 0; off < bytes; off += kChunk, b ^= 1) {
        const size_t n = std::min(kChunk, bytes - off);
        SSB_CUDA(cudaEventSynchronize(st.done[b]));  // the copy engine has drained this chunk
        par_memcpy(st.buf[b], static_cast<const char*>(host) + off, n);
        SSB_CUDA(cudaMemcpyAsync(static_cast<char*>(dev) + off, st.buf[b], n, cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaEventRecord(st.done[b], s));
    }
}

void copy_d2h(void* host, const void* dev, size_t bytes, cudaStream_t s) {
    if (bytes < (4u << 20) || pinned(host)) {
        SSB_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    Staging& st = staging();
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t k) {
        const size_t off = k * kChunk, n = std::min(kChunk, bytes - off);
        SSB_CUDA(cudaMemcpyAsync(st.buf[k & 1], static_cast<const char*>(dev) + off, n, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaEventRecord(st.done[k & 1], s));
    };
    issue(0);
    for (size_t k = 0; k < nch; ++k) {
        if (k + 1 < nch) issue(k + 1);  // the next chunk moves while this one is drained
        SSB_CUDA(cudaEventSynchronize(st.done[k & 1]));
        const size_t off = k * kChunk, n = std::min(kChunk, bytes - off);
        par_memcpy(static_cast<char*>(host) + off, st.buf[k & 1], n);
    }
}

}  // namespace ssb
