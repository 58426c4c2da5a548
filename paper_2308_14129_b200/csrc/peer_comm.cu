// Peer-memory transport: see peer_comm.hpp.
#include "peer_comm.hpp"

#include <cstring>
#include <string>

#include "cuda_util.hpp"
#include "host.hpp"
#include "pdl.cuh"

#include <atomic>

namespace spd {

extern std::atomic<std::uint64_t> g_kernel_launches;  // (tgn_trainer.cu)

namespace {
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// sequence numbers are compared wrap-safe
__device__ __forceinline__ bool reached(unsigned have, unsigned want) { return int(have - want) >= 0; }

// lane r < world: publish `kind` = seq into rank r's flag slot of this rank
__global__ void k_peer_signal(PeerView v, int kind, const std::uint64_t* seq_dev, std::uint64_t seq,
                              std::int64_t offset) {
    const int r = threadIdx.x;
    const unsigned s = unsigned((seq_dev ? *seq_dev : seq) + offset);
    __threadfence_system();  // this rank's earlier writes (gradients, exchange data) first
    if (r < v.world) st_release_sys(v.flags_of[r] + kind * kMaxPeers + v.rank, s);
}
// lane r < world: wait until rank r published `kind` >= seq
__global__ void k_peer_wait(PeerView v, int kind, const std::uint64_t* seq_dev, std::uint64_t seq,
                            std::int64_t offset) {
    const int r = threadIdx.x;
    const unsigned s = unsigned((seq_dev ? *seq_dev : seq) + offset);
    if (r < v.world)
        while (!reached(ld_acquire_sys(v.flags + kind * kMaxPeers + r), s)) __nanosleep(256);
    __syncwarp();
    __threadfence_system();
}

template <class T>
__device__ __forceinline__ T peer_op(T a, T b, int op) {
    return op == kOpSum ? a + b : op == kOpMin ? (b < a ? b : a) : (b > a ? b : a);
}
template <class T>
__global__ void k_peer_reduce(PeerView v, T* out, std::size_t n, int op) {
    for (std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (std::size_t)gridDim.x * blockDim.x) {
        T acc = __ldcg(reinterpret_cast<const T*>(v.sbuf[0]) + i);
        for (int r = 1; r < v.world; ++r) acc = peer_op(acc, __ldcg(reinterpret_cast<const T*>(v.sbuf[r]) + i), op);
        out[i] = acc;
    }
}
}  // namespace

// Gradient all-reduce fused with Adam: g = (sum over ranks in rank order of
// each rank's flat gradient, read from its HBM) / scale, then the update of
// tgn_kernels.cu k_adam. Identical inputs and order on every rank, so the
// replicated parameters stay bit-identical across ranks.
__global__ void k_adam_peer(float* p, PeerView v, float* m, float* vv, std::size_t n, float scale,
                            float lr, float b1, float one_m_b1, float b2, float one_m_b2,
                            const float* bc, float eps, float* p_tc) {
    pdl_entry();
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float gs = __ldcg(v.grads[0] + i);
    for (int r = 1; r < v.world; ++r) gs += __ldcg(v.grads[r] + i);
    const float bc1 = bc[0], bc2 = bc[1];
    const float gi = gs / scale;
    const float mi = b1 * m[i] + one_m_b1 * gi;
    const float vi = b2 * vv[i] + one_m_b2 * gi * gi;
    m[i] = mi;
    vv[i] = vi;
    const float pn = p[i] - lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
    p[i] = pn;
    if (p_tc) {
        std::uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(pn));
        p_tc[i] = __uint_as_float(r);
    }
}

PeerComm::PeerComm(int rank, int world, int device, const float* grads, std::size_t sbuf_bytes)
    : rank_(rank), world_(world), device_(device), sbuf_bytes_(sbuf_bytes) {
    if (world < 2 || world > kMaxPeers || rank < 0 || rank >= world)
        usage_error("peer transport: need 2 <= world <= 8 and 0 <= rank < world");
    DeviceGuard g(device);
    SPD_CUDA(cudaMalloc(&flags_, sizeof(unsigned) * kFlagKinds * kMaxPeers));
    SPD_CUDA(cudaMemset(flags_, 0, sizeof(unsigned) * kFlagKinds * kMaxPeers));
    SPD_CUDA(cudaMalloc(&sbuf_, sbuf_bytes_ ? sbuf_bytes_ : 256));
    SPD_CUDA(cudaDeviceSynchronize());
    v_.world = world;
    v_.rank = rank;
    v_.flags = flags_;
    v_.own_sbuf = sbuf_;
    v_.grads[rank] = grads;
    v_.flags_of[rank] = flags_;
    v_.sbuf[rank] = sbuf_;
}

PeerComm::~PeerComm() {
    DeviceGuard g(device_);
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (sbuf_) cudaFree(sbuf_);
    if (flags_) cudaFree(flags_);
}

void PeerComm::export_blob(unsigned char* out) const {
    DeviceGuard g(device_);
    cudaIpcMemHandle_t h[3];
    SPD_CUDA(cudaIpcGetMemHandle(&h[0], const_cast<float*>(v_.grads[rank_])));
    SPD_CUDA(cudaIpcGetMemHandle(&h[1], flags_));
    SPD_CUDA(cudaIpcGetMemHandle(&h[2], sbuf_));
    std::memcpy(out, h, sizeof h);
    const std::int32_t meta[2] = {rank_, world_};
    const std::uint64_t sb = sbuf_bytes_;
    std::memcpy(out + 3 * 64, meta, sizeof meta);
    std::memcpy(out + 3 * 64 + 8, &sb, sizeof sb);
}

void PeerComm::connect(const unsigned char* blobs) {
    if (connected_) usage_error("peer transport already connected");
    DeviceGuard g(device_);
    for (int r = 0; r < world_; ++r) {
        const unsigned char* b = blobs + std::size_t(r) * kBlobBytes;
        std::int32_t meta[2];
        std::uint64_t sb;
        std::memcpy(meta, b + 3 * 64, sizeof meta);
        std::memcpy(&sb, b + 3 * 64 + 8, sizeof sb);
        if (meta[0] != r || meta[1] != world_ || sb != sbuf_bytes_)
            data_error("ConfigMismatch", "peer blob " + std::to_string(r) + " is not rank " +
                                             std::to_string(r) + " of this world / configuration");
        if (r == rank_) continue;
        cudaIpcMemHandle_t h[3];
        std::memcpy(h, b, sizeof h);
        void* p[3];
        for (int k = 0; k < 3; ++k) {
            SPD_CUDA(cudaIpcOpenMemHandle(&p[k], h[k], cudaIpcMemLazyEnablePeerAccess));
            opened_.push_back(p[k]);
        }
        v_.grads[r] = static_cast<const float*>(p[0]);
        v_.flags_of[r] = static_cast<unsigned*>(p[1]);
        v_.sbuf[r] = static_cast<const unsigned char*>(p[2]);
    }
    connected_ = true;
}

void PeerComm::signal(int kind, const std::uint64_t* seq_dev, std::int64_t offset, cudaStream_t st) {
    k_peer_signal<<<1, 32, 0, st>>>(v_, kind, seq_dev, 0, offset);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    SPD_CUDA(cudaGetLastError());
}
void PeerComm::wait(int kind, const std::uint64_t* seq_dev, std::int64_t offset, cudaStream_t st) {
    k_peer_wait<<<1, 32, 0, st>>>(v_, kind, seq_dev, 0, offset);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    SPD_CUDA(cudaGetLastError());
}

void PeerComm::adam_step(const std::uint64_t* seq_dev, float* p, float* m, float* v, std::size_t n,
                         float scale, float lr, float b1, float one_m_b1, float b2, float one_m_b2,
                         const float* bc, float eps, float* p_tc, cudaStream_t st) {
    if (!connected_) usage_error("peer transport not connected (spd_tgn_peer_connect)");
    signal(kReady, seq_dev, 0, st);
    wait(kReady, seq_dev, 0, st);
    k_adam_peer<<<unsigned((n + 255) / 256), 256, 0, st>>>(p, v_, m, v, n, scale, lr, b1, one_m_b1, b2,
                                                           one_m_b2, bc, eps, p_tc);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    SPD_CUDA(cudaGetLastError());
    signal(kDone, seq_dev, 0, st);
}

void PeerComm::allreduce(void* data, std::size_t count, int type, int op, cudaStream_t st) {
    if (!connected_) usage_error("peer transport not connected (spd_tgn_peer_connect)");
    const std::size_t esz = type == kF64 ? 8 : 4;
    if (count * esz > sbuf_bytes_) internal_error("InvalidParams", "peer collective exceeds the exchange buffer");
    if (!count) return;
    const std::uint64_t seq = ++sync_seq_;
    // every peer has finished reading my exchange buffer (previous collective)
    k_peer_wait<<<1, 32, 0, st>>>(v_, kSyncDone, nullptr, seq - 1, 0);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    SPD_CUDA(cudaMemcpyAsync(sbuf_, data, count * esz, cudaMemcpyDeviceToDevice, st));
    k_peer_signal<<<1, 32, 0, st>>>(v_, kSyncReady, nullptr, seq, 0);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_peer_wait<<<1, 32, 0, st>>>(v_, kSyncReady, nullptr, seq, 0);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    const unsigned grid = unsigned(std::min<std::size_t>((count + 255) / 256, 1184));
    if (type == kF32) k_peer_reduce<float><<<grid, 256, 0, st>>>(v_, static_cast<float*>(data), count, op);
    else if (type == kF64) k_peer_reduce<double><<<grid, 256, 0, st>>>(v_, static_cast<double*>(data), count, op);
    else k_peer_reduce<int><<<grid, 256, 0, st>>>(v_, static_cast<int*>(data), count, op);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_peer_signal<<<1, 32, 0, st>>>(v_, kSyncDone, nullptr, seq, 0);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    SPD_CUDA(cudaGetLastError());
}

}  // namespace spd
