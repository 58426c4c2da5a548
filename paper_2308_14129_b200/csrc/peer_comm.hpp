// Peer-memory transport for the multi-process TGN trainer (one process per
// partition / GPU): the per-step gradient all-reduce is fused with Adam — each
// rank reads every rank's flat gradient buffer straight from its peer's HBM
// (CUDA IPC mappings: NVLink P2P across GPUs, the same HBM for ranks sharing
// one GPU), sums in rank order (bit-identical on every rank) and applies the
// update, so no separate reduce pass or staging copy exists. Ranks order
// themselves with monotonic per-step sequence flags in each other's memory
// (release / acquire at system scope): READY (my gradients of step s are
// final), DONE (I have finished reading your gradients of step s; you may
// clear them). The epoch-end shared-hub sync (pac_sim.cpp:162-203) uses the
// same flags around an exchange buffer.
//
// Alternative to NCCL (tgn_trainer.cu): selected when a trainer with world > 1
// is created without an NCCL id; the caller exchanges the export blobs of all
// ranks (any host channel: torch.distributed gloo, MPI, files) and connects.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace spd {

constexpr int kMaxPeers = 8;

// Device view (kernel parameter). Flag array of rank q: [kind][kMaxPeers]
// unsigned, slot [kind][r] written by rank r.
struct PeerView {
    int world = 1, rank = 0;
    const float* grads[kMaxPeers] = {};
    unsigned* flags_of[kMaxPeers] = {};      // every rank's flag array (mapped)
    const unsigned* flags = nullptr;         // own flag array
    const unsigned char* sbuf[kMaxPeers] = {};  // every rank's exchange buffer (mapped)
    unsigned char* own_sbuf = nullptr;
};
enum PeerFlag : int { kReady = 0, kDone = 1, kSyncReady = 2, kSyncDone = 3, kFlagKinds = 4 };
enum PeerOp : int { kOpSum = 0, kOpMin = 1, kOpMax = 2 };
enum PeerType : int { kF32 = 0, kF64 = 1, kI32 = 2 };

class PeerComm {
public:
    PeerComm(int rank, int world, int device, const float* grads, std::size_t sbuf_bytes);
    ~PeerComm();
    PeerComm(const PeerComm&) = delete;
    PeerComm& operator=(const PeerComm&) = delete;

    static constexpr std::size_t kBlobBytes = 3 * 64 + 16;
    void export_blob(unsigned char* out) const;  // kBlobBytes
    void connect(const unsigned char* blobs);    // world * kBlobBytes, rank order
    bool connected() const { return connected_; }
    const PeerView& view() const { return v_; }

    // In-graph step protocol (seq read from *seq_dev, the step's control word)
    void signal(int kind, const std::uint64_t* seq_dev, std::int64_t offset, cudaStream_t st);
    void wait(int kind, const std::uint64_t* seq_dev, std::int64_t offset, cudaStream_t st);
    // Eager collective over the ranks (epoch-end sync): data[0, count) of
    // `type` reduced with `op` in rank order into data on every rank.
    void allreduce(void* data, std::size_t count, int type, int op, cudaStream_t st);
    // The step's fused gradient all-reduce + Adam (k_adam_peer): READY(seq),
    // wait for every rank's READY(seq), read-sum-update, DONE(seq). The
    // caller's next gradient clear waits for DONE(seq) of every rank
    // (wait(kDone, seq_dev, -1) at step start).
    void adam_step(const std::uint64_t* seq_dev, float* p, float* m, float* v, std::size_t n,
                   float scale, float lr, float b1, float one_m_b1, float b2, float one_m_b2,
                   const float* bc, float eps,
                   float* p_tc, cudaStream_t st);

private:
    int rank_, world_, device_;
    bool connected_ = false;
    unsigned* flags_ = nullptr;  // [kFlagKinds][kMaxPeers]
    unsigned char* sbuf_ = nullptr;
    std::size_t sbuf_bytes_;
    std::uint64_t* seq_host_ = nullptr;  // eager collectives' sequence (device word)
    std::uint64_t sync_seq_ = 0;
    std::vector<void*> opened_;
    PeerView v_;
};

}  // namespace spd
