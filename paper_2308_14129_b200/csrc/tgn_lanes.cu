// Concurrent local workers (spd_tgn_config::concurrent, world 1): several SEP
// partitions on one GPU train at the same time instead of one after another.
// Each local worker becomes a "lane" — a child TGNTrainer with its own
// streams, step scratch, CUDA graphs and parameter / Adam replica — and the
// lanes form an in-process peer group (peer_comm.cu connect_local): every
// step's gradient all-reduce is the fused peer Adam (each lane reads every
// lane's gradients in lane order, so the replicas stay bit-identical) and the
// epoch-end shared-hub sync (pac_sim.cpp:162-203) runs over the same
// mappings. This is the multi-rank design of DESIGN.md §6 with ranks as
// streams of one process, so a small-batch step (launch/latency bound, one
// batch far from filling the GPU) overlaps with the other partitions' steps.
//
// Host discipline: a lane's step enqueues waits for its peers' flags, so every
// lane's work of a global step is enqueued before the host waits on any lane.
#include "pdl.cuh"
#include "tgn.hpp"

namespace spd {

void TGNTrainer::build_lanes(const SubGraphs& subs, const std::vector<int>& workers,
                             NodeId node_count) {
    const int W = static_cast<int>(workers.size());
    if (W > kMaxPeers) data_error("InvalidParams", "concurrent workers: at most 8 per process");
    spd_tgn_config c = cfg_;
    c.concurrent = 0;
    for (int i = 0; i < W; ++i)
        lanes_.emplace_back(std::make_unique<TGNTrainer>(c, subs, std::vector<int>{workers[i]}, shared_,
                                                         node_count, i, W, nullptr, device_));
    std::vector<PeerComm*> all;
    for (auto& l : lanes_) all.push_back(l->peer_.get());
    for (auto& l : lanes_) l->peer_->connect_local(all);
    // no programmatic dependent launch: early-launched dependents waiting on a
    // spinning peer wait would hold the SM slots the other lanes need to
    // raise its flag (pdl.cuh; process-wide, SPD_PDL=1 overrides at your risk)
    pdl_auto() = false;
    epoch_steps_ = lanes_[0]->epoch_steps_;
    total_workers_ = lanes_[0]->total_workers_;
}

TGNTrainer* TGNTrainer::lane_of(int gid) {
    for (auto& l : lanes_)
        for (auto& w : l->workers_)
            if (w->gid == gid) return l.get();
    usage_error("worker " + std::to_string(gid) + " is not owned by this trainer");
}

void TGNTrainer::lanes_wait() {
    for (auto& l : lanes_) SPD_CUDA(cudaStreamSynchronize(l->stream_));
}

void TGNTrainer::lanes_losses(float* loss_out) {
    // after every lane's step is enqueued: each lane's (single-worker) loss
    for (std::size_t k = 0; k < lanes_.size(); ++k) {
        TGNTrainer& l = *lanes_[k];
        float v = 0.f;
        SPD_CUDA(cudaMemcpyAsync(&v, l.loss_dev(), sizeof(float), cudaMemcpyDeviceToHost, l.stream_));
        SPD_CUDA(cudaStreamSynchronize(l.stream_));
        loss_out[k] = l.workers_[0]->batches > 0 ? v : std::nanf("");
    }
}

void TGNTrainer::lanes_step(float* loss_out) {
    for (auto& l : lanes_) l->step(nullptr);
    if (loss_out) lanes_losses(loss_out);
}

float TGNTrainer::lanes_run_steps(std::uint64_t n) {
    lanes_wait();
    cudaEvent_t a;
    SPD_CUDA(cudaEventCreate(&a));
    SPD_CUDA(cudaEventRecord(a, lanes_[0]->stream_));
    for (std::uint64_t k = 0; k < n; ++k) {
        if (lanes_[0]->step_in_epoch_ >= epoch_steps_) {
            end_epoch();
            begin_epoch(lanes_[0]->epoch_ + 1);
        }
        lanes_step(nullptr);
    }
    float ms = 0.f;
    for (auto& l : lanes_) {  // elapsed until the last lane's end
        cudaEvent_t b;
        SPD_CUDA(cudaEventCreate(&b));
        SPD_CUDA(cudaEventRecord(b, l->stream_));
        SPD_CUDA(cudaEventSynchronize(b));
        float t = 0.f;
        SPD_CUDA(cudaEventElapsedTime(&t, a, b));
        ms = std::max(ms, t);
        cudaEventDestroy(b);
    }
    cudaEventDestroy(a);
    return ms;
}

}  // namespace spd
