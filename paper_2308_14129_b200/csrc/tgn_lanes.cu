// Concurrent local workers (spd_tgn_config::concurrent, world 1): several SEP
// partitions on one GPU train at the same time instead of one after another.
// Each local worker becomes a "lane" — a child TGNTrainer with its own
// streams, step scratch, CUDA graph and parameter replica — whose step runs
// everything up to its gradient (the lane skips Adam and the shared-hub sync).
// The parent joins the lanes with CUDA events (stream-ordered dependencies
// only, nothing spins), runs ONE Adam on the sum of the lanes' gradients in
// lane order on lane 0's stream (k_adam_multi), copies the new parameters to
// the other replicas, and every lane's next step waits for that. The
// epoch-end restore + shared-hub sync (pac_sim.cpp:162-203) runs over all
// lanes' workers in worker order, exactly as for local workers of one trainer.
//
// So a small-batch step (launch/latency bound: one batch far from filling the
// GPU) overlaps with the other partitions' steps.
#include <atomic>
#include <cmath>

#include "tgn.hpp"

namespace spd {

extern std::atomic<std::uint64_t> g_kernel_launches;  // (tgn_trainer.cu)

void TGNTrainer::build_lanes(const SubGraphs& subs, const std::vector<int>& workers,
                             NodeId node_count) {
    const int W = static_cast<int>(workers.size());
    if (W > 8) data_error("InvalidParams", "concurrent workers: at most 8 per process");
    spd_tgn_config c = cfg_;
    c.concurrent = 0;
    for (int i = 0; i < W; ++i) {
        lanes_.emplace_back(std::make_unique<TGNTrainer>(c, subs, std::vector<int>{workers[i]}, shared_,
                                                         node_count, 0, 1, nullptr, device_));
        lanes_.back()->lane_ = true;
    }
    epoch_steps_ = lanes_[0]->epoch_steps_;
    total_workers_ = lanes_[0]->total_workers_;
    lane_end_.resize(W);
    for (auto& e : lane_end_) SPD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SPD_CUDA(cudaEventCreateWithFlags(&lanes_adam_, cudaEventDisableTiming));
    lanes_adam_valid_ = false;
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

// every other lane's stream waits for the point `ev` of lane 0's stream
void TGNTrainer::lanes_after(cudaEvent_t ev) {
    for (std::size_t k = 1; k < lanes_.size(); ++k) SPD_CUDA(cudaStreamWaitEvent(lanes_[k]->stream_, ev, 0));
}

// lane 0's stream waits for every other lane's current point
void TGNTrainer::lanes_join() {
    for (std::size_t k = 1; k < lanes_.size(); ++k) {
        SPD_CUDA(cudaEventRecord(lane_end_[k], lanes_[k]->stream_));
        SPD_CUDA(cudaStreamWaitEvent(lanes_[0]->stream_, lane_end_[k], 0));
    }
}

void TGNTrainer::lanes_losses(float* loss_out) {
    for (std::size_t k = 0; k < lanes_.size(); ++k) {
        TGNTrainer& l = *lanes_[k];
        float v = 0.f;
        SPD_CUDA(cudaMemcpyAsync(&v, l.loss_dev(), sizeof(float), cudaMemcpyDeviceToHost, l.stream_));
        SPD_CUDA(cudaStreamSynchronize(l.stream_));
        loss_out[k] = l.workers_[0]->batches > 0 ? v : std::nanf("");
    }
}

void TGNTrainer::lanes_step(float* loss_out) {
    // the previous step's Adam wrote every replica's parameters and read
    // every lane's gradients: each lane's step starts after it
    if (lanes_adam_valid_) lanes_after(lanes_adam_);
    for (auto& l : lanes_) l->step(nullptr);
    lanes_adam_step();
    if (loss_out) lanes_losses(loss_out);
}

// after every lane's step is enqueued: join them on lane 0's stream, Adam on
// the lane-ordered gradient sum, copy the parameters to the other replicas
void TGNTrainer::lanes_adam_step() {
    TGNTrainer& l0 = *lanes_[0];
    lanes_join();
    // one Adam on the lane-ordered gradient sum (lane 0's replica, moments
    // and bias corrections), then the replicas
    tgnk::GradList gl{};
    gl.n = static_cast<int>(lanes_.size());
    for (int k = 0; k < gl.n; ++k) gl.g[k] = lanes_[k]->grads_.p;
    const double b1 = cfg_.beta1, b2 = cfg_.beta2;
    const bool tc = cfg_.gemm_mode == 1;
    const std::size_t n = lay_.total;
    tgnk::k_adam_multi<<<unsigned((n + 255) / 256), 256, 0, l0.stream_>>>(
        l0.params_.p, gl, l0.adam_m_.p, l0.adam_v_.p, n, float(total_workers_), cfg_.lr, cfg_.beta1,
        static_cast<float>(1.0 - b1), cfg_.beta2, static_cast<float>(1.0 - b2), l0.adam_bc_, cfg_.adam_eps,
        tc ? l0.params_tc_.p : nullptr);
    SPD_CUDA(cudaGetLastError());
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    for (std::size_t k = 1; k < lanes_.size(); ++k) {
        SPD_CUDA(cudaMemcpyAsync(lanes_[k]->params_.p, l0.params_.p, n * sizeof(float),
                                 cudaMemcpyDeviceToDevice, l0.stream_));
        if (tc)
            SPD_CUDA(cudaMemcpyAsync(lanes_[k]->params_tc_.p, l0.params_tc_.p, n * sizeof(float),
                                     cudaMemcpyDeviceToDevice, l0.stream_));
    }
    SPD_CUDA(cudaEventRecord(lanes_adam_, l0.stream_));
    lanes_adam_valid_ = true;
    // loop ends of this step: flush the pending messages with the NEW
    // parameters, then snapshot (pac_sim.cpp:248-255), after the Adam
    bool any = false;
    for (auto& l : lanes_)
        for (auto& w : l->workers_) any = any || w->flush_due;
    if (!any) return;
    lanes_after(lanes_adam_);
    for (auto& l : lanes_)
        for (auto& w : l->workers_)
            if (w->flush_due) l->loop_end_flush(*w);
}

// epoch end: every lane restores its loop-end snapshot, then the shared-hub
// sync over all lanes' workers (worker order) on lane 0's stream
void TGNTrainer::lanes_end_epoch(bool wait) {
    if (lanes_adam_valid_) lanes_after(lanes_adam_);
    for (auto& l : lanes_) l->end_epoch(false);
    lanes_join();
    std::vector<Worker*> ws;
    for (auto& l : lanes_)
        for (auto& w : l->workers_) ws.push_back(w.get());
    lanes_[0]->sync_workers(ws, lanes_[0]->stream_);
    SPD_CUDA(cudaEventRecord(lanes_adam_, lanes_[0]->stream_));  // (the sync's end)
    lanes_adam_valid_ = true;
    lanes_after(lanes_adam_);
    if (wait) lanes_wait();
}

float TGNTrainer::lanes_run_steps(std::uint64_t n) {
    lanes_wait();
    cudaEvent_t a, b;
    SPD_CUDA(cudaEventCreate(&a));
    SPD_CUDA(cudaEventCreate(&b));
    SPD_CUDA(cudaEventRecord(a, lanes_[0]->stream_));
    for (std::uint64_t k = 0; k < n; ++k) {
        if (lanes_[0]->step_in_epoch_ >= epoch_steps_) {
            end_epoch();
            begin_epoch(lanes_[0]->epoch_ + 1);
        }
        lanes_step(nullptr);
    }
    // lane 0's stream ends with the step's Adam, after every lane's step
    SPD_CUDA(cudaEventRecord(b, lanes_[0]->stream_));
    SPD_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    SPD_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    lanes_wait();
    return ms;
}

}  // namespace spd
