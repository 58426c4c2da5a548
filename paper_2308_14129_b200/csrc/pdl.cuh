// Programmatic dependent launch (PDL): kernels of the training step may be
// launched with cudaLaunchAttributeProgrammaticStreamSerialization, so their
// dependents begin launching at once and each kernel waits for its
// predecessors' completion and memory before its first global access.
// On every stream: slower on the GDELT step (B = 2000: waiting dependent CTAs
// hold SM slots the side-stream weight-gradient GEMMs would use, 0.525 vs
// 0.500 ms), faster on small batches whose step is launch-latency bound
// (B = 200: Reddit 0.197 -> 0.186 ms, LastFM 0.180 -> 0.174 ms): on for
// batches <= 512 (set by the trainer); SPD_PDL=1 / SPD_PDL=0 force it. On the
// critical-path streams only: see pdl_main_only.
// Without the attribute both device instructions are no-ops.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace spd {

__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
// The two halves of pdl_entry, for a kernel with a prologue that reads only
// data no kernel of the current step writes: parameters, whose writer (the
// optimizer, or the lanes' replica copy) is always followed by non-GEMM
// kernels (gathers, persist) before any kernel that prefetches them, so it
// has completed when such a kernel launches (k_decoder, umma_gru_kernel,
// umma_gemm_kernel with Args::b_static).
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline int pdl_forced() {  // -1 auto, 0 off, 1 on
    static const int m = [] {
        const char* e = std::getenv("SPD_PDL");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return m;
}
inline bool& pdl_auto() {
    static bool on = false;
    return on;
}
inline bool pdl_enabled() {
    const int m = pdl_forced();
    return m >= 0 ? m == 1 : pdl_auto();
}
// PDL on the high-priority (critical-path) streams at every batch size: their
// kernels' launches overlap their predecessors' tails while the side streams'
// kernels launch normally and hold no SM slots waiting (GDELT B = 2000:
// 0.349 vs 0.364 ms per step). SPD_PDL_MAIN=0 turns it off.
inline bool pdl_main_only() {
    static const bool on = [] {
        const char* e = std::getenv("SPD_PDL_MAIN");
        return !(e && e[0] == '0');
    }();
    return on;
}
// whether a launch on a stream of priority `prio` uses PDL
inline bool pdl_for(int prio) {
    if (pdl_enabled()) return true;
    if (!pdl_main_only()) return false;
    static const int hi = [] {
        int lo = 0, h = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &h);
        return h;
    }();
    return prio == hi;
}

}  // namespace spd
