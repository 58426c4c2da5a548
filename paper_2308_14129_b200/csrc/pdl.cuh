// Programmatic dependent launch (PDL), opt-in (SPD_PDL=1): kernels of the
// training step are then launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, their dependents may
// begin launching at once and each kernel waits for its predecessors'
// completion and memory before its first global access. Measured on the
// GDELT step it is slower (0.525 vs 0.500 ms: waiting dependent CTAs hold SM
// slots the side-stream weight-gradient GEMMs would use), so it is off by
// default; without the attribute both instructions are no-ops.
#pragma once

#include <cstdlib>

namespace spd {

__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SPD_PDL");
        return e && e[0] == '1';
    }();
    return on;
}

}  // namespace spd
