// Definitions of the opaque C-ABI handle types and the exception guard shared
// by the extern "C" translation units.
#pragma once

#include <functional>
#include <memory>

#include "host.hpp"

namespace spd {
int guarded_call(const std::function<void()>& f);
}  // namespace spd

#define GUARD(...) return spd::guarded_call([&]() __VA_ARGS__)

struct spd_assignment {
    spd::Assignment a;
};
struct spd_eval_routing {
    spd::EvalRouting r;
};
struct spd_subgraphs {
    spd::SubGraphs s;
};
