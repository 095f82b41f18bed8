// Instantiations of k_refine (NEXT-f3 stages ②③, traverse_kernel.cuh) for
// METRIC = 1, split from stages23.cu so the two metrics compile in parallel.
#include "traverse_kernel.cuh"

namespace pa {
namespace trav {
namespace {
template <int VIS>
void* pick_smax(int cap, int D) {
    auto nvr = [&](auto smax) -> void* {
        constexpr int SM = decltype(smax)::value;
        if (D == 96) return (void*)k_refine<1, VIS, SM, 24>;
        return (void*)k_refine<1, VIS, SM, 0>;
    };
    if (cap <= 64) return nvr(std::integral_constant<int, 2>{});
    if (cap <= 96) return nvr(std::integral_constant<int, 3>{});
    if (cap <= 128) return nvr(std::integral_constant<int, 4>{});
    if (cap <= 256) return nvr(std::integral_constant<int, 8>{});
    return nvr(std::integral_constant<int, 16>{});
}
}  // namespace

void* refine_pick_m1(int cap, int D, bool compact) {
    return compact ? pick_smax<1>(cap, D) : pick_smax<0>(cap, D);
}
}  // namespace trav
}  // namespace pa
