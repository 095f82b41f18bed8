// Instantiations of k_traverse for METRIC = 0, 32-bit visited table.
#include "traverse_kernel.cuh"

namespace pa {
namespace trav {
// Trace mode (parity tests, never timed) uses the generic-row-length variant only.
template <int METRIC, bool COMPACT, int SMAX>
void* pick4(int dps, bool trace) {
    if (trace) return (void*)k_traverse<METRIC, COMPACT, SMAX, 0, true>;
    switch (dps) {
        case 32: return (void*)k_traverse<METRIC, COMPACT, SMAX, 8, false>;
        case 48: return (void*)k_traverse<METRIC, COMPACT, SMAX, 12, false>;
        case 64: return (void*)k_traverse<METRIC, COMPACT, SMAX, 16, false>;
        case 128: return (void*)k_traverse<METRIC, COMPACT, SMAX, 32, false>;
        default: return (void*)k_traverse<METRIC, COMPACT, SMAX, 0, false>;
    }
}
void* traverse_pick_0w(int ef, int dps, bool trace) {
    constexpr int METRIC = 0;
    constexpr bool COMPACT = false;
    if (ef <= 64) return pick4<METRIC, COMPACT, 2>(dps, trace);
    if (ef <= 96) return pick4<METRIC, COMPACT, 3>(dps, trace);
    if (ef <= 128) return pick4<METRIC, COMPACT, 4>(dps, trace);
    return pick4<METRIC, COMPACT, 8>(dps, trace);
}
}  // namespace trav
}  // namespace pa
