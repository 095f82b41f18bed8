// Instantiations of k_traverse: METRIC = 1, 16-bit visited table,
// binary16 reduced rows.  `d` = row length in elements (d' rounded).
#include "traverse_kernel.cuh"

namespace pa {
namespace trav {
namespace {
template <int METRIC, int VIS, int SMAX>
void* pick4(int d, bool trace) {
    if (trace) return (void*)k_traverse<METRIC, VIS, SMAX, 0, true, true>;
    switch (d) {
        case 32: return (void*)k_traverse<METRIC, VIS, SMAX, 4, false, true>;
        case 48: return (void*)k_traverse<METRIC, VIS, SMAX, 6, false, true>;
        case 64: return (void*)k_traverse<METRIC, VIS, SMAX, 8, false, true>;
        case 128: return (void*)k_traverse<METRIC, VIS, SMAX, 16, false, true>;
        default: return (void*)k_traverse<METRIC, VIS, SMAX, 0, false, true>;
    }
}
template <int METRIC, int VIS, int SMAX>
void* pick4p(int d, bool trace) {
    if (trace) return (void*)k_traverse_pipe<METRIC, VIS, SMAX, 0, true, true>;
    switch (d) {
        case 32: return (void*)k_traverse_pipe<METRIC, VIS, SMAX, 4, false, true>;
        case 48: return (void*)k_traverse_pipe<METRIC, VIS, SMAX, 6, false, true>;
        case 64: return (void*)k_traverse_pipe<METRIC, VIS, SMAX, 8, false, true>;
        case 96: return (void*)k_traverse_pipe<METRIC, VIS, SMAX, 12, false, true>;
        case 128: return (void*)k_traverse_pipe<METRIC, VIS, SMAX, 16, false, true>;
        default: return (void*)k_traverse_pipe<METRIC, VIS, SMAX, 0, false, true>;
    }
}
}  // namespace

void* traverse_pick_1ch(int ef, int d, bool trace) {
    constexpr int METRIC = 1;
    constexpr int VIS = 1;
    if (ef <= 64) return pick4<METRIC, VIS, 2>(d, trace);
    if (ef <= 96) return pick4<METRIC, VIS, 3>(d, trace);
    if (ef <= 128) return pick4<METRIC, VIS, 4>(d, trace);
    return pick4<METRIC, VIS, 8>(d, trace);
}
void* traverse_pick_pipe_1ch(int ef, int d, bool trace) {
    constexpr int METRIC = 1;
    constexpr int VIS = 1;
    if (ef <= 64) return pick4p<METRIC, VIS, 2>(d, trace);
    if (ef <= 96) return pick4p<METRIC, VIS, 3>(d, trace);
    if (ef <= 128) return pick4p<METRIC, VIS, 4>(d, trace);
    return pick4p<METRIC, VIS, 8>(d, trace);
}
}  // namespace trav
}  // namespace pa
