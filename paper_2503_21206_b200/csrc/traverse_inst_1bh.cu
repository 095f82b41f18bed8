// Instantiations of k_traverse_pipe: METRIC = 1, bloom-filter visited set
// (NEXT-f1), binary16 reduced rows.  `d` = row length in elements.
#include "traverse_kernel.cuh"

namespace pa {
namespace trav {
namespace {
template <int METRIC, int SMAX>
void* pick4p(int d, bool trace) {
    if (trace) return (void*)k_traverse_pipe<METRIC, 2, SMAX, 0, true, true>;
    switch (d) {
        case 32: return (void*)k_traverse_pipe<METRIC, 2, SMAX, 4, false, true>;
        case 48: return (void*)k_traverse_pipe<METRIC, 2, SMAX, 6, false, true>;
        case 64: return (void*)k_traverse_pipe<METRIC, 2, SMAX, 8, false, true>;
        case 96: return (void*)k_traverse_pipe<METRIC, 2, SMAX, 12, false, true>;
        case 128: return (void*)k_traverse_pipe<METRIC, 2, SMAX, 16, false, true>;
        default: return (void*)k_traverse_pipe<METRIC, 2, SMAX, 0, false, true>;
    }
}
}  // namespace

void* traverse_pick_pipe_1bh(int ef, int d, bool trace) {
    if (ef <= 64) return pick4p<1, 2>(d, trace);
    if (ef <= 96) return pick4p<1, 3>(d, trace);
    if (ef <= 128) return pick4p<1, 4>(d, trace);
    return pick4p<1, 8>(d, trace);
}
}  // namespace trav
}  // namespace pa
