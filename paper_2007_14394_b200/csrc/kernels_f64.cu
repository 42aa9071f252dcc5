// kernels_f64.cu — FP64 parity-mode instantiations. Compiled with -fmad=false so
// every product and sum rounds separately, matching the reference built with
// -ffp-contract=off (SURVEY §7 hard part 1); sqrt and division are IEEE.
#include "kernels_impl.cuh"

namespace sdfgi_dev {

__global__ void __launch_bounds__(128) k_query_points(QueryParams P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    Counters c;
    V3<double> p = mk(P.pts[3 * i], P.pts[3 * i + 1], P.pts[3 * i + 2]);
    double init = P.init ? P.init[i] : INFINITY;
    int owner = -1;
    P.outD[i] = query<double, false>(P.scene, p, init, &owner, &c);
    P.outOwner[i] = owner >= 0 ? P.scene.orig[owner] : -1;
}

void launch_relocate(const RelocParams& p, int nProbes, bool stats, cudaStream_t st) {
    const int blocks = (nProbes + 127) / 128;
    if (stats)
        k_relocate<true><<<blocks, 128, 0, st>>>(p);
    else
        k_relocate<false><<<blocks, 128, 0, st>>>(p);
}

void launch_query_points(const QueryParams& p, cudaStream_t st) {
    k_query_points<<<(p.n + 127) / 128, 128, 0, st>>>(p);
}

template void launch_probe_update<double>(const UpdateParams<double>&, int, int, bool, cudaStream_t);
template void launch_trace_debug<double>(const UpdateParams<double>&, int, cudaStream_t);

}  // namespace sdfgi_dev
