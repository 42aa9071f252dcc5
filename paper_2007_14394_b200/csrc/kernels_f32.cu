// kernels_f32.cu — FP32 perf-mode instantiations (FMA contraction allowed). Probe
// positions, stencils, MVC, atlas lookups and relocation stay FP64; the sphere
// traces, soft shadows and the texel convolution run in FP32.
#include "kernels_impl.cuh"

namespace sdfgi_dev {

template void launch_probe_update<float>(const UpdateParams<float>&, int, int, bool, cudaStream_t);
template void launch_trace_debug<float>(const UpdateParams<float>&, int, cudaStream_t);

}  // namespace sdfgi_dev
