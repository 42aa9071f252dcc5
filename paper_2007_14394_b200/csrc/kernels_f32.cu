// kernels_f32.cu — FP32 perf-mode instantiations (FMA contraction allowed). Probe
// positions, the stencil's cell selection and trilinear weights, atlas lookups and
// relocation stay FP64; the sphere traces, soft shadows, the MVC weights and the
// texel convolution run in FP32.
#include "kernels_impl.cuh"
#include "gather_impl.cuh"

namespace sdfgi_dev {

template void launch_wavefront<float>(const WaveParams<float>&, int, bool, cudaStream_t, const cudaEvent_t*,
                                      long long*);

template void launch_gather<float>(const GatherParams<float>&, int, bool, cudaStream_t);
template void launch_contact<float>(const WaveParams<float>&, bool, cudaStream_t, long long*);
template void launch_compose<float>(const WaveParams<float>&, bool, cudaStream_t, long long*);
template void launch_batch<float>(const WaveParams<float>&, int, bool, cudaStream_t, long long*);

}  // namespace sdfgi_dev
