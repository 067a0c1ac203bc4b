// conv_tc.cu -- tcgen05 implicit-GEMM convolution kernels (sm_100a).  Placeholder.
#include "tc.hpp"
namespace lrcnn {
bool tc_available() { return false; }
bool tc_conv_fwd(const ConvFwdArgs &, cudaStream_t) { return false; }
bool tc_conv_dgrad(const DgradArgs &, cudaStream_t) { return false; }
bool tc_conv_wgrad(const WgradArgs &, cudaStream_t) { return false; }
}  // namespace lrcnn
