// tc.hpp -- tensor-core (tcgen05 / TMEM / TMA) kernels for sm_100a (internal).
// Each launcher returns true when it took the op (shape supported) and enqueued
// the kernel; false means the shape was declined (the caller may run the SIMT kernel) unless
// tc_take_error() reports a launch / attribute failure.
#pragma once
#include "kernels.hpp"

namespace lrcnn {
bool tc_available();
bool tc_conv_fwd(const ConvFwdArgs &a, cudaStream_t st);
bool tc_conv_dgrad(const DgradArgs &a, cudaStream_t st);
bool tc_conv_wgrad(const WgradArgs &a, cudaStream_t st);
// fused 1x1 stride-1 dgrad + wgrad (both results; sets a.db_done / dg_done, d.add_done) or false
bool tc_conv_dwgrad(const WgradArgs &a, const DgradArgs &d, cudaStream_t st);
// name of the last tcgen05 kernel this host thread launched (per-kernel profile), or nullptr
const char *tc_last_kernel();
void tc_clear_last_kernel();
// true (and cleared) if a launcher failed for a reason other than declining the shape: the
// engine reports LRCNN_E_CUDA instead of falling back to SIMT
bool tc_take_error();
// programmatic dependent launch on (default) / off (per-launch event profiling) for this host thread
void tc_set_pdl(bool on);
}  // namespace lrcnn
