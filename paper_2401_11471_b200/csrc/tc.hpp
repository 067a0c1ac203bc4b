// tc.hpp -- tensor-core (tcgen05 / TMEM / TMA) kernels for sm_100a (internal).
// Each launcher returns true when it took the op (shape supported) and enqueued
// the kernel; false means the shape was declined (the caller may run the SIMT kernel) unless
// tc_take_error() reports a launch / attribute failure.
#pragma once
#include <cuda.h>

#include <utility>

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
// fused identity bottleneck forward (bneck_tc.cu), or false (shape declined / launch failed)
bool tc_bneck_fwd(const BneckArgs &a, cudaStream_t st);

// ---- shared launcher helpers (conv_tc.cu) for the other tcgen05 translation units
bool tc_smem_attr(const void *kern, int bytes);   // MaxDynamicSharedMemorySize once per (kernel, device)
int tc_num_sms();
// 4D map over a band View (Cp, W, rows, B), box (kc, TW*es, TH*es, 1), swizzle by kc (64/32/16 ch)
bool tc_encode_view(CUtensorMap *m, const View &v, int B, int TW, int TH, int es, int kc);
// 3D map over OHWI weights [rows][taps][cin_p], box (kc, 1, BN)
bool tc_encode_w(CUtensorMap *m, const void *w, int rows, int taps, int cin_p, int BN, int kc);
bool tc_pdl_on();
void tc_note_launch(const void *fn, bool ok);   // last-kernel name (profiling) / launch error flag
template <typename... KArgs, typename... Args>
static inline bool tc_launch(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = tc_pdl_on() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const bool ok = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...) == cudaSuccess;
    tc_note_launch((const void *)kern, ok);
    return ok;
}
}  // namespace lrcnn
