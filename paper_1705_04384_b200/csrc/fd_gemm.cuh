// Host-side dispatch of the DMMA mode-product GEMM (fd_gemm.cu): tile configurations, launch,
// and a setup-time autotuner that picks the fastest tile shape for each mode-product shape.
#pragma once
#include "common.cuh"
#include "dmma_gemm.cuh"

namespace fdiga {

// Number of tile configurations for a layout (indices 0 .. n-1; 0 is the 128x128 default).
int gemm_num_configs(BLayout L);
const char* gemm_config_name(BLayout L, int cfg);
// Launch config `cfg` on `stream` (p.tiles_* are filled here).  Chooses the 16-/8-byte cp.async
// variant from the operand alignment.
int gemm_launch(fdiga_ctx* ctx, cudaStream_t stream, BLayout L, int cfg, GemmParams p);
// Time every configuration on `p` (operands must be valid device buffers; their contents are
// overwritten in C) and return the fastest index.  Setup-time only.
int gemm_autotune(fdiga_ctx* ctx, BLayout L, const GemmParams& p, int* best_cfg, float* best_ms);

}  // namespace fdiga
