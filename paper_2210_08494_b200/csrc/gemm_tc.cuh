// tcgen05 3xTF32 GEMM (placeholder until the kernel lands).
#pragma once
namespace bkfac {
inline bool tc_init_attributes() { return true; }
#define BKFAC_GEMM_PATH "SIMT fp32 (CUDA cores)"
}
