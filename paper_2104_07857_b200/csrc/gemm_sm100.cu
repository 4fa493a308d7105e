// Placeholder until the tcgen05 tile GEMM lands (memory-centric tiling row).
#include "common.cuh"
extern "C" int zi_linear_fwd(const void*, const void*, const void*, void*, int, int, int, int,
                             int, int, void*) {
  zi::set_error("zi_linear_fwd: not built yet");
  return ZI_EINVAL;
}
