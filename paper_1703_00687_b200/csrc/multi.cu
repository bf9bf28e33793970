// Multi-GPU path (radsort_sort_multi): placeholder until the NCCL exchange lands.
#include <cuda_runtime.h>
#include "../../include/radsort.h"
extern "C" radsort_status radsort_sort_multi(void*, void*, uint64_t, uint64_t, uint64_t*, uint32_t, uint32_t, void*, void*) {
  return RADSORT_ERR_UNSUPPORTED;
}
