// Instantiation of the radsort level loop for rec_size=16, key_size=8.
#include "sorter.cuh"
namespace radsort {
template radsort_status run_layout<16, 8>(Context*, uint8_t*, uint8_t*, uint32_t, cudaStream_t, radsort_stats&);
}
