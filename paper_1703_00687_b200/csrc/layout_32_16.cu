// Instantiation of the radsort level loop for rec_size=32, key_size=16.
#include "sorter.cuh"
namespace radsort {
template radsort_status run_layout<32, 16>(Context*, uint8_t*, uint8_t*, uint32_t, cudaStream_t, radsort_stats&);
}
