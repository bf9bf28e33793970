// Instantiation of the radsort level loop and multi-GPU building blocks for
// rec_size=32, key_size=8.
#include "sorter.cuh"
namespace radsort {
// the (key, index) records of the key + index sort are sorted by layout_16_8.cu's instantiation
extern template radsort_status run_layout<16, 8>(Context*, uint8_t*, uint8_t*, uint32_t, cudaStream_t, radsort_stats&);
template radsort_status run_layout_segs<32, 8>(Context*, uint8_t*, uint8_t*, uint32_t, const uint32_t*,
                                                  const uint32_t*, uint32_t, uint32_t, cudaStream_t, radsort_stats&);
template radsort_status run_layout<32, 8>(Context*, uint8_t*, uint8_t*, uint32_t, cudaStream_t, radsort_stats&);
template radsort_status multi_hist<32, 8>(Context*, const uint8_t*, uint32_t, uint32_t, cudaStream_t, uint64_t*,
                                           uint64_t*);
template radsort_status multi_scatter<32, 8>(Context*, uint8_t*, uint8_t*, uint32_t, uint32_t, const uint64_t*,
                                              cudaStream_t);
template radsort_status multi_bounds<32, 8>(Context*, const uint8_t*, const uint32_t*, const uint32_t*,
                                             const uint64_t*, uint32_t, cudaStream_t, uint64_t*, uint64_t*);
template radsort_status multi_piece_hist<32, 8>(Context*, PieceWs&, const uint8_t*, const uint32_t*,
                                                const uint32_t*, uint32_t, uint32_t, cudaStream_t, uint32_t*);
template radsort_status multi_piece_scatter<32, 8>(Context*, PieceWs&, const uint8_t*, const uint32_t*,
                                                   const uint64_t*, cudaStream_t);
}
