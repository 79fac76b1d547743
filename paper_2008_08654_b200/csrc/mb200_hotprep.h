// mb200_hotprep.h -- host interface of the heavy-hitter selection kernels
// (kernels_hotprep.cu), called by run_hot (kernels_hot.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace mb200 {

// workspace words of one call (carved by run_hot from its stream-ordered allocation;
// tc .. fill are zeroed per call, tk is set to the empty key)
template <typename KeyT>
struct HotPrepWs {
    KeyT* tk;             // sample count table: keys (open addressing, `slots` entries)
    uint32_t* tc;         //                     counts
    uint32_t slots;
    uint32_t* hist;       // [256] histogram of min(count, 255)
    uint32_t* hot_count;  // [0] keys listed
    uint32_t* hot_sum;    // sampled items the listed keys cover
    uint32_t* fill;       // [256] per-level fill counters of the ordered selection
    uint32_t* go;         // [0] 1: the sample shows heavy hitters, [1] covered, [2] ticket
    uint32_t* placed;     // keys the layout placed (hot stats)
    KeyT* hot;            // the hot list, hottest first (kCap entries)
};

// probe -> count -> histogram -> ordered selection (w.hot, w.hot_count[0])
template <typename KeyT>
cudaError_t launch_hot_select(const KeyT* keys, uint64_t n, uint32_t sample, const HotPrepWs<KeyT>& w, cudaStream_t s);
// the two-choice table layout every scatter CTA copies (layout: keys per slot,
// tags: the tagged slot words of u32 keys, else null)
template <typename KeyT>
cudaError_t launch_hot_layout(const HotPrepWs<KeyT>& w, KeyT* layout, uint32_t* tags, const uint32_t* priv_go,
                              cudaStream_t s);

}  // namespace mb200
