// roll.hpp -- K10 (k_roll.cu): resize chains over a periodic column map.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/dpcuda.h"

namespace dpk {

// Launches K10 for a chain with a resize and at most one pixel op after it
// when the column map is periodic (or, with allow_general, any other ratio)
// and the buffers qualify (16-byte aligned, images in HBM or pinned host
// memory); returns 1 (nothing launched) when the chain is not K10's, DP_OK
// after the launch, or an error status.
int roll_chain_batch(const uint8_t* images, int64_t num_images, const int64_t* order, int64_t first, int64_t rows,
                     int64_t id_base, int64_t id_stride, int64_t id_block, const dp_image_chain* chain, int out_h,
                     int out_w, int64_t* out_ids, float* out, cudaStream_t stream, bool allow_general);

// The chain runs on K10 for HBM-resident, 16-byte aligned buffers.
bool roll_chain_eligible(const dp_image_chain* chain, int out_h, int out_w, bool allow_general);

}  // namespace dpk
