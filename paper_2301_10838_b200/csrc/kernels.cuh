// kernels.cuh -- host launchers of the sm_100a kernels (internal to libmt_b200).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "mt.h"

namespace mt {

// tile shape (32 x ty x tz, 4096 vertices) for a grid with nz planes
void tile_shape(uint32_t nz, uint32_t* ty, uint32_t* tz);

// K1 + K2 + in-tile K3/K4: keys, steepest descent, tile-local merge tree (tile_tmt.cu)
void launch_tile_tmt(const float* f, Cell* C, uint32_t nx, uint32_t ny, uint32_t nz, uint32_t flip,
                     unsigned long long* counters, unsigned long long* stats, cudaStream_t stream);

// K3: merge of the tile-crossing grid edges on the global store (merge_cross.cu)
void launch_merge_cross(Cell* C, uint32_t nx, uint32_t ny, uint32_t nz, unsigned long long* fetch,
                        unsigned long long* stats, int num_sms, cudaStream_t stream);

// K4+K5: repair fused with the ordered diagram compaction (repair_diagram.cu)
uint64_t repair_tiles(uint64_t n);
void launch_repair_diagram(Cell* C, uint64_t* T, const float* f, uint64_t n, unsigned long long* counters,
                           uint64_t* status, mt_pair* out, uint64_t out_cap, mt_pair* ess, uint32_t ess_cap,
                           unsigned long long* stats, cudaStream_t stream);
void launch_finish_diagram(unsigned long long* counters, mt_pair* out, uint64_t out_cap, mt_pair* ess,
                           uint32_t ess_cap, cudaStream_t stream);

}  // namespace mt
