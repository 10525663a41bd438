// kernels.cuh -- host launchers of the sm_100a kernels (internal to libmt_b200).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "mt.h"

namespace mt {

// K1+K2: keys + steepest-descent init with tile-local descent (init_descent.cu)
void launch_init_descent(const float* f, Cell* C, uint32_t nx, uint32_t ny, uint32_t nz, uint32_t flip,
                         unsigned long long* counters, cudaStream_t stream);

// K4 (compress mode): point every regular cell at its basin minimum (init_descent.cu)
void launch_compress(Cell* C, uint64_t n, int num_sms, cudaStream_t stream);

// K3: concurrent CAS edge merge over the +x/+y/+z grid edges (merge_edges.cu);
// with guard != NULL it only runs when the edge queue overflowed (*guard > guard_cap)
void launch_merge_edges(Cell* C, uint32_t nx, uint32_t ny, uint32_t nz, int num_sms, unsigned long long* stats,
                        const unsigned long long* guard, uint64_t guard_cap, cudaStream_t stream);

// K3 as filter + persistent state-machine merge over the inter-basin edge queue (merge_queue.cu)
size_t queue_entry_bytes();
void launch_filter_edges(const Cell* C, uint32_t nx, uint32_t ny, uint32_t nz, void* q, uint64_t cap,
                         unsigned long long* qctl, int num_sms, cudaStream_t stream);
void launch_merge_queue(Cell* C, const void* q, uint64_t cap, unsigned long long* qctl, unsigned long long* stats,
                        int num_sms, cudaStream_t stream);

// K4+K5: repair fused with the ordered diagram compaction (repair_diagram.cu)
uint64_t repair_tiles(uint64_t n);
void launch_repair_diagram(Cell* C, uint64_t* T, const float* f, uint64_t n, unsigned long long* counters,
                           uint64_t* status, mt_pair* out, uint64_t out_cap, mt_pair* ess, uint32_t ess_cap,
                           unsigned long long* stats, cudaStream_t stream);
void launch_finish_diagram(unsigned long long* counters, mt_pair* out, uint64_t out_cap, mt_pair* ess,
                           uint32_t ess_cap, cudaStream_t stream);

}  // namespace mt
