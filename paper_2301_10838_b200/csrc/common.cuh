// common.cuh -- device helpers shared by the sm_100a kernels of libmt_b200.
//
// Total order (step a1, SURVEY.md 8a / DESIGN.md "K1"): the paper compares raw
// values f(u) < f(v) and never resolves ties;
// reading R1 breaks ties by vertex id, i.e. vertices are ordered by the 64-bit
// key  key(u) = ord(f[u]) << 32 | u  compared as an unsigned integer, where
// ord() maps IEEE float32 bits to uint32 monotonically (-0.0 canonicalised to
// +0.0 first, reading R2).  For the split tree (reading R16)
// ord is complemented: ~ord(x) orders like ord(-x) and ids stay ascending.
#pragma once
#include <cstdint>

namespace mt {

constexpr uint32_t FULL_MASK = 0xffffffffu;

// uint32 whose unsigned order equals the IEEE order of finite floats.
__device__ __forceinline__ uint32_t ord32(float x) {
    uint32_t b = __float_as_uint(x);
    b = (b == 0x80000000u) ? 0u : b;                     // -0.0 -> +0.0
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ bool nonfinite(float x) {
    return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u;
}

// ord of f[x] with the split-tree complement mask (0 or ~0) applied.
__device__ __forceinline__ uint32_t ordf(const float* __restrict__ f, uint32_t x, uint32_t flip) {
    return ord32(__ldg(f + x)) ^ flip;
}

__device__ __forceinline__ uint64_t key_of(uint32_t ord, uint32_t id) {
    return (static_cast<uint64_t>(ord) << 32) | id;
}

__device__ __forceinline__ uint64_t keyf(const float* __restrict__ f, uint32_t x, uint32_t flip) {
    return key_of(ordf(f, x, flip), x);
}

// Packed triplet cell (reading R11): s high, v low.
__device__ __forceinline__ uint64_t pack(uint32_t s, uint32_t v) {
    return (static_cast<uint64_t>(s) << 32) | v;
}
__device__ __forceinline__ uint32_t cell_s(uint64_t c) { return static_cast<uint32_t>(c >> 32); }
__device__ __forceinline__ uint32_t cell_v(uint64_t c) { return static_cast<uint32_t>(c); }

// Coherent (L1-bypassing) loads/stores of cells that other threads CAS
// concurrently: a plain ld.global may hit a stale L1 line and livelock a CAS
// retry loop (reading R8).
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t cas64(uint64_t* p, uint64_t expected, uint64_t desired) {
    return atomicCAS(reinterpret_cast<unsigned long long*>(p), expected, desired);
}

// Error bits (sticky, in the workspace counters).
constexpr uint32_t ERR_NONFINITE = 1u;
constexpr uint32_t ERR_CAPACITY = 2u;
constexpr uint32_t ERR_ESS_CAPACITY = 4u;

// Workspace counter slots (uint64 each).
enum CounterSlot : int {
    CTR_TICKET = 0,     // dynamic tile ticket of the repair/diagram kernel
    CTR_ERR = 1,        // error bits
    CTR_ESS = 2,        // number of essential classes found
    CTR_FIN = 3,        // number of finite pairs (written by the last tile)
    CTR_CAP = 4,        // capacity (records) of the diagram target buffer
    CTR_COUNT = 8
};

}  // namespace mt
