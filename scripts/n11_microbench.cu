// n11_microbench.cu -- secondary ceilings of the hot path (SURVEY.md 8d "microbenchmark N11"):
// the merge phase (Alg. 2/3) and the repair walks (Alg. 4/5)
// are dependent random 8/16-byte gathers and 64/128-bit compare-and-swaps on cells spread over
// an array much larger than L2, not streams.  Their ceilings on this B200:
//   gather8 / gather16  -- independent random loads (all lanes, many in flight), loads/s and the
//                          32-B DRAM sector rate they imply;
//   chase16             -- dependent random 16-B loads (pointer chasing): latency per hop;
//   cas64 / cas128      -- uncontended atom.cas on random distinct cells (always succeeding);
//   cas128_hot          -- contended: every CAS on one of H hot cells (retry until success).
// One JSON line per test.  Build + run: python scripts/n11.py (nvcc, sm_100a).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct C16 {
    uint64_t lo, hi;
};

__global__ void init_kernel(C16* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        a[i] = C16{i, mix(i) % n};   // hi: a random successor for the chase
}

template <int W>   // W = 8 or 16 bytes per load
__global__ void gather_kernel(const C16* __restrict__ a, uint64_t n, uint64_t per_thread, uint64_t* sink) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    uint64_t acc = 0;
#pragma unroll 8
    for (uint64_t k = 0; k < per_thread; ++k) {
        const uint64_t i = mix(t * per_thread + k) % n;
        if (W == 8) {
            acc += __ldcg(reinterpret_cast<const unsigned long long*>(a + i));
        } else {
            uint64_t lo, hi;
            asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(a + i));
            acc += lo ^ hi;
        }
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

__global__ void chase_kernel(const C16* __restrict__ a, uint64_t n, uint64_t hops, uint64_t* sink) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    uint64_t x = mix(t) % n;
    for (uint64_t k = 0; k < hops; ++k) {
        uint64_t lo, hi;
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(a + x) : "memory");
        x = hi;
    }
    if (x == 0x123456789ull) sink[0] = x;
}

template <int W>
__global__ void cas_kernel(C16* a, uint64_t n, uint64_t per_thread, uint64_t salt, uint64_t* sink) {
    // uncontended: thread t's k-th CAS hits cell perm(t, k) (a bijection on [0, n) when
    // n is a power of two: odd multiplier), whose current value is known, so every CAS succeeds
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    const uint64_t nthreads = uint64_t(gridDim.x) * blockDim.x;
    uint64_t fails = 0;
    for (uint64_t k = 0; k < per_thread; ++k) {
        const uint64_t j = (t + k * nthreads);
        const uint64_t i = (j * 0x9E3779B97F4A7C15ull + salt) & (n - 1);
        if (W == 8) {
            const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(&a[i].lo), i, i);
            fails += old != i;
        } else {
            uint64_t olo, ohi;
            asm volatile(
                "{\n\t.reg .b128 d, c, v;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 v, {%2, %3};\n\t"
                "atom.relaxed.gpu.global.cas.b128 d, [%4], c, v;\n\tmov.b128 {%0, %1}, d;\n\t}"
                : "=l"(olo), "=l"(ohi)
                : "l"(i), "l"(mix(i) % n), "l"(a + i)
                : "memory");
            fails += olo != i;
        }
    }
    if (fails) atomicAdd(reinterpret_cast<unsigned long long*>(sink), fails);
}

__global__ void cas_hot_kernel(C16* a, uint64_t hot, uint64_t per_thread, uint64_t* sink) {
    // contended: H hot cells; each CAS increments the cell's lo (read, CAS, retry on failure)
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    uint64_t tries = 0;
    for (uint64_t k = 0; k < per_thread; ++k) {
        C16* p = a + (mix(t * per_thread + k) % hot) * 8;   // 128 B apart
        uint64_t lo, hi;
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
        while (true) {
            uint64_t olo, ohi;
            asm volatile(
                "{\n\t.reg .b128 d, c, v;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 v, {%4, %3};\n\t"
                "atom.relaxed.gpu.global.cas.b128 d, [%5], c, v;\n\tmov.b128 {%0, %1}, d;\n\t}"
                : "=l"(olo), "=l"(ohi)
                : "l"(lo), "l"(hi), "l"(lo + 1), "l"(p)
                : "memory");
            ++tries;
            if (olo == lo && ohi == hi) break;
            lo = olo;
            hi = ohi;
        }
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(sink), tries);
}

int main(int argc, char** argv) {
    const uint64_t n = 1ull << 30;   // 16 GiB of 16-B cells (c5's working-cell array), >> L2
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    C16* a;
    uint64_t* sink;
    CK(cudaMalloc(&a, n * sizeof(C16)));
    CK(cudaMalloc(&sink, 64));
    CK(cudaMemset(sink, 0, 64));
    init_kernel<<<sms * 8, 256>>>(a, n);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timed = [&](auto launch) {
        launch();   // warm-up
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        CK(cudaGetLastError());
        return double(best);
    };
    const int blocks = sms * 8, threads = 256;
    const uint64_t nt = uint64_t(blocks) * threads;
    {
        const uint64_t per = 256, ops = nt * per;
        double ms = timed([&] { gather_kernel<8><<<blocks, threads>>>(a, n, per, sink); });
        printf("{\"test\": \"gather8\", \"ops\": %llu, \"ms\": %.4f, \"Gops\": %.3f, \"sector_GBps\": %.1f}\n",
               (unsigned long long)ops, ms, ops / ms / 1e6, ops * 32.0 / ms / 1e6);
        ms = timed([&] { gather_kernel<16><<<blocks, threads>>>(a, n, per, sink); });
        printf("{\"test\": \"gather16\", \"ops\": %llu, \"ms\": %.4f, \"Gops\": %.3f, \"sector_GBps\": %.1f}\n",
               (unsigned long long)ops, ms, ops / ms / 1e6, ops * 32.0 / ms / 1e6);
    }
    {
        const uint64_t hops = 64;
        for (int bl : {sms, sms * 8, sms * 32}) {
            const uint64_t ops = uint64_t(bl) * threads * hops;
            double ms = timed([&] { chase_kernel<<<bl, threads>>>(a, n, hops, sink); });
            printf("{\"test\": \"chase16\", \"threads\": %llu, \"ops\": %llu, \"ms\": %.4f, \"Gops\": %.3f, "
                   "\"ns_per_hop\": %.1f}\n",
                   (unsigned long long)(uint64_t(bl) * threads), (unsigned long long)ops, ms, ops / ms / 1e6,
                   ms * 1e6 / hops);
        }
    }
    {
        const uint64_t per = 64, ops = nt * per;
        uint64_t salt = 1;
        double ms = timed([&] { cas_kernel<8><<<blocks, threads>>>(a, n, per, salt, sink); });
        printf("{\"test\": \"cas64\", \"ops\": %llu, \"ms\": %.4f, \"Gops\": %.3f}\n", (unsigned long long)ops, ms,
               ops / ms / 1e6);
        ms = timed([&] { cas_kernel<16><<<blocks, threads>>>(a, n, per, salt, sink); });
        printf("{\"test\": \"cas128\", \"ops\": %llu, \"ms\": %.4f, \"Gops\": %.3f}\n", (unsigned long long)ops, ms,
               ops / ms / 1e6);
    }
    for (uint64_t hot : {1ull << 10, 1ull << 16}) {
        const uint64_t per = 8, ops = nt * per;
        CK(cudaMemset(sink, 0, 64));
        double ms = timed([&] { cas_hot_kernel<<<blocks, threads>>>(a, hot, per, sink); });
        uint64_t tries = 0;
        CK(cudaMemcpy(&tries, sink, 8, cudaMemcpyDeviceToHost));
        printf("{\"test\": \"cas128_hot\", \"hot_cells\": %llu, \"ops\": %llu, \"ms\": %.4f, \"Gops\": %.3f, "
               "\"tries_per_op\": %.2f}\n",
               (unsigned long long)hot, (unsigned long long)ops, ms, ops / ms / 1e6, double(tries) / (4.0 * ops));
    }
    return 0;
}
