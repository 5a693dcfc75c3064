// microbench.cu -- B200 facts the MTGP32 kernel design depends on (run under gpurun).
//   1. HBM write-only peak: coalesced STG.128 grid-stride stores, and cudaMemsetAsync
//   2. MIO pipe: SHFL.IDX and LDS.128 / LDS.32 throughput per SM per clock
//   3. STG.128 with a 32-byte lane stride (a lane owning 8 consecutive words) vs contiguous,
//      and the same 8 words as one 256-bit store (sm_100)
//   4. TMA bulk stores (cp.async.bulk.global.shared::cta, 16 KB per op) from a double-buffered
//      shared-memory stage -- the store path north_star names, against direct STG.128
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));           \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__global__ void store_peak(uint4* __restrict__ p, size_t n4, uint32_t v) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n4; i += stride) __stcs(p + i, make_uint4(v, v ^ (uint32_t)i, v + 1, v + 2));
}

__global__ void store_stride32(uint4* __restrict__ p, size_t n4, uint32_t v) {
    // lane owns 8 words (32 B): two STG.128 per lane per 1 KB warp chunk
    const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t c = warp; c * 64 < n4; c += nwarps) {
        uint4* q = p + c * 64 + lane * 2;
        __stcs(q, make_uint4(v, lane, v, v));
        __stcs(q + 1, make_uint4(v, lane, v + 1, v));
    }
}

__global__ void store_256(uint4* __restrict__ p, size_t n4, uint32_t v) {
    // lane owns 8 words (32 B) as ONE 256-bit store (STG.E.EF.ENL2.256, sm_100): 1 KB per warp instr
    const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t c = warp; c * 64 < n4; c += nwarps) {
        uint4* q = p + c * 64 + lane * 2;
        asm volatile("st.global.cs.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(q), "r"(v), "r"(lane),
                     "r"(v), "r"(v), "r"(v), "r"(lane), "r"(v + 1), "r"(v)
                     : "memory");
    }
}

// Each CTA fills a 16 KB shared-memory stage (STS.128) and one thread bulk-stores it with TMA;
// two stages, so filling one overlaps the bulk store of the other.
constexpr uint32_t kTmaChunk = 16384;
__global__ void __launch_bounds__(256) store_tma(char* __restrict__ p, size_t bytes, uint32_t v) {
    extern __shared__ __align__(128) uint4 stage[];
    const size_t nch = bytes / kTmaChunk;
    uint32_t b = 0;
    for (size_t c = blockIdx.x; c < nch; c += gridDim.x, b ^= 1u) {
        uint4* s = stage + b * (kTmaChunk / 16);
        // the bulk store issued two chunks ago (same stage) must have finished reading it
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < kTmaChunk / 16; i += blockDim.x) s[i] = make_uint4(v, i, v + 1, (uint32_t)c);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t saddr = static_cast<uint32_t>(__cvta_generic_to_shared(s));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + c * kTmaChunk),
                         "r"(saddr), "r"(kTmaChunk)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void shfl_tput(uint32_t* out, int iters) {
    uint32_t a[8];
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 7 + k;
    const uint32_t tb = threadIdx.x * 0x9E3779B9u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __shfl_sync(0xffffffffu, tb, a[k] & 15, 16) ^ a[k];
    }
    uint32_t r = 0;
    for (int k = 0; k < 8; ++k) r ^= a[k];
    if (r == 0x12345678u) out[0] = r;
}

__global__ void lds128_tput(uint32_t* out, int iters) {
    __shared__ uint4 sm[1024];
    for (int j = threadIdx.x; j < 1024; j += blockDim.x) sm[j] = make_uint4(j, j + 1, j + 2, j + 3);
    __syncthreads();
    uint32_t acc[4] = {0, 0, 0, 0};
    uint32_t idx = threadIdx.x & 31;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint4 v = sm[(idx + k * 32 + (i & 7) * 128) & 1023];
            acc[k] ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if ((acc[0] ^ acc[1] ^ acc[2] ^ acc[3]) == 0x12345678u) out[0] = 1;
}

__global__ void lds32_tput(uint32_t* out, int iters) {
    __shared__ uint32_t sm[4096];
    for (int j = threadIdx.x; j < 4096; j += blockDim.x) sm[j] = j * 3;
    __syncthreads();
    uint32_t acc[8] = {0};
    uint32_t idx = threadIdx.x & 31;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] ^= sm[(idx + k * 32 + (i & 15) * 256) & 4095];
    }
    uint32_t r = 0;
    for (int k = 0; k < 8; ++k) r ^= acc[k];
    if (r == 0x12345678u) out[0] = 1;
}

int main() {
    int dev = 0;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    int clk_khz = 0;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", prop.name, prop.multiProcessorCount, clk_khz);
    const size_t bytes = 16ull << 30;  // 16 GiB
    uint4* buf;
    CK(cudaMalloc(&buf, bytes));
    uint32_t* o;
    CK(cudaMalloc(&o, 64));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float ms;
    const int sms = prop.multiProcessorCount;

    // 1. write peak
    for (int pass = 0; pass < 3; ++pass) {
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(a));
            if (pass == 0)
                store_peak<<<sms * 8, 512>>>(buf, bytes / 16, r);
            else if (pass == 1)
                store_stride32<<<sms * 8, 512>>>(buf, bytes / 16, r);
            else
                store_256<<<sms * 8, 512>>>(buf, bytes / 16, r);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            if (ms < best) best = ms;
        }
        printf(", \"%s_GBps\": %.1f", pass == 0 ? "stg128_coalesced" : pass == 1 ? "stg128_stride32" : "stg256_coalesced",
               bytes / (best * 1e6));
    }
    {
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(a));
            CK(cudaMemsetAsync(buf, r, bytes));
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            if (ms < best) best = ms;
        }
        printf(", \"memset_GBps\": %.1f", bytes / (best * 1e6));
    }
    // 4. TMA bulk stores, 2..6 CTAs (32 KB stage each) per SM
    CK(cudaFuncSetAttribute(store_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kTmaChunk));
    for (int per_sm : {2, 4, 6}) {
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(a));
            store_tma<<<sms * per_sm, 256, 2 * kTmaChunk>>>(reinterpret_cast<char*>(buf), bytes, r);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            if (ms < best) best = ms;
        }
        printf(", \"tma_bulk_store_%dcta_GBps\": %.1f", per_sm, bytes / (best * 1e6));
    }
    // 2. MIO throughput; report per-SM ops per ns (divide by GHz for per-clock)
    const int iters = 20000;
    for (int which = 0; which < 3; ++which) {
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            CK(cudaEventRecord(a));
            if (which == 0) shfl_tput<<<sms * 4, 256>>>(o, iters);
            if (which == 1) lds128_tput<<<sms * 4, 256>>>(o, iters);
            if (which == 2) lds32_tput<<<sms * 4, 256>>>(o, iters);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            if (ms < best) best = ms;
        }
        const double warp_instr = (double)sms * 4 * 8 * iters * (which == 1 ? 4 : 8);
        printf(", \"%s_warp_instr_per_ns_per_sm\": %.3f", which == 0 ? "shfl" : which == 1 ? "lds128" : "lds32",
               warp_instr / (best * 1e6) / sms);
    }
    printf("}\n");
    CK(cudaFree(buf));
    return 0;
}
