// mtgp_v1.cu -- reference-shaped MTGP32 kernel: one CTA per parameter set.
//
// This is the straightforward block-per-stream design of the MTGP paper and of cuRAND's
// device API (curand_mtgp32_kernel.h:196-228): the CTA keeps the set's state in a
// power-of-two shared-memory ring, and each pass computes d = min(blockDim, N - pos) new words
// in parallel (any d <= N - pos consecutive words are independent), tempers
// them and stores them coalesced. One __syncthreads per pass (a ring of >= N + d words makes
// the second barrier cuRAND needs unnecessary).
//
// It is kept as the correctness baseline (MTGP_OPT_KERNEL = 1) and for small requests; the
// throughput path is mtgp_v2.cu (warp teams + jump-ahead pieces).
#include "mtgp_internal.cuh"

namespace mtgpb {

template <int KIND, bool CKSUM>
__global__ void __launch_bounds__(256) mtgp_v1_kernel(const DevParams* __restrict__ params,
                                                      uint32_t* __restrict__ win, uint32_t N,
                                                      uint32_t ring_mask, void* __restrict__ out,
                                                      uint64_t L, DevCksum* __restrict__ ck) {
    extern __shared__ uint32_t ring[];
    __shared__ uint32_t s_tbl[16], s_tmp[16];
    __shared__ unsigned long long s_sum;
    __shared__ unsigned int s_xor;

    const uint32_t set = blockIdx.x;
    const uint32_t t = threadIdx.x;
    const DevParams& p = params[set];
    const uint32_t pos = p.pos, sh1 = p.sh1, sh2 = p.sh2, mask = p.mask;
    uint32_t* w = win + (size_t)set * N;

    for (uint32_t j = t; j < N; j += blockDim.x) ring[j] = w[j];
    if (t < 16) {
        s_tbl[t] = p.tbl[t];
        s_tmp[t] = p.tmp[t];
    }
    if (t == 0) {
        s_sum = 0;
        s_xor = 0;
    }
    __syncthreads();

    const uint32_t d = min((uint32_t)blockDim.x, N - pos);
    uint32_t* o = reinterpret_cast<uint32_t*>(out) + (size_t)set * L;
    unsigned long long sum = 0;
    uint32_t xr = 0;

    for (uint64_t base = 0; base < L; base += d) {
        const uint32_t off = (uint32_t)base + t;
        if (t < d && base + t < L) {
            const uint32_t a = ring[off & ring_mask];
            const uint32_t b = ring[(off + 1) & ring_mask];
            const uint32_t c = ring[(off + pos) & ring_mask];
            uint32_t tt = ring[(off + pos - 1) & ring_mask];
            uint32_t x = (a & mask) ^ b;
            x ^= x << sh1;
            const uint32_t y = x ^ (c >> sh2);
            const uint32_t r = y ^ s_tbl[y & 15u];
            ring[(off + N) & ring_mask] = r;
            tt ^= tt >> 16;
            tt ^= tt >> 8;
            uint32_t v = r ^ s_tmp[tt & 15u];
            if (KIND == MTGP_F64_01) {
                // next_f64_01: u32 * 2^-32 (proj/include/twistsieve/generator.hpp:39-41)
                __stcs(reinterpret_cast<double*>(out) + (size_t)set * L + base + t, (double)v * 0x1p-32);
            } else {
                if (KIND != MTGP_U32) {
                    v = (v >> 9) | 0x3F800000u;
                    if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));
                }
                __stcs(o + base + t, v);
            }
            if (CKSUM) {
                sum += v;
                xr ^= v;
            }
        }
        __syncthreads();
    }

    for (uint32_t j = t; j < N; j += blockDim.x) w[j] = ring[((uint32_t)L + j) & ring_mask];

    if (CKSUM) {
        for (int sft = 16; sft > 0; sft >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, sft);
            xr ^= __shfl_xor_sync(0xffffffffu, xr, sft);
        }
        if ((t & 31) == 0) {
            atomicAdd(&s_sum, sum);
            atomicXor(&s_xor, xr);
        }
        __syncthreads();
        if (t == 0) {
            atomicAdd(&ck[set].sum64, s_sum);
            atomicXor(&ck[set].xor32, s_xor);
            atomicAdd(&ck[set].words, (unsigned long long)L);
        }
    }
}

template <int KIND, bool CK>
static cudaError_t launch_v1_t(const DevParams* params, uint32_t* win, uint32_t n_sets, uint32_t N,
                               void* out, uint64_t L, DevCksum* ck, cudaStream_t st) {
    const uint32_t R = next_pow2(N + 256);
    const size_t smem = (size_t)R * 4;
    auto k = mtgp_v1_kernel<KIND, CK>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<n_sets, 256, smem, st>>>(params, win, N, R - 1, out, L, ck);
    return cudaGetLastError();
}

cudaError_t launch_v1(int kind, bool cksum, const DevParams* params, uint32_t* win, uint32_t n_sets,
                      uint32_t N, void* out, uint64_t L, DevCksum* ck, cudaStream_t st) {
    switch (kind * 2 + (cksum ? 1 : 0)) {
        case 0: return launch_v1_t<MTGP_U32, false>(params, win, n_sets, N, out, L, ck, st);
        case 1: return launch_v1_t<MTGP_U32, true>(params, win, n_sets, N, out, L, ck, st);
        case 2: return launch_v1_t<MTGP_F32_12, false>(params, win, n_sets, N, out, L, ck, st);
        case 3: return launch_v1_t<MTGP_F32_12, true>(params, win, n_sets, N, out, L, ck, st);
        case 4: return launch_v1_t<MTGP_F32_01OC, false>(params, win, n_sets, N, out, L, ck, st);
        case 5: return launch_v1_t<MTGP_F32_01OC, true>(params, win, n_sets, N, out, L, ck, st);
        case 6: return launch_v1_t<MTGP_F64_01, false>(params, win, n_sets, N, out, L, ck, st);
        case 7: return launch_v1_t<MTGP_F64_01, true>(params, win, n_sets, N, out, L, ck, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace mtgpb
