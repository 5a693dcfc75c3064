// mtgp_mt.cu -- the reference's own generic MT engine (Engine::mt) on the B200.
//
// Reference semantics (proj/src/generator.cpp): seeding :37-52, refill :68-88, temper :7-13,
// next_u32 = temper of the refilled state in order (generator.hpp:33-36). In sequence form,
// with x_0..x_{n-1} the seeded state:
//     y       = (x_i & upper) | (x_{i+1} & lower)          upper = 0xFFFFFFFF << r
//     x_{i+n} = x_{i+m} ^ (y >> 1) ^ (y & 1 ? a : 0)
//     out_i   = temper(x_{i+n})
// Any d <= n - m consecutive new words are independent (x_{i+m} is at distance n - m), so a
// CTA per stream computes d = min(256, n - m) words per pass from a shared-memory ring of
// >= n + d words with one barrier per pass -- the block-per-stream shape of the MTGP paper,
// applied to the reference's recurrence. Tempering (u, s, t, l, b, c are per status) and the
// float conversions are fused; checksums are accumulated like the MTGP kernels.
#include "mtgp_mt.cuh"

namespace mtgpb {

template <int KIND, bool CK>
__global__ void __launch_bounds__(256) mt_v1_kernel(const DevMtParams* __restrict__ params, uint32_t* __restrict__ win,
                                                   uint32_t nmax, uint32_t ring_mask, void* __restrict__ out,
                                                   uint64_t L, DevCksum* __restrict__ ck) {
    extern __shared__ uint32_t ring[];
    __shared__ unsigned long long s_sum;
    __shared__ unsigned int s_xor;
    const uint32_t set = blockIdx.x;
    const uint32_t t = threadIdx.x;
    const DevMtParams p = params[set];
    const uint32_t n = p.n, m = p.m;
    const uint32_t upper = p.r ? (0xFFFFFFFFu << p.r) : 0xFFFFFFFFu;
    const uint32_t lower = ~upper;
    uint32_t* w = win + (size_t)set * nmax;
    for (uint32_t j = t; j < n; j += blockDim.x) ring[j] = w[j];
    if (t == 0) {
        s_sum = 0;
        s_xor = 0;
    }
    __syncthreads();
    const uint32_t d = min((uint32_t)blockDim.x, n - m);
    uint32_t* o = reinterpret_cast<uint32_t*>(out) + (size_t)set * L;
    unsigned long long sum = 0;
    uint32_t xr = 0;
    for (uint64_t base = 0; base < L; base += d) {
        const uint32_t i = (uint32_t)base + t;
        if (t < d && base + t < L) {
            const uint32_t y = (ring[i & ring_mask] & upper) | (ring[(i + 1) & ring_mask] & lower);
            const uint32_t x = ring[(i + m) & ring_mask] ^ (y >> 1) ^ ((y & 1u) ? p.a : 0u);
            ring[(i + n) & ring_mask] = x;
            uint32_t v = x;
            v ^= v >> p.u;
            v ^= (v << p.s) & p.b;
            v ^= (v << p.t) & p.c;
            v ^= v >> p.l;
            if (KIND == MTGP_F64_01) {
                // Generator::next_f64_01: u32 * 2^-32 (proj/include/twistsieve/generator.hpp:39-41)
                __stcs(reinterpret_cast<double*>(out) + (size_t)set * L + base + t, (double)v * 0x1p-32);
            } else {
                if (KIND != MTGP_U32) {
                    v = (v >> 9) | 0x3F800000u;
                    if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));
                }
                __stcs(o + base + t, v);
            }
            if (CK) {
                sum += v;
                xr ^= v;
            }
        }
        __syncthreads();
    }
    for (uint32_t j = t; j < n; j += blockDim.x) w[j] = ring[((uint32_t)L + j) & ring_mask];
    if (CK) {
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
static cudaError_t launch_mt_t(const DevMtParams* params, uint32_t* win, uint32_t n_sets, uint32_t nmax, void* out,
                               uint64_t L, DevCksum* ck, cudaStream_t st) {
    const uint32_t R = next_pow2(nmax + 256);
    const size_t smem = (size_t)R * 4;
    auto k = mt_v1_kernel<KIND, CK>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<n_sets, 256, smem, st>>>(params, win, nmax, R - 1, out, L, ck);
    return cudaGetLastError();
}

cudaError_t launch_mt_v1(int kind, bool cksum, const DevMtParams* params, uint32_t* win, uint32_t n_sets,
                         uint32_t nmax, void* out, uint64_t L, DevCksum* ck, cudaStream_t st) {
    switch (kind * 2 + (cksum ? 1 : 0)) {
        case 0: return launch_mt_t<MTGP_U32, false>(params, win, n_sets, nmax, out, L, ck, st);
        case 1: return launch_mt_t<MTGP_U32, true>(params, win, n_sets, nmax, out, L, ck, st);
        case 2: return launch_mt_t<MTGP_F32_12, false>(params, win, n_sets, nmax, out, L, ck, st);
        case 3: return launch_mt_t<MTGP_F32_12, true>(params, win, n_sets, nmax, out, L, ck, st);
        case 4: return launch_mt_t<MTGP_F32_01OC, false>(params, win, n_sets, nmax, out, L, ck, st);
        case 5: return launch_mt_t<MTGP_F32_01OC, true>(params, win, n_sets, nmax, out, L, ck, st);
        case 6: return launch_mt_t<MTGP_F64_01, false>(params, win, n_sets, nmax, out, L, ck, st);
        case 7: return launch_mt_t<MTGP_F64_01, true>(params, win, n_sets, nmax, out, L, ck, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace mtgpb
