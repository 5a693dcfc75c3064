// pipes.cu -- per-SM throughput of the integer instructions the MTGP kernels are built from
// (LOP3, SHF, IMAD, IMAD.HI, IMAD.WIDE, SEL, mixes). 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipes tools/pipes.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int OP>
__global__ void k(uint32_t* out, int iters, uint32_t m1, uint32_t m2) {
    uint32_t a[8];
    uint64_t w[8];
    for (int i = 0; i < 8; ++i) {
        a[i] = threadIdx.x * 131 + i * 7;
        w[i] = a[i];
    }
    const bool p = (threadIdx.x & 7) < 3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = (a[i] & m1) ^ (a[i] >> 3) ^ m2;                 // LOP3 + SHF
            if (OP == 1) a[i] = (a[i] ^ m1) & (a[i] | m2);                        // LOP3 only (2)
            if (OP == 2) a[i] = a[i] * m1 + m2;                                   // IMAD
            if (OP == 3) a[i] = __umulhi(a[i], m1) ^ m2;                           // IMAD.HI + LOP3
            if (OP == 4) w[i] = (uint64_t)a[i] * m1 + w[i], a[i] += (uint32_t)w[i];  // IMAD.WIDE
            if (OP == 5) a[i] = (p ? a[i] : m1) ^ (a[i] >> m2);                    // SEL + SHF + LOP3
            if (OP == 6) a[i] = a[i] >> m2;                                       // SHF only
        }
    }
    uint32_t r = 0;
    for (int i = 0; i < 8; ++i) r ^= a[i] ^ (uint32_t)w[i];
    if (r == 0x12345678u) out[0] = r;
}

int main() {
    uint32_t* o;
    cudaMalloc(&o, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"lop3+shf", "lop3x2", "imad", "imadhi+lop3", "imadwide+iadd", "sel+shf+lop3", "shf"};
    const int iters = 4096;
    printf("{");
    for (int op = 0; op < 7; ++op) {
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            switch (op) {
                case 0: k<0><<<sms * 8, 256>>>(o, iters, 0x5bd1e995u, 7u); break;
                case 1: k<1><<<sms * 8, 256>>>(o, iters, 0x5bd1e995u, 7u); break;
                case 2: k<2><<<sms * 8, 256>>>(o, iters, 0x5bd1e995u, 7u); break;
                case 3: k<3><<<sms * 8, 256>>>(o, iters, 0x5bd1e995u, 7u); break;
                case 4: k<4><<<sms * 8, 256>>>(o, iters, 0x5bd1e995u, 7u); break;
                case 5: k<5><<<sms * 8, 256>>>(o, iters, 0x5bd1e995u, 7u); break;
                case 6: k<6><<<sms * 8, 256>>>(o, iters, 0x5bd1e995u, 7u); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        // "iterations of one 8-chain body" per ns per SM; divide by GHz for per-clock
        const double bodies = (double)sms * 8 * 256 / 32 * iters * 8;  // warp-level chain-steps
        printf("%s\"%s\": %.3f", op ? ", " : "", names[op], bodies / (best * 1e6) / sms);
    }
    printf(", \"unit\": \"warp chain-steps per ns per SM\"}\n");
    return 0;
}
