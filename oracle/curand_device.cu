// curand_device.cu -- cuRAND's own DEVICE MTGP32 on the B200: a second, on-device independent
// pin of the generation path, and the GPU-library baseline it is measured against.
// TEST / MEASUREMENT INFRASTRUCTURE ONLY (never linked into the product).
//
// besides cuRAND's headers compiled host-side (oracle/curand_pin.cpp),
// the device-API curand() kernel itself -- one curandStateMtgp32_t per thread block, 256
// threads, its 1024-word ring and two barriers per 256-word step (curand_mtgp32_kernel.h:196-228)
// -- generates the 200 certified MTGP32-11213 streams on the GPU. State setup is cuRAND's:
// curandMakeMTGP32Constants (curand_mtgp32_host.h:348-456) and curandMakeMTGP32KernelState
// (:482-510), which seeds stream i with (u32)(seed ^ (seed >> 32)) + i + 1.
//
//   curand_device words <L> <seed>   per-stream {sum64, xor32, first 8, last} of L words (JSON)
//   curand_device time <L> [reps]    Gsamples/s of the device API (state in shared / global
//                                    memory) and of the host API curandGenerate(MTGP32)
//
// Build (oracle/Makefile): nvcc -gencode arch=compute_100a,code=sm_100a -O3 ... -lcurand
#include <cuda_runtime.h>
#include <curand.h>
#include <curand_kernel.h>
#include <curand_mtgp32_host.h>
#include <curand_mtgp32dc_p_11213.h>

#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            std::exit(2);                                                                       \
        }                                                                                       \
    } while (0)
#define CR(x)                                                                     \
    do {                                                                          \
        curandStatus_t s_ = (x);                                                  \
        if (s_ != CURAND_STATUS_SUCCESS) {                                        \
            std::fprintf(stderr, "%s:%d %s: curand %d\n", __FILE__, __LINE__, #x, (int)s_); \
            std::exit(2);                                                         \
        }                                                                         \
    } while (0)

constexpr int kSets = CURAND_NUM_MTGP32_PARAMS;  // 200
constexpr int kThreads = 256;                    // curand()'s maximum block size

// Stream blockIdx.x: `steps` 256-word steps into out[blockIdx.x * L + ...], state held in
// shared memory for the call (the cuRAND documentation's recommended pattern), written back.
__global__ void __launch_bounds__(kThreads) gen_shared(curandStateMtgp32_t* st, uint32_t* out, uint64_t L,
                                                        uint64_t steps) {
    __shared__ curandStateMtgp32_t s;
    const int b = blockIdx.x;
    for (int i = threadIdx.x; i < MTGP32_STATE_SIZE; i += blockDim.x) s.s[i] = st[b].s[i];
    if (threadIdx.x == 0) {
        s.offset = st[b].offset;
        s.pIdx = st[b].pIdx;
        s.k = st[b].k;
    }
    __syncthreads();
    uint32_t* o = out + (size_t)b * L + threadIdx.x;
    for (uint64_t k = 0; k < steps; ++k) o[k * kThreads] = curand(&s);
    __syncthreads();
    for (int i = threadIdx.x; i < MTGP32_STATE_SIZE; i += blockDim.x) st[b].s[i] = s.s[i];
    if (threadIdx.x == 0) st[b].offset = s.offset;
}

// The same with the state left in global memory (the cuRAND documentation's minimal example).
__global__ void __launch_bounds__(kThreads) gen_global(curandStateMtgp32_t* st, uint32_t* out, uint64_t L,
                                                        uint64_t steps) {
    uint32_t* o = out + (size_t)blockIdx.x * L + threadIdx.x;
    for (uint64_t k = 0; k < steps; ++k) o[k * kThreads] = curand(&st[blockIdx.x]);
}

struct Dev {
    curandStateMtgp32_t* st = nullptr;
    mtgp32_kernel_params_t* kp = nullptr;
    explicit Dev(unsigned long long seed) {
        CK(cudaMalloc(&st, sizeof(curandStateMtgp32_t) * kSets));
        CK(cudaMalloc(&kp, sizeof(mtgp32_kernel_params_t)));
        CR(curandMakeMTGP32Constants(mtgp32dc_params_fast_11213, kp));
        CR(curandMakeMTGP32KernelState(st, mtgp32dc_params_fast_11213, kp, kSets, seed));
    }
    ~Dev() {
        cudaFree(st);
        cudaFree(kp);
    }
};

static int cmd_words(uint64_t L, unsigned long long seed) {
    if (L % kThreads) {
        std::fprintf(stderr, "L must be a multiple of %d\n", kThreads);
        return 1;
    }
    Dev d(seed);
    uint32_t* out = nullptr;
    CK(cudaMalloc(&out, sizeof(uint32_t) * kSets * L));
    gen_shared<<<kSets, kThreads>>>(d.st, out, L, L / kThreads);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> h((size_t)kSets * L);
    CK(cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost));
    cudaFree(out);
    std::printf("{\"generator\": \"cuRAND device API curand(curandStateMtgp32_t*), 256 threads/block, state in "
                "shared memory\", \"L\": %" PRIu64 ", \"seed\": %llu, \"streams\": [", L, seed);
    for (int s = 0; s < kSets; ++s) {
        const uint32_t* w = h.data() + (size_t)s * L;
        uint64_t sum = 0;
        uint32_t x = 0;
        for (uint64_t i = 0; i < L; ++i) {
            sum += w[i];
            x ^= w[i];
        }
        std::printf("%s{\"set\": %d, \"seed\": %u, \"sum64\": %" PRIu64 ", \"xor32\": %u, \"last\": %u, \"first\": [",
                    s ? ", " : "", s, (unsigned)(seed ^ (seed >> 32)) + s + 1, sum, x, w[L - 1]);
        for (int i = 0; i < 8; ++i) std::printf("%s%u", i ? ", " : "", w[i]);
        std::printf("]}");
    }
    std::printf("]}\n");
    return 0;
}

static double time_kernel(bool shared, Dev& d, uint32_t* out, uint64_t L, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto launch = [&] {
        if (shared)
            gen_shared<<<kSets, kThreads>>>(d.st, out, L, L / kThreads);
        else
            gen_global<<<kSets, kThreads>>>(d.st, out, L, L / kThreads);
    };
    launch();  // warm
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return (double)kSets * L * reps / (ms / 1e3) / 1e9;
}

static int cmd_time(uint64_t L, int reps) {
    Dev d(0);
    uint32_t* out = nullptr;
    CK(cudaMalloc(&out, sizeof(uint32_t) * kSets * L));
    const double g_sh = time_kernel(true, d, out, L, reps);
    const double g_gl = time_kernel(false, d, out, L / 16, reps);  // far slower: a shorter run
    // host API: the library's own MTGP32 bulk generator (its launch geometry, its ordering)
    curandGenerator_t gen;
    CR(curandCreateGenerator(&gen, CURAND_RNG_PSEUDO_MTGP32));
    CR(curandSetPseudoRandomGeneratorSeed(gen, 1));
    // the host API overflows past 2^31 outputs per call (illegal address at 200 x 2^24): the
    // same volume as chunks of 2^28 outputs into consecutive slices of the buffer
    const size_t n = (size_t)kSets * L, chunk = std::min<size_t>(n, size_t{1} << 28);
    auto host_api = [&] {
        for (size_t done = 0; done < n; done += chunk)
            CR(curandGenerate(gen, out + done, std::min(chunk, n - done)));
    };
    host_api();  // warm
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) host_api();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double g_host = (double)n * reps / (ms / 1e3) / 1e9;
    CR(curandDestroyGenerator(gen));
    cudaFree(out);
    int dev = 0;
    cudaDeviceProp prop;
    CK(cudaGetDevice(&dev));
    CK(cudaGetDeviceProperties(&prop, dev));
    std::printf("{\"device\": \"%s\", \"words_per_stream\": %" PRIu64 ", \"streams\": %d, \"reps\": %d, "
                "\"device_api_shared_state_gsamples\": %.3f, \"device_api_global_state_gsamples\": %.3f, "
                "\"host_api_curandGenerate_mtgp32_gsamples\": %.3f, \"unit\": \"Gsamples/s (u32)\"}\n",
                prop.name, L, kSets, reps, g_sh, g_gl, g_host);
    return 0;
}

int main(int argc, char** argv) {
    if (argc >= 4 && !std::strcmp(argv[1], "words"))
        return cmd_words(std::strtoull(argv[2], nullptr, 0), std::strtoull(argv[3], nullptr, 0));
    if (argc >= 3 && !std::strcmp(argv[1], "time"))
        return cmd_time(std::strtoull(argv[2], nullptr, 0), argc > 3 ? std::atoi(argv[3]) : 3);
    std::fprintf(stderr, "usage: curand_device words <L> <seed> | time <L> [reps]\n");
    return 1;
}
