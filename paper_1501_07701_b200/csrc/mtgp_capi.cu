// mtgp_capi.cu -- the C-ABI (include/mtgp_b200.h): contexts, validation, seeding, state
// save/restore, host<->device staging, and dispatch to the generation kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "mtgp_ctx.h"

using namespace mtgpb;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(e == cudaErrorMemoryAllocation ? MTGP_ENOMEM : MTGP_ECUDA, "%s: %s", what,
                cudaGetErrorString(e));
}

#define CK(call, what)                                    \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

// MTGP32 exponents whose state shape we support (the MTGP32 family, Saito & Matsumoto).
const uint32_t kMtgpMexp[] = {3217, 4253, 4423, 9689, 9941, 11213, 19937, 21701, 23209, 44497};

bool supported_mexp(uint32_t m) {
    for (uint32_t e : kMtgpMexp)
        if (e == m) return true;
    return false;
}

// Appendix A "Init(seed)"; external pin curand_mtgp32_host.h:155-172.
void seed_window(const mtgp_params& p, uint32_t seed, uint32_t* x) {
    const uint32_t n = state_words(p.mexp);
    const uint32_t hidden = p.tbl[4] ^ (p.tbl[8] << 16);
    uint32_t c = hidden;
    c += c >> 16;
    c += c >> 8;
    const uint32_t fillw = (c & 0xffu) * 0x01010101u;
    for (uint32_t i = 0; i < n; ++i) x[i] = fillw;
    x[0] = seed;
    x[1] = hidden;
    for (uint32_t i = 1; i < n; ++i) x[i] ^= 1812433253u * (x[i - 1] ^ (x[i - 1] >> 30)) + i;
}

}  // namespace

namespace mtgpb {
int set_error(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
int cuda_error(cudaError_t e, const char* what) { return cuda_fail(e, what); }
}  // namespace mtgpb

extern "C" {

int mtgp_abi_version(void) { return MTGP_ABI_VERSION; }
const char* mtgp_last_error(void) { return g_err.c_str(); }

int mtgp_validate_params(const mtgp_params* p) {
    if (!p) return fail(MTGP_EINVAL, "null parameter set");
    if (!supported_mexp(p->mexp)) return fail(MTGP_EINVAL, "unsupported period exponent %u", p->mexp);
    const uint32_t n = state_words(p->mexp);
    const uint32_t r = 32 * n - p->mexp;
    const uint32_t mask = r ? (0xFFFFFFFFu << r) : 0xFFFFFFFFu;
    if (p->mask != mask) return fail(MTGP_EINVAL, "mask must be 0x%08x for mexp %u", mask, p->mexp);
    if (p->sh1 < 1 || p->sh1 > 31 || p->sh2 < 1 || p->sh2 > 31)
        return fail(MTGP_EINVAL, "shifts must be in [1, 31]");
    if (p->pos < 3 || p->pos + 32 > n)
        return fail(MTGP_EINVAL, "pick-up position must satisfy 3 <= pos <= N - 32 (N=%u)", n);
    for (int i = 0; i < 16; ++i) {
        uint32_t t = 0, m = 0;
        for (int b = 0; b < 4; ++b)
            if (i & (1 << b)) {
                t ^= p->tbl[1 << b];
                m ^= p->tmp_tbl[1 << b];
            }
        if (p->tbl[i] != t || p->tmp_tbl[i] != m)
            return fail(MTGP_EINVAL, "tables must be GF(2)-linear in their index (entry %d)", i);
        if (p->flt_tmp_tbl[i] != ((p->tmp_tbl[i] >> 9) | 0x3F800000u))
            return fail(MTGP_EINVAL, "flt_tmp_tbl[%d] must equal (tmp_tbl>>9)|0x3F800000", i);
    }
    return MTGP_OK;
}

int mtgp_ctx_create(mtgp_ctx** out, int device, const mtgp_params* sets, uint32_t n_sets,
                    const uint32_t* seeds, void* stream) {
    if (!out || !sets || !seeds || n_sets == 0) return fail(MTGP_EINVAL, "null argument or n_sets == 0");
    *out = nullptr;
    for (uint32_t s = 0; s < n_sets; ++s) {
        int rc = mtgp_validate_params(&sets[s]);
        if (rc) return fail(rc, "set %u: %s", s, g_err.c_str());
        if (sets[s].mexp != sets[0].mexp) return fail(MTGP_EINVAL, "all sets of a context must share mexp");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(MTGP_ECUDA, "no CUDA device (there is no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(MTGP_EINVAL, "device %d out of range", device);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10) return fail(MTGP_ECUDA, "device %d is sm_%d%d; this library is built for sm_100a", device, prop.major, prop.minor);
    CK(cudaSetDevice(device), "cudaSetDevice");

    auto ctx = std::make_unique<mtgp_ctx>();
    ctx->device = device;
    ctx->n_sets = n_sets;
    ctx->mexp = sets[0].mexp;
    ctx->N = state_words(ctx->mexp);
    ctx->sets.assign(sets, sets + n_sets);
    ctx->position.assign(n_sets, 0);
    if (stream) {
        ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        ctx->own_stream = true;
    }
    CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&ctx->ev_gen[i], cudaEventDisableTiming), "cudaEventCreate");
        CK(cudaEventCreateWithFlags(&ctx->ev_copy[i], cudaEventDisableTiming), "cudaEventCreate");
    }

    std::vector<DevParams> dp(n_sets);
    for (uint32_t s = 0; s < n_sets; ++s) {
        dp[s].pos = sets[s].pos;
        dp[s].sh1 = sets[s].sh1;
        dp[s].sh2 = sets[s].sh2;
        dp[s].mask = sets[s].mask;
        dp[s].mul1 = 1u << sets[s].sh1;
        dp[s].mulhi2 = 1u << (32 - sets[s].sh2);
        dp[s].m16 = 1u << 16;
        dp[s].m24 = 1u << 24;
        dp[s].m23 = 1u << 23;
        dp[s].one = 1;
        dp[s].pad0 = dp[s].pad1 = 0;
        std::memcpy(dp[s].tbl, sets[s].tbl, sizeof(dp[s].tbl));
        std::memcpy(dp[s].tmp, sets[s].tmp_tbl, sizeof(dp[s].tmp));
    }
    std::vector<uint32_t> win((size_t)n_sets * ctx->N);
    for (uint32_t s = 0; s < n_sets; ++s) seed_window(sets[s], seeds[s], win.data() + (size_t)s * ctx->N);

    CK(cudaMalloc(&ctx->d_params, sizeof(DevParams) * n_sets), "cudaMalloc params");
    CK(cudaMalloc(&ctx->d_win, sizeof(uint32_t) * win.size()), "cudaMalloc state");
    CK(cudaMalloc(&ctx->d_ck, sizeof(DevCksum) * n_sets), "cudaMalloc checksums");
    CK(cudaMemcpyAsync(ctx->d_params, dp.data(), sizeof(DevParams) * n_sets, cudaMemcpyHostToDevice, ctx->stream), "upload params");
    CK(cudaMemcpyAsync(ctx->d_win, win.data(), sizeof(uint32_t) * win.size(), cudaMemcpyHostToDevice, ctx->stream), "upload state");
    CK(cudaMemsetAsync(ctx->d_ck, 0, sizeof(DevCksum) * n_sets, ctx->stream), "memset checksums");
    CK(cudaStreamSynchronize(ctx->stream), "sync");
    ctx->planner = std::make_unique<Planner>(ctx->sets, prop.multiProcessorCount);
    *out = ctx.release();
    return MTGP_OK;
}

// ---- Engine::mt (proj/src/params.cpp:23-39 validation, generator.cpp:37-52 seeding) ----
int mtgp_mt_validate_params(const mtgp_mt_params* p) {
    static const uint32_t kSupported[] = {89, 127, 521, 607, 1279, 2203, 2281, 3217, 19937, 23209};
    if (!p) return fail(MTGP_EINVAL, "null parameter set");
    if (p->n < 2) return fail(MTGP_EINVAL, "state length n must be >= 2");
    if (p->r >= 32) return fail(MTGP_EINVAL, "split position r must be < 32");
    if (32 * p->n - p->r != p->mexp) return fail(MTGP_EINVAL, "32*n - r must equal mexp");
    bool ok = false;
    for (uint32_t e : kSupported) ok = ok || e == p->mexp;
    if (!ok) return fail(MTGP_EINVAL, "unsupported period exponent %u", p->mexp);
    if (p->m < 1 || p->m >= p->n) return fail(MTGP_EINVAL, "middle offset m must satisfy 1 <= m < n");
    if ((p->a & 0xFFFFu) != p->id) return fail(MTGP_EINVAL, "low 16 bits of twist coefficient must carry the id");
    for (uint32_t sh : {p->temper_u, p->temper_s, p->temper_t, p->temper_l})
        if (sh < 1 || sh > 31) return fail(MTGP_EINVAL, "tempering shifts must be in [1, 31]");
    return MTGP_OK;
}

int mtgp_mt_ctx_create(mtgp_ctx** out, int device, const mtgp_mt_params* sets, uint32_t n_sets,
                       const uint32_t* seeds, void* stream) {
    if (!out || !sets || !seeds || n_sets == 0) return fail(MTGP_EINVAL, "null argument or n_sets == 0");
    *out = nullptr;
    uint32_t nmax = 0;
    for (uint32_t s = 0; s < n_sets; ++s) {
        int rc = mtgp_mt_validate_params(&sets[s]);
        if (rc) return fail(rc, "set %u: %s", s, g_err.c_str());
        nmax = std::max(nmax, sets[s].n);
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(MTGP_ECUDA, "no CUDA device (there is no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(MTGP_EINVAL, "device %d out of range", device);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10) return fail(MTGP_ECUDA, "device %d is sm_%d%d; this library is built for sm_100a", device, prop.major, prop.minor);
    CK(cudaSetDevice(device), "cudaSetDevice");
    auto ctx = std::make_unique<mtgp_ctx>();
    ctx->engine = 1;
    ctx->device = device;
    ctx->n_sets = n_sets;
    ctx->mexp = sets[0].mexp;
    ctx->N = nmax;
    ctx->mt_sets.assign(sets, sets + n_sets);
    ctx->position.assign(n_sets, 0);
    if (stream) {
        ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        ctx->own_stream = true;
    }
    CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&ctx->ev_gen[i], cudaEventDisableTiming), "cudaEventCreate");
        CK(cudaEventCreateWithFlags(&ctx->ev_copy[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    std::vector<DevMtParams> dp(n_sets);
    std::vector<uint32_t> win((size_t)n_sets * nmax, 0);
    for (uint32_t s = 0; s < n_sets; ++s) {
        const mtgp_mt_params& p = sets[s];
        dp[s] = DevMtParams{p.n, p.m, p.r, p.a, p.temper_b, p.temper_c, p.temper_u, p.temper_s, p.temper_t, p.temper_l,
                            1u << p.temper_s, 1u << p.temper_t};  // shifts validated in [1, 31]
        uint32_t* x = win.data() + (size_t)s * nmax;
        x[0] = seeds[s];
        for (uint32_t i = 1; i < p.n; ++i) x[i] = 1812433253u * (x[i - 1] ^ (x[i - 1] >> 30)) + i;
    }
    CK(cudaMalloc(&ctx->d_mt, sizeof(DevMtParams) * n_sets), "cudaMalloc params");
    CK(cudaMalloc(&ctx->d_win, sizeof(uint32_t) * win.size()), "cudaMalloc state");
    CK(cudaMalloc(&ctx->d_ck, sizeof(DevCksum) * n_sets), "cudaMalloc checksums");
    CK(cudaMemcpyAsync(ctx->d_mt, dp.data(), sizeof(DevMtParams) * n_sets, cudaMemcpyHostToDevice, ctx->stream), "upload params");
    CK(cudaMemcpyAsync(ctx->d_win, win.data(), sizeof(uint32_t) * win.size(), cudaMemcpyHostToDevice, ctx->stream), "upload state");
    CK(cudaMemsetAsync(ctx->d_ck, 0, sizeof(DevCksum) * n_sets, ctx->stream), "memset checksums");
    CK(cudaStreamSynchronize(ctx->stream), "sync");
    // jump-ahead pieces + warp teams when the statuses share one shape (Planner(mt_sets))
    ctx->planner = std::make_unique<Planner>(ctx->mt_sets, prop.multiProcessorCount);
    *out = ctx.release();
    return MTGP_OK;
}

int mtgp_ctx_destroy(mtgp_ctx* ctx) {
    delete ctx;  // ~mtgp_ctx releases everything (also on ctx_create's error paths)
    return MTGP_OK;
}

int mtgp_ctx_info(const mtgp_ctx* ctx, uint32_t* n_sets, uint32_t* state_words_out, uint32_t* mexp) {
    if (!ctx) return fail(MTGP_EINVAL, "null context");
    if (n_sets) *n_sets = ctx->n_sets;
    if (state_words_out) *state_words_out = ctx->N;
    if (mexp) *mexp = ctx->mexp;
    return MTGP_OK;
}

int mtgp_position(const mtgp_ctx* ctx, uint32_t s, uint64_t* words) {
    if (!ctx || !words) return fail(MTGP_EINVAL, "null argument");
    if (s >= ctx->n_sets) return fail(MTGP_EINVAL, "stream %u out of range", s);
    *words = ctx->position[s];
    return MTGP_OK;
}

int mtgp_ctx_stream(const mtgp_ctx* ctx, void** stream) {
    if (!ctx || !stream) return fail(MTGP_EINVAL, "null argument");
    *stream = ctx->stream;
    return MTGP_OK;
}

int mtgp_set_option(mtgp_ctx* ctx, int option, int64_t value) {
    if (!ctx) return fail(MTGP_EINVAL, "null context");
    switch (option) {
        case MTGP_OPT_CHECKSUM:
            if (value < 0 || value > 2) return fail(MTGP_EINVAL, "checksum must be 0 (off), 1 (sum64) or 2 (sum32)");
            ctx->cksum = value != 0;
            ctx->ck32 = value == 2;
            return MTGP_OK;
        case MTGP_OPT_KERNEL:
            if (value < 0 || value > 6) return fail(MTGP_EINVAL, "kernel must be 0 (auto) or 1 .. 6");
            ctx->kernel = (int)value;
            return MTGP_OK;
        case MTGP_OPT_MAX_PIECES:
            if (value < 0) return fail(MTGP_EINVAL, "max_pieces must be >= 0");
            ctx->max_pieces = (uint32_t)value;
            return MTGP_OK;
        case MTGP_OPT_MIN_PIECE_WORDS:
            if (value < 0) return fail(MTGP_EINVAL, "min_piece_words must be >= 0 (0 = auto)");
            ctx->min_piece_words = (uint64_t)value;
            return MTGP_OK;
        case MTGP_OPT_TIMING: ctx->timing = value != 0; return MTGP_OK;
        case MTGP_OPT_HOST_CHUNK:
            if (value < 1) return fail(MTGP_EINVAL, "host chunk must be >= 1");
            ctx->host_chunk = (uint64_t)value;
            return MTGP_OK;
        case MTGP_OPT_PREJUMP:
            if (value < 0 || value > 2) return fail(MTGP_EINVAL, "prejump must be 0 (auto), 1 (off) or 2 (on)");
            ctx->prejump = (int)value;
            return MTGP_OK;
        case MTGP_OPT_JUMP:
            if (value < 0 || value > 2) return fail(MTGP_EINVAL, "jump must be 0 (auto), 1 (direct) or 2 (split)");
            ctx->jump_mode = (int)value;
            if (ctx->planner) ctx->planner->set_jump_mode((int)value);
            return MTGP_OK;
    }
    return fail(MTGP_EINVAL, "unknown option %d", option);
}

}  // extern "C"

namespace {

int generate_device_impl(mtgp_ctx* ctx, int kind, void* out, uint64_t L);

// One device-side generation of L words per stream into device memory `out`.
int generate_device(mtgp_ctx* ctx, int kind, void* out, uint64_t L) {
    if (L == 0) return MTGP_OK;
    const int rc = generate_device_impl(ctx, kind, out, L);
    ++ctx->state_epoch;  // whatever ran (or failed half-way), the next call starts a new epoch
    return rc;
}

int generate_device_impl(mtgp_ctx* ctx, int kind, void* out, uint64_t L) {
    if (kind >= kKindBitmapBit0 && (ctx->kernel == 1 || !ctx->planner || !ctx->planner->v2_supported() ||
                                    (ctx->engine == 1 && (ctx->kernel == 5 || !ctx->planner->mt3_supported(kind, L, out)))))
        return fail(MTGP_EINVAL, "bitmap output needs the register-resident warp-team kernels");
    // Engine::mt f64 (next_f64_01) rides the teams only on the register-resident kernel's shape
    const bool mt_teams = ctx->engine == 1 && ctx->kernel != 1 && ctx->planner && ctx->planner->v2_supported() &&
                          (kind != MTGP_F64_01 || ctx->kernel == 6 ||
                           (ctx->kernel != 5 && ctx->planner->mt3_supported(kind, L, out)));
    if (ctx->engine == 1 && !mt_teams) {
        size_t e0 = 0, e1 = 0;
        if (ctx->timing) ctx->pool.record(ctx->stream, &e0);
        cudaError_t e = launch_mt_v1(kind, ctx->cksum, ctx->d_mt, ctx->d_win, ctx->n_sets, ctx->N, out, L, ctx->d_ck,
                                     ctx->stream);
        if (e != cudaSuccess) return cuda_fail(e, "Engine::mt generation kernel");
        if (ctx->timing) {
            ctx->pool.record(ctx->stream, &e1);
            ctx->pool.gen.push_back({e0, e1});
        }
        ctx->total_launches += 1;
        ctx->last_pieces = ctx->n_sets;
        ctx->last_warps = 8;
        ctx->last_kernel = 1;
        for (auto& p : ctx->position) p += L;
        return MTGP_OK;
    }
    // doubles (8 B/sample, the reference's next_f64_01) are produced by the stream-per-CTA kernel
    const bool use_v1 = !mt_teams && (ctx->kernel == 1 || !ctx->planner->v2_supported() || kind == MTGP_F64_01);
    if (use_v1) {
        size_t e0 = 0, e1 = 0;
        if (ctx->timing) ctx->pool.record(ctx->stream, &e0);
        cudaError_t e = launch_v1(kind, ctx->cksum, ctx->d_params, ctx->d_win, ctx->n_sets, ctx->N, out, L,
                                  ctx->d_ck, ctx->stream);
        if (e != cudaSuccess) return cuda_fail(e, "v1 generation kernel");
        if (ctx->timing) {
            ctx->pool.record(ctx->stream, &e1);
            ctx->pool.gen.push_back({e0, e1});
        }
        ctx->total_launches += 1;
        ctx->last_pieces = ctx->n_sets;
        ctx->last_warps = 8;
        ctx->last_kernel = 1;
    } else {
        PlanRun run;
        run.kind = kind;
        run.cksum = ctx->cksum;
        run.ck32 = ctx->ck32;
        if (ctx->cksum && ctx->ck32) ctx->ck_sum_mod32 = true;
        run.params = ctx->engine == 1 ? static_cast<const void*>(ctx->d_mt) : static_cast<const void*>(ctx->d_params);
        run.win = ctx->d_win;
        run.ck = ctx->d_ck;
        run.out = out;
        run.L = L;
        run.stream = ctx->stream;
        run.max_pieces = ctx->max_pieces;
        run.min_piece_words = ctx->min_piece_words;
        run.words_done = ctx->position.empty() ? 0 : *std::min_element(ctx->position.begin(), ctx->position.end());
        run.pred = ctx->bm_pred;
        run.timing = ctx->timing ? &ctx->pool : nullptr;
        // Engine::mt contexts: 5 / 6 pick the warp-team kernel, the MTGP kernel numbers mean auto
        run.want_kernel = ctx->engine == 1 ? (ctx->kernel >= 5 ? ctx->kernel : 0) : ctx->kernel;
        run.prejump = ctx->prejump;
        run.epoch = ctx->state_epoch;
        std::string err;
        cudaError_t e = ctx->planner->run(run, err);
        if (e != cudaSuccess) return fail(e == cudaErrorMemoryAllocation ? MTGP_ENOMEM : MTGP_ECUDA, "v2 generation: %s (%s)", err.c_str(), cudaGetErrorString(e));
        if (!err.empty()) return fail(MTGP_EINVAL, "v2 generation: %s", err.c_str());
        ctx->total_launches += run.launches;
        ctx->last_pieces = run.pieces;
        ctx->last_warps = run.warps_per_piece;
        ctx->last_kernel = (uint32_t)run.version;
    }
    for (auto& p : ctx->position) p += L;
    return MTGP_OK;
}

}  // namespace

int mtgpb::ctx_generate_device(mtgp_ctx* ctx, int kind, void* out, uint64_t L) {
    return generate_device(ctx, kind, out, L);
}

int mtgpb::ctx_generate_bitmap(mtgp_ctx* ctx, int kind, uint32_t* bitmap, uint64_t L, const BitmapPred& pred) {
    ctx->bm_pred = pred;
    return generate_device(ctx, kind, bitmap, L);
}

namespace {
int generate_impl(mtgp_ctx* ctx, int kind, void* out, uint64_t L, int out_is_device, bool wait);
}

extern "C" {

int mtgp_generate(mtgp_ctx* ctx, int kind, void* out, uint64_t L, int out_is_device) {
    return generate_impl(ctx, kind, out, L, out_is_device, true);
}

int mtgp_generate_async(mtgp_ctx* ctx, int kind, void* out, uint64_t L, int out_is_device) {
    return generate_impl(ctx, kind, out, L, out_is_device, false);
}

}  // extern "C"

namespace {
int generate_impl(mtgp_ctx* ctx, int kind, void* out, uint64_t L, int out_is_device, bool wait) {
    if (!ctx) return fail(MTGP_EINVAL, "null context");
    if (kind < MTGP_U32 || kind > MTGP_F64_01) return fail(MTGP_EINVAL, "unknown output kind %d", kind);
    if (!out && L) return fail(MTGP_EINVAL, "null output");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (out_is_device) return generate_device(ctx, kind, out, L);

    // Host output: generate chunks of Lc words per stream into a double-buffered device stage
    // and copy each chunk out with one strided 2-D copy, overlapping generation of chunk c+1
    // with the copy of chunk c.
    const size_t es = kind == MTGP_F64_01 ? 8 : 4;  // bytes per sample
    // chunk lengths are multiples of 4 (the register-resident kernels need L % 4 == 0 per call),
    // so the device path a request takes does not depend on the staging size
    uint64_t Lc = std::min<uint64_t>(L, std::max<uint64_t>(4, ctx->host_chunk & ~3ull));
    // Few streams (a GpuWordSource refill): one device call for the whole request when it is at
    // most 2^24 words, so the call can split each stream into jump-ahead pieces over many warps and
    // its plan (cached per request length) is reused refill after refill; no ramp.
    const bool single = (uint64_t)ctx->n_sets * L <= (1ull << 24) && L % 4 == 0;
    if (single) Lc = L;
    const size_t chunk_bytes = (size_t)Lc * ctx->n_sets * es;
    if (ctx->stage_bytes < 2 * chunk_bytes) {
        CK(cudaStreamSynchronize(ctx->copy_stream), "sync");
        cudaFree(ctx->d_stage);
        ctx->d_stage = nullptr;
        ctx->stage_bytes = 0;
        CK(cudaMalloc(&ctx->d_stage, 2 * chunk_bytes), "cudaMalloc stage");
        ctx->stage_bytes = 2 * chunk_bytes;
    }
    char* host = static_cast<char*>(out);
    // Chunk sizes ramp up 16x per chunk from a small first chunk: the copy engine starts after
    // ~1/64 of a chunk's generation instead of a whole one (generation outruns PCIe ~20x, so
    // the ramp never starves the copy). Lengths stay multiples of 4 words (v3 eligibility).
    uint64_t next_len = single ? Lc : std::max<uint64_t>(std::min<uint64_t>(Lc, 4096), (Lc >> 6) & ~3ull);
    for (uint64_t done = 0, len = 0; done < L; done += len) {
        len = std::min<uint64_t>(next_len, L - done);
        next_len = std::min<uint64_t>(Lc, next_len * 16);
        const int b = (int)(ctx->stage_next++ & 1);
        // halves of the stage at fixed offsets: a chunk never overlaps the other half, whose copy
        // may still be in flight from an earlier (asynchronous) call with another chunk size
        char* stage = static_cast<char*>(ctx->d_stage) + b * (ctx->stage_bytes / 2);
        // buffer b is free once its previous copy finished
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_copy[b], 0), "wait");
        int rc = generate_device(ctx, kind, stage, len);
        if (rc) return rc;
        CK(cudaEventRecord(ctx->ev_gen[b], ctx->stream), "event");
        CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_gen[b], 0), "wait");
        CK(cudaMemcpy2DAsync(host + done * es, (size_t)L * es, stage, (size_t)len * es, (size_t)len * es,
                             ctx->n_sets, cudaMemcpyDeviceToHost, ctx->copy_stream),
           "D2H copy");
        CK(cudaEventRecord(ctx->ev_copy[b], ctx->copy_stream), "event");
    }
    if (wait) CK(cudaStreamSynchronize(ctx->copy_stream), "sync");
    return MTGP_OK;
}
}  // namespace

extern "C" {

int mtgp_generate_u32(mtgp_ctx* ctx, uint32_t* out, uint64_t L, int out_is_device) {
    return mtgp_generate(ctx, MTGP_U32, out, L, out_is_device);
}
int mtgp_generate_f32_12(mtgp_ctx* ctx, float* out, uint64_t L, int out_is_device) {
    return mtgp_generate(ctx, MTGP_F32_12, out, L, out_is_device);
}
int mtgp_generate_f32_01oc(mtgp_ctx* ctx, float* out, uint64_t L, int out_is_device) {
    return mtgp_generate(ctx, MTGP_F32_01OC, out, L, out_is_device);
}

int mtgp_skip(mtgp_ctx* ctx, uint64_t words) {
    if (!ctx) return fail(MTGP_EINVAL, "null context");
    if (words == 0) return MTGP_OK;
    ++ctx->state_epoch;
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (words < 4096 || !ctx->planner || !ctx->planner->v2_supported()) {
        // Short skips (and shapes without a planner: mixed Engine::mt statuses): generate into a
        // scratch buffer in chunks; generating is cheaper than a jump for short distances.
        // The scratch is context-owned and reused: its contents are never read, and every write
        // to it is ordered on the context stream, so no synchronisation is needed between skips.
        const uint64_t chunk = std::min<uint64_t>(words, 1ull << 20);
        const size_t need = (size_t)chunk * ctx->n_sets * 4;
        if (ctx->skip_bytes < need) {
            if (ctx->d_skip) {
                cudaStreamSynchronize(ctx->stream);
                cudaFree(ctx->d_skip);
                ctx->d_skip = nullptr;
                ctx->skip_bytes = 0;
            }
            CK(cudaMalloc(&ctx->d_skip, need), "cudaMalloc skip scratch");
            ctx->skip_bytes = need;
        }
        void* scratch = ctx->d_skip;
        const bool ck = ctx->cksum;
        const int kern = ctx->kernel;
        ctx->cksum = false;
        ctx->kernel = 0;  // internal scratch generation: any kernel that takes the shape
        int rc = MTGP_OK;
        for (uint64_t done = 0; done < words && rc == MTGP_OK; done += chunk)
            rc = generate_device(ctx, MTGP_U32, scratch, std::min<uint64_t>(chunk, words - done));
        ctx->cksum = ck;
        ctx->kernel = kern;
        return rc;
    }
    std::string err;
    const void* prm = ctx->engine == 1 ? static_cast<const void*>(ctx->d_mt) : static_cast<const void*>(ctx->d_params);
    cudaError_t e = ctx->planner->skip(prm, ctx->d_win, words, ctx->stream, err);
    if (e != cudaSuccess) return fail(MTGP_ECUDA, "skip: %s (%s)", err.c_str(), cudaGetErrorString(e));
    if (!err.empty()) return fail(MTGP_EINVAL, "skip: %s", err.c_str());
    for (auto& p : ctx->position) p += words;
    return MTGP_OK;
}

int mtgp_charpoly_sha1(mtgp_ctx* ctx, char* out) {
    if (!ctx || !out) return fail(MTGP_EINVAL, "null argument");
    if (ctx->engine != 0) return fail(MTGP_EINVAL, "charpoly digests are implemented for MTGP32 contexts");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    std::vector<std::string> d;
    std::string err;
    cudaError_t e = ctx->planner->charpoly_sha1(ctx->d_params, ctx->d_win, ctx->stream, d, err);
    if (e != cudaSuccess) return cuda_fail(e, "charpoly analysis");
    if (!err.empty()) return fail(MTGP_EINVAL, "%s", err.c_str());
    for (uint32_t s = 0; s < ctx->n_sets; ++s) {
        std::memset(out + 41 * s, 0, 41);
        std::memcpy(out + 41 * s, d[s].data(), std::min<size_t>(40, d[s].size()));
    }
    return MTGP_OK;
}

int mtgp_state_save(mtgp_ctx* ctx, uint32_t* windows, uint64_t* positions) {
    if (!ctx || !windows) return fail(MTGP_EINVAL, "null argument");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(cudaMemcpyAsync(windows, ctx->d_win, (size_t)ctx->n_sets * ctx->N * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H state");
    CK(cudaStreamSynchronize(ctx->stream), "sync");
    if (positions) std::copy(ctx->position.begin(), ctx->position.end(), positions);
    return MTGP_OK;
}

int mtgp_state_restore(mtgp_ctx* ctx, const uint32_t* windows, const uint64_t* positions) {
    if (!ctx || !windows) return fail(MTGP_EINVAL, "null argument");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(cudaMemcpyAsync(ctx->d_win, windows, (size_t)ctx->n_sets * ctx->N * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D state");
    CK(cudaStreamSynchronize(ctx->stream), "sync");
    if (positions) std::copy(positions, positions + ctx->n_sets, ctx->position.begin());
    if (ctx->planner) ctx->planner->invalidate();
    ++ctx->state_epoch;
    return MTGP_OK;
}

int mtgp_checksums(mtgp_ctx* ctx, mtgp_cksum* out) {
    if (!ctx || !out) return fail(MTGP_EINVAL, "null argument");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    std::vector<DevCksum> h(ctx->n_sets);
    CK(cudaMemcpyAsync(h.data(), ctx->d_ck, sizeof(DevCksum) * ctx->n_sets, cudaMemcpyDeviceToHost, ctx->stream), "D2H checksums");
    CK(cudaStreamSynchronize(ctx->stream), "sync");
    for (uint32_t s = 0; s < ctx->n_sets; ++s) {
        out[s].sum64 = ctx->ck_sum_mod32 ? (h[s].sum64 & 0xFFFFFFFFull) : h[s].sum64;
        out[s].words = h[s].words;
        out[s].xor32 = h[s].xor32;
        out[s].pad = 0;
    }
    return MTGP_OK;
}

int mtgp_checksums_reset(mtgp_ctx* ctx) {
    if (!ctx) return fail(MTGP_EINVAL, "null context");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(cudaMemsetAsync(ctx->d_ck, 0, sizeof(DevCksum) * ctx->n_sets, ctx->stream), "memset");
    ctx->ck_sum_mod32 = false;
    return MTGP_OK;
}

int mtgp_host_alloc(size_t bytes, void** out) {
    if (!out) return fail(MTGP_EINVAL, "null output pointer");
    *out = nullptr;
    if (bytes == 0) return MTGP_OK;
    CK(cudaHostAlloc(out, bytes, cudaHostAllocPortable), "cudaHostAlloc");
    return MTGP_OK;
}

int mtgp_host_free(void* p) {
    if (p) CK(cudaFreeHost(p), "cudaFreeHost");
    return MTGP_OK;
}

int mtgp_sync(mtgp_ctx* ctx) {
    if (!ctx) return fail(MTGP_EINVAL, "null context");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(cudaStreamSynchronize(ctx->stream), "sync");
    CK(cudaStreamSynchronize(ctx->copy_stream), "sync");
    return MTGP_OK;
}

int mtgp_kernel_timing(mtgp_ctx* ctx, double* gen_ms, uint64_t* gen_launches, double* jump_ms,
                       uint64_t* jump_launches) {
    if (!ctx) return fail(MTGP_EINVAL, "null context");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(ctx->pool.resolve(&ctx->gen_ms, &ctx->gen_launches, &ctx->jump_ms, &ctx->jump_launches), "event resolve");
    if (gen_ms) *gen_ms = ctx->gen_ms;
    if (gen_launches) *gen_launches = ctx->gen_launches;
    if (jump_ms) *jump_ms = ctx->jump_ms;
    if (jump_launches) *jump_launches = ctx->jump_launches;
    return MTGP_OK;
}

int mtgp_kernel_timing_reset(mtgp_ctx* ctx) {
    if (!ctx) return fail(MTGP_EINVAL, "null context");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    double a = 0, b = 0;
    uint64_t c = 0, d = 0;
    CK(ctx->pool.resolve(&a, &c, &b, &d), "event resolve");
    ctx->gen_ms = ctx->jump_ms = 0;
    ctx->gen_launches = ctx->jump_launches = 0;
    return MTGP_OK;
}

int mtgp_launch_count(const mtgp_ctx* ctx, uint64_t* launches) {
    if (!ctx || !launches) return fail(MTGP_EINVAL, "null argument");
    *launches = ctx->total_launches;
    return MTGP_OK;
}

int mtgp_last_plan(const mtgp_ctx* ctx, uint32_t* pieces, uint32_t* warps, uint32_t* kernel_version) {
    if (!ctx) return fail(MTGP_EINVAL, "null context");
    if (pieces) *pieces = ctx->last_pieces;
    if (warps) *warps = ctx->last_warps;
    if (kernel_version) *kernel_version = ctx->last_kernel;
    return MTGP_OK;
}

}  // extern "C"
