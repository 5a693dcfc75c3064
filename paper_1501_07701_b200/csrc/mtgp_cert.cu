// mtgp_cert.cu -- parameter-set certification and the reference's charpoly digests
// ("table tooling": digest verification and a faster certifier).
//
// The reference accepts a status in its dynamic creator when the minimal polynomial probed from
// the generator has degree mexp and is irreducible (proj/src/dynamic_creator.cpp:79-81,
// gf2poly.cpp:342-383), and re-checks stored statuses by digest (verify_digest,
// dynamic_creator.cpp:99-103). Here:
//   MTGP32 contexts: the minimal polynomial is the jump planner's annihilator (Berlekamp-Massey
//     over dense word functionals of GPU-generated state words, csrc/mtgp_plan.cu);
//   Engine::mt contexts: the reference's own probe -- bit 0 of the next 2*mexp + 64 outputs,
//     generated on the GPU, then Berlekamp-Massey on the host -- digested in the reference's
//     poly_digest format, so it reproduces statuses' charpoly_digest bit for bit.
// Irreducibility: Rabin's test with PCLMUL/Barrett squaring (csrc/gf2.cpp), one host thread per
// stream. Context state and checksums are left unchanged.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gf2.h"
#include "mtgp_ctx.h"

namespace mtgpb {
namespace {

template <class F>
void for_streams(size_t n, F&& f) {
    const size_t nt = std::max<size_t>(1, std::min<size_t>(n, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    std::atomic<size_t> next{0};
    for (size_t t = 0; t < nt; ++t)
        th.emplace_back([&] {
            for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
        });
    for (auto& x : th) x.join();
}

// probe_minimal_polynomial (dynamic_creator.cpp:33-38) for every Engine::mt stream of ctx, from
// its current state; the state is restored afterwards.
int mt_probe(mtgp_ctx* ctx, std::vector<gf2::Poly>& polys) {
    const uint32_t S = ctx->n_sets;
    uint32_t max_mexp = 0;
    for (const auto& p : ctx->mt_sets) max_mexp = std::max(max_mexp, p.mexp);
    const uint64_t L = 2ull * max_mexp + 64;
    const size_t win_bytes = (size_t)S * ctx->N * 4;
    void* d_words = nullptr;
    void* d_win = nullptr;
    cudaError_t e = cudaMalloc(&d_words, (size_t)S * L * 4);
    if (e == cudaSuccess) e = cudaMalloc(&d_win, win_bytes);
    if (e != cudaSuccess) {
        cudaFree(d_words);
        return cuda_error(e, "cudaMalloc probe");
    }
    const std::vector<uint64_t> pos = ctx->position;
    const bool ck = ctx->cksum;
    cudaMemcpyAsync(d_win, ctx->d_win, win_bytes, cudaMemcpyDeviceToDevice, ctx->stream);
    ctx->cksum = false;
    int rc = ctx_generate_device(ctx, MTGP_U32, d_words, L);
    std::vector<uint32_t> h((size_t)S * L);
    if (rc == MTGP_OK) {
        e = cudaMemcpyAsync(h.data(), d_words, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) rc = cuda_error(e, "probe copy");
    }
    cudaMemcpyAsync(ctx->d_win, d_win, win_bytes, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    ++ctx->state_epoch;  // the window went back: no speculative windows apply
    ctx->position = pos;
    ctx->cksum = ck;
    cudaFree(d_words);
    cudaFree(d_win);
    if (rc != MTGP_OK) return rc;
    polys.assign(S, gf2::Poly());
    for_streams(S, [&](size_t s) {
        const size_t nbits = 2 * (size_t)ctx->mt_sets[s].mexp + 64;
        std::vector<uint64_t> bits(nbits / 64 + 1, 0);
        const uint32_t* w = h.data() + s * L;
        for (size_t k = 0; k < nbits; ++k)
            if (w[k] & 1u) bits[k >> 6] |= 1ull << (k & 63);
        polys[s] = gf2::berlekamp_massey(bits, nbits);
    });
    return MTGP_OK;
}

}  // namespace
}  // namespace mtgpb

extern "C" int mtgp_certify(mtgp_ctx* ctx, int32_t* out) {
    using namespace mtgpb;
    if (!ctx || !out) return set_error(MTGP_EINVAL, "null argument");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    if (ctx->engine == 1) {
        std::vector<gf2::Poly> polys;
        const int rc = mt_probe(ctx, polys);
        if (rc) return rc;
        for_streams(ctx->n_sets, [&](size_t s) {
            const gf2::Poly& P = polys[s];
            out[s] = P.degree() == (int)ctx->mt_sets[s].mexp && gf2::is_irreducible(P) ? 1 : 0;
        });
        return MTGP_OK;
    }
    std::vector<int> c;
    std::string err;
    e = ctx->planner->certify(ctx->d_params, ctx->d_win, ctx->stream, c, err);
    if (e != cudaSuccess) return cuda_error(e, "certify analysis");
    if (!err.empty()) return set_error(MTGP_EINVAL, "%s", err.c_str());
    for (uint32_t s = 0; s < ctx->n_sets; ++s) out[s] = c[s];
    return MTGP_OK;
}

extern "C" int mtgp_mt_charpoly_digest(mtgp_ctx* ctx, char* out) {
    using namespace mtgpb;
    if (!ctx || !out) return set_error(MTGP_EINVAL, "null argument");
    if (ctx->engine != 1) return set_error(MTGP_EINVAL, "reference-format digests are for Engine::mt contexts");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    std::vector<gf2::Poly> polys;
    const int rc = mt_probe(ctx, polys);
    if (rc) return rc;
    for (uint32_t s = 0; s < ctx->n_sets; ++s) {
        const std::string d = gf2::reference_digest(polys[s]);
        std::memset(out + 41 * s, 0, 41);
        std::memcpy(out + 41 * s, d.data(), std::min<size_t>(40, d.size()));
    }
    return MTGP_OK;
}

extern "C" int mtgp_gf2_is_irreducible(const uint8_t* coeff_bits, uint64_t n, int32_t* out) {
    using namespace mtgpb;
    if ((!coeff_bits && n) || !out) return set_error(MTGP_EINVAL, "null argument");
    gf2::Poly p;
    for (uint64_t i = 0; i < n; ++i)
        if (coeff_bits[i]) p.set((int)i);
    p.trim();
    if (p.degree() < 1) return set_error(MTGP_EINVAL, "constant polynomial");
    *out = gf2::is_irreducible(p) ? 1 : 0;
    return MTGP_OK;
}
