// curand_pin.cpp -- independent MTGP32 known-answer generator. TEST INFRASTRUCTURE ONLY.
//
// Compiles NVIDIA's cuRAND MTGP32 headers host-side (no GPU; SURVEY.md Appendix B recipe) and
// prints golden vectors as JSON. cuRAND plays the role std::mt19937 plays for the reference's
// own engine (proj/tests/test_generator.cpp:17-24): an independently written implementation
// of the same published algorithm. tests/golden/make_goldens.py runs this and freezes the
// output into tests/golden/mtgp32_11213_curand.json, against which oracle/mtgp32_oracle.c
// (and through it the CUDA path) is pinned.
//
//   g++ -std=c++17 -O2 -I/usr/local/cuda/include oracle/curand_pin.cpp -o oracle/_ref/curand_pin
//
// `curand_pin --large` (stdin: parameter sets, one per line) pins the larger exponents
// (MTGP32-23209, N = 726; MTGP32-44497, N = 1391), for which cuRAND ships no tables and its
// curand() hard-codes N = 351 (MTGPDC_N). cuRAND's own N-independent pieces still define the
// algorithm: mtgp32_init_state (curand_mtgp32_host.h:155-172, sizes the state from para->mexp),
// para_rec, temper and temper_single (curand_mtgp32_kernel.h:137-183), with each set loaded
// into an mtgp32_kernel_params_t slot exactly as curandMakeMTGP32Constants does. Only the ring
// stepping -- word t of a step reads x[t], x[t+1], x[t+pos], x[t+pos-1] and writes x[t+N]
// (curand_mtgp32_kernel.h:196-228) -- is restated here with N a variable, over a 4096-word ring.
#include <cuda_runtime.h>

const dim3 blockDim(1, 1, 1);
const uint3 threadIdx = {0, 0, 0};

#include <curand_mtgp32_host.h>
#include <curand_mtgp32dc_p_11213.h>
#include <curand_mtgp32_kernel.h>

#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <vector>

static mtgp32_kernel_params_t g_k;

static void fill_kernel_params() {
    for (int i = 0; i < CURAND_NUM_MTGP32_PARAMS; ++i) {
        const mtgp32_params_fast_t& p = mtgp32dc_params_fast_11213[i];
        g_k.pos_tbl[i] = p.pos;
        g_k.sh1_tbl[i] = p.sh1;
        g_k.sh2_tbl[i] = p.sh2;
        for (int j = 0; j < 16; ++j) {
            g_k.param_tbl[i][j] = p.tbl[j];
            g_k.temper_tbl[i][j] = p.tmp_tbl[j];
            g_k.single_temper_tbl[i][j] = p.flt_tmp_tbl[j];
        }
    }
    g_k.mask[0] = mtgp32dc_params_fast_11213[0].mask;
}

struct Stream {
    curandStateMtgp32_t st;
    explicit Stream(int set, unsigned seed) {
        std::memset(&st, 0, sizeof(st));
        st.k = &g_k;
        st.pIdx = set;
        st.offset = 0;
        mtgp32_init_state(st.s, &mtgp32dc_params_fast_11213[set], seed);
    }
    unsigned next() { return curand(&st); }
    // One step through cuRAND's own para_rec + temper_single (the [1,2) float path),
    // stepping the ring exactly as curand() does.
    unsigned next_single_bits() {
        const int pos = st.k->pos_tbl[st.pIdx];
        const unsigned t = 0;
        const unsigned r = para_rec(st.k, st.s[(t + st.offset) & MTGP32_STATE_MASK],
                                    st.s[(t + st.offset + 1) & MTGP32_STATE_MASK],
                                    st.s[(t + st.offset + pos) & MTGP32_STATE_MASK], st.pIdx);
        st.s[(t + st.offset + MTGPDC_N) & MTGP32_STATE_MASK] = r;
        const unsigned o = temper_single(st.k, r, st.s[(t + st.offset + pos - 1) & MTGP32_STATE_MASK],
                                         st.pIdx);
        st.offset = (st.offset + 1) & MTGP32_STATE_MASK;
        return o;
    }
};

// ---- --large: cuRAND's init / para_rec / temper / temper_single at any N ----
static mtgp32_kernel_params_t g_large;

struct LargeStream {
    unsigned s[4096];
    unsigned n, pos, off = 0;
    int bid;
    LargeStream(const mtgp32_params_fast_t& p, int slot, unsigned seed) : n(p.mexp / 32 + 1), pos(p.pos), bid(slot) {
        std::memset(s, 0, sizeof(s));
        mtgp32_init_state(s, &p, seed);  // cuRAND's seeding, sized by p.mexp
    }
    // one step through cuRAND's para_rec; returns the new state word and its tempering helper
    unsigned rec(unsigned* helper) {
        const unsigned r = para_rec(&g_large, s[off & 4095], s[(off + 1) & 4095], s[(off + pos) & 4095], bid);
        s[(off + n) & 4095] = r;
        *helper = s[(off + pos - 1) & 4095];
        ++off;
        return r;
    }
    unsigned next() {
        unsigned t;
        const unsigned r = rec(&t);
        return temper(&g_large, r, t, bid);
    }
    unsigned next_single_bits() {
        unsigned t;
        const unsigned r = rec(&t);
        return temper_single(&g_large, r, t, bid);
    }
};

// stdin: "mexp pos sh1 sh2 mask tbl[16] tmp_tbl[16] flt_tmp_tbl[16]" per line, all sets of one
// run sharing mexp (mtgp32_kernel_params_t has a single mask); seeds and lengths are fixed below.
static int run_large() {
    std::vector<mtgp32_params_fast_t> ps;
    for (;;) {
        mtgp32_params_fast_t p;
        std::memset(&p, 0, sizeof(p));
        unsigned v[5];
        if (std::scanf("%u %u %u %u %u", &v[0], &v[1], &v[2], &v[3], &v[4]) != 5) break;
        p.mexp = (int)v[0];
        p.pos = (int)v[1];
        p.sh1 = (int)v[2];
        p.sh2 = (int)v[3];
        p.mask = v[4];
        int got = 0;
        for (int j = 0; j < 16; ++j) got += std::scanf("%u", &p.tbl[j]);
        for (int j = 0; j < 16; ++j) got += std::scanf("%u", &p.tmp_tbl[j]);
        for (int j = 0; j < 16; ++j) got += std::scanf("%u", &p.flt_tmp_tbl[j]);
        if (got != 48) return 1;
        ps.push_back(p);
    }
    if (ps.empty() || ps.size() > CURAND_NUM_MTGP32_PARAMS) return 1;
    std::memset(&g_large, 0, sizeof(g_large));
    for (size_t i = 0; i < ps.size(); ++i) {  // curandMakeMTGP32Constants' layout
        g_large.pos_tbl[i] = ps[i].pos;
        g_large.sh1_tbl[i] = ps[i].sh1;
        g_large.sh2_tbl[i] = ps[i].sh2;
        for (int j = 0; j < 16; ++j) {
            g_large.param_tbl[i][j] = ps[i].tbl[j];
            g_large.temper_tbl[i][j] = ps[i].tmp_tbl[j];
            g_large.single_temper_tbl[i][j] = ps[i].flt_tmp_tbl[j];
        }
    }
    g_large.mask[0] = ps[0].mask;
    const unsigned seeds[] = {1, 0xFFFFFFFFu, 4357};
    std::printf("{\n  \"source\": \"cuRAND %d.%d.%d mtgp32_init_state / para_rec / temper / temper_single "
                "compiled host-side, N = mexp/32+1 ring (oracle/curand_pin.cpp --large)\",\n  \"cases\": [\n",
                CURAND_VER_MAJOR, CURAND_VER_MINOR, CURAND_VER_PATCH);
    bool first = true;
    for (size_t i = 0; i < ps.size(); ++i) {
        for (unsigned seed : seeds) {
            std::printf("%s    {\"mexp\": %d, \"set\": %zu, \"seed\": %u", first ? "" : ",\n", ps[i].mexp, i, seed);
            first = false;
            {
                LargeStream g(ps[i], (int)i, seed);
                std::printf(", \"init_x0_x1_last\": [%u, %u, %u]", g.s[0], g.s[1], g.s[g.n - 1]);
                std::printf(", \"u32\": [");
                for (int k = 0; k < 32; ++k) std::printf("%s%u", k ? ", " : "", g.next());
                std::printf("]");
                // checksums of the first 2^20 words (the 32 above included)
                uint64_t sum = 0;
                uint32_t x = 0, last = 0;
                LargeStream h(ps[i], (int)i, seed);
                for (int k = 0; k < (1 << 20); ++k) {
                    const uint32_t v = h.next();
                    sum += v;
                    x ^= v;
                    last = v;
                }
                std::printf(", \"n\": %d, \"sum64\": %" PRIu64 ", \"xor32\": %u, \"last\": %u", 1 << 20, sum, x, last);
            }
            {
                LargeStream g(ps[i], (int)i, seed);
                std::printf(", \"single12_bits\": [");
                for (int k = 0; k < 32; ++k) std::printf("%s%u", k ? ", " : "", g.next_single_bits());
                std::printf("]}");
            }
        }
    }
    std::printf("\n  ]\n}\n");
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "--large") == 0) return run_large();
    fill_kernel_params();
    std::printf("{\n  \"source\": \"cuRAND %d.%d.%d MTGP32 headers compiled host-side (oracle/curand_pin.cpp)\",\n",
                CURAND_VER_MAJOR, CURAND_VER_MINOR, CURAND_VER_PATCH);

    {   // init state of set 0, seed 1
        unsigned s[MTGPDC_N];
        mtgp32_init_state(s, &mtgp32dc_params_fast_11213[0], 1);
        std::printf("  \"init_set0_seed1\": {\"x0\": %u, \"x1\": %u, \"x2\": %u, \"x3\": %u, \"x350\": %u},\n",
                    s[0], s[1], s[2], s[3], s[350]);
    }

    // first 32 words for several (set, seed) pairs
    const int sets[] = {0, 1, 2, 7, 63, 100, 199};
    const unsigned seeds[] = {1, 0, 5489, 0xFFFFFFFFu, 12345};
    std::printf("  \"first32\": [\n");
    bool first = true;
    for (int set : sets) {
        for (unsigned seed : seeds) {
            Stream g(set, seed);
            std::printf("%s    {\"set\": %d, \"seed\": %u, \"u32\": [", first ? "" : ",\n", set, seed);
            first = false;
            for (int i = 0; i < 32; ++i) std::printf("%s%u", i ? ", " : "", g.next());
            std::printf("]}");
        }
    }
    std::printf("\n  ],\n");

    // float [1,2) through cuRAND's own temper_single, first 32 of set 0 / set 5, seed 1
    std::printf("  \"single12\": [\n");
    for (int set : {0, 5}) {
        Stream g(set, 1);
        std::printf("    {\"set\": %d, \"seed\": 1, \"bits\": [", set);
        for (int i = 0; i < 32; ++i) std::printf("%s%u", i ? ", " : "", g.next_single_bits());
        std::printf("]}%s\n", set == 0 ? "," : "");
    }
    std::printf("  ],\n");

    // long-stream checksums (sum64, xor32, last, poly31) at several lengths and offsets
    struct Case { int set; unsigned seed; uint64_t skip; uint64_t n; };
    const Case cases[] = {
        {0, 1, 0, 1u << 20}, {1, 1, 0, 1u << 20}, {199, 1, 0, 1u << 20},
        {42, 7, 1000003, 1u << 18}, {150, 0xDEADBEEFu, 123456789, 4096},
    };
    std::printf("  \"checksums\": [\n");
    for (size_t c = 0; c < sizeof(cases) / sizeof(cases[0]); ++c) {
        Stream g(cases[c].set, cases[c].seed);
        for (uint64_t i = 0; i < cases[c].skip; ++i) g.next();
        uint64_t sum = 0;
        uint32_t x = 0, last = 0, h = 0;
        for (uint64_t i = 0; i < cases[c].n; ++i) {
            const uint32_t v = g.next();
            sum += v; x ^= v; last = v; h = h * 31u + v;
        }
        std::printf("    {\"set\": %d, \"seed\": %u, \"skip\": %" PRIu64 ", \"n\": %" PRIu64
                    ", \"sum64\": %" PRIu64 ", \"xor32\": %u, \"last\": %u, \"poly31\": %u}%s\n",
                    cases[c].set, cases[c].seed, cases[c].skip, cases[c].n, sum, x, last, h,
                    c + 1 < sizeof(cases) / sizeof(cases[0]) ? "," : "");
    }
    std::printf("  ],\n");

    // all 200 sets, seed 1, 2^16 words each: sum_s (s+1) * sum64_s mod 2^64, and per-set sum64
    uint64_t weighted = 0;
    std::printf("  \"all200_seed1_n65536_sum64\": [");
    for (int s = 0; s < CURAND_NUM_MTGP32_PARAMS; ++s) {
        Stream g(s, 1);
        uint64_t sum = 0;
        for (int i = 0; i < 65536; ++i) sum += g.next();
        weighted += (uint64_t)(s + 1) * sum;
        std::printf("%s%" PRIu64, s ? ", " : "", sum);
    }
    std::printf("],\n  \"all200_seed1_n65536_weighted\": %" PRIu64 "\n}\n", weighted);
    return 0;
}
