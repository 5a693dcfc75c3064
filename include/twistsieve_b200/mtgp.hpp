// twistsieve_b200/mtgp.hpp -- C++ drop-in for the reference's generation path, MTGP32 on B200.
//
// Mirrors the reference's C++ API shape (the reference binds its generation path in C++, not
// through an FFI):
//   ParameterizedStatus + validate()         proj/include/twistsieve/params.hpp:21-42,
//                                            proj/src/params.cpp:23-39      -> MtgpStatus
//   WordSource::fill(std::span<uint32_t>)    proj/include/twistsieve/word_source.hpp:21-25
//                                                                           -> GpuWordSource
//   make_word_source(params, seed)           word_source.hpp:75-76, word_source.cpp:5-16
//   Generator::next_u32 / next_f64_01        generator.hpp:33-41             -> GpuWordSource
//   StatusRecord / read_status_file / status_from_line / status_to_json_line
//                                            proj/include/twistsieve/status_io.hpp:13-27
//   splitmix64 / derive_seed                 word_source.cpp:18-27
// Error behaviour follows the reference: std::invalid_argument for invalid parameters or
// arguments, std::runtime_error for everything else (CUDA failures, I/O) -- translated from
// the C-ABI's status codes (include/mtgp_b200.h).
//
// WordSource: by default this header declares a WordSource with the reference's exact virtual
// interface. Define TWISTSIEVE_B200_WITH_REFERENCE before including it (and put the reference's
// include/ directory on the include path) to derive from twistsieve::WordSource itself, so a
// GpuWordSource plugs into BufferedStream and the sieve unchanged.
#pragma once

#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mtgp_b200.h"

#ifdef TWISTSIEVE_B200_WITH_REFERENCE
#include "twistsieve/word_source.hpp"
#endif

namespace twistsieve_b200 {

#ifdef TWISTSIEVE_B200_WITH_REFERENCE
using WordSource = twistsieve::WordSource;
#else
/// Campaign-facing word producer (same virtual interface as proj/include/twistsieve/word_source.hpp:21-25).
class WordSource {
public:
    virtual ~WordSource() = default;
    virtual void fill(std::span<std::uint32_t> out) = 0;
};
#endif

/// Output conversions of one MTGP32 stream.
enum class OutputKind { u32 = MTGP_U32, f32_12 = MTGP_F32_12, f32_01oc = MTGP_F32_01OC };

/// One MTGP32 parameter set -- the Engine::mtgp32 counterpart of ParameterizedStatus.
struct MtgpStatus {
    std::uint32_t id = 0;
    std::uint32_t mexp = 0;
    std::uint32_t pos = 0;
    std::uint32_t sh1 = 0;
    std::uint32_t sh2 = 0;
    std::uint32_t mask = 0;
    std::uint32_t tbl[16] = {};
    std::uint32_t tmp_tbl[16] = {};
    std::uint32_t flt_tmp_tbl[16] = {};
    std::string poly_sha1;  // hex SHA-1 of the characteristic polynomial (cuRAND table), may be empty
    bool certified = false; // full period certified by the table's authors

    std::uint32_t n() const { return mexp / 32 + 1; }
    /// Throws std::invalid_argument on any violated invariant (mtgp_validate_params).
    void validate() const;
    mtgp_params to_c() const;
    bool operator==(const MtgpStatus&) const = default;
};

/// Engine::mt status: the recurrence fields of the reference's ParameterizedStatus
/// (proj/include/twistsieve/params.hpp:21-42), generated on the GPU bit-exactly.
struct MtStatus {
    std::uint32_t id = 0;
    std::uint32_t mexp = 0;
    std::uint32_t n = 0;
    std::uint32_t m = 0;
    std::uint32_t r = 0;
    std::uint32_t a = 0;
    std::uint32_t temper_b = 0;
    std::uint32_t temper_c = 0;
    std::uint32_t temper_u = 11;
    std::uint32_t temper_s = 7;
    std::uint32_t temper_t = 15;
    std::uint32_t temper_l = 18;
    /// Throws std::invalid_argument like ParameterizedStatus::validate (params.cpp:23-39).
    void validate() const;
    mtgp_mt_params to_c() const;
    bool operator==(const MtStatus&) const = default;
};

/// The MT19937 preset (proj/src/params.cpp:63-77).
MtStatus mt19937_status();

/// Stable identifier for reports, e.g. "mtgp11213-id7" (cf. status_display_id, params.hpp:45).
std::string status_display_id(const MtgpStatus& p);

/// The 200 certified MTGP32-11213 sets shipped with the CUDA toolkit
/// (curand_mtgp32dc_p_11213.h), read from `header` or from $CUDA_HOME/include.
std::vector<MtgpStatus> curand_mtgp32_11213(const std::string& header = "");

/// Deterministic MTGP-shaped set #idx for `mexp` with UNCERTIFIED period;
/// identical to paper_1501_07701_b200.tables.synthetic_set.
MtgpStatus synthetic_status(std::uint32_t mexp, std::uint32_t idx, std::uint64_t family_seed = 0x4D544750ull);

// ---- parameter-set table file (extends proj/src/status_io.cpp:15-141) ----
struct StatusRecord {
    MtgpStatus status;
    std::optional<std::uint32_t> seed;
};
std::string status_to_json_line(const StatusRecord& rec);
StatusRecord status_from_line(const std::string& line);  // JSON or key=value; validates
std::vector<StatusRecord> read_status_file(const std::filesystem::path& path);
void write_status_file(const std::filesystem::path& path, const std::vector<StatusRecord>& records);

// ---- seeds (proj/src/word_source.cpp:18-27) ----
std::uint64_t splitmix64(std::uint64_t x);
std::uint32_t derive_seed(std::uint64_t source, std::uint32_t j);
/// cuRAND's convention (curandMakeMTGP32KernelState, curand_mtgp32_host.h:482-510): stream i is
/// seeded with (u32)(seed ^ (seed >> 32)) + i + 1.
std::vector<std::uint32_t> curand_kernel_state_seeds(std::uint64_t seed, std::uint32_t n);

/// RAII owner of a C-ABI context: many independent streams on one GPU.
class StreamBatch {
public:
    StreamBatch(const std::vector<MtgpStatus>& sets, const std::vector<std::uint32_t>& seeds, int device = 0);
    /// Engine::mt streams (the reference's classic recurrence).
    StreamBatch(const std::vector<MtStatus>& sets, const std::vector<std::uint32_t>& seeds, int device = 0);
    ~StreamBatch();
    StreamBatch(const StreamBatch&) = delete;
    StreamBatch& operator=(const StreamBatch&) = delete;
    StreamBatch(StreamBatch&&) noexcept;
    StreamBatch& operator=(StreamBatch&&) noexcept;

    std::uint32_t size() const { return n_sets_; }
    std::uint32_t state_words() const { return n_; }
    /// words_per_stream outputs of every stream into host memory out[s*L + j] (s-major).
    void generate_host(OutputKind kind, void* out, std::uint64_t words_per_stream);
    /// same into device memory (asynchronous on the context stream).
    void generate_device(OutputKind kind, void* device_out, std::uint64_t words_per_stream);
    /// generate_host without waiting (mtgp_generate_async): out is valid after synchronize().
    void generate_host_async(OutputKind kind, void* out, std::uint64_t words_per_stream);
    void skip(std::uint64_t words);
    std::uint64_t position(std::uint32_t s) const;
    std::vector<mtgp_cksum> checksums() const;
    /// Per stream: minimal polynomial (from the current state) of degree mexp and irreducible,
    /// the reference dynamic creator's acceptance test (dynamic_creator.cpp:79-81).
    std::vector<bool> certify();
    /// Engine::mt batches: the reference's poly_digest of each stream's probed minimal polynomial.
    std::vector<std::string> mt_charpoly_digests();
    void set_option(int option, std::int64_t value);
    void synchronize();
    mtgp_ctx* handle() { return ctx_; }

private:
    mtgp_ctx* ctx_ = nullptr;
    std::uint32_t n_sets_ = 0, n_ = 0;
};

/// Several GPUs in one process (C-ABI mtgp_multi): n sets split into contiguous balanced ID
/// ranges, one context and one host thread per device, no collective on the hot path, the
/// per-stream checksums all-gathered over NCCL (north_star (5)). The reference's
/// parallelism is its worker pool over independent statuses (proj/src/sieve.cpp:170-177).
class MultiGpuBatch {
public:
    enum class Gather { automatic = 0, nccl = 1, host = 2 };
    MultiGpuBatch(const std::vector<MtgpStatus>& sets, const std::vector<std::uint32_t>& seeds,
                  const std::vector<int>& devices, Gather gather = Gather::automatic);
    ~MultiGpuBatch();
    MultiGpuBatch(const MultiGpuBatch&) = delete;
    MultiGpuBatch& operator=(const MultiGpuBatch&) = delete;
    std::uint32_t devices() const { return n_dev_; }
    bool nccl() const { return nccl_; }
    /// global set IDs [first, first + count) of device slot r
    std::pair<std::uint32_t, std::uint32_t> range(std::uint32_t r) const;
    /// words_per_stream outputs of every stream; device slot r writes its streams into device
    /// memory outs[r] (per-stream contiguous). Returns when every device is done.
    void generate_device(OutputKind kind, const std::vector<void*>& outs, std::uint64_t words_per_stream);
    /// all streams' checksums in global set order (the all-gather)
    std::vector<mtgp_cksum> checksums();
    mtgp_ctx* context(std::uint32_t r);

private:
    mtgp_multi* m_ = nullptr;
    std::uint32_t n_dev_ = 0, n_sets_ = 0;
    bool nccl_ = false;
};

/// One MTGP32 stream served from device-generated chunks -- the GPU counterpart of
/// MtWordSource (word_source.hpp:27-37): fill() returns the next words of the stream exactly
/// as successive next_u32() calls would.
class GpuWordSource final : public WordSource {
public:
    /// kind != u32 makes fill() return the stream's single-float bit patterns instead.
    GpuWordSource(const MtgpStatus& params, std::uint32_t seed, OutputKind kind = OutputKind::u32,
                  int device = 0, std::size_t chunk_words = std::size_t{1} << 20);
    /// Engine::mt stream: the GPU counterpart of MtWordSource itself (word_source.hpp:27-37).
    GpuWordSource(const MtStatus& params, std::uint32_t seed, OutputKind kind = OutputKind::u32,
                  int device = 0, std::size_t chunk_words = std::size_t{1} << 20);
    ~GpuWordSource() override;
    GpuWordSource(const GpuWordSource&) = delete;
    GpuWordSource& operator=(const GpuWordSource&) = delete;
    void fill(std::span<std::uint32_t> out) override;
    std::uint32_t next_u32();
    /// next_u32() / 2^32 in [0, 1), draw for draw (generator.hpp:39-41).
    double next_f64_01() { return static_cast<double>(next_u32()) * (1.0 / 4294967296.0); }
    std::uint64_t position() const { return consumed_; }

private:
    void refill();
    StreamBatch batch_;
    OutputKind kind_;
    // two refill buffers in page-locked memory (mtgp_host_alloc): the consumer reads buf_[cur_]
    // while the next chunk is generated and copied into buf_[cur_ ^ 1] (mtgp_generate_async)
    struct PinnedFree {
        void operator()(std::uint32_t* p) const;
    };
    std::unique_ptr<std::uint32_t[], PinnedFree> buf_[2];
    int cur_ = 0;
    bool pending_ = false;  // a chunk is in flight into buf_[cur_ ^ 1]
    std::size_t cap_ = 0;
    std::size_t pos_ = 0, len_ = 0;
    std::uint64_t consumed_ = 0;
};

/// verify_digest (proj/src/dynamic_creator.cpp:99-103) on the GPU: the digest of the status's
/// minimal polynomial probed from a generator seeded with kDefaultProbeSeed (1) equals `digest`.
bool verify_digest(const MtStatus& status, const std::string& digest, int device = 0);

/// Factory with the reference's shape (word_source.cpp:5-16).
std::unique_ptr<WordSource> make_word_source(const MtgpStatus& params, std::uint32_t seed);
std::unique_ptr<WordSource> make_word_source(const MtStatus& params, std::uint32_t seed);

#ifdef TWISTSIEVE_B200_WITH_REFERENCE
/// The recurrence fields of a reference status (proj/include/twistsieve/params.hpp:21-42).
MtStatus from_reference(const twistsieve::ParameterizedStatus& p);

/// The reference's own factory signature (word_source.hpp:75-76), dispatching on
/// ParameterizedStatus::engine like proj/src/word_source.cpp:5-16, with the Engine::mt branch
/// served by the GPU: a GpuWordSource over the status's own recurrence, word for word what
/// MtWordSource would fill. The planted calibration engines (constant, lfsr16) go to the
/// reference's make_word_source unchanged. MTGP32 parameter sets have no Engine value in the
/// reference; the MtgpStatus overload above is their tag. Throws std::invalid_argument for an
/// invalid status (the reference's own ParameterizedStatus::validate), std::runtime_error when
/// no sm_100 device is usable (there is no CPU fallback). Call it qualified
/// (twistsieve_b200::make_word_source): argument-dependent lookup also finds the reference's.
std::unique_ptr<twistsieve::WordSource> make_word_source(const twistsieve::ParameterizedStatus& params,
                                                         std::uint32_t seed);
#endif

}  // namespace twistsieve_b200
