// twistsieve_b200.cpp -- implementation of include/twistsieve_b200/mtgp.hpp over the C-ABI.
#include "twistsieve_b200/mtgp.hpp"

#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>

namespace twistsieve_b200 {

namespace {

// C-ABI status -> the reference's exception types (std::invalid_argument for bad input,
// std::runtime_error otherwise; proj/src/params.cpp:23-39, proj/src/cli.cpp:429-435).
void check(int rc, const char* what) {
    if (rc == MTGP_OK) return;
    std::string msg = std::string(what) + ": " + mtgp_last_error();
    if (rc == MTGP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

constexpr std::uint32_t kMask32 = 0xFFFFFFFFu;

std::uint32_t state_mask(std::uint32_t mexp) {
    const std::uint32_t r = 32 * (mexp / 32 + 1) - mexp;
    return r ? (kMask32 << r) : kMask32;
}

void linear_tables(const std::uint32_t bt[4], const std::uint32_t bm[4], MtgpStatus& p) {
    for (int i = 0; i < 16; ++i) {
        std::uint32_t t = 0, m = 0;
        for (int b = 0; b < 4; ++b)
            if (i >> b & 1) {
                t ^= bt[b];
                m ^= bm[b];
            }
        p.tbl[i] = t;
        p.tmp_tbl[i] = m;
        p.flt_tmp_tbl[i] = (m >> 9) | 0x3F800000u;
    }
}

// ---------------- minimal flat JSON (numbers, strings, bools, arrays of numbers) ----------------
struct JVal {
    enum Kind { num, str, boolean, arr } kind = num;
    std::uint64_t n = 0;
    std::string s;
    bool b = false;
    std::vector<std::uint64_t> a;
};

struct JParser {
    const std::string& t;
    std::size_t i = 0;
    explicit JParser(const std::string& s) : t(s) {}
    [[noreturn]] void bad(const char* why) {
        throw std::invalid_argument(std::string("bad status JSON (") + why + ") at offset " + std::to_string(i));
    }
    void ws() {
        while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
    }
    char peek() {
        ws();
        return i < t.size() ? t[i] : '\0';
    }
    void expect(char c) {
        if (peek() != c) bad("unexpected character");
        ++i;
    }
    std::string str() {
        expect('"');
        std::string out;
        while (i < t.size() && t[i] != '"') {
            if (t[i] == '\\' && i + 1 < t.size()) ++i;
            out += t[i++];
        }
        if (i >= t.size()) bad("unterminated string");
        ++i;
        return out;
    }
    std::uint64_t number() {
        ws();
        std::size_t j = i;
        while (j < t.size() && (std::isdigit(static_cast<unsigned char>(t[j])))) ++j;
        if (j == i) bad("number expected");
        const std::uint64_t v = std::stoull(t.substr(i, j - i));
        i = j;
        return v;
    }
    JVal value() {
        JVal v;
        const char c = peek();
        if (c == '"') {
            v.kind = JVal::str;
            v.s = str();
        } else if (c == '[') {
            v.kind = JVal::arr;
            ++i;
            if (peek() == ']') {
                ++i;
                return v;
            }
            for (;;) {
                v.a.push_back(number());
                if (peek() == ',') {
                    ++i;
                    continue;
                }
                expect(']');
                break;
            }
        } else if (t.compare(i, 4, "true") == 0) {
            v.kind = JVal::boolean;
            v.b = true;
            i += 4;
        } else if (t.compare(i, 5, "false") == 0) {
            v.kind = JVal::boolean;
            i += 5;
        } else {
            v.n = number();
        }
        return v;
    }
    std::map<std::string, JVal> object() {
        std::map<std::string, JVal> m;
        expect('{');
        if (peek() == '}') {
            ++i;
            return m;
        }
        for (;;) {
            const std::string k = str();
            expect(':');
            m[k] = value();
            if (peek() == ',') {
                ++i;
                continue;
            }
            expect('}');
            break;
        }
        return m;
    }
};

std::uint64_t parse_uint(const std::string& v) {
    std::size_t used = 0;
    const std::uint64_t out = std::stoull(v, &used, 0);  // base 0: 0x accepted (status_io.cpp:36-41)
    if (used != v.size()) throw std::invalid_argument("bad numeric value: " + v);
    return out;
}

std::vector<std::uint64_t> parse_list(const std::string& v) {
    std::vector<std::uint64_t> out;
    std::stringstream ss(v);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(parse_uint(item));
    return out;
}

void copy16(std::uint32_t* dst, const std::vector<std::uint64_t>& src, const char* name) {
    if (src.size() != 16) throw std::invalid_argument(std::string(name) + " must have 16 entries");
    for (int i = 0; i < 16; ++i) dst[i] = static_cast<std::uint32_t>(src[i]);
}

}  // namespace

// ---------------------------------------------------------------------------------------------
void MtgpStatus::validate() const {
    const mtgp_params c = to_c();
    check(mtgp_validate_params(&c), "invalid MTGP32 status");
}

mtgp_params MtgpStatus::to_c() const {
    mtgp_params c{};
    c.mexp = mexp;
    c.pos = pos;
    c.sh1 = sh1;
    c.sh2 = sh2;
    c.mask = mask;
    std::memcpy(c.tbl, tbl, sizeof(tbl));
    std::memcpy(c.tmp_tbl, tmp_tbl, sizeof(tmp_tbl));
    std::memcpy(c.flt_tmp_tbl, flt_tmp_tbl, sizeof(flt_tmp_tbl));
    return c;
}

void MtStatus::validate() const {
    const mtgp_mt_params c = to_c();
    check(mtgp_mt_validate_params(&c), "invalid MT status");
}

mtgp_mt_params MtStatus::to_c() const {
    return mtgp_mt_params{id, mexp, n, m, r, a, temper_b, temper_c, temper_u, temper_s, temper_t, temper_l};
}

MtStatus mt19937_status() {
    MtStatus p;
    p.id = 0xB0DF;
    p.mexp = 19937;
    p.n = 624;
    p.m = 397;
    p.r = 31;
    p.a = 0x9908B0DF;
    p.temper_b = 0x9D2C5680;
    p.temper_c = 0xEFC60000;
    return p;
}

std::string status_display_id(const MtgpStatus& p) {
    return "mtgp" + std::to_string(p.mexp) + "-id" + std::to_string(p.id);
}

std::vector<MtgpStatus> curand_mtgp32_11213(const std::string& header) {
    std::string path = header;
    if (path.empty()) {
        for (const char* env : {"CUDA_HOME", "CUDA_PATH"}) {
            const char* v = std::getenv(env);
            if (v && *v) {
                path = std::string(v) + "/include/curand_mtgp32dc_p_11213.h";
                if (std::ifstream(path)) break;
                path.clear();
            }
        }
        if (path.empty()) path = "/usr/local/cuda/include/curand_mtgp32dc_p_11213.h";
    }
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    std::size_t i = text.find("mtgp32dc_params_fast_11213[]");
    if (i == std::string::npos) throw std::runtime_error("no MTGP32 table in " + path);
    // numbers of the initializer list, skipping comments (which hold "No.k delta:.. weight:..")
    std::vector<std::uint64_t> nums;
    const std::size_t end = text.find("};", i);
    i = text.find('{', i);
    while (i < end) {
        if (text.compare(i, 2, "/*") == 0) {
            i = text.find("*/", i) + 2;
            continue;
        }
        if (std::isdigit(static_cast<unsigned char>(text[i]))) {
            std::size_t used = 0;
            nums.push_back(std::stoull(text.substr(i, 24), &used, 0));
            i += used;
            continue;
        }
        ++i;
    }
    constexpr std::size_t kRec = 4 + 48 + 1 + 21;
    if (nums.size() != 200 * kRec) throw std::runtime_error("unexpected MTGP32 table layout in " + path);
    std::vector<MtgpStatus> out(200);
    for (std::size_t k = 0; k < 200; ++k) {
        const std::uint64_t* v = nums.data() + k * kRec;
        MtgpStatus& p = out[k];
        p.id = static_cast<std::uint32_t>(k);
        p.mexp = static_cast<std::uint32_t>(v[0]);
        p.pos = static_cast<std::uint32_t>(v[1]);
        p.sh1 = static_cast<std::uint32_t>(v[2]);
        p.sh2 = static_cast<std::uint32_t>(v[3]);
        for (int j = 0; j < 16; ++j) {
            p.tbl[j] = static_cast<std::uint32_t>(v[4 + j]);
            p.tmp_tbl[j] = static_cast<std::uint32_t>(v[20 + j]);
            p.flt_tmp_tbl[j] = static_cast<std::uint32_t>(v[36 + j]);
        }
        p.mask = static_cast<std::uint32_t>(v[52]);
        static const char* hex = "0123456789abcdef";
        for (int j = 0; j < 20; ++j) {
            p.poly_sha1 += hex[(v[53 + j] >> 4) & 15];
            p.poly_sha1 += hex[v[53 + j] & 15];
        }
        p.certified = true;
    }
    return out;
}

MtgpStatus synthetic_status(std::uint32_t mexp, std::uint32_t idx, std::uint64_t family_seed) {
    MtgpStatus p;
    p.id = idx;
    p.mexp = mexp;
    const std::uint32_t n = mexp / 32 + 1;
    const std::uint32_t team = mexp == 11213 ? 256 : mexp == 23209 ? 512 : mexp == 44497 ? 1024 : 256;
    std::uint64_t ctr = splitmix64(family_seed) ^ (static_cast<std::uint64_t>(mexp) << 32) ^
                        (static_cast<std::uint64_t>(idx) * 0x100000001B3ull);
    auto draw = [&] { return splitmix64(++ctr); };
    const std::uint32_t pos_max = std::max<std::uint32_t>(3, n > team ? n - team : 0);
    p.pos = 3 + static_cast<std::uint32_t>(draw() % (pos_max - 3 + 1));
    p.sh1 = 1 + static_cast<std::uint32_t>(draw() % 30);
    p.sh2 = 1 + static_cast<std::uint32_t>(draw() % 19);
    std::uint32_t bt[4], bm[4];
    for (auto& b : bt) b = static_cast<std::uint32_t>(draw() & kMask32);
    for (auto& b : bm) b = static_cast<std::uint32_t>(draw() & kMask32);
    linear_tables(bt, bm, p);
    p.mask = state_mask(mexp);
    p.certified = false;
    return p;
}

// ---------------------------------------------------------------------------------------------
std::string status_to_json_line(const StatusRecord& rec) {
    const MtgpStatus& p = rec.status;
    std::ostringstream o;
    auto arr = [&](const std::uint32_t* v) {
        o << '[';
        for (int i = 0; i < 16; ++i) o << (i ? "," : "") << v[i];
        o << ']';
    };
    o << "{\"id\":" << p.id << ",\"engine\":\"mtgp32\",\"mexp\":" << p.mexp << ",\"pos\":" << p.pos
      << ",\"sh1\":" << p.sh1 << ",\"sh2\":" << p.sh2 << ",\"mask\":" << p.mask << ",\"tbl\":";
    arr(p.tbl);
    o << ",\"tmp_tbl\":";
    arr(p.tmp_tbl);
    o << ",\"flt_tmp_tbl\":";
    arr(p.flt_tmp_tbl);
    o << ",\"poly_sha1\":\"" << p.poly_sha1 << "\",\"certified\":" << (p.certified ? "true" : "false");
    if (rec.seed) o << ",\"seed\":" << *rec.seed;
    o << '}';
    return o.str();
}

StatusRecord status_from_line(const std::string& line) {
    StatusRecord rec;
    MtgpStatus& p = rec.status;
    const auto first = line.find_first_not_of(" \t");
    bool have_flt = false, have_mask = false;
    if (first != std::string::npos && line[first] == '{') {
        JParser jp(line);
        jp.i = first;
        auto m = jp.object();
        auto need = [&](const char* k) -> JVal& {
            auto it = m.find(k);
            if (it == m.end()) throw std::invalid_argument(std::string("missing status field: ") + k);
            return it->second;
        };
        if (m.count("engine") && m["engine"].s != "mtgp32")
            throw std::invalid_argument("not an mtgp32 status: engine=" + m["engine"].s);
        p.id = m.count("id") ? static_cast<std::uint32_t>(m["id"].n) : 0;
        p.mexp = static_cast<std::uint32_t>(need("mexp").n);
        p.pos = static_cast<std::uint32_t>(need("pos").n);
        p.sh1 = static_cast<std::uint32_t>(need("sh1").n);
        p.sh2 = static_cast<std::uint32_t>(need("sh2").n);
        copy16(p.tbl, need("tbl").a, "tbl");
        copy16(p.tmp_tbl, need("tmp_tbl").a, "tmp_tbl");
        if (m.count("flt_tmp_tbl")) {
            copy16(p.flt_tmp_tbl, m["flt_tmp_tbl"].a, "flt_tmp_tbl");
            have_flt = true;
        }
        if (m.count("mask")) {
            p.mask = static_cast<std::uint32_t>(m["mask"].n);
            have_mask = true;
        }
        if (m.count("poly_sha1")) p.poly_sha1 = m["poly_sha1"].s;
        if (m.count("certified")) p.certified = m["certified"].b;
        if (m.count("seed")) rec.seed = static_cast<std::uint32_t>(m["seed"].n);
    } else {
        std::istringstream in(line);
        std::string token;
        while (in >> token) {
            const auto eq = token.find('=');
            if (eq == std::string::npos) throw std::invalid_argument("expected key=value, got: " + token);
            const std::string key = token.substr(0, eq), value = token.substr(eq + 1);
            if (key == "id") p.id = static_cast<std::uint32_t>(parse_uint(value));
            else if (key == "engine") {
                if (value != "mtgp32") throw std::invalid_argument("not an mtgp32 status: engine=" + value);
            } else if (key == "mexp") p.mexp = static_cast<std::uint32_t>(parse_uint(value));
            else if (key == "pos") p.pos = static_cast<std::uint32_t>(parse_uint(value));
            else if (key == "sh1") p.sh1 = static_cast<std::uint32_t>(parse_uint(value));
            else if (key == "sh2") p.sh2 = static_cast<std::uint32_t>(parse_uint(value));
            else if (key == "mask") {
                p.mask = static_cast<std::uint32_t>(parse_uint(value));
                have_mask = true;
            } else if (key == "tbl") copy16(p.tbl, parse_list(value), "tbl");
            else if (key == "tmp_tbl") copy16(p.tmp_tbl, parse_list(value), "tmp_tbl");
            else if (key == "flt_tmp_tbl") {
                copy16(p.flt_tmp_tbl, parse_list(value), "flt_tmp_tbl");
                have_flt = true;
            } else if (key == "poly_sha1") p.poly_sha1 = value;
            else if (key == "certified") p.certified = value == "1" || value == "true" || value == "yes";
            else if (key == "seed") rec.seed = static_cast<std::uint32_t>(parse_uint(value));
            else throw std::invalid_argument("unknown status field: " + key);
        }
    }
    if (!have_flt)
        for (int i = 0; i < 16; ++i) p.flt_tmp_tbl[i] = (p.tmp_tbl[i] >> 9) | 0x3F800000u;
    if (!have_mask) p.mask = state_mask(p.mexp);
    p.validate();
    return rec;
}

std::vector<StatusRecord> read_status_file(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open status file: " + path.string());
    std::vector<StatusRecord> out;
    std::string line;
    std::size_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        const auto first = line.find_first_not_of(" \t\r");
        if (first == std::string::npos || line[first] == '#') continue;
        try {
            out.push_back(status_from_line(line));
        } catch (const std::exception& e) {
            throw std::runtime_error(path.string() + ":" + std::to_string(lineno) + ": " + e.what());
        }
    }
    return out;
}

void write_status_file(const std::filesystem::path& path, const std::vector<StatusRecord>& records) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write status file: " + path.string());
    for (const auto& rec : records) out << status_to_json_line(rec) << '\n';
    if (!out) throw std::runtime_error("write failed: " + path.string());
}

std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

std::vector<std::uint32_t> curand_kernel_state_seeds(std::uint64_t seed, std::uint32_t n) {
    const auto base = static_cast<std::uint32_t>(seed ^ (seed >> 32));
    std::vector<std::uint32_t> out(n);
    for (std::uint32_t i = 0; i < n; ++i) out[i] = base + i + 1;
    return out;
}

std::uint32_t derive_seed(std::uint64_t source, std::uint32_t j) {
    return static_cast<std::uint32_t>(splitmix64(source + j));
}

// ---------------------------------------------------------------------------------------------
StreamBatch::StreamBatch(const std::vector<MtgpStatus>& sets, const std::vector<std::uint32_t>& seeds, int device) {
    if (sets.empty()) throw std::invalid_argument("no parameter sets");
    if (sets.size() != seeds.size()) throw std::invalid_argument("one seed per parameter set");
    std::vector<mtgp_params> c;
    c.reserve(sets.size());
    for (const auto& s : sets) c.push_back(s.to_c());
    check(mtgp_ctx_create(&ctx_, device, c.data(), static_cast<std::uint32_t>(c.size()), seeds.data(), nullptr),
          "mtgp_ctx_create");
    check(mtgp_ctx_info(ctx_, &n_sets_, &n_, nullptr), "mtgp_ctx_info");
}

StreamBatch::StreamBatch(const std::vector<MtStatus>& sets, const std::vector<std::uint32_t>& seeds, int device) {
    if (sets.empty()) throw std::invalid_argument("no parameter sets");
    if (sets.size() != seeds.size()) throw std::invalid_argument("one seed per parameter set");
    std::vector<mtgp_mt_params> c;
    c.reserve(sets.size());
    for (const auto& s : sets) c.push_back(s.to_c());
    check(mtgp_mt_ctx_create(&ctx_, device, c.data(), static_cast<std::uint32_t>(c.size()), seeds.data(), nullptr),
          "mtgp_mt_ctx_create");
    check(mtgp_ctx_info(ctx_, &n_sets_, &n_, nullptr), "mtgp_ctx_info");
}

StreamBatch::~StreamBatch() {
    if (ctx_) mtgp_ctx_destroy(ctx_);
}

StreamBatch::StreamBatch(StreamBatch&& o) noexcept : ctx_(o.ctx_), n_sets_(o.n_sets_), n_(o.n_) { o.ctx_ = nullptr; }

StreamBatch& StreamBatch::operator=(StreamBatch&& o) noexcept {
    if (this != &o) {
        if (ctx_) mtgp_ctx_destroy(ctx_);
        ctx_ = o.ctx_;
        n_sets_ = o.n_sets_;
        n_ = o.n_;
        o.ctx_ = nullptr;
    }
    return *this;
}

void StreamBatch::generate_host(OutputKind kind, void* out, std::uint64_t words) {
    check(mtgp_generate(ctx_, static_cast<int>(kind), out, words, 0), "mtgp_generate");
}

void StreamBatch::generate_host_async(OutputKind kind, void* out, std::uint64_t words) {
    check(mtgp_generate_async(ctx_, static_cast<int>(kind), out, words, 0), "mtgp_generate_async");
}

void StreamBatch::generate_device(OutputKind kind, void* out, std::uint64_t words) {
    check(mtgp_generate(ctx_, static_cast<int>(kind), out, words, 1), "mtgp_generate");
}

void StreamBatch::skip(std::uint64_t words) { check(mtgp_skip(ctx_, words), "mtgp_skip"); }

std::uint64_t StreamBatch::position(std::uint32_t s) const {
    std::uint64_t v = 0;
    check(mtgp_position(ctx_, s, &v), "mtgp_position");
    return v;
}

std::vector<bool> StreamBatch::certify() {
    std::vector<std::int32_t> c(n_sets_);
    check(mtgp_certify(ctx_, c.data()), "mtgp_certify");
    return std::vector<bool>(c.begin(), c.end());
}

std::vector<std::string> StreamBatch::mt_charpoly_digests() {
    std::vector<char> buf(41 * (size_t)n_sets_);
    check(mtgp_mt_charpoly_digest(ctx_, buf.data()), "mtgp_mt_charpoly_digest");
    std::vector<std::string> out;
    for (std::uint32_t s = 0; s < n_sets_; ++s) out.emplace_back(buf.data() + 41 * (size_t)s);
    return out;
}

bool verify_digest(const MtStatus& status, const std::string& digest, int device) {
    StreamBatch b(std::vector<MtStatus>{status}, {1u}, device);  // kDefaultProbeSeed
    return b.mt_charpoly_digests()[0] == digest;
}

std::vector<mtgp_cksum> StreamBatch::checksums() const {
    std::vector<mtgp_cksum> v(n_sets_);
    check(mtgp_checksums(ctx_, v.data()), "mtgp_checksums");
    return v;
}

void StreamBatch::set_option(int option, std::int64_t value) {
    check(mtgp_set_option(ctx_, option, value), "mtgp_set_option");
}

void StreamBatch::synchronize() { check(mtgp_sync(ctx_), "mtgp_sync"); }

// ---------------------------------------------------------------------------------------------
void GpuWordSource::PinnedFree::operator()(std::uint32_t* p) const { mtgp_host_free(p); }

namespace {
std::uint32_t* pinned_words(std::size_t n) {
    void* p = nullptr;
    check(mtgp_host_alloc(n * sizeof(std::uint32_t), &p), "mtgp_host_alloc");
    return static_cast<std::uint32_t*>(p);
}
}  // namespace

// chunk_words is rounded up to a multiple of 4: the register-resident kernels take L % 4 == 0
GpuWordSource::GpuWordSource(const MtgpStatus& params, std::uint32_t seed, OutputKind kind, int device,
                             std::size_t chunk_words)
    : batch_({params}, {seed}, device), kind_(kind), cap_((std::max<std::size_t>(chunk_words, 256) + 3) & ~std::size_t{3}) {
    buf_[0].reset(pinned_words(cap_));
    buf_[1].reset(pinned_words(cap_));
}

GpuWordSource::GpuWordSource(const MtStatus& params, std::uint32_t seed, OutputKind kind, int device,
                             std::size_t chunk_words)
    : batch_(std::vector<MtStatus>{params}, {seed}, device), kind_(kind),
      cap_((std::max<std::size_t>(chunk_words, 256) + 3) & ~std::size_t{3}) {
    buf_[0].reset(pinned_words(cap_));
    buf_[1].reset(pinned_words(cap_));
}

GpuWordSource::~GpuWordSource() {
    // a chunk may still be in flight into a buffer that is about to be freed
    if (pending_) mtgp_sync(batch_.handle());
}

// The stream's words arrive chunk by chunk: buf_[cur_] (being read), then the chunk in flight
// into buf_[cur_ ^ 1]. A refill waits for that chunk, switches to it, and starts the next one.
void GpuWordSource::refill() {
    if (!pending_) {  // first refill: nothing in flight yet
        batch_.generate_host_async(kind_, buf_[cur_ ^ 1].get(), cap_);
        pending_ = true;
    }
    batch_.synchronize();
    cur_ ^= 1;
    pos_ = 0;
    len_ = cap_;
    batch_.generate_host_async(kind_, buf_[cur_ ^ 1].get(), cap_);
}

void GpuWordSource::fill(std::span<std::uint32_t> out) {
    // every word passes through the page-locked buffers: a direct device->host copy into the
    // caller's (pageable) span is slower than the copy out of a pinned buffer
    std::size_t done = 0;
    while (done < out.size()) {
        if (pos_ == len_) refill();
        const std::size_t n = std::min(len_ - pos_, out.size() - done);
        std::memcpy(out.data() + done, buf_[cur_].get() + pos_, n * sizeof(std::uint32_t));
        pos_ += n;
        done += n;
    }
    consumed_ += out.size();
}

std::uint32_t GpuWordSource::next_u32() {
    if (pos_ == len_) refill();
    ++consumed_;
    return buf_[cur_][pos_++];
}

MultiGpuBatch::MultiGpuBatch(const std::vector<MtgpStatus>& sets, const std::vector<std::uint32_t>& seeds,
                             const std::vector<int>& devices, Gather gather) {
    if (sets.size() != seeds.size()) throw std::invalid_argument("one seed per parameter set");
    std::vector<mtgp_params> c;
    c.reserve(sets.size());
    for (const auto& s : sets) c.push_back(s.to_c());
    check(mtgp_multi_create(&m_, devices.data(), static_cast<std::uint32_t>(devices.size()), c.data(),
                            static_cast<std::uint32_t>(c.size()), seeds.data(), static_cast<int>(gather)),
          "mtgp_multi_create");
    int nccl = 0;
    check(mtgp_multi_info(m_, &n_dev_, &nccl), "mtgp_multi_info");
    nccl_ = nccl != 0;
    n_sets_ = static_cast<std::uint32_t>(sets.size());
}

MultiGpuBatch::~MultiGpuBatch() {
    if (m_) mtgp_multi_destroy(m_);
}

std::pair<std::uint32_t, std::uint32_t> MultiGpuBatch::range(std::uint32_t r) const {
    mtgp_ctx* ctx = nullptr;
    std::uint32_t f = 0, n = 0;
    check(mtgp_multi_context(m_, r, &ctx, &f, &n), "mtgp_multi_context");
    return {f, n};
}

mtgp_ctx* MultiGpuBatch::context(std::uint32_t r) {
    mtgp_ctx* ctx = nullptr;
    check(mtgp_multi_context(m_, r, &ctx, nullptr, nullptr), "mtgp_multi_context");
    return ctx;
}

void MultiGpuBatch::generate_device(OutputKind kind, const std::vector<void*>& outs, std::uint64_t words_per_stream) {
    if (outs.size() != n_dev_) throw std::invalid_argument("one output buffer per device");
    check(mtgp_multi_generate(m_, static_cast<int>(kind), outs.data(), words_per_stream), "mtgp_multi_generate");
}

std::vector<mtgp_cksum> MultiGpuBatch::checksums() {
    std::vector<mtgp_cksum> out(n_sets_);
    check(mtgp_multi_checksums(m_, out.data()), "mtgp_multi_checksums");
    return out;
}

std::unique_ptr<WordSource> make_word_source(const MtgpStatus& params, std::uint32_t seed) {
    return std::make_unique<GpuWordSource>(params, seed);
}

std::unique_ptr<WordSource> make_word_source(const MtStatus& params, std::uint32_t seed) {
    return std::make_unique<GpuWordSource>(params, seed);
}

#ifdef TWISTSIEVE_B200_WITH_REFERENCE
MtStatus from_reference(const twistsieve::ParameterizedStatus& p) {
    MtStatus s;
    s.id = p.id;
    s.mexp = p.mexp;
    s.n = p.n;
    s.m = p.m;
    s.r = p.r;
    s.a = p.a;
    s.temper_b = p.temper_b;
    s.temper_c = p.temper_c;
    s.temper_u = p.temper_u;
    s.temper_s = p.temper_s;
    s.temper_t = p.temper_t;
    s.temper_l = p.temper_l;
    return s;
}

std::unique_ptr<twistsieve::WordSource> make_word_source(const twistsieve::ParameterizedStatus& params,
                                                         std::uint32_t seed) {
    if (params.engine != twistsieve::Engine::mt) return twistsieve::make_word_source(params, seed);
    params.validate();  // the reference's own invariants and messages (proj/src/params.cpp:23-39)
    return std::make_unique<GpuWordSource>(from_reference(params), seed);
}
#endif

}  // namespace twistsieve_b200
