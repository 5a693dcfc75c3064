// mtgp_multi.cu -- one process, several GPUs: the C-ABI mtgp_multi_* (include/mtgp_b200.h).
//
// Parameter-set IDs are split into contiguous balanced ranges, one per device (mtgp_multi.h,
// DESIGN.md §6); each device owns an ordinary context for its range, and every generation call
// runs one host thread per device (each thread drives its own context and stream, so devices
// generate concurrently with no collective on the hot path -- the streams are independent,
// PAPER.md:80). The only collective is the final per-stream checksum
// all-gather: NCCL (ncclCommInitAll over the devices, ncclAllGather of the padded checksum
// blocks on every device's stream, over NVLink / NVSwitch) when libnccl is loadable, else a
// host concatenation. NCCL is loaded with dlopen, so the library has no link-time dependency
// on it and a machine without NCCL still gathers.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "mtgp_ctx.h"
#include "mtgp_multi.h"

using mtgpb::set_error;

namespace {

// ---- NCCL, resolved at run time ----
struct NcclApi {
    void* handle = nullptr;
    decltype(&ncclCommInitAll) commInitAll = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    bool ok() const { return commInitAll && commDestroy && allGather && groupStart && groupEnd && errorString; }
};

const NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            a.handle = dlopen(name, RTLD_NOW | RTLD_LOCAL);
            if (a.handle) break;
        }
        if (!a.handle) return a;
        a.commInitAll = reinterpret_cast<decltype(a.commInitAll)>(dlsym(a.handle, "ncclCommInitAll"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(a.handle, "ncclCommDestroy"));
        a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(a.handle, "ncclAllGather"));
        a.groupStart = reinterpret_cast<decltype(a.groupStart)>(dlsym(a.handle, "ncclGroupStart"));
        a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(dlsym(a.handle, "ncclGroupEnd"));
        a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(a.handle, "ncclGetErrorString"));
        return a;
    }();
    return api;
}

// ncclAllGather of equal byte blocks, one rank per device, each on its context's stream
struct NcclGather final : mtgpb::GatherComm {
    std::vector<int> devs;
    std::vector<cudaStream_t> streams;
    std::vector<ncclComm_t> comms;
    std::vector<void*> d_send, d_recv;
    std::vector<size_t> cap;

    uint32_t world() const override { return (uint32_t)devs.size(); }
    const char* name() const override { return "nccl"; }

    int init(const std::vector<int>& d, const std::vector<cudaStream_t>& st) {
        const NcclApi& api = nccl_api();
        if (!api.ok()) return set_error(MTGP_ECUDA, "NCCL is not loadable");
        devs = d;
        streams = st;
        comms.assign(devs.size(), nullptr);
        d_send.assign(devs.size(), nullptr);
        d_recv.assign(devs.size(), nullptr);
        cap.assign(devs.size(), 0);
        const ncclResult_t r = api.commInitAll(comms.data(), (int)devs.size(), devs.data());
        if (r != ncclSuccess) {
            comms.clear();
            return set_error(MTGP_ECUDA, "ncclCommInitAll: %s", api.errorString(r));
        }
        return MTGP_OK;
    }

    int all_gather(const std::vector<std::vector<uint8_t>>& send, std::vector<uint8_t>& recv0) override {
        const NcclApi& api = nccl_api();
        const size_t bytes = send.empty() ? 0 : send[0].size();
        const uint32_t w = world();
        for (uint32_t r = 0; r < w; ++r) {
            cudaSetDevice(devs[r]);
            if (cap[r] < bytes) {
                cudaFree(d_send[r]);
                cudaFree(d_recv[r]);
                d_send[r] = d_recv[r] = nullptr;
                if (cudaMalloc(&d_send[r], bytes) != cudaSuccess || cudaMalloc(&d_recv[r], bytes * w) != cudaSuccess)
                    return set_error(MTGP_ENOMEM, "checksum gather buffers");
                cap[r] = bytes;
            }
            if (cudaMemcpyAsync(d_send[r], send[r].data(), bytes, cudaMemcpyHostToDevice, streams[r]) != cudaSuccess)
                return set_error(MTGP_ECUDA, "checksum gather upload");
        }
        api.groupStart();
        for (uint32_t r = 0; r < w; ++r) {
            const ncclResult_t e = api.allGather(d_send[r], d_recv[r], bytes, ncclUint8, comms[r], streams[r]);
            if (e != ncclSuccess) {
                api.groupEnd();
                return set_error(MTGP_ECUDA, "ncclAllGather: %s", api.errorString(e));
            }
        }
        const ncclResult_t e = api.groupEnd();
        if (e != ncclSuccess) return set_error(MTGP_ECUDA, "ncclGroupEnd: %s", api.errorString(e));
        recv0.resize(bytes * w);
        cudaSetDevice(devs[0]);
        if (cudaMemcpyAsync(recv0.data(), d_recv[0], bytes * w, cudaMemcpyDeviceToHost, streams[0]) != cudaSuccess)
            return set_error(MTGP_ECUDA, "checksum gather download");
        for (uint32_t r = 0; r < w; ++r) {
            cudaSetDevice(devs[r]);
            if (cudaStreamSynchronize(streams[r]) != cudaSuccess) return set_error(MTGP_ECUDA, "checksum gather sync");
        }
        return MTGP_OK;
    }

    ~NcclGather() override {
        const NcclApi& api = nccl_api();
        for (size_t r = 0; r < comms.size(); ++r)
            if (comms[r]) api.commDestroy(comms[r]);
        for (size_t r = 0; r < d_send.size(); ++r) {
            cudaSetDevice(devs[r]);
            cudaFree(d_send[r]);
            cudaFree(d_recv[r]);
        }
    }
};

// host concatenation (no NCCL, or the same device listed more than once)
struct HostGather final : mtgpb::GatherComm {
    uint32_t w = 0;
    uint32_t world() const override { return w; }
    const char* name() const override { return "host"; }
    int all_gather(const std::vector<std::vector<uint8_t>>& send, std::vector<uint8_t>& recv0) override {
        recv0.clear();
        for (const auto& b : send) recv0.insert(recv0.end(), b.begin(), b.end());
        return MTGP_OK;
    }
};

}  // namespace

struct mtgp_multi {
    std::vector<int> devices;
    std::vector<uint32_t> first, count;
    std::vector<mtgp_ctx*> ctxs;
    std::unique_ptr<mtgpb::GatherComm> comm;
    ~mtgp_multi() {
        comm.reset();
        for (mtgp_ctx* c : ctxs)
            if (c) mtgp_ctx_destroy(c);
    }
};

extern "C" {

int mtgp_shard_range(uint32_t n_sets, uint32_t world, uint32_t rank, uint32_t* first, uint32_t* count) {
    if (!first || !count || world == 0 || rank >= world) return set_error(MTGP_EINVAL, "bad shard arguments");
    mtgpb::shard_range(n_sets, world, rank, first, count);
    return MTGP_OK;
}

int mtgp_multi_create(mtgp_multi** out, const int* devices, uint32_t n_devices, const mtgp_params* sets,
                      uint32_t n_sets, const uint32_t* seeds, int gather) {
    if (!out || !devices || !sets || !seeds || n_devices == 0) return set_error(MTGP_EINVAL, "null argument");
    *out = nullptr;
    if (n_sets < n_devices) return set_error(MTGP_EINVAL, "fewer parameter sets (%u) than devices (%u)", n_sets, n_devices);
    if (gather < 0 || gather > 2) return set_error(MTGP_EINVAL, "gather must be 0 (auto), 1 (NCCL) or 2 (host)");
    auto m = std::make_unique<mtgp_multi>();
    m->devices.assign(devices, devices + n_devices);
    for (uint32_t r = 0; r < n_devices; ++r) {
        uint32_t f, c;
        mtgpb::shard_range(n_sets, n_devices, r, &f, &c);
        m->first.push_back(f);
        m->count.push_back(c);
        mtgp_ctx* ctx = nullptr;
        const int rc = mtgp_ctx_create(&ctx, devices[r], sets + f, c, seeds + f, nullptr);
        if (rc) return set_error(rc, "device %d (sets %u..%u): %s", devices[r], f, f + c - 1, mtgp_last_error());
        m->ctxs.push_back(ctx);
    }
    bool distinct = true;
    for (uint32_t a = 0; a < n_devices; ++a)
        for (uint32_t b = a + 1; b < n_devices; ++b) distinct &= devices[a] != devices[b];
    if (gather != 2 && distinct && nccl_api().ok()) {
        auto g = std::make_unique<NcclGather>();
        std::vector<cudaStream_t> st;
        for (mtgp_ctx* c : m->ctxs) st.push_back(c->stream);
        const int rc = g->init(m->devices, st);
        if (rc == MTGP_OK)
            m->comm = std::move(g);
        else if (gather == 1)
            return rc;
    } else if (gather == 1) {
        return set_error(MTGP_EINVAL, distinct ? "NCCL is not loadable" : "NCCL needs distinct devices");
    }
    if (!m->comm) {
        auto h = std::make_unique<HostGather>();
        h->w = n_devices;
        m->comm = std::move(h);
    }
    *out = m.release();
    return MTGP_OK;
}

int mtgp_multi_destroy(mtgp_multi* m) {
    delete m;
    return MTGP_OK;
}

int mtgp_multi_info(const mtgp_multi* m, uint32_t* n_devices, int* nccl) {
    if (!m) return set_error(MTGP_EINVAL, "null handle");
    if (n_devices) *n_devices = (uint32_t)m->devices.size();
    if (nccl) *nccl = std::string(m->comm->name()) == "nccl" ? 1 : 0;
    return MTGP_OK;
}

int mtgp_multi_context(mtgp_multi* m, uint32_t rank, mtgp_ctx** ctx, uint32_t* first_set, uint32_t* n_sets) {
    if (!m || !ctx) return set_error(MTGP_EINVAL, "null argument");
    if (rank >= m->ctxs.size()) return set_error(MTGP_EINVAL, "rank %u out of range", rank);
    *ctx = m->ctxs[rank];
    if (first_set) *first_set = m->first[rank];
    if (n_sets) *n_sets = m->count[rank];
    return MTGP_OK;
}

int mtgp_multi_generate(mtgp_multi* m, int kind, void* const* outs, uint64_t words_per_stream) {
    if (!m || !outs) return set_error(MTGP_EINVAL, "null argument");
    const size_t w = m->ctxs.size();
    std::vector<int> rc(w, MTGP_OK);
    std::vector<std::string> err(w);
    std::vector<std::thread> th;
    th.reserve(w);
    for (size_t r = 0; r < w; ++r)
        th.emplace_back([&, r] {  // one host thread per device: its own context, its own stream
            rc[r] = mtgp_generate(m->ctxs[r], kind, outs[r], words_per_stream, 1);
            if (rc[r] == MTGP_OK) rc[r] = mtgp_sync(m->ctxs[r]);
            if (rc[r]) err[r] = mtgp_last_error();  // thread-local: carry it to the caller's thread
        });
    for (auto& t : th) t.join();
    for (size_t r = 0; r < w; ++r)
        if (rc[r]) return set_error(rc[r], "device %d: %s", m->devices[r], err[r].c_str());
    return MTGP_OK;
}

int mtgp_multi_checksums(mtgp_multi* m, mtgp_cksum* out) {
    if (!m || !out) return set_error(MTGP_EINVAL, "null argument");
    std::vector<std::vector<mtgp_cksum>> per(m->ctxs.size());
    for (size_t r = 0; r < m->ctxs.size(); ++r) {
        per[r].resize(m->count[r]);
        const int rc = mtgp_checksums(m->ctxs[r], per[r].data());
        if (rc) return rc;
    }
    std::vector<mtgp_cksum> all;
    const int rc = mtgpb::gather_checksums(*m->comm, per, all);
    if (rc) return rc;
    std::copy(all.begin(), all.end(), out);
    return MTGP_OK;
}

}  // extern "C"
