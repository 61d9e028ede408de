// SPDX-License-Identifier: Apache-2.0
// DeviceContext: binds a rank to its GPU and to its peers' memory, bootstrapped over the
// reference's Transport (control plane only). See gflow/device.hpp.
#include "gflow/device.hpp"

#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>

#include "gflow/errors.hpp"

namespace gflow {

void check(int status, const char* what) {
    if (status == GF_OK) return;
    std::string msg = std::string(what ? what : "gflow_b200") + ": " + gf_last_error();
    switch (status) {
        case GF_ERR_CONFIG: throw ConfigError(msg);
        case GF_ERR_PROTOCOL: throw ProtocolError(msg);
        case GF_ERR_TRAINING: throw TrainingError(msg);
        default: throw TransportError(msg);  // transport + CUDA failures
    }
}

namespace {

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw TransportError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Hello {
    std::int64_t pid;
    std::int32_t device;      // chosen device of the sender
    std::int32_t device_count;
};

template <typename T>
std::vector<std::byte> pod_bytes(const T& v) {
    std::vector<std::byte> b(sizeof(T));
    std::memcpy(b.data(), &v, sizeof(T));
    return b;
}
template <typename T>
T from_pod(const std::vector<std::byte>& b) {
    if (b.size() != sizeof(T)) throw ProtocolError("device bootstrap: malformed control message");
    T v;
    std::memcpy(&v, b.data(), sizeof(T));
    return v;
}

// All-to-all of one fixed-size record through the control plane.
template <typename T>
std::vector<T> allgather(Transport& tp, const T& mine, std::uint32_t tag) {
    const int n = tp.world_size(), r = tp.rank();
    std::vector<T> all(static_cast<std::size_t>(n));
    all[static_cast<std::size_t>(r)] = mine;
    const auto bytes = pod_bytes(mine);
    for (int q = 0; q < n; ++q)
        if (q != r) tp.control_send(q, tag, bytes);
    for (int q = 0; q < n; ++q)
        if (q != r) all[static_cast<std::size_t>(q)] = from_pod<T>(tp.control_recv(q, tag));
    return all;
}

constexpr std::uint32_t kBootTag = 0xFFF00000u;

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

// ---- colocated ranks: one launch per collective over every rank's buffer ------------------
struct ColocatedGroup {
    explicit ColocatedGroup(int w) : world(w), slots(static_cast<std::size_t>(w), nullptr) {}
    int world;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<void*> slots;
    int arrived = 0;
    std::uint64_t generation = 0;
    int status = GF_OK;
    std::string error;

    // Every rank deposits its pointer; the last one runs `fn(slots)` for all of them.
    template <typename F>
    void run(int rank, void* ptr, std::chrono::milliseconds timeout, F&& fn) {
        std::unique_lock lock(mu);
        slots[static_cast<std::size_t>(rank)] = ptr;
        const std::uint64_t mine = generation;
        if (++arrived == world) {
            status = GF_OK;
            try {
                fn(slots);
            } catch (const std::exception& e) {
                status = GF_ERR_TRANSPORT;
                error = e.what();
            }
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else if (!cv.wait_for(lock, timeout, [&] { return generation != mine; })) {
            throw TransportError("colocated collective timed out at rank " + std::to_string(rank) +
                                 " (a rank never reached it)");
        }
        if (status != GF_OK) throw TransportError(error);
    }
};

namespace {
std::mutex g_groups_mu;
std::map<std::uintptr_t, std::shared_ptr<ColocatedGroup>> g_groups;
}  // namespace

DeviceContext::DeviceContext(Transport& tp, int device) : tp_(tp), rank_(tp.rank()), world_(tp.world_size()) {
    int count = 0;
    cuda_ok(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    int cur = 0;
    cuda_ok(cudaGetDevice(&cur), "cudaGetDevice");
    device_ = device >= 0 ? device : cur;
    if (device_ >= count) throw ConfigError("device " + std::to_string(device_) + " not present");
    Hello me{static_cast<std::int64_t>(::getpid()), device_, count};
    const auto all = allgather(tp_, me, kBootTag | 1u);
    bool same_proc = true, all_same_dev = true, distinct = true;
    for (int r = 0; r < world_; ++r) {
        same_proc &= all[r].pid == me.pid;
        all_same_dev &= all[r].device == all[0].device;
        for (int q = 0; q < r; ++q) distinct &= all[q].device != all[r].device;
    }
    if (world_ == 1) {
        mode_ = Mode::kSolo;
    } else if (same_proc && distinct) {
        mode_ = Mode::kLocal;
    } else if (same_proc && all_same_dev) {
        mode_ = Mode::kColocated;
    } else if (!same_proc && distinct) {
        mode_ = Mode::kIpc;
    } else {
        throw ConfigError("unsupported rank placement: ranks must each own a distinct GPU, or (in one "
                          "process) all share one GPU");
    }
    DeviceGuard g(device_);
    cudaStream_t st = nullptr;
    cuda_ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreateWithFlags");
    stream_ = st;
    cudaEvent_t e1 = nullptr, e2 = nullptr;
    cuda_ok(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming), "event");
    cuda_ok(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming), "event");
    ev_client_ = e1;
    ev_done_ = e2;
    if (mode_ == Mode::kColocated) {
        std::uintptr_t key = 0;
        if (rank_ == 0) {
            auto grp = std::make_shared<ColocatedGroup>(world_);
            key = reinterpret_cast<std::uintptr_t>(grp.get());
            std::lock_guard lk(g_groups_mu);
            g_groups[key] = grp;
        }
        const auto keys = allgather(tp_, key, kBootTag | 2u);
        std::lock_guard lk(g_groups_mu);
        group_ = g_groups.at(keys[0]);
        return;
    }
    check(gf_comm_create(world_, rank_, device_, 0, &comm_), "gf_comm_create");
    check(gf_comm_set_timeout_ms(comm_, static_cast<std::uint64_t>(tp_.timeout().count())), "timeout");
    if (mode_ == Mode::kLocal) {
        const auto comms = allgather(tp_, reinterpret_cast<std::uintptr_t>(comm_), kBootTag | 3u);
        if (rank_ == 0) {
            std::vector<gf_comm*> cs;
            for (auto c : comms) cs.push_back(reinterpret_cast<gf_comm*>(c));
            check(gf_comm_connect_local(cs.data(), world_), "gf_comm_connect_local");
        }
        // nobody launches before rank 0 connected every comm
        allgather(tp_, std::uint8_t{1}, kBootTag | 4u);
    } else if (mode_ == Mode::kIpc) {
        struct H {
            char b[GF_IPC_HANDLE_BYTES];
        } h;
        check(gf_comm_export_handle(comm_, h.b), "gf_comm_export_handle");
        const auto hs = allgather(tp_, h, kBootTag | 5u);
        std::vector<char> flat(static_cast<std::size_t>(world_) * GF_IPC_HANDLE_BYTES);
        for (int r = 0; r < world_; ++r) std::memcpy(flat.data() + r * GF_IPC_HANDLE_BYTES, hs[r].b, GF_IPC_HANDLE_BYTES);
        check(gf_comm_connect_ipc(comm_, flat.data()), "gf_comm_connect_ipc");
    }
}

DeviceContext::~DeviceContext() {
    DeviceGuard g(device_);
    cudaDeviceSynchronize();
    for (auto& [k, base] : ipc_cache_) gf_ipc_close(comm_, base);
    for (auto& s : scratch_) cudaFree(s.first);
    if (comm_) gf_comm_destroy(comm_);
    if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
    if (ev_client_) cudaEventDestroy(static_cast<cudaEvent_t>(ev_client_));
    if (ev_done_) cudaEventDestroy(static_cast<cudaEvent_t>(ev_done_));
    if (group_) {
        std::lock_guard lk(g_groups_mu);
        for (auto it = g_groups.begin(); it != g_groups.end(); ++it) {
            if (it->second == group_ && it->second.use_count() <= 2) {
                g_groups.erase(it);
                break;
            }
        }
    }
}

const char* DeviceContext::mode_name() const {
    switch (mode_) {
        case Mode::kSolo: return "solo";
        case Mode::kLocal: return "local-p2p";
        case Mode::kIpc: return "ipc-p2p";
        case Mode::kColocated: return "colocated";
    }
    return "?";
}

void DeviceContext::activate() const { cudaSetDevice(device_); }

void* DeviceContext::scratch(std::size_t bytes, int slot) {
    std::lock_guard lk(mu_);
    if (scratch_.size() <= static_cast<std::size_t>(slot)) scratch_.resize(static_cast<std::size_t>(slot) + 1, {nullptr, 0});
    auto& s = scratch_[static_cast<std::size_t>(slot)];
    if (s.second < bytes) {
        DeviceGuard g(device_);
        if (s.first) cudaFree(s.first);
        s.first = nullptr;
        cuda_ok(cudaMalloc(&s.first, std::max<std::size_t>(bytes, 256)), "cudaMalloc scratch");
        s.second = std::max<std::size_t>(bytes, 256);
    }
    return s.first;
}

std::vector<void*> DeviceContext::exchange(void* mine, std::uint32_t tag, std::uint64_t agree) {
    if (mode_ == Mode::kSolo) return {mine};
    // every rank must describe the same collective (sizes, windows): the reference fails a
    // mismatch at its first exchange (collectives.cpp:21-27); here, at the pointer exchange
    auto check_agree = [&](auto get) {
        for (int q = 0; q < world_; ++q)
            if (get(q) != agree)
                throw ProtocolError("collective mismatch across ranks at rank " + std::to_string(rank_) +
                                    " (rank " + std::to_string(q) + " describes a different buffer / windows)");
    };
    if (mode_ != Mode::kIpc) {
        struct Ptr {
            std::uintptr_t p;
            std::uint64_t agree;
        };
        const auto all = allgather(tp_, Ptr{reinterpret_cast<std::uintptr_t>(mine), agree}, tag);
        check_agree([&](int q) { return all[static_cast<std::size_t>(q)].agree; });
        std::vector<void*> out;
        for (auto& p : all) out.push_back(reinterpret_cast<void*>(p.p));
        return out;
    }
    struct Reg {
        char h[GF_IPC_HANDLE_BYTES];
        std::uint64_t off;
        std::uint64_t agree;
    } r{};
    check(gf_ipc_export(mine, r.h, &r.off), "gf_ipc_export");
    r.agree = agree;
    const auto all = allgather(tp_, r, tag);
    check_agree([&](int q) { return all[static_cast<std::size_t>(q)].agree; });
    std::vector<void*> out(static_cast<std::size_t>(world_));
    for (int q = 0; q < world_; ++q) {
        if (q == rank_) {
            out[static_cast<std::size_t>(q)] = mine;
            continue;
        }
        const std::string key(all[q].h, GF_IPC_HANDLE_BYTES);
        void* base = nullptr;
        {
            std::lock_guard lk(mu_);
            auto it = ipc_cache_.find(key);
            if (it == ipc_cache_.end()) {
                check(gf_ipc_open(comm_, all[q].h, &base), "gf_ipc_open");
                ipc_cache_[key] = base;
            } else {
                base = it->second;
            }
        }
        out[static_cast<std::size_t>(q)] = static_cast<char*>(base) + all[q].off;
    }
    return out;
}

void DeviceContext::ring_allreduce(ScalarBuffer buf, const std::vector<int>& ring,
                                   const std::vector<std::pair<std::size_t, std::size_t>>& windows,
                                   std::uint32_t tag) {
    if (world_ == 1 || windows.empty()) return;
    DeviceGuard g(device_);
    const auto st = static_cast<cudaStream_t>(stream_);
    const std::size_t es = element_size(buf.type);
    // Peers' buffers must share this buffer's 16-byte misalignment so one aligned base plus
    // shifted windows describes every rank; otherwise the collective runs in aligned scratch.
    std::uint64_t agree = 1469598103934665603ull;  // FNV-1a of (type, windows): same on every rank
    auto mix = [&](std::uint64_t v) {
        for (int b = 0; b < 8; ++b) {
            agree ^= (v >> (8 * b)) & 0xFFu;
            agree *= 1099511628211ull;
        }
    };
    mix(static_cast<std::uint64_t>(buf.type));
    for (auto& w : windows) {
        mix(w.first);
        mix(w.second);
    }
    auto ptrs = exchange(buf.data, tag, agree);
    const std::uintptr_t mis = reinterpret_cast<std::uintptr_t>(buf.data) & 15u;
    bool same = mis % es == 0;
    for (void* p : ptrs) same &= (reinterpret_cast<std::uintptr_t>(p) & 15u) == mis;
    std::size_t lo = windows.front().first, hi = 0;
    for (auto& w : windows) {
        lo = std::min(lo, w.first);
        hi = std::max(hi, w.first + w.second);
    }
    std::vector<std::uint64_t> ws, wl;
    std::byte* staged = nullptr;
    if (same) {
        for (auto& p : ptrs) p = static_cast<char*>(p) - mis;
        for (auto& w : windows) {
            ws.push_back(w.first + mis / es);
            wl.push_back(w.second);
        }
    } else {
        staged = static_cast<std::byte*>(scratch((hi - lo) * es, 1));
        cuda_ok(cudaMemcpyAsync(staged, buf.data + lo * es, (hi - lo) * es, cudaMemcpyDefault, st), "stage");
        ptrs = exchange(staged, tag | 0x80u, agree);
        for (auto& w : windows) {
            ws.push_back(w.first - lo);
            wl.push_back(w.second);
        }
    }
    const int dt = static_cast<int>(buf.type);
    if (mode_ == Mode::kColocated) {
        group_->run(rank_, ptrs[static_cast<std::size_t>(rank_)], tp_.timeout(), [&](std::vector<void*>& slots) {
            std::vector<void*> b = slots;  // each rank's own view of its buffer (same device)
            check(gf_ring_allreduce_colocated(dt, b.data(), world_, ring.data(), ws.data(), wl.data(),
                                              static_cast<int>(ws.size()), st),
                  "gf_ring_allreduce_colocated");
            cuda_ok(cudaStreamSynchronize(st), "colocated ring");
        });
    } else {
        check(gf_comm_set_ring_order(comm_, ring.data()), "ring order");
        check(gf_ring_allreduce_ptrs(comm_, dt, ptrs.data(), ws.data(), wl.data(), static_cast<int>(ws.size()), st),
              "gf_ring_allreduce_ptrs");
        cuda_ok(cudaStreamSynchronize(st), "ring allreduce");
        check(gf_comm_status(comm_), "ring allreduce");
    }
    if (staged) {
        cuda_ok(cudaMemcpyAsync(buf.data + lo * es, staged, (hi - lo) * es, cudaMemcpyDefault, st), "unstage");
        cuda_ok(cudaStreamSynchronize(st), "unstage");
    }
}

void DeviceContext::ring_allreduce_async(ElementType type, const std::vector<void*>& rank_bufs,
                                         const std::vector<int>& ring,
                                         const std::vector<std::pair<std::size_t, std::size_t>>& windows,
                                         void* client) {
    if (world_ == 1 || windows.empty()) return;
    if (!async_collectives()) throw ConfigError("ring_allreduce_async needs peer-mapped ranks on distinct GPUs");
    DeviceGuard g(device_);
    const auto cs = static_cast<cudaStream_t>(stream_);
    if (client) {
        cuda_ok(cudaEventRecord(static_cast<cudaEvent_t>(ev_client_), static_cast<cudaStream_t>(client)), "event");
        cuda_ok(cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(ev_client_), 0), "wait");
    }
    std::vector<std::uint64_t> ws, wl;
    for (auto& w : windows) {
        ws.push_back(w.first);
        wl.push_back(w.second);
    }
    check(gf_comm_set_ring_order(comm_, ring.data()), "ring order");
    std::vector<void*> b = rank_bufs;
    check(gf_ring_allreduce_ptrs(comm_, static_cast<int>(type), b.data(), ws.data(), wl.data(),
                                 static_cast<int>(ws.size()), stream_),
          "gf_ring_allreduce_ptrs");
    if (client) {
        cuda_ok(cudaEventRecord(static_cast<cudaEvent_t>(ev_done_), cs), "event");
        cuda_ok(cudaStreamWaitEvent(static_cast<cudaStream_t>(client), static_cast<cudaEvent_t>(ev_done_), 0), "wait");
    }
}

}  // namespace gflow
