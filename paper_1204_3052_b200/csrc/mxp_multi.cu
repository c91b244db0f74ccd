// mxp_power_multi: A^k on several GPUs from ONE process.
//
// Composed from the single-GPU C ABI, one handle (stream, workspaces, graph
// cache) per device:
//   * batch >= 2: the batch is split into contiguous shards (the same
//     shard_range as bench.py / distributed.py), one host thread per device
//     runs mxp_power_batched on its shard — no communication, results
//     bitwise equal to one device;
//   * batch == 1, FP32, n > 128, k >= 2: the matrix is row-sharded.  Every
//     device holds the base and ping/pong 3xTF32 planes of the whole (padded)
//     matrix; at each plan step device g computes its 256-row blocks with the
//     CTA-pair kernel (mxp_gemm_rows_planes_peers) whose epilogue stores the
//     new rows straight into EVERY device's next planes over NVLink (peer
//     access), tile by tile, so the exchange overlaps the MMAs still running.
//     CUDA events order the steps across the devices' streams (each stream
//     waits for every device's previous step before it overwrites their
//     planes).  Every element's dot product is computed on one device with
//     the single-GPU kernel and k-order, so the result is bitwise equal to
//     mxp_power on the 3xTF32 datapath (MXP_DATAPATH_3XTF32: the same
//     CTA-pair kernel, n % 256 == 0, n >= 1024; the default single-GPU chain
//     at these sizes is K1PH, equal within the tolerance);
//   * batch == 1, FP32 at the K1PH sizes (n > 1408, or roundup(n, 128) a
//     multiple of 256 >= 1024): the same row shards on scaled fp16x2 planes
//     (power_multi_rows_f16): each device computes its fp32 rows with the
//     K1PH row-block GEMM, the row maxima meet in every device's chain state
//     (system-scope atomicMax over peer access), and each device splits its
//     rows at the global exact scale straight into every device's next
//     planes (peer stores) — bitwise the single-device K1PH chain; a chain
//     that loses dynamic range is recomputed on the 3xTF32 row shards;
//   * batch == 1, FP64, n >= 256, k >= 2: row-sharded with the DMMA row-block
//     GEMM and peer copies of each device's rows (power_multi_rows_f64);
//   * anything else (n <= 128 FP32, small FP64, k <= 1) is too small to
//     shard: it runs on devices[0] (replicas only).
// The reference has no multi-device path (its
// device is one queue, gpu-backend/src/device.ts:6-8); this entry keeps the
// reference call's semantics (plan, k = 0 / 1, errors) on top.
#include <array>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "matexpo_b200.h"
#include "mxp_internal.h"

// defined in mxp_api.cu: the library's (thread-local) error slot
int mxp_internal_fail(int code, const char* fmt, ...);

namespace {

constexpr int kMaxDevices = 8;  // the fused epilogue's peer table (kMaxPeers)

// (device, occurrence) -> handle: a device listed twice gets two handles
// (two streams), which is how the sharding runs on a one-GPU machine.
std::mutex g_mu;
std::map<std::pair<int, int>, mxp_handle> g_handles;

int get_handles(int ngpus, const int* devices, std::vector<mxp_handle>& hs) {
    std::map<int, int> seen;
    hs.assign(ngpus, nullptr);
    for (int g = 0; g < ngpus; ++g) {
        const int dev = devices ? devices[g] : g;
        const std::pair<int, int> key(dev, seen[dev]++);
        auto it = g_handles.find(key);
        if (it == g_handles.end()) {
            mxp_handle h = nullptr;
            const int rc = mxp_create(dev, &h);
            if (rc) return rc;
            it = g_handles.emplace(key, h).first;
        }
        hs[g] = it->second;
    }
    return MXP_OK;
}

void shard_range(int64_t total, int r, int world, int64_t* lo, int64_t* hi) {
    const int64_t base = total / world, rem = total % world;
    *lo = r * base + (r < rem ? r : rem);
    *hi = *lo + base + (r < rem ? 1 : 0);
}

std::string last_error_string() {
    char buf[512];
    mxp_last_error(buf, sizeof buf);
    return buf;
}

int64_t plan_len(int64_t k, int64_t* squares) {
    *squares = 0;
    if (k <= 1) return 0;
    int64_t len = 0;
    for (int shift = 62; shift >= 0; --shift) {
        if ((k >> shift) & 1) {
            for (int s = shift - 1; s >= 0; --s) {
                ++len;
                ++*squares;
                if ((k >> s) & 1) ++len;
            }
            break;
        }
    }
    return len;
}

// ---- batch shards --------------------------------------------------------
int power_multi_batched(const std::vector<mxp_handle>& hs, int mode, int64_t n, int64_t batch,
                        int64_t k, const void* hA, void* hOut, mxp_stats* st) {
    const int G = static_cast<int>(hs.size());
    const size_t mat = static_cast<size_t>(n) * n * (mode == MXP_F64 ? 8 : 4);
    std::vector<int> rc(G, MXP_OK);
    std::vector<std::string> msg(G);
    std::vector<mxp_stats> sub(G);
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g) {
        int64_t lo, hi;
        shard_range(batch, g, G, &lo, &hi);
        th.emplace_back([&, g, lo, hi] {
            std::memset(&sub[g], 0, sizeof sub[g]);
            sub[g].failed_step = -1;
            if (hi == lo) return;
            rc[g] = mxp_power_batched(hs[g], mode, n, hi - lo, k,
                                      static_cast<const char*>(hA) + lo * mat,
                                      static_cast<char*>(hOut) + lo * mat, &sub[g]);
            if (rc[g]) msg[g] = last_error_string();
        });
    }
    for (auto& t : th) t.join();
    for (int g = 0; g < G; ++g) {
        if (rc[g]) {
            if (st) st->failed_step = sub[g].failed_step;
            return mxp_internal_fail(rc[g], "device shard %d: %s", g, msg[g].c_str());
        }
    }
    if (st) {
        int64_t sq = 0;
        const int64_t m = plan_len(k, &sq);
        st->multiply_count = m * batch;
        st->square_count = sq * batch;
        for (int g = 0; g < G; ++g) {
            st->launches += sub[g].launches;
            st->h2d += sub[g].h2d;  // one upload per device that holds a shard
            st->d2h += sub[g].d2h;
            st->h2d_bytes += sub[g].h2d_bytes;
            st->d2h_bytes += sub[g].d2h_bytes;
            if (sub[g].device_ms > st->device_ms) st->device_ms = sub[g].device_ms;  // max over devices
        }
    }
    return MXP_OK;
}

// peer access between distinct devices (UVA pointers then work across them)
int enable_peers(const std::vector<int>& dev) {
    const int G = static_cast<int>(dev.size());
    for (int g = 0; g < G; ++g)
        for (int q = 0; q < G; ++q) {
            if (dev[g] == dev[q]) continue;
            int ok = 0;
            if (cudaDeviceCanAccessPeer(&ok, dev[g], dev[q]) != cudaSuccess || !ok)
                return mxp_internal_fail(MXP_E_UNSUPPORTED,
                                         "device %d cannot access device %d (no P2P / NVLink)",
                                         dev[g], dev[q]);
            cudaSetDevice(dev[g]);
            cudaError_t e = cudaDeviceEnablePeerAccess(dev[q], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
            } else if (e != cudaSuccess) {
                return mxp_internal_fail(MXP_E_CUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s",
                                         dev[g], dev[q], cudaGetErrorString(e));
            }
        }
    return MXP_OK;
}

// every device's stream waits for every other device's work so far
int cross_fence(const std::vector<int>& dev, const std::vector<cudaStream_t>& stream,
                const std::vector<cudaEvent_t>& ev) {
    const int G = static_cast<int>(dev.size());
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(dev[g]);
        if (cudaEventRecord(ev[g], stream[g]) != cudaSuccess)
            return mxp_internal_fail(MXP_E_CUDA, "event record on device %d", dev[g]);
    }
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(dev[g]);
        for (int q = 0; q < G; ++q)
            if (q != g && cudaStreamWaitEvent(stream[g], ev[q], 0) != cudaSuccess)
                return mxp_internal_fail(MXP_E_CUDA, "stream wait on device %d", dev[g]);
    }
    return MXP_OK;
}

// ---- one FP64 matrix, row shards -----------------------------------------
// tcgen05 has no f64 kind and the DMMA kernel has no fused peer epilogue:
// each device computes its contiguous row block with the public row-block
// GEMM (mxp_gemm_prepare_rhs + mxp_gemm_rows_prepared: the single-GPU kernel
// and k-order, so every row is bitwise the single-device chain's), then
// copies the block into every other device's next buffer over NVLink
// (cudaMemcpyAsync between peers on its own stream); CUDA events order the
// steps.  SURVEY §8(e) C4: "same scheme, optional".
int power_multi_rows_f64(const std::vector<mxp_handle>& hs, const int* devices, int64_t n,
                         int64_t k, const void* hA, void* hOut, mxp_stats* st) {
    const int G = static_cast<int>(hs.size());
    const size_t mat = static_cast<size_t>(n) * n * 8;
    std::vector<int> dev(G);
    for (int g = 0; g < G; ++g) dev[g] = devices ? devices[g] : g;
    int rc = enable_peers(dev);
    if (rc) return rc;
    struct Guard {
        const std::vector<mxp_handle>& hs;
        std::vector<std::array<void*, 3>> buf;  // base, ping, pong
        std::vector<cudaEvent_t> ev;
        explicit Guard(const std::vector<mxp_handle>& h) : hs(h), buf(h.size()), ev(h.size()) {
            for (auto& b : buf) b = {nullptr, nullptr, nullptr};
        }
        ~Guard() {
            for (size_t g = 0; g < buf.size(); ++g) {
                mxp_synchronize(hs[g]);
                for (void* p : buf[g])
                    if (p) mxp_free(hs[g], p);
                if (ev[g]) cudaEventDestroy(ev[g]);
            }
        }
    } guard(hs);
    std::vector<cudaStream_t> stream(G);
    for (int g = 0; g < G && rc == MXP_OK; ++g) {
        void* s = nullptr;
        rc = mxp_get_stream(hs[g], &s);
        stream[g] = static_cast<cudaStream_t>(s);
        for (int i = 0; i < 3 && rc == MXP_OK; ++i) rc = mxp_alloc(hs[g], mat, &guard.buf[g][i]);
        if (rc == MXP_OK) {
            cudaSetDevice(dev[g]);
            if (cudaEventCreateWithFlags(&guard.ev[g], cudaEventDisableTiming) != cudaSuccess)
                rc = mxp_internal_fail(MXP_E_CUDA, "event creation on device %d", dev[g]);
        }
    }
    if (rc) return rc;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    cudaSetDevice(dev[0]);
    if (cudaEventCreate(&t0) != cudaSuccess || cudaEventCreate(&t1) != cudaSuccess)
        return mxp_internal_fail(MXP_E_CUDA, "event creation");
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() {
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } evg{t0, t1};
    cudaEventRecord(t0, stream[0]);
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(dev[g]);
        cudaError_t e = cudaMemcpyAsync(guard.buf[g][0], hA, mat, cudaMemcpyHostToDevice, stream[g]);
        if (e != cudaSuccess)
            return mxp_internal_fail(MXP_E_CUDA, "upload to device %d: %s", dev[g],
                                     cudaGetErrorString(e));
    }
    if ((rc = cross_fence(dev, stream, guard.ev))) return rc;
    int64_t sq = 0;
    const int64_t m = plan_len(k, &sq);
    int cur = 0, launches = 0;
    int64_t bit = 62;
    while (!((k >> bit) & 1)) --bit;
    int64_t step = 0;
    for (int64_t s = bit - 1; s >= 0; --s) {
        for (int mult = 0; mult < 2; ++mult) {
            if (mult && !((k >> s) & 1)) break;
            const int nxt = cur == 1 ? 2 : 1;
            for (int g = 0; g < G; ++g) {
                int64_t lo, hi;
                shard_range(n, g, G, &lo, &hi);
                if (hi == lo) continue;
                const size_t off = static_cast<size_t>(lo) * n * 8;
                char* c_cur = static_cast<char*>(guard.buf[g][cur]);
                char* c_nxt = static_cast<char*>(guard.buf[g][nxt]);
                rc = mxp_gemm_prepare_rhs(hs[g], MXP_F64, n, guard.buf[g][mult ? 0 : cur]);
                if (rc == MXP_OK)
                    rc = mxp_gemm_rows_prepared(hs[g], MXP_F64, n, hi - lo, c_cur + off, c_nxt + off);
                if (rc) {
                    if (st) st->failed_step = step;
                    return rc;
                }
                launches += 4;  // rhs pad, rows pad, GEMM, unpad
                cudaSetDevice(dev[g]);
                for (int q = 0; q < G; ++q) {
                    if (q == g) continue;
                    cudaError_t e = cudaMemcpyAsync(static_cast<char*>(guard.buf[q][nxt]) + off,
                                                    c_nxt + off, static_cast<size_t>(hi - lo) * n * 8,
                                                    cudaMemcpyDefault, stream[g]);
                    if (e != cudaSuccess) {
                        if (st) st->failed_step = step;
                        return mxp_internal_fail(MXP_E_CUDA, "row exchange %d -> %d: %s", dev[g],
                                                 dev[q], cudaGetErrorString(e));
                    }
                }
            }
            if ((rc = cross_fence(dev, stream, guard.ev))) return rc;
            cur = nxt;
            ++step;
        }
    }
    cudaSetDevice(dev[0]);
    cudaEventRecord(t1, stream[0]);
    cudaError_t e = cudaMemcpyAsync(hOut, guard.buf[0][cur], mat, cudaMemcpyDeviceToHost, stream[0]);
    for (int g = 0; g < G && e == cudaSuccess; ++g) {
        cudaSetDevice(dev[g]);
        e = cudaStreamSynchronize(stream[g]);
    }
    if (e != cudaSuccess)
        return mxp_internal_fail(MXP_E_CUDA, "row-sharded FP64 chain: %s", cudaGetErrorString(e));
    if (st) {
        st->multiply_count = m;
        st->square_count = sq;
        st->launches = launches;
        st->h2d = G;
        st->d2h = 1;
        st->h2d_bytes = static_cast<int64_t>(G * mat);
        st->d2h_bytes = static_cast<int64_t>(mat);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t0, t1);
        st->device_ms = ms;
    }
    return MXP_OK;
}

// ---- one matrix, row shards, exchange fused into the GEMM epilogue ------
struct RowBufs {
    void* base = nullptr;               // n_p x n_p fp32 (zero padded input)
    void* plane[6] = {};                // base hi/lo, p0 hi/lo, p1 hi/lo (tf32 bits)
    void* out = nullptr;                // n_p x n_p fp32 (final rows of every device)
    cudaEvent_t ev = nullptr;           // end of this device's current step
};

int power_multi_rows(const std::vector<mxp_handle>& hs, const int* devices, int64_t n, int64_t k,
                     const void* hA, void* hOut, mxp_stats* st) {
    const int G = static_cast<int>(hs.size());
    // padded order: 256-row CTA-pair blocks per device and n_p >= 1024 (the
    // pair kernel's range) — distributed.fused_layout
    int64_t n_p = (n + 256 * G - 1) / (256 * G) * (256 * G);
    if (n_p < 1024) n_p = (1024 + 256 * G - 1) / (256 * G) * (256 * G);
    const int64_t rows = n_p / G;
    const size_t plane = static_cast<size_t>(n_p) * n_p * 4;
    std::vector<int> dev(G);
    for (int g = 0; g < G; ++g) dev[g] = devices ? devices[g] : g;
    int rc = enable_peers(dev);
    if (rc) return rc;
    // buffers, freed on every exit path
    struct Guard {
        const std::vector<mxp_handle>& hs;
        std::vector<RowBufs> b;
        explicit Guard(const std::vector<mxp_handle>& h) : hs(h), b(h.size()) {}
        ~Guard() {
            for (size_t g = 0; g < b.size(); ++g) {
                mxp_synchronize(hs[g]);
                if (b[g].base) mxp_free(hs[g], b[g].base);
                for (void* p : b[g].plane)
                    if (p) mxp_free(hs[g], p);
                if (b[g].out) mxp_free(hs[g], b[g].out);
                if (b[g].ev) cudaEventDestroy(b[g].ev);
            }
        }
    } guard(hs);
    auto& B = guard.b;
    std::vector<cudaStream_t> stream(G);
    for (int g = 0; g < G && rc == MXP_OK; ++g) {
        void* s = nullptr;
        rc = mxp_get_stream(hs[g], &s);
        stream[g] = static_cast<cudaStream_t>(s);
        if (rc == MXP_OK) rc = mxp_alloc(hs[g], plane, &B[g].base);
        for (int i = 0; i < 6 && rc == MXP_OK; ++i) rc = mxp_alloc(hs[g], plane, &B[g].plane[i]);
        if (rc == MXP_OK) rc = mxp_alloc(hs[g], plane, &B[g].out);
        if (rc == MXP_OK) {
            cudaSetDevice(dev[g]);
            if (cudaEventCreateWithFlags(&B[g].ev, cudaEventDisableTiming) != cudaSuccess)
                rc = mxp_internal_fail(MXP_E_CUDA, "event creation on device %d", dev[g]);
        }
    }
    if (rc) return rc;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    cudaSetDevice(dev[0]);
    if (cudaEventCreate(&t0) != cudaSuccess || cudaEventCreate(&t1) != cudaSuccess)
        return mxp_internal_fail(MXP_E_CUDA, "event creation");
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() {
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } evg{t0, t1};
    cudaEventRecord(t0, stream[0]);
    // upload (one H2D per device) into the zero-padded base, split into the
    // base and first ping planes
    for (int g = 0; g < G && rc == MXP_OK; ++g) {
        cudaSetDevice(dev[g]);
        cudaError_t e = cudaMemsetAsync(B[g].base, 0, plane, stream[g]);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(B[g].base, n_p * 4, hA, n * 4, n * 4, n, cudaMemcpyHostToDevice,
                                  stream[g]);
        if (e != cudaSuccess) return mxp_internal_fail(MXP_E_CUDA, "upload to device %d: %s",
                                                       dev[g], cudaGetErrorString(e));
        rc = mxp_split_planes(hs[g], n_p, B[g].base, B[g].plane[0], B[g].plane[1]);
        if (rc == MXP_OK) rc = mxp_split_planes(hs[g], n_p, B[g].base, B[g].plane[2], B[g].plane[3]);
    }
    if (rc) return rc;
    // every device's planes are initialised before anyone stores into them
    auto step_fence = [&]() -> int {
        for (int g = 0; g < G; ++g) {
            cudaSetDevice(dev[g]);
            if (cudaEventRecord(B[g].ev, stream[g]) != cudaSuccess)
                return mxp_internal_fail(MXP_E_CUDA, "event record on device %d", dev[g]);
        }
        for (int g = 0; g < G; ++g) {
            cudaSetDevice(dev[g]);
            for (int q = 0; q < G; ++q)
                if (q != g && cudaStreamWaitEvent(stream[g], B[q].ev, 0) != cudaSuccess)
                    return mxp_internal_fail(MXP_E_CUDA, "stream wait on device %d", dev[g]);
        }
        return MXP_OK;
    };
    if ((rc = step_fence())) return rc;
    int64_t sq = 0;
    const int64_t m = plan_len(k, &sq);
    int cur = 1, launches = 0;  // plane pair index: 0 base, 1 p0, 2 p1
    int64_t bit = 62;
    while (!((k >> bit) & 1)) --bit;
    int64_t step = 0;
    std::vector<void*> dhi(G), dlo(G), df32(G);
    for (int64_t s = bit - 1; s >= 0; --s) {
        for (int mult = 0; mult < 2; ++mult) {
            if (mult && !((k >> s) & 1)) break;
            const bool last = step == m - 1;
            const int nxt = cur == 1 ? 2 : 1;
            for (int q = 0; q < G; ++q) {
                dhi[q] = last ? nullptr : B[q].plane[2 * nxt];
                dlo[q] = last ? nullptr : B[q].plane[2 * nxt + 1];
                df32[q] = last ? B[q].out : nullptr;
            }
            for (int g = 0; g < G; ++g) {
                const int rhs = mult ? 0 : cur;
                rc = mxp_gemm_rows_planes_peers(hs[g], n_p, rows, g * rows, B[g].plane[2 * cur],
                                                B[g].plane[2 * cur + 1], B[g].plane[2 * rhs],
                                                B[g].plane[2 * rhs + 1], G,
                                                last ? nullptr : dhi.data(),
                                                last ? nullptr : dlo.data(),
                                                last ? df32.data() : nullptr);
                if (rc) {
                    if (st) st->failed_step = step;
                    return rc;
                }
                ++launches;
            }
            if ((rc = step_fence())) return rc;
            cur = nxt;
            ++step;
        }
    }
    // every device holds the whole result: read it back once, from devices[0]
    cudaSetDevice(dev[0]);
    cudaEventRecord(t1, stream[0]);
    cudaError_t e = cudaMemcpy2DAsync(hOut, n * 4, B[0].out, n_p * 4, n * 4, n,
                                      cudaMemcpyDeviceToHost, stream[0]);
    for (int g = 0; g < G && e == cudaSuccess; ++g) {
        cudaSetDevice(dev[g]);
        e = cudaStreamSynchronize(stream[g]);
    }
    if (e != cudaSuccess) return mxp_internal_fail(MXP_E_CUDA, "row-sharded chain: %s",
                                                   cudaGetErrorString(e));
    if (st) {
        st->multiply_count = m;
        st->square_count = sq;
        st->launches = launches + 2 * G;  // + the splits
        st->h2d = G;                      // one upload per device
        st->d2h = 1;
        st->h2d_bytes = static_cast<int64_t>(G) * n * n * 4;
        st->d2h_bytes = n * n * 4;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t0, t1);
        st->device_ms = ms;
    }
    return MXP_OK;
}

// ---- one FP32 matrix, row shards on scaled fp16x2 planes (K1PH) ---------
// Returns MXP_OK with *raised = 1 when the chain lost dynamic range (the
// caller then recomputes on the 3xTF32 row shards).
bool k1ph_multi_eligible(int64_t n) {
    const int64_t p128 = (n + 127) / 128 * 128;
    return (p128 >= 1024 && p128 % 256 == 0) || n > 1408;
}

int power_multi_rows_f16(const std::vector<mxp_handle>& hs, const int* devices, int64_t n,
                         int64_t k, const void* hA, void* hOut, mxp_stats* st, int* raised) {
    using namespace mxp;
    const int G = static_cast<int>(hs.size());
    *raised = 0;
    // the single-device chain's padded order when it is a multiple of 256 G
    // (results are bitwise the single-device chain's for any padding: zero
    // rows and columns only add exact zeros in the same k-blocks)
    int64_t n_p = (n + 256 * G - 1) / (256 * G) * (256 * G);
    if (n_p < 1024) n_p = (1024 + 256 * G - 1) / (256 * G) * (256 * G);
    const int64_t rows = n_p / G;
    const size_t n2 = static_cast<size_t>(n_p) * n_p;
    std::vector<int> dev(G);
    for (int g = 0; g < G; ++g) dev[g] = devices ? devices[g] : g;
    int rc = enable_peers(dev);
    if (rc) return rc;
    struct Bufs {
        void* plane[6] = {};  // h0/h1 of base, p0, p1 (fp16, n_p x n_p)
        void* rowsf = nullptr;  // this device's fp32 rows of the running product
        void* state = nullptr;
        void* out = nullptr;    // the final fp32 rows of every device (devices[0])
        cudaEvent_t ev = nullptr;
        F16Maps maps[3];
    };
    struct Guard {
        const std::vector<mxp_handle>& hs;
        std::vector<Bufs> b;
        explicit Guard(const std::vector<mxp_handle>& h) : hs(h), b(h.size()) {}
        ~Guard() {
            for (size_t g = 0; g < b.size(); ++g) {
                mxp_synchronize(hs[g]);
                for (void* p : b[g].plane)
                    if (p) mxp_free(hs[g], p);
                for (void* p : {b[g].rowsf, b[g].state, b[g].out})
                    if (p) mxp_free(hs[g], p);
                if (b[g].ev) cudaEventDestroy(b[g].ev);
            }
        }
    } guard(hs);
    auto& B = guard.b;
    std::vector<cudaStream_t> stream(G);
    std::vector<int> sms(G);
    for (int g = 0; g < G && rc == MXP_OK; ++g) {
        void* s = nullptr;
        rc = mxp_get_stream(hs[g], &s);
        stream[g] = static_cast<cudaStream_t>(s);
        if (rc == MXP_OK) rc = mxp_num_sms(hs[g], &sms[g]);
        for (int i = 0; i < 6 && rc == MXP_OK; ++i) rc = mxp_alloc(hs[g], n2 * 2, &B[g].plane[i]);
        if (rc == MXP_OK) rc = mxp_alloc(hs[g], static_cast<size_t>(rows) * n_p * 4, &B[g].rowsf);
        if (rc == MXP_OK) rc = mxp_alloc(hs[g], f16_chain_state_bytes(), &B[g].state);
        if (rc == MXP_OK && g == 0) rc = mxp_alloc(hs[g], static_cast<size_t>(n) * n * 4, &B[g].out);
        if (rc == MXP_OK) {
            cudaSetDevice(dev[g]);
            if (cudaEventCreateWithFlags(&B[g].ev, cudaEventDisableTiming) != cudaSuccess)
                rc = mxp_internal_fail(MXP_E_CUDA, "event creation on device %d", dev[g]);
            for (int i = 0; i < 3 && rc == MXP_OK; ++i) {
                F16Maps& m = B[g].maps[i];
                if (!encode_plane16_map(&m.a0, B[g].plane[2 * i], (int)n_p, 128) ||
                    !encode_plane16_map(&m.a1, B[g].plane[2 * i + 1], (int)n_p, 128) ||
                    !encode_plane16_map(&m.b0, B[g].plane[2 * i], (int)n_p, 64) ||
                    !encode_plane16_map(&m.b1, B[g].plane[2 * i + 1], (int)n_p, 64))
                    rc = mxp_internal_fail(MXP_E_CUDA, "cuTensorMapEncodeTiled (fp16) failed");
            }
        }
    }
    if (rc) return rc;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    cudaSetDevice(dev[0]);
    if (cudaEventCreate(&t0) != cudaSuccess || cudaEventCreate(&t1) != cudaSuccess)
        return mxp_internal_fail(MXP_E_CUDA, "event creation");
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() {
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } evg{t0, t1};
    auto fence = [&]() -> int {
        for (int g = 0; g < G; ++g) {
            cudaSetDevice(dev[g]);
            if (cudaEventRecord(B[g].ev, stream[g]) != cudaSuccess)
                return mxp_internal_fail(MXP_E_CUDA, "event record on device %d", dev[g]);
        }
        for (int g = 0; g < G; ++g) {
            cudaSetDevice(dev[g]);
            for (int q = 0; q < G; ++q)
                if (q != g && cudaStreamWaitEvent(stream[g], B[q].ev, 0) != cudaSuccess)
                    return mxp_internal_fail(MXP_E_CUDA, "stream wait on device %d", dev[g]);
        }
        return MXP_OK;
    };
    cudaEventRecord(t0, stream[0]);
    // every device: A uploaded into a temporary, its state reset, the base
    // planes and max computed locally (identical on every device)
    std::vector<void*> a_dev(G, nullptr);
    for (int g = 0; g < G && rc == MXP_OK; ++g) {
        rc = mxp_alloc(hs[g], static_cast<size_t>(n) * n * 4, &a_dev[g]);
        if (rc) break;
        cudaSetDevice(dev[g]);
        cudaError_t e = cudaMemsetAsync(B[g].state, 0, f16_chain_state_bytes(), stream[g]);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(a_dev[g], hA, static_cast<size_t>(n) * n * 4, cudaMemcpyHostToDevice,
                                stream[g]);
        // the base planes and max, identical on every device
        if (e == cudaSuccess)
            e = launch_split16(static_cast<const float*>(a_dev[g]), (int)n, (int)n, B[g].plane[0],
                               B[g].plane[1], (int)n_p, B[g].state, 0, -1, -1, stream[g]);
        if (e != cudaSuccess)
            rc = mxp_internal_fail(MXP_E_CUDA, "upload / split on device %d: %s", dev[g],
                                   cudaGetErrorString(e));
    }
    auto free_a = [&]() {
        for (int g = 0; g < G; ++g)
            if (a_dev[g]) {
                mxp_synchronize(hs[g]);
                mxp_free(hs[g], a_dev[g]);
                a_dev[g] = nullptr;
            }
    };
    // every state is reset before any device's maxima reach it
    if (rc == MXP_OK) rc = fence();
    if (rc) {
        free_a();
        return rc;
    }
    int64_t sq = 0;
    const int64_t m = plan_len(k, &sq);
    int cur = 0, cur_i = 0, launches = 0;  // plane pair of the running power, its state index
    int64_t bit = 62;
    while (!((k >> bit) & 1)) --bit;
    int64_t step = 0;
    std::vector<void*> states(G), dh0(G), dh1(G);
    for (int g = 0; g < G; ++g) states[g] = B[g].state;
    for (int64_t s = bit - 1; s >= 0 && rc == MXP_OK; --s) {
        for (int mult = 0; mult < 2 && rc == MXP_OK; ++mult) {
            if (mult && !((k >> s) & 1)) break;
            const bool last = step == m - 1;
            const int nxt = cur == 1 ? 2 : 1;
            const int rhs = mult ? 0 : cur, rhs_i = mult ? 0 : cur_i;
            const int oi = static_cast<int>(step) + 1;
            for (int g = 0; g < G && rc == MXP_OK; ++g) {
                cudaSetDevice(dev[g]);
                const int64_t row0 = g * rows;
                // last step: this device's rows of the result straight into
                // devices[0]'s n x n output (peer stores, rows < n only)
                float* out = last ? static_cast<float*>(B[0].out) + row0 * n
                                  : static_cast<float*>(B[g].rowsf);
                cudaError_t e = cudaSuccess;
                if (!last || row0 < n)
                    e = launch_k1ph_gemm(B[g].maps[cur], B[g].maps[rhs], (int)n_p, out,
                                         last ? (int)n : (int)n_p, last ? (int)n : (int)n_p,
                                         B[g].state, cur_i, rhs_i, last ? -1 : oi, sms[g], stream[g],
                                         (int)rows, (int)row0);
                if (e == cudaSuccess && !last) e = launch_max_to_peers(B[g].state, oi, states.data(), G, stream[g]);
                if (e != cudaSuccess) {
                    if (st) st->failed_step = step;
                    rc = mxp_internal_fail(MXP_E_CUDA, "k1ph row block on device %d: %s", dev[g],
                                           cudaGetErrorString(e));
                }
                launches += last ? 1 : 2;
            }
            if (rc == MXP_OK && !last) {
                // every device's max is global: split the rows into everyone's planes
                if ((rc = fence())) break;
                for (int q = 0; q < G; ++q) {
                    dh0[q] = B[q].plane[2 * nxt];
                    dh1[q] = B[q].plane[2 * nxt + 1];
                }
                for (int g = 0; g < G && rc == MXP_OK; ++g) {
                    cudaSetDevice(dev[g]);
                    cudaError_t e = launch_split16_rows_peers(
                        static_cast<const float*>(B[g].rowsf), (int)rows, (int)(g * rows), (int)n_p,
                        (int)n, B[g].state, oi, cur_i, rhs_i, dh0.data(), dh1.data(), G, stream[g]);
                    if (e != cudaSuccess) {
                        if (st) st->failed_step = step;
                        rc = mxp_internal_fail(MXP_E_CUDA, "row split on device %d: %s", dev[g],
                                               cudaGetErrorString(e));
                    }
                    ++launches;
                }
            }
            if (rc == MXP_OK) rc = fence();
            cur = nxt;
            cur_i = oi;
            ++step;
        }
    }
    if (rc) {
        free_a();
        return rc;
    }
    cudaSetDevice(dev[0]);
    cudaEventRecord(t1, stream[0]);
    cudaError_t e = cudaMemcpyAsync(hOut, B[0].out, static_cast<size_t>(n) * n * 4,
                                    cudaMemcpyDeviceToHost, stream[0]);
    for (int g = 0; g < G && e == cudaSuccess; ++g) {
        cudaSetDevice(dev[g]);
        e = cudaStreamSynchronize(stream[g]);
    }
    free_a();
    if (e != cudaSuccess)
        return mxp_internal_fail(MXP_E_CUDA, "row-sharded K1PH chain: %s", cudaGetErrorString(e));
    int flag = 0;
    cudaSetDevice(dev[0]);
    if (cudaMemcpy(&flag, f16_chain_flag(B[0].state), sizeof flag, cudaMemcpyDeviceToHost) != cudaSuccess)
        return mxp_internal_fail(MXP_E_CUDA, "flag readback");
    *raised = flag != 0;
    if (st) {
        st->multiply_count = m;
        st->square_count = sq;
        st->launches = launches + 3 * G;  // + each device's base max / split / state reset
        st->h2d = G;
        st->d2h = 1;
        st->h2d_bytes = static_cast<int64_t>(G) * n * n * 4;
        st->d2h_bytes = n * n * 4;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t0, t1);
        st->device_ms = ms;
    }
    return MXP_OK;
}

}  // namespace

extern "C" int mxp_power_multi(int ngpus, const int* devices, int mode, int64_t n, int64_t batch,
                               int64_t k, const void* hA, void* hOut, mxp_stats* st) {
    if (st) {
        std::memset(st, 0, sizeof *st);
        st->failed_step = -1;
    }
    if (ngpus < 1 || ngpus > kMaxDevices)
        return mxp_internal_fail(MXP_E_VALIDATION, "1 <= ngpus <= %d, got %d", kMaxDevices, ngpus);
    if (mode != MXP_F32 && mode != MXP_F64)
        return mxp_internal_fail(MXP_E_VALIDATION, "unknown element mode %d", mode);
    if (n < 1) return mxp_internal_fail(MXP_E_VALIDATION, "n must be >= 1, got %lld", (long long)n);
    if (k < 0) return mxp_internal_fail(MXP_E_VALIDATION, "power must be >= 0, got %lld", (long long)k);
    if (batch < 1) return mxp_internal_fail(MXP_E_VALIDATION, "batch must be >= 1, got %lld", (long long)batch);
    if (!hA || !hOut) return mxp_internal_fail(MXP_E_VALIDATION, "null host pointer");
    std::lock_guard<std::mutex> lock(g_mu);  // the handles are single-caller
    std::vector<mxp_handle> hs;
    int rc = get_handles(ngpus, devices, hs);
    if (rc) return rc;
    if (batch >= 2) {
        if (batch < ngpus) hs.resize(static_cast<size_t>(batch));
        return power_multi_batched(hs, mode, n, batch, k, hA, hOut, st);
    }
    if (ngpus >= 2 && mode == MXP_F32 && n > 128 && k >= 2) {
        if (k1ph_multi_eligible(n)) {
            int raised = 0;
            rc = power_multi_rows_f16(hs, devices, n, k, hA, hOut, st, &raised);
            // a product lost dynamic range: the 3xTF32 row shards recompute it
            // (bitwise the single-device chain's 3xTF32 recomputation)
            if (rc != MXP_OK || !raised) return rc;
            if (st) {
                std::memset(st, 0, sizeof *st);
                st->failed_step = -1;
            }
        }
        return power_multi_rows(hs, devices, n, k, hA, hOut, st);
    }
    if (ngpus >= 2 && mode == MXP_F64 && n >= 256 && k >= 2)
        return power_multi_rows_f64(hs, devices, n, k, hA, hOut, st);
    return mxp_power(hs[0], mode, n, k, hA, hOut, st);  // replicas only
}

extern "C" int mxp_multi_release(void) {
    std::lock_guard<std::mutex> lock(g_mu);
    int rc = MXP_OK;
    for (auto& kv : g_handles) {
        const int r = mxp_destroy(kv.second);
        if (r && rc == MXP_OK) rc = r;
    }
    g_handles.clear();
    return rc;
}
