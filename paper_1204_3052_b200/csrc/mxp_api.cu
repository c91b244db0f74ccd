// C-ABI shim (include/matexpo_b200.h): validation, workspace, the CUDA-graph
// square-and-multiply scheduler, and dispatch to the sm_100a kernels.
//
// The scheduler replaces the reference's host loop (expo.py:131-138) and the
// device chain of gpuExponentiate (gpu-backend/src/host.ts:106-141): the plan
// (expo.py:60-75) is baked into one captured CUDA graph of m GEMM launches
// over ping-pong buffers in HBM; the graph is cached per (mode, n, k, in, out)
// and replayed.
#include <condition_variable>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/matexpo_b200.h"
#include "mxp_internal.h"

// host batched pipeline chunk (MB): small enough that the PCIe fill and drain
// (one chunk each way) stay short, large enough for a full persistent kernel
#ifndef MXP_E2E_CHUNK_MB
#define MXP_E2E_CHUNK_MB 64
#endif

namespace mxp {

cudaError_t prepare_tf32_kernels();
cudaError_t prepare_f64_kernels();
cudaError_t prepare_kernels() {
    cudaError_t e = prepare_tf32_kernels();
    if (e == cudaSuccess) e = prepare_f64_kernels();
    if (e == cudaSuccess) e = prepare_k3b_kernel();
    if (e == cudaSuccess) e = prepare_k3h_kernel();
    if (e == cudaSuccess) e = prepare_mod_i8_kernel();
    if (e == cudaSuccess) e = prepare_f16x2_kernels();
    return e;
}

PlanBits make_plan(int64_t k) {
    PlanBits p{};
    if (k <= 1) return p;
    int top = 63;
    while (!((k >> top) & 1)) --top;
    for (int shift = top - 1; shift >= 0; --shift) {
        p.len++;  // SQUARE
        p.squares++;
        if ((k >> shift) & 1) {
            p.mult[p.len >> 6] |= 1ull << (p.len & 63);
            p.len++;
        }
    }
    return p;
}

}  // namespace mxp

using namespace mxp;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(MXP_E_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define MXP_CUDA(expr)                                         \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);    \
    } while (0)

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct GraphKey {
    int mode;
    int64_t n, k;
    const void* in;
    void* out;
    bool operator<(const GraphKey& o) const {
        return std::tie(mode, n, k, in, out) < std::tie(o.mode, o.n, o.k, o.in, o.out);
    }
};

// A small pool of host threads for copies between pageable caller memory
// and pinned staging buffers (mxp_power_batched with ordinary numpy arrays:
// the DMA engines only stream from pinned pages, and the driver's own
// pageable path is single-threaded).  run(f) calls f(i, n) on every worker
// i in [0, n) and returns when all have finished.
class HostPool {
  public:
    explicit HostPool(int n) : n_(n) {
        for (int i = 0; i < n_; ++i) threads_.emplace_back([this, i] { loop(i); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    int size() const { return n_; }
    void run(const std::function<void(int, int)>& f) {
        std::unique_lock<std::mutex> g(m_);
        job_ = &f;
        pending_ = n_;
        ++gen_;
        cv_.notify_all();
        done_cv_.wait(g, [this] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int, int)>* job;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                job = job_;
            }
            (*job)(i, n_);
            {
                std::lock_guard<std::mutex> g(m_);
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }
    int n_;
    std::vector<std::thread> threads_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int, int)>* job_ = nullptr;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// Copy up to two independent ranges with every pool thread (each thread takes
// its slice of both, 4 KB-aligned).
struct CopyJob {
    void* dst;
    const void* src;
    size_t bytes;
};
void pool_copy(HostPool& pool, const CopyJob* jobs, int njobs) {
    pool.run([&](int i, int n) {
        for (int j = 0; j < njobs; ++j) {
            const size_t per = ((jobs[j].bytes + n - 1) / n + 4095) & ~size_t(4095);
            const size_t lo = per * i;
            if (lo >= jobs[j].bytes) continue;
            const size_t len = (lo + per <= jobs[j].bytes) ? per : jobs[j].bytes - lo;
            std::memcpy(static_cast<char*>(jobs[j].dst) + lo,
                        static_cast<const char*>(jobs[j].src) + lo, len);
        }
    });
}

bool is_pageable(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

}  // namespace

struct mxp_handle_s {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    // fp32 single-matrix workspace: 6 tf32 planes (base, ping, pong) x (hi, lo)
    int64_t ws32_pad = 0;  // padded order the planes are currently laid out for
    int64_t ws32_cap = 0;  // padded order they are allocated for (>= ws32_pad)
    uint32_t* planes[6] = {};
    int splits = 1;  // split-K factor of the 1-CTA K1 tiles at ws32_pad
    unsigned int* bar_ctr = nullptr;  // grid-barrier counter of the one-launch chain (K1C)
    CUtensorMap map_a[6], map_b[6];
    // right-hand side prepared by mxp_gemm_prepare_rhs (planes[2..3] / f64buf[1]);
    // any other use of the workspace invalidates it
    int rhs_mode = -1;
    int64_t rhs_n = 0;
    // K1PH workspace (scaled fp16x2 chain): h0/h1 planes of base, ping, pong
    // and the chain state (kernels_f16x2.cu: F16Chain)
    int f32_datapath = MXP_DATAPATH_AUTO;
    int64_t ws16_pad = 0;  // padded order the maps are encoded for
    int64_t ws16_cap = 0;  // padded order the buffers are allocated for
    void* planes16[6] = {};
    float* fbuf = nullptr;     // the fp32 product of the running step
    void* f16state = nullptr;  // the chain state (maxima, plane exponents, bounds, flag)
    F16Maps maps16[3];
    bool f16_ran = false;  // the last chain ran K1PH (mxp_last_f32_fallback)
    // fp64 workspace: base, ping, pong (n_pad^2 doubles)
    int64_t ws64_pad = 0;
    double* f64buf[3] = {};
    // modular workspace: base limbs (3), acc limbs (3), T0..T2 (3), n_pad^2 doubles each
    int64_t wsmod_pad = 0;
    double* modbuf[9] = {};
    // INT8 modular workspace: byte limb planes (4 each) of base, ping, pong
    int64_t wsi8_pad = 0;
    uint8_t* i8buf[12] = {};
    // plan-step progress of the running chain (pinned, mapped): kernels store
    // step+1 at the start of each step, so after an asynchronous device fault
    // the host still reads which step failed (BackendStepError, errors.py:43-49)
    uint32_t* progress_host = nullptr;
    uint32_t* progress_dev = nullptr;
    int fault_step = -1;  // test hook (mxp_debug_inject_fault): trap at this step
    // in-kernel clock of the last batched K3H launch: {clock64, globaltimer}
    // at the start and the end of CTA 0 (mxp_last_kernel_clock)
    unsigned long long* stamps = nullptr;
    bool stamps_valid = false;
    // K3H's dynamic-range fixup list: fix[0] = count, fix[1 ..] matrix indices
    int* fix = nullptr;
    int64_t fix_cap = 0;
    // host-API staging device buffers
    size_t io_bytes = 0;
    void* d_in = nullptr;
    void* d_in2 = nullptr;
    void* d_out = nullptr;
    // pinned staging for pageable host buffers (mxp_power_batched): two in and
    // two out slots of stage_bytes each, and the copy threads
    size_t stage_bytes = 0;
    char* stage_in = nullptr;
    char* stage_out = nullptr;
    HostPool* pool = nullptr;

    // captured chains, keyed by (mode, n, k, in, out); bounded LRU (callers that
    // pass fresh buffers every call would otherwise grow it without limit)
    struct CachedGraph {
        cudaGraphExec_t exec;
        int64_t launches;
        uint64_t last_use;
    };
    std::map<GraphKey, CachedGraph> graphs;
    uint64_t graph_clock = 0;
    static constexpr size_t kMaxGraphs = 32;

    void drop_graphs() {
        for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
        graphs.clear();
    }
    void evict_lru() {
        while (graphs.size() >= kMaxGraphs) {
            auto victim = graphs.begin();
            for (auto it = graphs.begin(); it != graphs.end(); ++it)
                if (it->second.last_use < victim->second.last_use) victim = it;
            // a graph still queued on the stream must not be destroyed under it
            cudaStreamSynchronize(stream);
            cudaGraphExecDestroy(victim->second.exec);
            graphs.erase(victim);
        }
    }
};

namespace {

int check_handle(mxp_handle h) {
    if (h == nullptr) return fail(MXP_E_VALIDATION, "null handle");
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    return MXP_OK;
}

int validate(int mode, int64_t n, int64_t k) {
    if (mode != MXP_F32 && mode != MXP_F64)
        return fail(MXP_E_VALIDATION, "unknown element mode %d (expected MXP_F32 or MXP_F64)", mode);
    if (n < 1) return fail(MXP_E_VALIDATION, "matrix order must be >= 1, got %lld", (long long)n);
    if (n > 32768)
        return fail(MXP_E_UNSUPPORTED, "matrix order %lld exceeds the supported 32768",
                    (long long)n);
    if (k < 0) return fail(MXP_E_VALIDATION, "power must be >= 0, got %lld", (long long)k);
    return MXP_OK;
}

size_t elem_size(int mode) { return mode == MXP_F64 ? 8 : 4; }

void stats_reset(mxp_stats* st) {
    if (!st) return;
    std::memset(st, 0, sizeof *st);
    st->failed_step = -1;
}

// The fp32 workspace for padded order n_pad: 6 planes (allocated for the
// largest order seen, used with stride n_pad), the split-K factor of n_pad
// (and, for the two-launch split-K, its partial-sum buffer).  Every call
// runs at its own n_pad, whatever larger order the handle served before, so
// a result does not depend on the handle's history.
int ensure_ws32(mxp_handle h, int64_t n_pad) {
    h->rhs_mode = -1;
    if (h->ws32_cap < n_pad) {
        for (auto& p : h->planes) {
            if (p) cudaFree(p);
            p = nullptr;
        }
        h->drop_graphs();
        h->ws32_cap = 0;
        h->ws32_pad = 0;
        const size_t bytes = static_cast<size_t>(n_pad) * n_pad * 4;
        for (auto& p : h->planes) MXP_CUDA(cudaMalloc(&p, bytes));
        h->ws32_cap = n_pad;
    }
    if (h->ws32_pad != n_pad) {
        h->splits = (k1_block_n((int)n_pad, h->num_sms) == 128)
                        ? k1_split_k((int)n_pad, (int)n_pad, h->num_sms)
                        : 1;
        h->ws32_pad = n_pad;
    }
    return MXP_OK;
}

// (Re-)encode the TMA maps of the 6 planes for the current n_pad.
int encode_ws32(mxp_handle h, int64_t n_pad) {
    for (int i = 0; i < 6; ++i) {
        if (!encode_plane_map(&h->map_a[i], h->planes[i], (int)n_pad, 32, 128, false) ||
            !encode_plane_map(&h->map_b[i], h->planes[i], (int)n_pad, 32, 32, true))
            return fail(MXP_E_CUDA, "cuTensorMapEncodeTiled failed (n_pad=%lld)", (long long)n_pad);
    }
    return MXP_OK;
}

// K1PH workspace for n_pad (allocated for the largest order seen; the TMA
// maps are re-encoded when the order changes — captured graphs keep their own
// copies, and the buffers they point into stay allocated).
int ensure_ws16(mxp_handle h, int64_t n_pad) {
    if (h->ws16_pad == n_pad) return MXP_OK;
    if (h->ws16_cap < n_pad) {
        h->drop_graphs();
        for (auto& p : h->planes16) {
            if (p) cudaFree(p);
            p = nullptr;
        }
        if (h->fbuf) cudaFree(h->fbuf);
        h->fbuf = nullptr;
        h->ws16_cap = h->ws16_pad = 0;
        const size_t n2 = static_cast<size_t>(n_pad) * n_pad;
        for (auto& p : h->planes16) MXP_CUDA(cudaMalloc(&p, n2 * 2));
        MXP_CUDA(cudaMalloc(&h->fbuf, n2 * 4));
        h->ws16_cap = n_pad;
    }
    if (!h->f16state) MXP_CUDA(cudaMalloc(&h->f16state, f16_chain_state_bytes()));
    for (int i = 0; i < 3; ++i) {
        F16Maps& m = h->maps16[i];
        if (!encode_plane16_map(&m.a0, h->planes16[2 * i], (int)n_pad, 128) ||
            !encode_plane16_map(&m.a1, h->planes16[2 * i + 1], (int)n_pad, 128) ||
            !encode_plane16_map(&m.b0, h->planes16[2 * i], (int)n_pad, 64) ||
            !encode_plane16_map(&m.b1, h->planes16[2 * i + 1], (int)n_pad, 64))
            return fail(MXP_E_CUDA, "cuTensorMapEncodeTiled (fp16) failed (n_pad=%lld)", (long long)n_pad);
    }
    h->ws16_pad = n_pad;
    return MXP_OK;
}

// Padded order a K1PH chain runs at, 0 when the chain stays on 3xTF32: the
// CTA-pair sizes (roundup(n, 128) a multiple of 256, >= 1024), and beyond
// K1C's one-launch range (n > 1408) every other order, padded to 256.
int64_t k1ph_pad(mxp_handle h, int64_t n) {
    if (h->f32_datapath != MXP_DATAPATH_AUTO || n <= kSmallMax) return 0;
    if (k1ph_eligible(round_up(n, 128))) return round_up(n, 128);
    return n > 1408 ? round_up(n, 256) : 0;
}
bool use_k1ph(mxp_handle h, int64_t n) { return k1ph_pad(h, n) != 0; }

int ensure_ws64(mxp_handle h, int64_t n_pad) {
    h->rhs_mode = -1;
    if (h->ws64_pad >= n_pad) return MXP_OK;
    for (auto& p : h->f64buf) {
        if (p) cudaFree(p);
        p = nullptr;
    }
    h->drop_graphs();
    h->ws64_pad = 0;
    const size_t bytes = static_cast<size_t>(n_pad) * n_pad * 8;
    for (auto& p : h->f64buf) MXP_CUDA(cudaMalloc(&p, bytes));
    h->ws64_pad = n_pad;
    return MXP_OK;
}

int ensure_io(mxp_handle h, size_t bytes) {
    if (h->io_bytes >= bytes) return MXP_OK;
    // graphs captured on the old staging buffers would replay into freed memory
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    h->drop_graphs();
    if (h->d_in) cudaFree(h->d_in);
    if (h->d_in2) cudaFree(h->d_in2);
    if (h->d_out) cudaFree(h->d_out);
    h->d_in = h->d_in2 = h->d_out = nullptr;
    h->io_bytes = 0;
    MXP_CUDA(cudaMalloc(&h->d_in, bytes));
    MXP_CUDA(cudaMalloc(&h->d_in2, bytes));
    MXP_CUDA(cudaMalloc(&h->d_out, bytes));
    h->io_bytes = bytes;
    return MXP_OK;
}

// ---- enqueue helpers (no validation; stream = h->stream) -----------------

int enqueue_chain_tf32(mxp_handle h, int64_t n, const PlanBits& plan, const float* dA,
                       float* dOut, int64_t* launches, int64_t* failed, const int* gate);

// K1PH chain (scaled fp16x2 planes, one exponent per matrix), then the 3xTF32
// chain gated on the dynamic-range flag the GEMMs raise (no-op launches
// unless a product lost range).  Planes: 0 base, 1 ping, 2 pong; chain state
// index 0 = the base, s + 1 = the product of step s.
int enqueue_chain_f16x2(mxp_handle h, int64_t n, const PlanBits& plan, const float* dA,
                        float* dOut, int64_t* launches, int64_t* failed) {
    const int64_t n_pad = k1ph_pad(h, n);
    int rc = ensure_ws16(h, n_pad);
    if (rc) return rc;
    const int np = (int)n_pad;
    void* st = h->f16state;
    cudaError_t e = cudaMemsetAsync(st, 0, f16_chain_state_bytes(), h->stream);
    if (e == cudaSuccess)
        e = launch_split16(dA, (int)n, (int)n, h->planes16[0], h->planes16[1], np, st, 0, -1, -1,
                           h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "k1ph split");
    *launches += 2;
    int acc = 0, acc_i = 0;  // plane pair of the running power, its state index
    for (int s = 0; s < plan.len; ++s) {
        const bool mult = plan_is_mult(plan, s);
        const bool last = (s == plan.len - 1);
        const int dst = (acc == 1) ? 2 : 1;
        const int rhs = mult ? 0 : acc, rhs_i = mult ? 0 : acc_i;
        e = launch_progress_mark(h->progress_dev, static_cast<uint32_t>(s + 1), s == h->fault_step,
                                 h->stream);
        if (e == cudaSuccess)
            e = launch_k1ph_gemm(h->maps16[acc], h->maps16[rhs], np, last ? dOut : h->fbuf,
                                 last ? (int)n : np, last ? (int)n : np, st, acc_i, rhs_i,
                                 last ? -1 : s + 1, h->num_sms, h->stream);
        if (e == cudaSuccess && !last)
            e = launch_split16(h->fbuf, np, np, h->planes16[2 * dst], h->planes16[2 * dst + 1], np, st,
                               s + 1, acc_i, rhs_i, h->stream);
        if (e != cudaSuccess) {
            *failed = s;
            return cuda_fail(e, "k1ph_gemm_f16x2");
        }
        *launches += last ? 2 : 3;
        acc = dst;
        acc_i = s + 1;
    }
    // the 3xTF32 recomputation, every launch gated on the flag
    int64_t gated = 0;
    rc = enqueue_chain_tf32(h, n, plan, dA, dOut, &gated, failed, f16_chain_flag(st));
    *launches += gated;
    return rc;
}

// Single-matrix FP32 chain for n > kSmallMax: K1PH at the CTA-pair sizes
// (MXP_DATAPATH_AUTO), else 3xTF32 through K1 / K1C / K1P.
int enqueue_chain_f32(mxp_handle h, int64_t n, const PlanBits& plan, const float* dA,
                      float* dOut, int64_t* launches, int64_t* failed) {
    h->f16_ran = use_k1ph(h, n);
    if (h->f16_ran) return enqueue_chain_f16x2(h, n, plan, dA, dOut, launches, failed);
    return enqueue_chain_tf32(h, n, plan, dA, dOut, launches, failed, nullptr);
}

// 3xTF32 chain for n > kSmallMax through K1, planes padded to 128.  gate
// (device, may be null): every launch is a no-op unless *gate != 0.
int enqueue_chain_tf32(mxp_handle h, int64_t n, const PlanBits& plan, const float* dA,
                       float* dOut, int64_t* launches, int64_t* failed, const int* gate) {
    const int64_t n_pad = round_up(n, 128);
    int rc = ensure_ws32(h, n_pad);
    if (rc) return rc;
    rc = encode_ws32(h, h->ws32_pad);
    if (rc) return rc;
    const int np = (int)h->ws32_pad;  // planes are laid out with the workspace stride
    const int bn = k1_block_n(np, h->num_sms);
    cudaError_t e = launch_split(dA, (int)n, (int)n, h->planes[0], h->planes[1], np, h->stream, gate);
    if (e != cudaSuccess) return cuda_fail(e, "split");
    ++*launches;
    if (bn == 128 && gate == nullptr) {
        // the whole chain in one launch when every split-K cluster fits at once
        e = launch_k1c_chain(h->map_a, h->map_b, h->planes, plan, np, h->splits, dOut, (int)n,
                             h->bar_ctr, h->progress_dev, h->fault_step, h->stream);
        if (e == cudaSuccess) {
            ++*launches;
            return MXP_OK;
        }
        if (e != cudaErrorNotSupported) return cuda_fail(e, "k1c_chain_3xtf32");
    }
    int acc = 0;  // plane pair index: 0 base, 1 ping, 2 pong
    for (int s = 0; s < plan.len; ++s) {
        const bool mult = plan_is_mult(plan, s);
        const bool last = (s == plan.len - 1);
        const int dst = (acc == 1) ? 2 : 1;
        const int rhs = mult ? 0 : acc;
        if (gate == nullptr) {  // (a gated recomputation keeps the K1PH chain's marks)
            e = launch_progress_mark(h->progress_dev, static_cast<uint32_t>(s + 1),
                                     s == h->fault_step, h->stream);
            if (e != cudaSuccess) {
                *failed = s;
                return cuda_fail(e, "progress mark");
            }
            ++*launches;
        }
        GemmPlanes m;
        m.a_hi = h->map_a[2 * acc];
        m.a_lo = h->map_a[2 * acc + 1];
        m.b_hi = h->map_b[2 * rhs];
        m.b_lo = h->map_b[2 * rhs + 1];
        e = launch_k1_gemm_rows(m, np, np, bn, last ? dOut : nullptr, (int)n, (int)n, (int)n,
                                last ? nullptr : h->planes[2 * dst],
                                last ? nullptr : h->planes[2 * dst + 1], h->stream, h->splits, gate);
        if (e != cudaSuccess) {
            *failed = s;
            return cuda_fail(e, "k1_gemm_3xtf32");
        }
        ++*launches;
        acc = dst;
    }
    return MXP_OK;
}

int enqueue_chain_f64(mxp_handle h, int64_t n, const PlanBits& plan, const double* dA,
                      double* dOut, int64_t* launches, int64_t* failed) {
    const int64_t n_pad = f64_pad((int)n);
    int rc = ensure_ws64(h, n_pad);
    if (rc) return rc;
    double** b = h->f64buf;
    cudaError_t e = launch_f64_pad(dA, (int)n, b[0], (int)n_pad, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "f64_pad");
    ++*launches;
    int acc = 0;
    for (int s = 0; s < plan.len; ++s) {
        const bool mult = plan_is_mult(plan, s);
        const int dst = (acc == 1) ? 2 : 1;
        e = launch_progress_mark(h->progress_dev, static_cast<uint32_t>(s + 1), s == h->fault_step,
                                 h->stream);
        if (e == cudaSuccess)
            e = launch_f64_gemm(b[acc], mult ? b[0] : b[acc], b[dst], (int)n_pad, h->stream);
        if (e != cudaSuccess) {
            *failed = s;
            return cuda_fail(e, "f64_gemm");
        }
        *launches += 2;
        acc = dst;
    }
    e = launch_f64_unpad(b[acc], (int)n_pad, dOut, (int)n, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "f64_unpad");
    ++*launches;
    return MXP_OK;
}

// Enqueue A^k for one matrix (k >= 2) on h->stream.
int enqueue_power(mxp_handle h, int mode, int64_t n, int64_t k, const void* dA, void* dOut,
                  int64_t* launches, int64_t* failed) {
    const PlanBits plan = make_plan(k);
    if (mode == MXP_F32) {
        if (n <= kSmallMax) {
            int variant = -1;
            cudaError_t e = launch_k3_batched(static_cast<const float*>(dA),
                                              static_cast<float*>(dOut), (int)n, 1, plan, 1,
                                              nullptr, &variant, h->fix, h->stream);
            if (e != cudaSuccess) {
                *failed = 0;
                return cuda_fail(e, "k3_batched_power");
            }
            *launches += (variant == 0) ? 2 : 1;  // K3H + its (usually empty) K3B fixup pass
            return MXP_OK;
        }
        return enqueue_chain_f32(h, n, plan, static_cast<const float*>(dA),
                                 static_cast<float*>(dOut), launches, failed);
    }
    return enqueue_chain_f64(h, n, plan, static_cast<const double*>(dA),
                             static_cast<double*>(dOut), launches, failed);
}

// k in {0, 1}: identity / bitwise copy, zero multiplies.
int enqueue_trivial(mxp_handle h, int mode, int64_t n, int64_t k, const void* dA, void* dOut,
                    int64_t batch, int64_t* launches) {
    const size_t bytes = static_cast<size_t>(n) * n * elem_size(mode);
    for (int64_t b = 0; b < batch; ++b) {
        void* o = static_cast<char*>(dOut) + b * bytes;
        const void* a = static_cast<const char*>(dA) + b * bytes;
        if (k == 1) {
            if (o != a) MXP_CUDA(cudaMemcpyAsync(o, a, bytes, cudaMemcpyDeviceToDevice, h->stream));
        } else {
            cudaError_t e = (mode == MXP_F64)
                                ? launch_identity_f64(static_cast<double*>(o), (int)n, h->stream)
                                : launch_identity_f32(static_cast<float*>(o), (int)n, h->stream);
            if (e != cudaSuccess) return cuda_fail(e, "identity");
            ++*launches;
        }
    }
    return MXP_OK;
}

// plan step index of the last progress mark (-1: none this call)
int64_t progress_step(mxp_handle h) {
    return static_cast<int64_t>(*reinterpret_cast<volatile uint32_t*>(h->progress_host)) - 1;
}

// errors an earlier kernel's fault leaves behind (sticky): they surface at
// whatever runtime call comes next, not at the launch that caused them
bool is_async_fault(cudaError_t e) {
    return e == cudaErrorLaunchFailure || e == cudaErrorIllegalAddress ||
           e == cudaErrorIllegalInstruction || e == cudaErrorMisalignedAddress ||
           e == cudaErrorHardwareStackError || e == cudaErrorAssert ||
           e == cudaErrorInvalidAddressSpace || e == cudaErrorInvalidPc ||
           e == cudaErrorLaunchTimeout;
}

void fill_plan_stats(mxp_stats* st, int64_t k, int64_t batch) {
    if (!st) return;
    const PlanBits p = make_plan(k);
    st->multiply_count = static_cast<int64_t>(p.len) * batch;
    st->square_count = static_cast<int64_t>(p.squares) * batch;
}

// Run A^k on device through a cached CUDA graph (single matrix).
int run_power_graph(mxp_handle h, int mode, int64_t n, int64_t k, const void* dA, void* dOut,
                    mxp_stats* st) {
    int64_t launches = 0, failed = -1;
    GraphKey key{mode, n, k, dA, dOut};
    auto it = h->graphs.find(key);
    if (it == h->graphs.end()) {
        // workspace must exist before capture (no cudaMalloc inside capture)
        if (mode == MXP_F32 && n > kSmallMax) {
            int rc = ensure_ws32(h, round_up(n, 128));
            if (rc == MXP_OK && use_k1ph(h, n)) rc = ensure_ws16(h, k1ph_pad(h, n));
            if (rc) return rc;
        } else if (mode == MXP_F64) {
            int rc = ensure_ws64(h, f64_pad((int)n));
            if (rc) return rc;
        }
        cudaGraph_t g = nullptr;
        MXP_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_power(h, mode, n, k, dA, dOut, &launches, &failed);
        cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
        if (rc) {
            if (g) cudaGraphDestroy(g);
            if (st) st->failed_step = failed;
            return rc;
        }
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
        cudaGraphExec_t ge = nullptr;
        ce = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate");
        h->evict_lru();
        it = h->graphs.emplace(key, mxp_handle_s::CachedGraph{ge, launches, 0}).first;
    }
    // the chain overwrites the workspace planes a prepared right-hand side
    // lives in (cache hit or miss alike)
    h->rhs_mode = -1;
    h->f16_ran = mode == MXP_F32 && use_k1ph(h, n);
    it->second.last_use = ++h->graph_clock;
    cudaError_t e = cudaGraphLaunch(it->second.exec, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
    if (st) st->launches += it->second.launches;
    return MXP_OK;
}

}  // namespace

// for the other translation units of the library (mxp_multicast.cu)
int mxp_internal_fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
int mxp_internal_device(mxp_handle h) { return h->device; }

// =====================================================================
extern "C" {

int mxp_debug_inject_fault(mxp_handle h, int64_t step) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (step < -1 || step > 127) return fail(MXP_E_VALIDATION, "fault step must be in [-1, 127]");
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    h->drop_graphs();  // captured chains carry the old setting
    h->fault_step = static_cast<int>(step);
    return MXP_OK;
}

int mxp_version(int* major, int* minor) {
    if (major) *major = 0;
    if (minor) *minor = 1;
    return MXP_OK;
}

const char* mxp_status_string(int status) {
    switch (status) {
        case MXP_OK: return "MXP_OK";
        case MXP_E_VALIDATION: return "MXP_E_VALIDATION";
        case MXP_E_UNSUPPORTED: return "MXP_E_UNSUPPORTED";
        case MXP_E_DEVICE_UNAVAILABLE: return "MXP_E_DEVICE_UNAVAILABLE";
        case MXP_E_CUDA: return "MXP_E_CUDA";
        case MXP_E_NCCL: return "MXP_E_NCCL";
        default: return "MXP_E_UNKNOWN";
    }
}

int mxp_last_error(char* buf, size_t len) {
    if (buf && len) {
        std::strncpy(buf, g_err.c_str(), len - 1);
        buf[len - 1] = '\0';
    }
    return MXP_OK;
}

int mxp_plan(int64_t k, char* steps, int64_t cap, int64_t* count) {
    if (k < 0) return fail(MXP_E_VALIDATION, "power must be >= 0, got %lld", (long long)k);
    const PlanBits p = make_plan(k);
    for (int s = 0; s < p.len && s < cap; ++s) steps[s] = plan_is_mult(p, s) ? 'M' : 'S';
    if (count) *count = p.len;
    return MXP_OK;
}

int mxp_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        if (count) *count = 0;
        return fail(MXP_E_DEVICE_UNAVAILABLE, "no CUDA device: %s", cudaGetErrorString(e));
    }
    if (count) *count = c;
    return MXP_OK;
}

int mxp_create(int device, mxp_handle* out) {
    if (!out) return fail(MXP_E_VALIDATION, "null output pointer");
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        return fail(MXP_E_DEVICE_UNAVAILABLE, "no CUDA device available");
    if (device < 0 || device >= count)
        return fail(MXP_E_VALIDATION, "device %d out of range [0, %d)", device, count);
    cudaDeviceProp prop;
    MXP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(MXP_E_DEVICE_UNAVAILABLE,
                    "device %d is sm_%d%d; this build targets sm_100a (B200) only", device,
                    prop.major, prop.minor);
    MXP_CUDA(cudaSetDevice(device));
    MXP_CUDA(prepare_kernels());
    auto* h = new mxp_handle_s();
    h->device = device;
    h->num_sms = prop.multiProcessorCount;
    cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->copy_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->copy_out, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev1);
    if (e == cudaSuccess) e = cudaMalloc(&h->bar_ctr, 256);
    if (e == cudaSuccess) e = cudaMemset(h->bar_ctr, 0, 256);  // K1C keeps it zero between launches
    if (e == cudaSuccess) e = cudaMalloc(&h->stamps, 64);
    if (e == cudaSuccess) e = cudaMalloc(&h->fix, (1 + 1024) * sizeof(int));
    if (e == cudaSuccess) {
        h->fix_cap = 1024;
        e = cudaMemset(h->fix, 0, sizeof(int));
    }
    if (e == cudaSuccess)
        e = cudaHostAlloc(reinterpret_cast<void**>(&h->progress_host), 64, cudaHostAllocMapped);
    if (e == cudaSuccess)
        e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->progress_dev), h->progress_host, 0);
    if (e != cudaSuccess) {
        delete h;
        return cuda_fail(e, "stream/event creation");
    }
    *out = h;
    return MXP_OK;
}

int mxp_destroy(mxp_handle h) {
    if (!h) return MXP_OK;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    h->drop_graphs();
    for (auto p : h->planes)
        if (p) cudaFree(p);
    for (auto p : h->planes16)
        if (p) cudaFree(p);
    if (h->fbuf) cudaFree(h->fbuf);
    if (h->f16state) cudaFree(h->f16state);
    if (h->bar_ctr) cudaFree(h->bar_ctr);
    if (h->stamps) cudaFree(h->stamps);
    if (h->fix) cudaFree(h->fix);
    if (h->progress_host) cudaFreeHost(h->progress_host);
    for (auto p : h->f64buf)
        if (p) cudaFree(p);
    for (auto p : h->modbuf)
        if (p) cudaFree(p);
    for (auto p : h->i8buf)
        if (p) cudaFree(p);
    if (h->d_in) cudaFree(h->d_in);
    if (h->d_in2) cudaFree(h->d_in2);
    if (h->d_out) cudaFree(h->d_out);
    if (h->stage_in) cudaFreeHost(h->stage_in);
    if (h->stage_out) cudaFreeHost(h->stage_out);
    delete h->pool;
    cudaEventDestroy(h->ev0);
    cudaEventDestroy(h->ev1);
    cudaStreamDestroy(h->stream);
    cudaStreamDestroy(h->copy_in);
    cudaStreamDestroy(h->copy_out);
    delete h;
    return MXP_OK;
}

int mxp_get_stream(mxp_handle h, void** stream) {
    if (!h || !stream) return fail(MXP_E_VALIDATION, "null argument");
    *stream = h->stream;
    return MXP_OK;
}

int mxp_num_sms(mxp_handle h, int* sms) {
    if (!h || !sms) return fail(MXP_E_VALIDATION, "null argument");
    *sms = h->num_sms;
    return MXP_OK;
}

int mxp_synchronize(mxp_handle h) {
    int rc = check_handle(h);
    if (rc) return rc;
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    return MXP_OK;
}

int mxp_alloc(mxp_handle h, size_t bytes, void** dptr) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!dptr) return fail(MXP_E_VALIDATION, "null output pointer");
    MXP_CUDA(cudaMalloc(dptr, bytes ? bytes : 16));
    return MXP_OK;
}

int mxp_free(mxp_handle h, void* dptr) {
    int rc = check_handle(h);
    if (rc) return rc;
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    MXP_CUDA(cudaFree(dptr));
    return MXP_OK;
}

int mxp_host_alloc(mxp_handle h, size_t bytes, void** hptr) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!hptr) return fail(MXP_E_VALIDATION, "null output pointer");
    MXP_CUDA(cudaHostAlloc(hptr, bytes ? bytes : 16, cudaHostAllocPortable));
    return MXP_OK;
}

int mxp_host_free(mxp_handle h, void* hptr) {
    int rc = check_handle(h);
    if (rc) return rc;
    MXP_CUDA(cudaFreeHost(hptr));
    return MXP_OK;
}

int mxp_upload(mxp_handle h, void* dst, const void* src, size_t bytes) {
    int rc = check_handle(h);
    if (rc) return rc;
    MXP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    return MXP_OK;
}

int mxp_download(mxp_handle h, void* dst, const void* src, size_t bytes) {
    int rc = check_handle(h);
    if (rc) return rc;
    MXP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    return MXP_OK;
}

int mxp_copy2d_device(mxp_handle h, void* dst, size_t dpitch, const void* src, size_t spitch,
                      size_t width, size_t rows) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!dst || !src) return fail(MXP_E_VALIDATION, "null device pointer");
    if (width > dpitch || width > spitch) return fail(MXP_E_VALIDATION, "width exceeds a pitch");
    MXP_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToDevice,
                               h->stream));
    return MXP_OK;
}

int mxp_gemm(mxp_handle h, int mode, int64_t n, const void* dA, const void* dB, void* dC) {
    int rc = check_handle(h);
    if (rc) return rc;
    rc = validate(mode, n, 2);
    if (rc) return rc;
    if (!dA || !dB || !dC) return fail(MXP_E_VALIDATION, "null device pointer");
    if (mode == MXP_F32) {
        const int64_t n_pad = round_up(n, 128);
        rc = ensure_ws32(h, n_pad);
        if (rc) return rc;
        rc = encode_ws32(h, h->ws32_pad);
        if (rc) return rc;
        const int np = (int)h->ws32_pad;
        cudaError_t e = launch_split(static_cast<const float*>(dA), (int)n, (int)n, h->planes[0],
                                     h->planes[1], np, h->stream);
        if (e == cudaSuccess)
            e = launch_split(static_cast<const float*>(dB), (int)n, (int)n, h->planes[2],
                             h->planes[3], np, h->stream);
        if (e != cudaSuccess) return cuda_fail(e, "split");
        GemmPlanes m{h->map_a[0], h->map_a[1], h->map_b[2], h->map_b[3]};
        e = launch_k1_gemm_rows(m, np, np, k1_block_n(np, h->num_sms), static_cast<float*>(dC),
                                (int)n, (int)n, (int)n, nullptr, nullptr, h->stream, h->splits);
        if (e != cudaSuccess) return cuda_fail(e, "k1_gemm_3xtf32");
        return MXP_OK;
    }
    const int64_t n_pad = f64_pad((int)n);
    rc = ensure_ws64(h, n_pad);
    if (rc) return rc;
    double** b = h->f64buf;
    cudaError_t e = launch_f64_pad(static_cast<const double*>(dA), (int)n, b[0], (int)n_pad, h->stream);
    if (e == cudaSuccess)
        e = launch_f64_pad(static_cast<const double*>(dB), (int)n, b[1], (int)n_pad, h->stream);
    if (e == cudaSuccess) e = launch_f64_gemm(b[0], b[1], b[2], (int)n_pad, h->stream);
    if (e == cudaSuccess)
        e = launch_f64_unpad(b[2], (int)n_pad, static_cast<double*>(dC), (int)n, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "f64 gemm");
    return MXP_OK;
}

// The right-hand side of a row-block multiply, prepared once (split into tf32
// hi/lo planes, or padded for FP64) in the handle's workspace.
int mxp_gemm_prepare_rhs(mxp_handle h, int mode, int64_t n, const void* dB) {
    int rc = check_handle(h);
    if (rc) return rc;
    rc = validate(mode, n, 2);
    if (rc) return rc;
    if (!dB) return fail(MXP_E_VALIDATION, "null device pointer");
    const int64_t n_pad = round_up(n, 128);
    if (mode == MXP_F32) {
        rc = ensure_ws32(h, n_pad);
        if (rc) return rc;
        cudaError_t e = launch_split(static_cast<const float*>(dB), (int)n, (int)n, h->planes[2],
                                     h->planes[3], (int)h->ws32_pad, h->stream);
        if (e != cudaSuccess) return cuda_fail(e, "split");
    } else {
        rc = ensure_ws64(h, n_pad);
        if (rc) return rc;
        cudaError_t e = launch_f64_pad(static_cast<const double*>(dB), (int)n, h->f64buf[1],
                                       (int)n_pad, h->stream);
        if (e != cudaSuccess) return cuda_fail(e, "f64 pad");
    }
    h->rhs_mode = mode;
    h->rhs_n = n;
    return MXP_OK;
}

// C[rows x n] = A[rows x n] * (the prepared right-hand side).
int mxp_gemm_rows_prepared(mxp_handle h, int mode, int64_t n, int64_t rows, const void* dA,
                           void* dC) {
    int rc = check_handle(h);
    if (rc) return rc;
    rc = validate(mode, n, 2);
    if (rc) return rc;
    if (rows < 1 || rows > n)
        return fail(MXP_E_VALIDATION, "row block must satisfy 1 <= rows <= n, got %lld", (long long)rows);
    if (!dA || !dC) return fail(MXP_E_VALIDATION, "null device pointer");
    if (h->rhs_mode != mode || h->rhs_n != n)
        return fail(MXP_E_VALIDATION, "no right-hand side prepared for this mode and n "
                                      "(call mxp_gemm_prepare_rhs first)");
    const int64_t n_pad = round_up(n, 128);
    int64_t r_pad = round_up(rows, 128);
    if (mode == MXP_F32) {
        const int np = (int)h->ws32_pad;
        const int bn = k1_block_n(np, h->num_sms);
        if (bn == 256) r_pad = round_up(rows, 256);  // CTA-pair tiles are 256 rows
        CUtensorMap a_hi, a_lo, b_hi, b_lo;
        if (!encode_plane_map(&a_hi, h->planes[0], np, 32, 128, false, (int)r_pad) ||
            !encode_plane_map(&a_lo, h->planes[1], np, 32, 128, false, (int)r_pad) ||
            !encode_plane_map(&b_hi, h->planes[2], np, 32, 32, true) ||
            !encode_plane_map(&b_lo, h->planes[3], np, 32, 32, true))
            return fail(MXP_E_CUDA, "cuTensorMapEncodeTiled failed");
        cudaError_t e = launch_split_rows(static_cast<const float*>(dA), (int)n, (int)n, (int)rows,
                                          h->planes[0], h->planes[1], np, (int)r_pad, h->stream);
        if (e != cudaSuccess) return cuda_fail(e, "split");
        GemmPlanes m{a_hi, a_lo, b_hi, b_lo};
        // same k-split as the full multiply / chain: bitwise-identical rows
        e = launch_k1_gemm_rows(m, np, (int)r_pad, bn, static_cast<float*>(dC), (int)n, (int)rows,
                                (int)n, nullptr, nullptr, h->stream, h->splits);
        if (e != cudaSuccess) return cuda_fail(e, "k1_gemm_3xtf32");
        return MXP_OK;
    }
    double** b = h->f64buf;
    cudaError_t e = launch_f64_pad_rows(static_cast<const double*>(dA), (int)n, (int)rows, b[0],
                                        (int)n_pad, (int)r_pad, h->stream);
    if (e == cudaSuccess) e = launch_f64_gemm_rows(b[0], b[1], b[2], (int)n_pad, (int)r_pad, h->stream);
    if (e == cudaSuccess)
        e = launch_f64_unpad_rows(b[2], (int)n_pad, static_cast<double*>(dC), (int)n, (int)rows,
                                  h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "f64 gemm rows");
    return MXP_OK;
}

// ---------------------------------------------------------------- fused row-sharded exchange
// cuMemGetAddressRange through the runtime's driver entry point (the library
// does not link libcuda directly: it must load on machines without a driver).
static int alloc_base(const void* p, CUdeviceptr* base) {
    using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static Fn fn = nullptr;
    if (fn == nullptr) {
        void* q = nullptr;
        cudaDriverEntryPointQueryResult r;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &q, cudaEnableDefault, &r) !=
                cudaSuccess ||
            r != cudaDriverEntryPointSuccess)
            return fail(MXP_E_CUDA, "cuMemGetAddressRange unavailable");
        fn = reinterpret_cast<Fn>(q);
    }
    size_t size = 0;
    if (fn(base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
        return fail(MXP_E_CUDA, "cuMemGetAddressRange failed");
    return MXP_OK;
}

// The exported handle is the CUDA IPC handle of the ALLOCATION that contains
// dptr plus dptr's byte offset inside it (sub-allocated pointers, e.g. from a
// caching allocator, map to the allocation base on the other side).
int mxp_ipc_get_handle(mxp_handle h, const void* dptr, void* handle_out) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!dptr || !handle_out) return fail(MXP_E_VALIDATION, "null pointer");
    cudaIpcMemHandle_t ih;
    MXP_CUDA(cudaIpcGetMemHandle(&ih, const_cast<void*>(dptr)));
    CUdeviceptr base = 0;
    rc = alloc_base(dptr, &base);
    if (rc) return rc;
    const uint64_t off = reinterpret_cast<uint64_t>(dptr) - static_cast<uint64_t>(base);
    static_assert(sizeof(ih) + sizeof(off) == MXP_IPC_HANDLE_BYTES, "ipc handle size");
    std::memcpy(handle_out, &ih, sizeof ih);
    std::memcpy(static_cast<char*>(handle_out) + sizeof ih, &off, sizeof off);
    return MXP_OK;
}

int mxp_ipc_open_handle(mxp_handle h, const void* handle, void** dptr) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!handle || !dptr) return fail(MXP_E_VALIDATION, "null pointer");
    cudaIpcMemHandle_t ih;
    uint64_t off = 0;
    std::memcpy(&ih, handle, sizeof ih);
    std::memcpy(&off, static_cast<const char*>(handle) + sizeof ih, sizeof off);
    void* base = nullptr;
    MXP_CUDA(cudaIpcOpenMemHandle(&base, ih, cudaIpcMemLazyEnablePeerAccess));
    *dptr = static_cast<char*>(base) + off;
    return MXP_OK;
}

int mxp_ipc_close_handle(mxp_handle h, void* dptr) {
    int rc = check_handle(h);
    if (rc) return rc;
    CUdeviceptr base = 0;
    rc = alloc_base(dptr, &base);
    if (rc) return rc;
    MXP_CUDA(cudaIpcCloseMemHandle(reinterpret_cast<void*>(base)));
    return MXP_OK;
}

int mxp_split_planes(mxp_handle h, int64_t n, const void* dA, void* d_hi, void* d_lo) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (n < 1) return fail(MXP_E_VALIDATION, "n must be >= 1, got %lld", (long long)n);
    if (!dA || !d_hi || !d_lo) return fail(MXP_E_VALIDATION, "null device pointer");
    cudaError_t e = launch_split(static_cast<const float*>(dA), (int)n, (int)n,
                                 static_cast<uint32_t*>(d_hi), static_cast<uint32_t*>(d_lo),
                                 (int)round_up(n, 128), h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "split");
    return MXP_OK;
}

int mxp_gemm_rows_planes_peers(mxp_handle h, int64_t n, int64_t rows, int64_t row0,
                               const void* a_hi, const void* a_lo, const void* b_hi,
                               const void* b_lo, int npeers, void* const* peer_hi,
                               void* const* peer_lo, void* const* peer_f32) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (n < 1024 || n % 256 != 0)
        return fail(MXP_E_UNSUPPORTED, "fused exchange needs n %% 256 == 0 and n >= 1024, got %lld",
                    (long long)n);
    if (rows < 256 || rows % 256 != 0 || row0 < 0 || row0 % 256 != 0 || row0 + rows > n)
        return fail(MXP_E_VALIDATION, "row block [%lld, +%lld) must be 256-aligned inside n",
                    (long long)row0, (long long)rows);
    if (npeers < 1 || npeers > kMaxPeers)
        return fail(MXP_E_VALIDATION, "1 <= npeers <= %d, got %d", kMaxPeers, npeers);
    if (!a_hi || !a_lo || !b_hi || !b_lo) return fail(MXP_E_VALIDATION, "null device pointer");
    PeerOut po;
    po.n = npeers;
    po.row0 = static_cast<int>(row0);
    for (int i = 0; i < npeers; ++i) {
        po.f32[i] = peer_f32 ? static_cast<float*>(peer_f32[i]) : nullptr;
        po.hi[i] = peer_hi ? static_cast<uint32_t*>(peer_hi[i]) : nullptr;
        po.lo[i] = peer_lo ? static_cast<uint32_t*>(peer_lo[i]) : nullptr;
        if (!po.f32[i] && (!po.hi[i] || !po.lo[i]))
            return fail(MXP_E_VALIDATION, "peer %d has no destination", i);
    }
    const size_t off = static_cast<size_t>(row0) * n;
    CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
    if (!encode_plane_map(&ma_hi, static_cast<const uint32_t*>(a_hi) + off, (int)n, 32, 128, false,
                          (int)rows) ||
        !encode_plane_map(&ma_lo, static_cast<const uint32_t*>(a_lo) + off, (int)n, 32, 128, false,
                          (int)rows) ||
        !encode_plane_map(&mb_hi, b_hi, (int)n, 32, 32, true) ||
        !encode_plane_map(&mb_lo, b_lo, (int)n, 32, 32, true))
        return fail(MXP_E_CUDA, "cuTensorMapEncodeTiled failed");
    GemmPlanes m{ma_hi, ma_lo, mb_hi, mb_lo};
    cudaError_t e = launch_k1p_gemm_peers(m, (int)n, (int)rows, (int)n, po, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "k1p_gemm_3xtf32 (fused exchange)");
    return MXP_OK;
}

int mxp_k1ph_state_bytes(size_t* bytes) {
    if (!bytes) return fail(MXP_E_VALIDATION, "null argument");
    *bytes = f16_chain_state_bytes();
    return MXP_OK;
}

namespace {
int k1ph_rows_check(int64_t n, int64_t rows, int64_t row0) {
    if (!k1ph_eligible(n))
        return fail(MXP_E_UNSUPPORTED, "K1PH row shards need n %% 256 == 0 and n >= 1024, got %lld",
                    (long long)n);
    if (rows < 256 || rows % 256 != 0 || row0 < 0 || row0 % 256 != 0 || row0 + rows > n)
        return fail(MXP_E_VALIDATION, "row block [%lld, +%lld) must be 256-aligned inside n",
                    (long long)row0, (long long)rows);
    return MXP_OK;
}
}  // namespace

int mxp_k1ph_split_base(mxp_handle h, int64_t n_true, int64_t n, const void* dA, void* h0, void* h1,
                        void* state) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!k1ph_eligible(n) || n_true < 1 || n_true > n)
        return fail(MXP_E_VALIDATION, "need n %% 256 == 0, n >= 1024 and 1 <= n_true <= n");
    if (!dA || !h0 || !h1 || !state) return fail(MXP_E_VALIDATION, "null device pointer");
    cudaError_t e = launch_split16(static_cast<const float*>(dA), (int)n_true, (int)n_true, h0, h1,
                                   (int)n, state, 0, -1, -1, h->stream);
    return e == cudaSuccess ? MXP_OK : cuda_fail(e, "k1ph base split");
}

int mxp_k1ph_gemm_rows(mxp_handle h, int64_t n, int64_t rows, int64_t row0, const void* x_h0,
                       const void* x_h1, const void* y_h0, const void* y_h1, void* out,
                       int64_t ld_out, int64_t n_out, void* state, int xi, int yi, int oi) {
    int rc = check_handle(h);
    if (rc) return rc;
    if ((rc = k1ph_rows_check(n, rows, row0))) return rc;
    if (!x_h0 || !x_h1 || !y_h0 || !y_h1 || !out || !state)
        return fail(MXP_E_VALIDATION, "null device pointer");
    if (xi < 0 || yi < 0 || xi > kF16MaxSteps || yi > kF16MaxSteps || oi > kF16MaxSteps || ld_out < 1)
        return fail(MXP_E_VALIDATION, "state index out of range");
    F16Maps x, y;
    if (!encode_plane16_map(&x.a0, x_h0, (int)n, 128) || !encode_plane16_map(&x.a1, x_h1, (int)n, 128) ||
        !encode_plane16_map(&y.b0, y_h0, (int)n, 64) || !encode_plane16_map(&y.b1, y_h1, (int)n, 64))
        return fail(MXP_E_CUDA, "cuTensorMapEncodeTiled (fp16) failed");
    cudaError_t e = launch_k1ph_gemm(x, y, (int)n, static_cast<float*>(out), (int)n_out, (int)ld_out,
                                     state, xi, yi, oi, h->num_sms, h->stream, (int)rows, (int)row0);
    return e == cudaSuccess ? MXP_OK : cuda_fail(e, "k1ph_gemm_f16x2 (row block)");
}

int mxp_k1ph_max_to_peers(mxp_handle h, const void* state, int i, int npeers,
                          void* const* peer_states) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!state || !peer_states || npeers < 1 || npeers > kF16MaxPeers || i < 0 || i > kF16MaxSteps)
        return fail(MXP_E_VALIDATION, "bad peer-state arguments");
    cudaError_t e = launch_max_to_peers(state, i, peer_states, npeers, h->stream);
    return e == cudaSuccess ? MXP_OK : cuda_fail(e, "k1ph max to peers");
}

int mxp_k1ph_split_rows_peers(mxp_handle h, int64_t n_true, int64_t n, int64_t rows, int64_t row0,
                              const void* rows_f32, void* state, int i, int xi, int yi, int npeers,
                              void* const* peer_h0, void* const* peer_h1) {
    int rc = check_handle(h);
    if (rc) return rc;
    if ((rc = k1ph_rows_check(n, rows, row0))) return rc;
    if (!rows_f32 || !state || !peer_h0 || !peer_h1 || npeers < 1 || npeers > kF16MaxPeers ||
        i < 1 || i > kF16MaxSteps || xi < 0 || yi < 0 || xi > kF16MaxSteps || yi > kF16MaxSteps ||
        n_true < 1 || n_true > n)
        return fail(MXP_E_VALIDATION, "bad split arguments");
    cudaError_t e = launch_split16_rows_peers(static_cast<const float*>(rows_f32), (int)rows, (int)row0,
                                              (int)n, (int)n_true, state, i, xi, yi, peer_h0, peer_h1,
                                              npeers, h->stream);
    return e == cudaSuccess ? MXP_OK : cuda_fail(e, "k1ph row split to peers");
}

int mxp_k1ph_read_flag(mxp_handle h, const void* state, int* raised) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!state || !raised) return fail(MXP_E_VALIDATION, "null argument");
    MXP_CUDA(cudaSetDevice(h->device));
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    int flag = 0;
    MXP_CUDA(cudaMemcpy(&flag, f16_chain_flag(const_cast<void*>(state)), sizeof flag,
                        cudaMemcpyDeviceToHost));
    *raised = flag != 0;
    return MXP_OK;
}

int mxp_gemm_rows_planes_mc(mxp_handle h, int64_t n, int64_t rows, int64_t row0, const void* a_hi,
                            const void* a_lo, const void* b_hi, const void* b_lo, void* mc_hi,
                            void* mc_lo, void* mc_f32) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (n < 1024 || n % 256 != 0)
        return fail(MXP_E_UNSUPPORTED, "fused exchange needs n %% 256 == 0 and n >= 1024, got %lld",
                    (long long)n);
    if (rows < 256 || rows % 256 != 0 || row0 < 0 || row0 % 256 != 0 || row0 + rows > n)
        return fail(MXP_E_VALIDATION, "row block [%lld, +%lld) must be 256-aligned inside n",
                    (long long)row0, (long long)rows);
    if (!a_hi || !a_lo || !b_hi || !b_lo) return fail(MXP_E_VALIDATION, "null device pointer");
    if (!mc_f32 && (!mc_hi || !mc_lo)) return fail(MXP_E_VALIDATION, "no multicast destination");
    PeerOut po;
    po.n = 1;
    po.mc = 1;
    po.row0 = static_cast<int>(row0);
    po.f32[0] = static_cast<float*>(mc_f32);
    po.hi[0] = static_cast<uint32_t*>(mc_hi);
    po.lo[0] = static_cast<uint32_t*>(mc_lo);
    const size_t off = static_cast<size_t>(row0) * n;
    CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
    if (!encode_plane_map(&ma_hi, static_cast<const uint32_t*>(a_hi) + off, (int)n, 32, 128, false,
                          (int)rows) ||
        !encode_plane_map(&ma_lo, static_cast<const uint32_t*>(a_lo) + off, (int)n, 32, 128, false,
                          (int)rows) ||
        !encode_plane_map(&mb_hi, b_hi, (int)n, 32, 32, true) ||
        !encode_plane_map(&mb_lo, b_lo, (int)n, 32, 32, true))
        return fail(MXP_E_CUDA, "cuTensorMapEncodeTiled failed");
    GemmPlanes m{ma_hi, ma_lo, mb_hi, mb_lo};
    cudaError_t e = launch_k1p_gemm_peers(m, (int)n, (int)rows, (int)n, po, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "k1p_gemm_3xtf32 (multicast exchange)");
    return MXP_OK;
}

int mxp_peer_barrier(mxp_handle h, int rank, int npeers, void* const* peer_flags, uint32_t epoch) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!peer_flags) return fail(MXP_E_VALIDATION, "null flag table");
    cudaError_t e = launch_peer_barrier(reinterpret_cast<uint32_t* const*>(peer_flags), npeers,
                                        rank, epoch, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "peer barrier");
    return MXP_OK;
}

int mxp_gemm_rows(mxp_handle h, int mode, int64_t n, int64_t rows, const void* dA, const void* dB,
                  void* dC) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (rows < 1 || rows > n)
        return fail(MXP_E_VALIDATION, "row block must satisfy 1 <= rows <= n, got %lld", (long long)rows);
    if (!dA || !dB || !dC) return fail(MXP_E_VALIDATION, "null device pointer");
    rc = mxp_gemm_prepare_rhs(h, mode, n, dB);
    if (rc) return rc;
    return mxp_gemm_rows_prepared(h, mode, n, rows, dA, dC);
}

int mxp_multiply(mxp_handle h, int mode, int64_t n, const void* hA, const void* hB, void* hC,
                 mxp_stats* st) {
    stats_reset(st);
    int rc = check_handle(h);
    if (rc) return rc;
    rc = validate(mode, n, 2);
    if (rc) return rc;
    if (!hA || !hB || !hC) return fail(MXP_E_VALIDATION, "null host pointer");
    const size_t bytes = static_cast<size_t>(n) * n * elem_size(mode);
    rc = ensure_io(h, bytes);
    if (rc) return rc;
    MXP_CUDA(cudaMemcpyAsync(h->d_in, hA, bytes, cudaMemcpyHostToDevice, h->stream));
    MXP_CUDA(cudaMemcpyAsync(h->d_in2, hB, bytes, cudaMemcpyHostToDevice, h->stream));
    MXP_CUDA(cudaEventRecord(h->ev0, h->stream));
    rc = mxp_gemm(h, mode, n, h->d_in, h->d_in2, h->d_out);
    if (rc) return rc;
    MXP_CUDA(cudaEventRecord(h->ev1, h->stream));
    MXP_CUDA(cudaMemcpyAsync(hC, h->d_out, bytes, cudaMemcpyDeviceToHost, h->stream));
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    if (st) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h->ev0, h->ev1);
        st->device_ms = ms;
        st->multiply_count = 1;
        st->launches = (mode == MXP_F32) ? 3 : 4;
        st->h2d = 2;
        st->d2h = 1;
        st->h2d_bytes = 2 * bytes;
        st->d2h_bytes = bytes;
    }
    return MXP_OK;
}

int mxp_power_device(mxp_handle h, int mode, int64_t n, int64_t k, const void* dA, void* dOut,
                     mxp_stats* st) {
    stats_reset(st);
    int rc = check_handle(h);
    if (rc) return rc;
    rc = validate(mode, n, k);
    if (rc) return rc;
    if (!dA || !dOut) return fail(MXP_E_VALIDATION, "null device pointer");
    fill_plan_stats(st, k, 1);
    if (k <= 1) {
        int64_t launches = 0;
        rc = enqueue_trivial(h, mode, n, k, dA, dOut, 1, &launches);
        if (st) st->launches = launches;
        return rc;
    }
    return run_power_graph(h, mode, n, k, dA, dOut, st);
}

int mxp_power(mxp_handle h, int mode, int64_t n, int64_t k, const void* hA, void* hOut,
              mxp_stats* st) {
    stats_reset(st);
    int rc = check_handle(h);
    if (rc) return rc;
    rc = validate(mode, n, k);
    if (rc) return rc;
    if (!hA || !hOut) return fail(MXP_E_VALIDATION, "null host pointer");
    const size_t bytes = static_cast<size_t>(n) * n * elem_size(mode);
    rc = ensure_io(h, bytes);
    if (rc) return rc;
    MXP_CUDA(cudaStreamSynchronize(h->stream));  // no earlier chain still writes progress marks
    *reinterpret_cast<volatile uint32_t*>(h->progress_host) = 0;
    MXP_CUDA(cudaMemcpyAsync(h->d_in, hA, bytes, cudaMemcpyHostToDevice, h->stream));
    MXP_CUDA(cudaEventRecord(h->ev0, h->stream));
    mxp_stats inner;
    rc = mxp_power_device(h, mode, n, k, h->d_in, h->d_out, &inner);
    if (rc) {
        if (st) st->failed_step = inner.failed_step;
        return rc;
    }
    // An asynchronous fault inside the chain surfaces at the first runtime
    // call after it: name the last plan step a kernel of this chain started
    // (-1: before the first step; the n <= 128 kernels run a whole chain per
    // CTA and leave no marks).
    cudaError_t e = cudaEventRecord(h->ev1, h->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(hOut, h->d_out, bytes, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
        if (st) st->failed_step = progress_step(h);
        return cuda_fail(e, "power chain");
    }
    if (st) {
        *st = inner;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h->ev0, h->ev1);
        st->device_ms = ms;
        st->h2d = 1;
        st->d2h = 1;
        st->h2d_bytes = bytes;
        st->d2h_bytes = bytes;
    }
    return MXP_OK;
}

int mxp_power_batched_device(mxp_handle h, int mode, int64_t n, int64_t batch, int64_t k,
                             const void* dA, void* dOut, mxp_stats* st) {
    stats_reset(st);
    int rc = check_handle(h);
    if (rc) return rc;
    rc = validate(mode, n, k);
    if (rc) return rc;
    if (batch < 0) return fail(MXP_E_VALIDATION, "batch must be >= 0, got %lld", (long long)batch);
    if (batch == 0) return MXP_OK;
    if (!dA || !dOut) return fail(MXP_E_VALIDATION, "null device pointer");
    fill_plan_stats(st, k, batch);
    int64_t launches = 0, failed = -1;
    if (k <= 1) {
        rc = enqueue_trivial(h, mode, n, k, dA, dOut, batch, &launches);
        if (st) st->launches = launches;
        return rc;
    }
    if (mode == MXP_F32 && n <= kSmallMax) {
        if (batch > h->fix_cap) {  // the fixup list holds up to one entry per matrix
            MXP_CUDA(cudaStreamSynchronize(h->stream));
            h->drop_graphs();  // captured n <= 128 chains point at the old list
            MXP_CUDA(cudaFree(h->fix));
            h->fix = nullptr;
            h->fix_cap = 0;
            MXP_CUDA(cudaMalloc(&h->fix, static_cast<size_t>(1 + batch) * sizeof(int)));
            h->fix_cap = batch;
        }
        int variant = -1;
        cudaError_t e = launch_k3_batched(static_cast<const float*>(dA), static_cast<float*>(dOut),
                                          (int)n, batch, make_plan(k), h->num_sms, h->stamps,
                                          &variant, h->fix, h->stream);
        if (e != cudaSuccess) {
            if (st) st->failed_step = 0;
            return cuda_fail(e, "k3_batched_power");
        }
        h->stamps_valid = (variant == 0);
        if (st) st->launches = (variant == 0) ? 2 : 1;
        return MXP_OK;
    }
    // n > 128 (or fp64): one chain per matrix, enqueued back to back.
    const size_t bytes = static_cast<size_t>(n) * n * elem_size(mode);
    for (int64_t b = 0; b < batch; ++b) {
        rc = enqueue_power(h, mode, n, k, static_cast<const char*>(dA) + b * bytes,
                           static_cast<char*>(dOut) + b * bytes, &launches, &failed);
        if (rc) {
            if (st) st->failed_step = failed;
            return rc;
        }
    }
    if (st) st->launches = launches;
    return MXP_OK;
}

int mxp_power_batched(mxp_handle h, int mode, int64_t n, int64_t batch, int64_t k,
                      const void* hA, void* hOut, mxp_stats* st) {
    stats_reset(st);
    int rc = check_handle(h);
    if (rc) return rc;
    rc = validate(mode, n, k);
    if (rc) return rc;
    if (batch < 0) return fail(MXP_E_VALIDATION, "batch must be >= 0, got %lld", (long long)batch);
    if (batch == 0) return MXP_OK;
    if (!hA || !hOut) return fail(MXP_E_VALIDATION, "null host pointer");
    const size_t mat = static_cast<size_t>(n) * n * elem_size(mode);
    // Pipeline in chunks: H2D (copy_in) | compute (stream) | D2H (copy_out),
    // double-buffered, so PCIe in both directions overlaps the tensor cores.
    const size_t chunk_target = size_t(MXP_E2E_CHUNK_MB) << 20;
    int64_t chunk = static_cast<int64_t>(chunk_target / mat);
    if (chunk < 1) chunk = 1;
    if (chunk > batch) chunk = batch;
    const size_t chunk_bytes = static_cast<size_t>(chunk) * mat;
    rc = ensure_io(h, 2 * chunk_bytes);  // d_in/d_out hold two chunk slots each
    if (rc) return rc;
    // Pageable caller memory goes through pinned staging slots, filled and
    // drained by the host thread pool while the GPU works on the neighbouring
    // chunk (chunk i is filled while chunk i-1 computes; it is drained two
    // chunks later, when its slot comes round again).
    const bool stage_in = is_pageable(hA), stage_out = is_pageable(hOut);
    if (stage_in || stage_out) {
        if (h->stage_bytes < chunk_bytes) {
            MXP_CUDA(cudaStreamSynchronize(h->copy_in));
            MXP_CUDA(cudaStreamSynchronize(h->copy_out));
            if (h->stage_in) cudaFreeHost(h->stage_in);
            if (h->stage_out) cudaFreeHost(h->stage_out);
            h->stage_in = h->stage_out = nullptr;
            h->stage_bytes = 0;
            MXP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h->stage_in), 2 * chunk_bytes,
                                   cudaHostAllocPortable));
            MXP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h->stage_out), 2 * chunk_bytes,
                                   cudaHostAllocPortable));
            h->stage_bytes = chunk_bytes;
        }
        if (h->pool == nullptr) {
            unsigned hw = std::thread::hardware_concurrency();
            h->pool = new HostPool(static_cast<int>(hw < 2 ? 2 : (hw > 16 ? 16 : hw)));
        }
    }
    const size_t sb = h->stage_bytes;
    // the pipeline's events, destroyed on every exit path
    struct Events {
        cudaEvent_t in_ready[2] = {}, comp_done[2] = {}, out_done[2] = {};
        ~Events() {
            for (int i = 0; i < 2; ++i) {
                if (in_ready[i]) cudaEventDestroy(in_ready[i]);
                if (comp_done[i]) cudaEventDestroy(comp_done[i]);
                if (out_done[i]) cudaEventDestroy(out_done[i]);
            }
        }
    } ev;
    cudaEvent_t* in_ready = ev.in_ready;
    cudaEvent_t* comp_done = ev.comp_done;
    cudaEvent_t* out_done = ev.out_done;
    for (int i = 0; i < 2; ++i) {
        MXP_CUDA(cudaEventCreateWithFlags(&in_ready[i], cudaEventDisableTiming));
        MXP_CUDA(cudaEventCreateWithFlags(&comp_done[i], cudaEventDisableTiming));
        MXP_CUDA(cudaEventCreateWithFlags(&out_done[i], cudaEventDisableTiming));
    }
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    auto chunk_len = [&](int64_t c) -> size_t {
        const int64_t b0 = c * chunk;
        return static_cast<size_t>((b0 + chunk <= batch) ? chunk : batch - b0) * mat;
    };
    MXP_CUDA(cudaEventRecord(h->ev0, h->stream));
    int64_t launches = 0;
    cudaError_t err = cudaSuccess;
    for (int64_t c = 0; c < nchunks && err == cudaSuccess; ++c) {
        const int slot = static_cast<int>(c & 1);
        const int64_t b0 = c * chunk;
        const int64_t nb = static_cast<int64_t>(chunk_len(c) / mat);
        const size_t nbytes = chunk_len(c);
        char* din = static_cast<char*>(h->d_in) + slot * chunk_bytes;
        char* dout = static_cast<char*>(h->d_out) + slot * chunk_bytes;
        const char* src = static_cast<const char*>(hA) + b0 * mat;
        if (stage_in || stage_out) {
            // the slot's previous chunk (c - 2) has left the staging buffers
            CopyJob jobs[2];
            int nj = 0;
            if (c >= 2) {
                if ((err = cudaEventSynchronize(in_ready[slot])) != cudaSuccess) break;
                if ((err = cudaEventSynchronize(out_done[slot])) != cudaSuccess) break;
                if (stage_out)
                    jobs[nj++] = {static_cast<char*>(hOut) + (c - 2) * chunk * mat,
                                  h->stage_out + slot * sb, chunk_len(c - 2)};
            }
            if (stage_in) {
                jobs[nj++] = {h->stage_in + slot * sb, src, nbytes};
                src = h->stage_in + slot * sb;
            }
            if (nj) pool_copy(*h->pool, jobs, nj);
        }
        if (c >= 2) MXP_CUDA(cudaStreamWaitEvent(h->copy_in, comp_done[slot], 0));
        MXP_CUDA(cudaMemcpyAsync(din, src, nbytes, cudaMemcpyHostToDevice, h->copy_in));
        MXP_CUDA(cudaEventRecord(in_ready[slot], h->copy_in));
        MXP_CUDA(cudaStreamWaitEvent(h->stream, in_ready[slot], 0));
        if (c >= 2) MXP_CUDA(cudaStreamWaitEvent(h->stream, out_done[slot], 0));
        mxp_stats inner;
        rc = mxp_power_batched_device(h, mode, n, nb, k, din, dout, &inner);
        if (rc) {
            cudaStreamSynchronize(h->copy_in);
            cudaStreamSynchronize(h->copy_out);
            if (st) st->failed_step = inner.failed_step;
            return rc;
        }
        launches += inner.launches;
        MXP_CUDA(cudaEventRecord(comp_done[slot], h->stream));
        MXP_CUDA(cudaStreamWaitEvent(h->copy_out, comp_done[slot], 0));
        void* dst = stage_out ? static_cast<void*>(h->stage_out + slot * sb)
                              : static_cast<void*>(static_cast<char*>(hOut) + b0 * mat);
        MXP_CUDA(cudaMemcpyAsync(dst, dout, nbytes, cudaMemcpyDeviceToHost, h->copy_out));
        MXP_CUDA(cudaEventRecord(out_done[slot], h->copy_out));
    }
    // drain the last (up to two) staged results
    if (stage_out && err == cudaSuccess) {
        for (int64_t c = (nchunks >= 2 ? nchunks - 2 : 0); c < nchunks && err == cudaSuccess; ++c) {
            const int slot = static_cast<int>(c & 1);
            if ((err = cudaEventSynchronize(out_done[slot])) != cudaSuccess) break;
            CopyJob job{static_cast<char*>(hOut) + c * chunk * mat, h->stage_out + slot * sb,
                        chunk_len(c)};
            pool_copy(*h->pool, &job, 1);
        }
    }
    if (err == cudaSuccess) {
        MXP_CUDA(cudaStreamWaitEvent(h->stream, out_done[0], 0));
        if (nchunks > 1) MXP_CUDA(cudaStreamWaitEvent(h->stream, out_done[1], 0));
        MXP_CUDA(cudaEventRecord(h->ev1, h->stream));
        err = cudaStreamSynchronize(h->stream);
    }
    if (err != cudaSuccess) return cuda_fail(err, "batched power");
    if (st) {
        fill_plan_stats(st, k, batch);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h->ev0, h->ev1);
        st->device_ms = ms;
        st->launches = launches;
        st->h2d = 1;
        st->d2h = 1;
        st->h2d_bytes = static_cast<int64_t>(batch * mat);
        st->d2h_bytes = static_cast<int64_t>(batch * mat);
    }
    return MXP_OK;
}

int mxp_random_device(mxp_handle h, int mode, int64_t n, int64_t batch, uint64_t seed0,
                      double lo, double hi, double scale, void* dOut) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (mode != MXP_F32 && mode != MXP_F64)
        return fail(MXP_E_VALIDATION, "unknown element mode %d", mode);
    if (n < 1) return fail(MXP_E_VALIDATION, "matrix order must be >= 1, got %lld", (long long)n);
    if (!(lo < hi)) return fail(MXP_E_VALIDATION, "need lo < hi, got [%g, %g)", lo, hi);
    if (batch < 0 || !dOut) return fail(MXP_E_VALIDATION, "bad batch or null pointer");
    if (batch == 0) return MXP_OK;
    cudaError_t e = launch_random(mode, n, batch, seed0, lo, hi, scale, dOut, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "random_kernel");
    return MXP_OK;
}

int mxp_small_kernel_for(int64_t n, int64_t k, int* kernel) {
    if (!kernel) return fail(MXP_E_VALIDATION, "null output pointer");
    if (n < 1 || n > kSmallMax || k < 2)
        return fail(MXP_E_VALIDATION, "needs 1 <= n <= %d and k >= 2", kSmallMax);
    *kernel = k3_route(static_cast<int>(n), make_plan(k)) == 0 ? MXP_KERNEL_K3H : MXP_KERNEL_K3B;
    return MXP_OK;
}

int mxp_set_f32_datapath(mxp_handle h, int datapath) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (datapath != MXP_DATAPATH_AUTO && datapath != MXP_DATAPATH_3XTF32)
        return fail(MXP_E_VALIDATION, "unknown f32 datapath %d", datapath);
    if (datapath != h->f32_datapath) {
        MXP_CUDA(cudaStreamSynchronize(h->stream));
        h->drop_graphs();  // cached chains were captured for the other datapath
        h->f32_datapath = datapath;
    }
    return MXP_OK;
}

int mxp_last_f32_fallback(mxp_handle h, int* raised) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!raised) return fail(MXP_E_VALIDATION, "null argument");
    if (!h->f16_ran || !h->f16state) return fail(MXP_E_UNSUPPORTED, "no K1PH chain ran on this handle");
    MXP_CUDA(cudaSetDevice(h->device));
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    int flag = 0;
    MXP_CUDA(cudaMemcpy(&flag, f16_chain_flag(h->f16state), sizeof(int), cudaMemcpyDeviceToHost));
    *raised = flag != 0;
    return MXP_OK;
}

int mxp_last_small_fixups(mxp_handle h, int64_t* count) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!count) return fail(MXP_E_VALIDATION, "null output pointer");
    int c = 0;
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    MXP_CUDA(cudaMemcpy(&c, h->fix, sizeof c, cudaMemcpyDeviceToHost));
    *count = c;
    return MXP_OK;
}

int mxp_last_kernel_clock(mxp_handle h, double* sm_mhz, double* kernel_ms) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (!h->stamps_valid)
        return fail(MXP_E_UNSUPPORTED, "no batched K3H launch on this handle yet");
    unsigned long long t[4];
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    MXP_CUDA(cudaMemcpy(t, h->stamps, sizeof t, cudaMemcpyDeviceToHost));
    const double cycles = static_cast<double>(t[2] - t[0]);
    const double ns = static_cast<double>(t[3] - t[1]);
    if (ns <= 0) return fail(MXP_E_CUDA, "globaltimer did not advance");
    if (sm_mhz) *sm_mhz = cycles / ns * 1e3;
    if (kernel_ms) *kernel_ms = ns * 1e-6;
    return MXP_OK;
}

int mxp_splitmix64_device(mxp_handle h, uint64_t seed, int64_t count, void* dOut) {
    int rc = check_handle(h);
    if (rc) return rc;
    if (count < 0) return fail(MXP_E_VALIDATION, "count must be >= 0, got %lld", (long long)count);
    if (count == 0) return MXP_OK;
    if (!dOut) return fail(MXP_E_VALIDATION, "null device pointer");
    cudaError_t e = launch_splitmix64(seed, count, static_cast<uint64_t*>(dOut), h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "splitmix64_kernel");
    return MXP_OK;
}

int mxp_power_mod_device(mxp_handle h, int64_t n, int64_t k, uint32_t p, const void* dA,
                         void* dOut, mxp_stats* st) {
    stats_reset(st);
    int rc = check_handle(h);
    if (rc) return rc;
    if (n < 1) return fail(MXP_E_VALIDATION, "matrix order must be >= 1, got %lld", (long long)n);
    if (n > 32768)
        return fail(MXP_E_UNSUPPORTED, "matrix order %lld exceeds the supported 32768", (long long)n);
    if (k < 0) return fail(MXP_E_VALIDATION, "power must be >= 0, got %lld", (long long)k);
    if (p < 2 || p >= (1u << 31))
        return fail(MXP_E_VALIDATION, "modulus must satisfy 2 <= p < 2^31, got %u", p);
    if (!dA || !dOut) return fail(MXP_E_VALIDATION, "null device pointer");
    fill_plan_stats(st, k, 1);
    const uint32_t* a = static_cast<const uint32_t*>(dA);
    uint32_t* out = static_cast<uint32_t*>(dOut);
    int64_t launches = 0;
    if (k <= 1) {
        cudaError_t e = launch_mod_trivial(out, a, (int)n, p, k == 1, h->stream);
        if (e != cudaSuccess) return cuda_fail(e, "mod_trivial");
        if (st) st->launches = 1;
        return MXP_OK;
    }
    if (round_up(n, 128) <= kModI8MaxN) {
        // INT8 tensor cores: 16 limb-pair GEMMs accumulated per diagonal (K5I)
        const int64_t np8 = round_up(n, 128);
        if (h->wsi8_pad < np8) {
            for (auto& q : h->i8buf) {
                if (q) cudaFree(q);
                q = nullptr;
            }
            h->wsi8_pad = 0;
            for (auto& q : h->i8buf) MXP_CUDA(cudaMalloc(&q, static_cast<size_t>(np8) * np8));
            h->wsi8_pad = np8;
        }
        uint8_t* const* L = h->i8buf;  // base 0..3, ping 4..7, pong 8..11
        // planes are laid out at np8 (a larger workspace is reused at this stride)
        cudaError_t e = launch_mod_split_u8(a, (int)n, p, L, (int)np8, h->stream);
        if (e != cudaSuccess) return cuda_fail(e, "mod_split_u8");
        ++launches;
        const PlanBits plan = make_plan(k);
        int acc = 0;  // limb set: 0 base, 1 ping, 2 pong
        for (int s = 0; s < plan.len; ++s) {
            const int rhs = plan_is_mult(plan, s) ? 0 : acc;
            const int dst = (acc == 1) ? 2 : 1;
            const bool last = (s == plan.len - 1);
            e = launch_progress_mark(h->progress_dev, static_cast<uint32_t>(s + 1), s == h->fault_step,
                                     h->stream);
            if (e == cudaSuccess)
                e = launch_mod_i8_gemm(L + 4 * acc, L + 4 * rhs, (int)np8, p,
                                       last ? nullptr : L + 4 * dst, last ? out : nullptr, (int)n,
                                       h->stream);
            if (e != cudaSuccess) {
                if (st) st->failed_step = is_async_fault(e) ? progress_step(h) : s;
                return cuda_fail(e, "modular multiply (int8)");
            }
            launches += 2;
            acc = dst;
        }
        if (st) st->launches = launches;
        return MXP_OK;
    }
    const int64_t n_pad = f64_pad((int)n);
    if (h->wsmod_pad < n_pad) {
        for (auto& q : h->modbuf) {
            if (q) cudaFree(q);
            q = nullptr;
        }
        h->wsmod_pad = 0;
        for (auto& q : h->modbuf)
            MXP_CUDA(cudaMalloc(&q, static_cast<size_t>(n_pad) * n_pad * sizeof(double)));
        h->wsmod_pad = n_pad;
    }
    const int np = (int)h->wsmod_pad;
    double** B = h->modbuf;  // base: 0..2, acc: 3..5, T0,T1,T2: 6..8
    cudaError_t e = launch_mod_split(a, (int)n, p, B[0], B[1], B[2], np, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "mod_split");
    ++launches;
    const PlanBits plan = make_plan(k);
    int acc = 0;  // limb set index: 0 = base planes, 3 = acc planes
    for (int s = 0; s < plan.len; ++s) {
        const int rhs = plan_is_mult(plan, s) ? 0 : acc;
        const bool last = (s == plan.len - 1);
        e = launch_progress_mark(h->progress_dev, static_cast<uint32_t>(s + 1), s == h->fault_step,
                                 h->stream);
        if (e == cudaSuccess)
            e = launch_f64_gemm(B[acc + 1], B[rhs + 1], B[7], np, h->stream);  // T1
        if (e == cudaSuccess) e = launch_f64_gemm(B[acc], B[rhs], B[6], np, h->stream);  // T0
        if (e == cudaSuccess) e = launch_f64_gemm(B[acc + 2], B[rhs + 2], B[8], np, h->stream);
        if (e == cudaSuccess)
            e = launch_mod_combine(B[6], B[7], B[8], p, np, B[3], B[4], B[5],
                                   last ? out : nullptr, (int)n, h->stream);
        if (e != cudaSuccess) {
            if (st) st->failed_step = is_async_fault(e) ? progress_step(h) : s;
            return cuda_fail(e, "modular multiply");
        }
        launches += 5;
        acc = 3;
    }
    if (st) st->launches = launches;
    return MXP_OK;
}

int mxp_power_mod(mxp_handle h, int64_t n, int64_t k, uint32_t p, const void* hA, void* hOut,
                  mxp_stats* st) {
    stats_reset(st);
    int rc = check_handle(h);
    if (rc) return rc;
    if (n < 1) return fail(MXP_E_VALIDATION, "matrix order must be >= 1, got %lld", (long long)n);
    if (!hA || !hOut) return fail(MXP_E_VALIDATION, "null host pointer");
    const size_t bytes = static_cast<size_t>(n) * n * 4;
    rc = ensure_io(h, bytes);
    if (rc) return rc;
    MXP_CUDA(cudaStreamSynchronize(h->stream));
    *reinterpret_cast<volatile uint32_t*>(h->progress_host) = 0;
    MXP_CUDA(cudaMemcpyAsync(h->d_in, hA, bytes, cudaMemcpyHostToDevice, h->stream));
    MXP_CUDA(cudaEventRecord(h->ev0, h->stream));
    mxp_stats inner;
    rc = mxp_power_mod_device(h, n, k, p, h->d_in, h->d_out, &inner);
    if (rc) {
        if (st) st->failed_step = inner.failed_step;
        return rc;
    }
    cudaError_t e = cudaEventRecord(h->ev1, h->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(hOut, h->d_out, bytes, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
        if (st) st->failed_step = progress_step(h);
        return cuda_fail(e, "modular power");
    }
    if (st) {
        *st = inner;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h->ev0, h->ev1);
        st->device_ms = ms;
        st->h2d = 1;
        st->d2h = 1;
        st->h2d_bytes = bytes;
        st->d2h_bytes = bytes;
    }
    return MXP_OK;
}

}  // extern "C"
