/*
 * matexpo_b200 — C ABI of the B200-native matrix-power engine (A^k).
 *
 * Drop-in boundary for the reference `matexpo` hot path
 * (/root/reference/pkg/src/matexpo).  Plain pointers and sizes only; no
 * torch or CUDA types cross this interface.  Every entry point returns an
 * MXP_* status; the message of the last failure on the calling thread is
 * available from mxp_last_error().
 *
 * Reference interface each entry point replaces:
 *   mxp_plan            <- plan_exponentiation        expo.py:60-75
 *   mxp_multiply        <- Backend.multiply(a, b)     expo.py:78-86 (backend
 *                          plugin called at expo.py:133-136); device-side
 *                          analogue gpuMatmul         gpu-backend/src/host.ts:67-95
 *   mxp_power           <- exponentiate(a, k, backend) expo.py:121-139 executed
 *                          on-device as in gpuExponentiate host.ts:106-141
 *                          (one upload, ping-pong chain, one readback)
 *   mxp_power_batched   <- exponentiate over independent matrices (BASELINE
 *                          config 3; no reference counterpart beyond the loop)
 *   mxp_alloc/free,     <- ComputeDevice.createBuffer / releaseBuffer /
 *   mxp_upload/download    writeBuffer / readBuffer  device.ts:25-39
 *   mxp_gemm_prepare_rhs,  the same, split so several row blocks share one
 *   mxp_gemm_rows_prepared right-hand side (row-sharded chain)
 *   mxp_gemm            <- ComputeDevice.dispatchMatmul(kernel, n, a, b, c)
 *                          device.ts:33-39 (device pointers, async)
 *   mxp_power_device    <- the gpuExponentiate step loop host.ts:126-131 on
 *                          caller-owned device buffers (async, graph replay)
 *   mxp_power_mod       <- (new) exact modular mode, no reference counterpart
 *   mxp_last_error      <- the message of the raised error (errors.py)
 *
 * Semantics kept from the reference:
 *   - row-major, element (i, j) at i*n + j (linalg.py:27-31); square only;
 *   - k = 0 -> identity (expo.py:128-129); k = 1 -> a bitwise copy of A with
 *     zero multiplies (expo.py:130, :139); k < 0 -> MXP_E_VALIDATION
 *     (expo.py:66-67);
 *   - exactly floor(log2 k) + popcount(k) - 1 multiplies (expo.py:44-46),
 *     reported in mxp_stats; host APIs move the input once and the result
 *     once (count_transfers, expo.py:159-169; host.test.ts:136-146);
 *   - all validation happens before any device work (host.ts:48-59);
 *   - a failing multiply inside a chain reports its plan step index in
 *     mxp_stats.failed_step (BackendStepError, errors.py:43-49).
 * Threading: one handle = one CUDA stream + workspace; use a handle from one
 * thread at a time (device.ts:6-8).
 */
#ifndef MATEXPO_B200_H
#define MATEXPO_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MXP_API __attribute__((visibility("default")))
#else
#define MXP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define MXP_OK 0
#define MXP_E_VALIDATION 1         /* ValueError family (ShapeError, InvalidDimensionError, ...) */
#define MXP_E_UNSUPPORTED 2        /* mode/size not supported (UnsupportedPowerError analogue) */
#define MXP_E_DEVICE_UNAVAILABLE 3 /* no usable sm_100 device (errors.ts DeviceUnavailableError) */
#define MXP_E_CUDA 4               /* CUDA runtime failure (-> BackendStepError inside a chain) */
#define MXP_E_NCCL 5               /* collective failure (multi-GPU paths) */

/* element modes */
#define MXP_F32 0     /* float32 in/out; split-fp32 on tcgen05 tensor cores (scaled
                         fp16x2 / bf16x3 for n <= 128; 3xTF32 for n > 128, scaled
                         fp16x2 for the CTA-pair sizes, see mxp_set_f32_datapath) */
#define MXP_F64 1     /* float64 in/out; DMMA tensor pipe */
#define MXP_U32_MOD 2 /* uint32 residues mod p; exact (see mxp_power_mod) */

typedef struct mxp_handle_s* mxp_handle;

typedef struct mxp_stats {
    int64_t multiply_count; /* plan multiplies executed (expo.py:52-53) */
    int64_t square_count;   /* SQUARE steps (expo.py:55-57) */
    int64_t launches;       /* kernels launched by this call */
    int64_t h2d;            /* host->device matrix transfers (logical) */
    int64_t d2h;            /* device->host matrix transfers (logical) */
    int64_t h2d_bytes;
    int64_t d2h_bytes;
    int64_t failed_step;    /* plan step index of a failed multiply, else -1 */
    double device_ms;       /* device time of the call (host APIs), else 0 */
} mxp_stats;

/* library / device */
MXP_API int mxp_version(int* major, int* minor);
MXP_API int mxp_device_count(int* count);
MXP_API int mxp_create(int device, mxp_handle* out);
MXP_API int mxp_destroy(mxp_handle h);
MXP_API int mxp_get_stream(mxp_handle h, void** stream);     /* cudaStream_t of the handle */
MXP_API int mxp_synchronize(mxp_handle h);
MXP_API int mxp_num_sms(mxp_handle h, int* sms);

/* device verbs (ComputeDevice, device.ts:20-40) */
MXP_API int mxp_alloc(mxp_handle h, size_t bytes, void** dptr);
MXP_API int mxp_free(mxp_handle h, void* dptr);
MXP_API int mxp_host_alloc(mxp_handle h, size_t bytes, void** hptr); /* pinned host memory */
MXP_API int mxp_host_free(mxp_handle h, void* hptr);
MXP_API int mxp_upload(mxp_handle h, void* dst, const void* src, size_t bytes);
MXP_API int mxp_download(mxp_handle h, void* dst, const void* src, size_t bytes);

/* the plan (expo.py:60-75): writes 'S'/'M' bytes, *count = multiply count */
MXP_API int mxp_plan(int64_t k, char* steps, int64_t cap, int64_t* count);

/* rows x width bytes, device to device (pitches in bytes), async on the handle stream */
MXP_API int mxp_copy2d_device(mxp_handle h, void* dst, size_t dpitch, const void* src,
                              size_t spitch, size_t width, size_t rows);

/* one multiply C = A * B */
MXP_API int mxp_gemm(mxp_handle h, int mode, int64_t n, const void* dA, const void* dB, void* dC);
/* a row block of one multiply: C[rows x n] = A[rows x n] * B[n x n] (row-major,
 * leading dimension n).  The building block of the row-sharded multi-GPU chain:
 * every element's arithmetic is the same as in mxp_gemm, so sharded results are
 * bitwise equal to the single-GPU ones. */
MXP_API int mxp_gemm_rows(mxp_handle h, int mode, int64_t n, int64_t rows, const void* dA,
                          const void* dB, void* dC);
/* the row-block multiply in two parts, so a caller can run several row blocks
 * against one right-hand side (the row-sharded multi-GPU chain computes its
 * rows in chunks and all-gathers each chunk while the next one computes):
 * prepare B once (split / pad into the handle's workspace), then any number
 * of C[rows x n] = A[rows x n] * B.  Any other call that uses the handle's
 * workspace invalidates the prepared B (E_VALIDATION until prepared again).
 * Arithmetic per element is identical to mxp_gemm_rows / mxp_gemm. */
MXP_API int mxp_gemm_prepare_rhs(mxp_handle h, int mode, int64_t n, const void* dB);
MXP_API int mxp_gemm_rows_prepared(mxp_handle h, int mode, int64_t n, int64_t rows,
                                   const void* dA, void* dC);
/* Fused exchange for the row-sharded chain: the CTA-pair GEMM
 * epilogue stores its output rows straight into every rank's buffers, tile by
 * tile, instead of a separate all-gather.  Ranks share buffers through CUDA
 * IPC handles (72 opaque bytes) and order their steps with a flag barrier in
 * peer-mapped memory.  MXP_F32 only; n % 256 == 0 and n >= 1024; planes are
 * tf32 hi/lo n x n (mxp_split_planes).  peer_f32 (or NULL): write fp32 rows
 * (leading dim n) instead of planes — the chain's last step. */
#define MXP_IPC_HANDLE_BYTES 72 /* cudaIpcMemHandle_t + byte offset in the allocation */
MXP_API int mxp_ipc_get_handle(mxp_handle h, const void* dptr, void* handle_out);
MXP_API int mxp_ipc_open_handle(mxp_handle h, const void* handle, void** dptr);
MXP_API int mxp_ipc_close_handle(mxp_handle h, void* dptr);
MXP_API int mxp_split_planes(mxp_handle h, int64_t n, const void* dA, void* d_hi, void* d_lo);
MXP_API int mxp_gemm_rows_planes_peers(mxp_handle h, int64_t n, int64_t rows, int64_t row0,
                                       const void* a_hi, const void* a_lo, const void* b_hi,
                                       const void* b_lo, int npeers, void* const* peer_hi,
                                       void* const* peer_lo, void* const* peer_f32);
MXP_API int mxp_peer_barrier(mxp_handle h, int rank, int npeers, void* const* peer_flags,
                             uint32_t epoch);
/* NVLS variant of the fused exchange: the ranks' plane / result buffers are
 * bound to multicast objects, and the epilogue stores each 16 bytes ONCE to
 * the multicast address (multimem.st); the NVSwitch writes every rank's copy.
 * Lifecycle: one rank mxp_mc_create (exports MXP_MC_HANDLE_BYTES of FABRIC
 * handle), the others mxp_mc_import it; once every rank has created or
 * imported, each calls mxp_mc_bind (its own device memory + a unicast and a
 * multicast mapping); mxp_mc_destroy when done. */
#define MXP_MC_HANDLE_BYTES 64
typedef struct mxp_mc_s* mxp_mc;
MXP_API int mxp_mc_supported(mxp_handle h, int* ok);
MXP_API int mxp_mc_create(mxp_handle h, int nranks, size_t bytes, void* handle_out, mxp_mc* out);
MXP_API int mxp_mc_import(mxp_handle h, const void* handle, size_t bytes, mxp_mc* out);
MXP_API int mxp_mc_size(mxp_mc mc, size_t* bytes);
MXP_API int mxp_mc_bind(mxp_mc mc, void** local_ptr, void** mc_ptr);
MXP_API int mxp_mc_destroy(mxp_mc mc);
MXP_API int mxp_gemm_rows_planes_mc(mxp_handle h, int64_t n, int64_t rows, int64_t row0,
                                    const void* a_hi, const void* a_lo, const void* b_hi,
                                    const void* b_lo, void* mc_hi, void* mc_lo, void* mc_f32);
MXP_API int mxp_multiply(mxp_handle h, int mode, int64_t n, const void* hA, const void* hB, void* hC,
                 mxp_stats* stats);

/* K1PH row shards across processes (distributed.RowShardedK1PH; one process
 * per GPU, peer buffers mapped with mxp_ipc_*).  A chain state (size from
 * mxp_k1ph_state_bytes, zeroed by the caller before a chain) holds the
 * maxima, plane exponents and the dynamic-range flag.  fp16 planes are
 * n x n (n % 256 == 0, n >= 1024), row-major.
 *   mxp_k1ph_split_base: dA (n_true x n_true fp32, dense) -> base planes at
 *     its exact scale (state index 0);
 *   mxp_k1ph_gemm_rows: rows [row0, row0 + rows) of P_xi * P_yi (fp32, out
 *     leading dim ld_out, entries of global row or column >= n_out skipped);
 *     oi >= 0: their max -> maxw[oi];
 *   mxp_k1ph_max_to_peers: this rank's maxw[i] into every peer state;
 *   mxp_k1ph_split_rows_peers: this rank's fp32 rows of P_i -> h0 / h1 rows in
 *     every peer's planes at the (global) exact scale, with the range test;
 *   mxp_k1ph_read_flag: the state's flag (synchronizes the handle stream). */
MXP_API int mxp_k1ph_state_bytes(size_t* bytes);
MXP_API int mxp_k1ph_split_base(mxp_handle h, int64_t n_true, int64_t n, const void* dA, void* h0,
                                void* h1, void* state);
MXP_API int mxp_k1ph_gemm_rows(mxp_handle h, int64_t n, int64_t rows, int64_t row0,
                               const void* x_h0, const void* x_h1, const void* y_h0,
                               const void* y_h1, void* out, int64_t ld_out, int64_t n_out,
                               void* state, int xi, int yi, int oi);
MXP_API int mxp_k1ph_max_to_peers(mxp_handle h, const void* state, int i, int npeers,
                                  void* const* peer_states);
MXP_API int mxp_k1ph_split_rows_peers(mxp_handle h, int64_t n_true, int64_t n, int64_t rows,
                                      int64_t row0, const void* rows_f32, void* state, int i,
                                      int xi, int yi, int npeers, void* const* peer_h0,
                                      void* const* peer_h1);
MXP_API int mxp_k1ph_read_flag(mxp_handle h, const void* state, int* raised);

/* A^k, whole chain on device */
MXP_API int mxp_power_device(mxp_handle h, int mode, int64_t n, int64_t k, const void* dA, void* dOut,
                     mxp_stats* stats);
MXP_API int mxp_power(mxp_handle h, int mode, int64_t n, int64_t k, const void* hA, void* hOut,
              mxp_stats* stats);

/* A_i^k for `batch` independent row-major n x n matrices stored back to back */
MXP_API int mxp_power_batched_device(mxp_handle h, int mode, int64_t n, int64_t batch, int64_t k,
                             const void* dA, void* dOut, mxp_stats* stats);
MXP_API int mxp_power_batched(mxp_handle h, int mode, int64_t n, int64_t batch, int64_t k,
                      const void* hA, void* hOut, mxp_stats* stats);

/* A^k on several GPUs from ONE process (SURVEY §8(b) mxp_power_multi; the
 * reference has no multi-device path: SPEC.md:447, device.ts:6-8).  devices:
 * ngpus device ordinals (NULL: 0 .. ngpus-1; a device may repeat, each
 * occurrence gets its own internal handle and stream), 1 <= ngpus <= 8.
 *   batch >= 2: contiguous batch shards, one host thread per device running
 *     mxp_power_batched — no communication, bitwise equal to one device;
 *   batch == 1, MXP_F32 at the K1PH sizes (see mxp_set_f32_datapath), k >= 2:
 *     row-sharded K1PH chain: each device's fp32 rows, the maxima met in every
 *     device's state (peer atomics), each device's rows split at the global
 *     scale into every device's planes (peer stores); bitwise the
 *     single-device K1PH chain (recomputed on the 3xTF32 row shards below if
 *     a product loses dynamic range);
 *   batch == 1, MXP_F32, other n > 128, k >= 2: row-sharded chain, each step's
 *     new rows stored by the CTA-pair GEMM epilogue straight into every
 *     device's next planes over NVLink (peer access), CUDA events between
 *     steps (3xTF32); bitwise equal to mxp_power on MXP_DATAPATH_3XTF32
 *     where that also runs the CTA-pair kernel (n % 256 == 0, n >= 1024);
 *   batch == 1, MXP_F64, n >= 256, k >= 2: row-sharded with the DMMA
 *     row-block GEMM and peer copies of each device's rows, bitwise equal to
 *     mxp_power;
 *   otherwise: devices[0] alone (replicas only).
 * Host buffers as mxp_power / mxp_power_batched.  stats: launches summed,
 * h2d = one per device used, device_ms = max over devices.
 * mxp_multi_release destroys the internal handles. */
MXP_API int mxp_power_multi(int ngpus, const int* devices, int mode, int64_t n, int64_t batch,
                            int64_t k, const void* hA, void* hOut, mxp_stats* stats);
MXP_API int mxp_multi_release(void);

/* exact modular mode: uint32 residues, result (A^k) mod p, 2 <= p < 2^31 */
MXP_API int mxp_power_mod_device(mxp_handle h, int64_t n, int64_t k, uint32_t p, const void* dA,
                         void* dOut, mxp_stats* stats);
MXP_API int mxp_power_mod(mxp_handle h, int64_t n, int64_t k, uint32_t p, const void* hA, void* hOut,
                  mxp_stats* stats);

/* inputs: the reference's SplitMix64 random_matrix (linalg.py:127-148) on
 * device, bit-identical; matrix b of the batch uses seed seed0 + b.  With
 * scale != 0 the value is fl(random_matrix(n, F64, seed, lo, hi) * scale)
 * (the configs' spectrally normalised recipe); with scale == 0 it is
 * random_matrix(n, mode's dtype, seed, lo, hi).  Async on the handle stream. */
MXP_API int mxp_random_device(mxp_handle h, int mode, int64_t n, int64_t batch, uint64_t seed0,
                              double lo, double hi, double scale, void* dOut);

/* the raw SplitMix64 stream (linalg.py:117-124 splitmix64(seed, count)):
 * count uint64 draws of `seed` into dOut.  Async on the handle stream. */
MXP_API int mxp_splitmix64_device(mxp_handle h, uint64_t seed, int64_t count, void* dOut);

/* Datapath of single-matrix FP32 chains at the CTA-pair sizes (roundup(n, 128)
 * a multiple of 256 and >= 1024, e.g. C5; and every n > 1408, padded to 256):
 *   MXP_DATAPATH_AUTO (default): K1PH — scaled fp16x2 planes, one exponent
 *     per matrix, half the tensor work of 3xTF32 at the same 22-bit operand
 *     precision; a chain whose product loses dynamic range (strong
 *     cancellation, zero or non-finite) is recomputed on 3xTF32 inside the
 *     same call (a gated chain enqueued behind it);
 *   MXP_DATAPATH_3XTF32: always 3xTF32 (an exponent per element) — the
 *     datapath of the row-sharded multi-GPU chains, so their results are
 *     bitwise this single-device chain's.
 * Other sizes and n <= 128 are unaffected.  Per handle; drops cached graphs. */
#define MXP_DATAPATH_AUTO 0
#define MXP_DATAPATH_3XTF32 1
MXP_API int mxp_set_f32_datapath(mxp_handle h, int datapath);
/* Whether the last K1PH chain of this handle raised its dynamic-range flag
 * (its result then came from the 3xTF32 recomputation).  Synchronizes. */
MXP_API int mxp_last_f32_fallback(mxp_handle h, int* raised);

/* Which persistent kernel an n <= 128 fp32 chain of power k runs on: the
 * scaled fp16x2 K3H, or the bf16x3 K3B when K3H's accumulated tensor-core
 * truncation bias, predicted as (k-1)(2.5e-8 + 1.05e-9 n), would exceed 60%
 * of the chain tolerance 16 m(k) sqrt(n) 2^-24.  Host-only (no device). */
#define MXP_KERNEL_K3H 0
#define MXP_KERNEL_K3B 1
MXP_API int mxp_small_kernel_for(int64_t n, int64_t k, int* kernel);

/* How many matrices of the last n <= 128 K3H launch were recomputed on K3B
 * because their chain hit strong cancellation (the scaled fp16 planes keep
 * one exponent per matrix; K3B keeps one per element).  Synchronizes. */
MXP_API int mxp_last_small_fixups(mxp_handle h, int64_t* count);

/* The SM clock the last batched n <= 128 launch (K3H) actually ran at:
 * clock64 and globaltimer stamped by CTA 0 at its start and end, so
 * *sm_mhz = cycles / ns (NVML samples miss short kernels).  Synchronizes
 * the handle's stream.  MXP_E_UNSUPPORTED if no such launch happened. */
MXP_API int mxp_last_kernel_clock(mxp_handle h, double* sm_mhz, double* kernel_ms);

/* Test hook (fault injection): chains captured after this call trap at plan
 * step `step` (-1 disables), so tests can check that an asynchronous device
 * fault inside a graph-replayed chain is reported with the right step index
 * (mxp_stats.failed_step -> BackendStepError, errors.py:43-49; the reference's
 * own test is test_expo.py:123-137).  The trap kills the CUDA context: use it
 * in a throw-away process. */
MXP_API int mxp_debug_inject_fault(mxp_handle h, int64_t step);

/* error reporting */
MXP_API int mxp_last_error(char* buf, size_t len); /* copies the thread's last message */
MXP_API const char* mxp_status_string(int status);

#ifdef __cplusplus
}
#endif

#endif /* MATEXPO_B200_H */
