// Internal launch interface between the C-ABI shim (mxp_api.cu) and the
// sm_100a kernels.  Not exported.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace mxp {

// Square-and-multiply plan (expo.py:60-75) as a bitmask: bit s set means step
// s is MULTIPLY_BASE, clear means SQUARE.  At most 126 steps (k < 2^63).
struct PlanBits {
    int32_t len;
    int32_t squares;
    uint64_t mult[2];
};
PlanBits make_plan(int64_t k);
// (select, not p.mult[s >> 6]: a runtime index would copy a kernel-parameter
// PlanBits into local memory)
__host__ __device__ inline bool plan_is_mult(const PlanBits& p, int s) {
    const uint64_t w = s < 64 ? p.mult[0] : p.mult[1];
    return (w >> (s & 63)) & 1ull;
}

// Set shared-memory attributes of every kernel on the current device (once
// per device, before any launch or graph capture).
cudaError_t prepare_kernels();

// ---- n <= 128: persistent batched chains --------------------------------
// launch_k3_batched (kernels_tf32.cu) routes a chain to K3H or K3B by its
// predicted accumulated truncation bias (k3_route: 0 = K3H, 2 = K3B).
// stamps (device, may be null): K3H's CTA 0 writes {clock64, globaltimer} at
// its start and end into stamps[0..3] (the in-kernel SM clock of the launch).
constexpr int kSmallMax = 128;
int k3_route(int n, const PlanBits& plan);
// fix (device, 1 + batch ints, may be null): the dynamic-range fixup list of
// K3H (count at fix[0]); when given, a K3B pass over the listed matrices is
// enqueued after K3H (two launches; the second exits at once when the list
// is empty).
cudaError_t launch_k3_batched(const float* in, float* out, int n, int64_t batch,
                              const PlanBits& plan, int grid, unsigned long long* stamps,
                              int* variant, int* fix, cudaStream_t s, cudaStream_t side = nullptr);
// K3B (kernels_k3b.cu): two chains per SM, bf16x3 split.
size_t k3b_smem_bytes();
cudaError_t prepare_k3b_kernel();
// idx/count (device, may be null): recompute only matrices idx[0 .. *count)
cudaError_t launch_k3b_batched(const float* in, float* out, int n, int64_t batch,
                               const PlanBits& plan, int grid, cudaStream_t s,
                               const int* idx = nullptr, const int* count = nullptr);
// K3H (kernels_k3h.cu): two chains per SM, scaled fp16x2 split.
size_t k3h_smem_bytes();
cudaError_t prepare_k3h_kernel();
// fix_idx/fix_count (device, may be null): matrices whose chain hit strong
// cancellation (a product more than 2^12 below its bound, where the fp16
// planes' range loses entries a later product depends on) are appended to
// fix_idx for K3B to recompute (launch_k3_batched enqueues that pass).
cudaError_t launch_k3h_batched(const float* in, float* out, int n, int64_t batch,
                               const PlanBits& plan, int grid, unsigned long long* stamps,
                               int* fix_idx, int* fix_count, cudaStream_t s);

// fp32 (n x n, leading dim ld) -> tf32 hi/lo planes (n_pad x n_pad, zero pad).
cudaError_t launch_split(const float* in, int n, int ld, uint32_t* hi, uint32_t* lo, int n_pad,
                         cudaStream_t s, const int* gate = nullptr);
// identity (k = 0) into an n x n fp32 / fp64 buffer
cudaError_t launch_identity_f32(float* out, int n, cudaStream_t s);
cudaError_t launch_identity_f64(double* out, int n, cudaStream_t s);

// K1: one 3xTF32 GEMM C = A * B over hi/lo planes (n_pad multiple of 128).
// Writes the product as hi/lo planes (out_hi/out_lo, may be null) and/or as
// fp32 into out_f32 (n_out x n_out, leading dim ld_out; may be null).
struct GemmPlanes {
    CUtensorMap a_hi, a_lo;  // box {32, 128}, SWIZZLE_128B (K-major left operand)
    CUtensorMap b_hi, b_lo;  // box {32, 32}, SWIZZLE_128B_ATOM_32B (MN-major right operand)
};
bool encode_tile_map(CUtensorMap* map, const void* base, int64_t rows);
bool encode_plane_map(CUtensorMap* map, const void* plane, int n_pad, int box_cols, int box_rows,
                      bool right_operand, int rows = 0);
int k1_block_n(int n_pad, int num_sms);
// Fused exchange (row-sharded multi-GPU chain): the CTA-pair kernel's epilogue
// stores its output rows straight into every rank's buffers (peer / IPC
// pointers), tile by tile, instead of a separate all-gather.
constexpr int kMaxPeers = 8;
struct PeerOut {
    int n = 0;     // destinations (0: the kernel's ordinary outputs)
    int row0 = 0;  // global row of this launch's row 0
    int mc = 0;    // 1: hi[0]/lo[0]/f32[0] are NVLS multicast addresses (n == 1):
                   // one multimem.st reaches every rank's copy through the switch
    uint32_t* hi[kMaxPeers] = {};
    uint32_t* lo[kMaxPeers] = {};
    float* f32[kMaxPeers] = {};  // fp32 rows (leading dim ld_out) instead of planes
};
cudaError_t launch_k1p_gemm_peers(const GemmPlanes& maps, int n_pad, int m_pad, int ld_out,
                                  const PeerOut& po, cudaStream_t s);
// Cross-process barrier over peer-mapped flag words: rank writes `epoch` into
// slot [rank] of every peer's flags (release, system scope), then waits until
// all npeers slots of its own flags reach `epoch` (acquire).
cudaError_t launch_peer_barrier(uint32_t* const* flags, int npeers, int rank, uint32_t epoch,
                                cudaStream_t s);
cudaError_t launch_k1_gemm(const GemmPlanes& maps, int n_pad, int block_n, float* out_f32,
                           int n_out, int ld_out, uint32_t* out_hi, uint32_t* out_lo,
                           cudaStream_t s);
// Row block: C[m_pad x n_pad] = A[m_pad x n_pad] * B[n_pad x n_pad].
// splits > 1 (1-CTA tiles): split-K over `splits` k-ranges, the splits of a
// tile launched as one cluster and reduced deterministically through DSMEM.
cudaError_t launch_k1_gemm_rows(const GemmPlanes& maps, int n_pad, int m_pad, int block_n,
                                float* out_f32, int n_out, int m_out, int ld_out, uint32_t* out_hi,
                                uint32_t* out_lo, cudaStream_t s, int splits = 1,
                                const int* gate = nullptr);
int k1_split_k(int n_pad, int m_pad, int num_sms);
// K1C: the whole 3xTF32 chain in one launch (kernels_tf32.cu);
// cudaErrorNotSupported / a launch error => run the per-step chain
// progress (host-mapped, may be null): every CTA stores step+1 at the start of
// each plan step; fault_step >= 0 makes CTA (0,0) trap there (test hook).
cudaError_t launch_k1c_chain(const CUtensorMap* map_a, const CUtensorMap* map_b,
                             uint32_t* const* planes, const PlanBits& plan, int n_pad, int splits,
                             float* out_f32, int n_out, unsigned int* bar_ctr, uint32_t* progress,
                             int fault_step, cudaStream_t s);
// one-thread kernel: *progress = value (host-mapped memory, survives a sticky
// device fault so the host can name the failing plan step); trap != 0 then
// executes a trap (the fault-injection test hook)
cudaError_t launch_progress_mark(uint32_t* progress, uint32_t value, int trap, cudaStream_t s);  // kernel launches one split-K multiply takes
// whether K1C runs the chain on 64-column tiles (2 x tiles x splits CTAs in one wave)
bool k1c_narrow(int n_pad, int splits);
cudaError_t launch_split_rows(const float* in, int n, int ld, int rows, uint32_t* hi, uint32_t* lo,
                              int n_pad, int rows_pad, cudaStream_t s, const int* gate = nullptr);

// ---- K1PH (kernels_f16x2.cu): the large-n chain on scaled fp16x2 planes ----
// gate (device, may be null) on the 3xTF32 launches above: the kernel does
// nothing unless *gate != 0 (the fallback chain enqueued behind a K1PH chain
// runs only when that chain raised its dynamic-range flag).
struct F16Maps {
    CUtensorMap a0, a1;  // h0 / h1 as the K-major left operand: box {64, 128}, SWIZZLE_128B
    CUtensorMap b0, b1;  // h0 / h1 as the MN-major right operand: box {64, 64}, SWIZZLE_128B
};
cudaError_t prepare_f16x2_kernels();
bool k1ph_eligible(int64_t n_pad);  // n_pad % 256 == 0 && n_pad >= 1024 (K1P's sizes)
bool encode_plane16_map(CUtensorMap* map, const void* plane, int n_pad, int box_rows);
// Chain state (device, f16_chain_state_bytes(), zeroed before a chain):
// index 0 = the base A, s + 1 = the product of plan step s; the flag word
// (f16_chain_flag) gates the 3xTF32 recomputation.
constexpr int kF16MaxSteps = 128;  // plan steps (k < 2^63: at most 126)
size_t f16_chain_state_bytes();
int* f16_chain_flag(void* state);
// fp32 P_i (n x n, leading dim ld) -> its h0 / h1 planes (n_pad x n_pad,
// zero padded) at the exact scale of maxw[i]; the base (xi < 0) measures its
// max first; a product P_i = P_xi P_yi is tested for lost dynamic range
cudaError_t launch_split16(const float* in, int n, int ld, void* h0, void* h1, int n_pad,
                           void* state, int i, int xi, int yi, cudaStream_t s);
// P_oi = P_xi P_yi (fp32 out: n_out x n_out, leading dim ld_out) from the
// planes of P_xi (left) and P_yi (right); oi >= 0: max |P_oi| -> maxw[oi]
// m_rows > 0: only rows [row0, row0 + m_rows) of the product (multiples of
// 256), out row r = global row row0 + r (row-sharded chains)
cudaError_t launch_k1ph_gemm(const F16Maps& x, const F16Maps& y, int n_pad, float* out, int n_out,
                             int ld_out, void* state, int xi, int yi, int oi, int num_sms,
                             cudaStream_t s, int m_rows = 0, int row0 = 0);
// Row-sharded K1PH chains (mxp_multi.cu): this device's max |P_i| into every
// device's state (system-scope atomicMax over peer access), then this
// device's fp32 rows of P_i split at the global exact scale into every
// device's h0 / h1 planes (peer stores), with the dynamic-range test.
constexpr int kF16MaxPeers = 8;
cudaError_t launch_max_to_peers(const void* state, int i, void* const* peer_states, int npeers,
                                cudaStream_t s);
cudaError_t launch_split16_rows_peers(const float* in, int m_rows, int row0, int n_pad, int n,
                                      void* state, int i, int xi, int yi, void* const* h0,
                                      void* const* h1, int npeers, cudaStream_t s);

// ---- generation (kernels_gen.cu) -------------------------------------------
// Reference random_matrix (linalg.py:127-148) on device; scale != 0 selects
// the scaled recipe fl(random_matrix(n, F64, seed, lo, hi) * scale).
// Matrix b of the batch uses seed seed0 + b.
cudaError_t launch_splitmix64(uint64_t seed, int64_t count, uint64_t* out, cudaStream_t s);
cudaError_t launch_random(int mode, int64_t n, int64_t batch, uint64_t seed0, double lo, double hi,
                          double scale, void* out, cudaStream_t s);

// ---- FP64 (kernels_f64.cu) ------------------------------------------------
cudaError_t launch_f64_gemm(const double* a, const double* b, double* c, int n, cudaStream_t s);
// Row block: C[m x n] = A[m x n] * B[n x n] (m, n multiples of 128).
cudaError_t launch_f64_gemm_rows(const double* a, const double* b, double* c, int n, int m,
                                 cudaStream_t s);
cudaError_t launch_f64_pad_rows(const double* in, int n, int rows, double* out, int n_pad,
                                int rows_pad, cudaStream_t s);
cudaError_t launch_f64_unpad_rows(const double* in, int n_pad, double* out, int n, int rows,
                                  cudaStream_t s);
cudaError_t launch_f64_pad(const double* in, int n, double* out, int n_pad, cudaStream_t s);
cudaError_t launch_f64_unpad(const double* in, int n_pad, double* out, int n, cudaStream_t s);
int f64_pad(int n);

// ---- exact modular mode (kernels_mod.cu): 16-bit limbs, Karatsuba, DMMA ---
// K5I (kernels_mod_i8.cu): one exact modular product on the INT8 tensor cores
// over byte limb planes (n_pad % 128 == 0, n_pad <= kModI8MaxN so that every
// s32 accumulator stays < 2^31).  Writes the next step's limb planes, or the
// final n x n uint32 residues when out != nullptr.
constexpr int kModI8MaxN = 8192;
cudaError_t prepare_mod_i8_kernel();
cudaError_t launch_mod_split_u8(const uint32_t* in, int n, uint32_t p, uint8_t* const* limb,
                                int n_pad, cudaStream_t s);
cudaError_t launch_mod_i8_gemm(uint8_t* const* a_limb, uint8_t* const* b_limb, int n_pad, uint32_t p,
                               uint8_t* const* out_limb, uint32_t* out, int n, cudaStream_t s);
cudaError_t launch_mod_split(const uint32_t* in, int n, uint32_t p, double* l0, double* l1,
                             double* ls, int n_pad, cudaStream_t s);
cudaError_t launch_mod_combine(const double* t0, const double* t1, const double* t2, uint32_t p,
                               int n_pad, double* l0, double* l1, double* ls, uint32_t* out,
                               int n, cudaStream_t s);
cudaError_t launch_mod_trivial(uint32_t* out, const uint32_t* a, int n, uint32_t p, int copy,
                               cudaStream_t s);

}  // namespace mxp
