// Shared internals of libddppo.so (not part of the ABI).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ddppo.h"

constexpr int kMaxPeers = 8;

struct ddppo_ctx {
  int rank = 0, world = 1, device = 0, sm_count = 148;
  ncclComm_t comm = nullptr;
  // device scratch
  int* d_err = nullptr;                // non-finite flag (bitmask of tensor ids)
  unsigned int* d_counters = nullptr;  // last-block-done counters (one slot per kernel family)
  double* d_partials = nullptr;        // per-block partial sums (fixed-order reductions)
  float* d_scalars = nullptr;          // clip coef etc.
  int32_t* d_i32 = nullptr;            // preemption poll buffer
  int64_t* d_i64 = nullptr;            // counts buffer
  std::string last_error;
  // NVLink peer memory (peer.cu): flag arrays of every rank, IPC mappings, the registered learner
  // workspace of every rank, the barrier epoch and the running minibatch counter (gradient parity)
  unsigned int* peer_flags[kMaxPeers] = {};
  unsigned int* own_flags = nullptr;
  std::vector<void*> ipc_opened;
  void* peer_ws = nullptr;
  char* peer_ws_base[kMaxPeers] = {};
  unsigned int* d_peer_epoch = nullptr;  // barrier epoch, advanced on the device by the barrier kernel
  unsigned int* d_cnt_epoch = nullptr;   // counts-exchange epoch (ddppo_allreduce_counts over NVLink)
  cudaStream_t cnt_stream = nullptr;     // its own non-blocking stream: not queued behind learner work
  int64_t* h_cnt = nullptr;              // pinned host result
  uint64_t peer_mb = 0;
  int a8_mode = DDPPO_A8_AUTO;          // ddppo_set_a8_mode
  int conv_engine = DDPPO_CONV_TMA;     // ddppo_set_conv_engine
  int fwd_planes = 2;                   // ddppo_set_fwd_planes: encoder forward operands bf16x3 (2) / bf16 (1)
  bool tconv_bn64 = getenv("DDPPO_TCONV_BN128") == nullptr;  // A/B switch for the conv kernel's N tile
  // programmatic dependent launch of the learner step's kernels (launch_k); DDPPO_PDL=0: plain launches
  bool pdl = getenv("DDPPO_PDL") == nullptr || atoi(getenv("DDPPO_PDL")) != 0;
  int* d_tile_cnt = nullptr;            // split-K tile arrival counters (tconv.cu), zero between kernels
  // learner runtime: Adam update count on the device; captured CUDA graph of the last learner step
  int* d_step = nullptr;
  int64_t step_expected = -1;       // value *d_step will hold once the enqueued work has run
  bool graphs = true;               // ddppo_set_graphs
  struct GraphCache;
  GraphCache* graph = nullptr;
  // side streams for work beside the recurrences (fork / join with events), created lazily
  cudaStream_t side[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> fork_events;
  size_t fork_next = 0;
  // measurement (ddppo_profile_*)
  bool prof = false;
  int64_t launches[DDPPO_K_COUNT] = {};
  double ms[DDPPO_K_COUNT] = {};
  double flops[DDPPO_K_COUNT] = {};            // algorithmic FLOPs issued (profiling mode)
  double smem_bytes[DDPPO_K_COUNT] = {};       // shared-memory bytes moved by the tensor-core kernels (idem)
  int cur_fam = DDPPO_K_OTHER;                 // family of the innermost open ProfScope
  void count(int n) { launches[cur_fam] += n; }  // launches made by shared launchers
  struct Rec { int fam; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get_event() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
};

// Counts `n` launches of family `fam`; when profiling is on, brackets the scope with events
// recorded on the launching stream.
struct ProfScope {
  ddppo_ctx* ctx;
  int fam;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  int prev_fam;
  ProfScope(ddppo_ctx* c, int f, cudaStream_t s, int n) : ctx(c), fam(f), st(s), prev_fam(c->cur_fam) {
    ctx->launches[fam] += n;
    ctx->cur_fam = fam;
    if (ctx->prof) {
      a = ctx->get_event();
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    ctx->cur_fam = prev_fam;
    if (ctx->prof && a) {
      cudaEvent_t b = ctx->get_event();
      cudaEventRecord(b, st);
      ctx->pending.push_back({fam, a, b});
    }
  }
};

enum { CNT_GAE = 0, CNT_LOSS = 1, CNT_NORM = 2, CNT_MISC = 3, CNT_NUM = 8 };
constexpr int kMaxPartials = 1 << 16;   // doubles
constexpr int kMaxCountVals = 64;
constexpr int kMaxTileCounters = 1 << 16;

enum { ERR_BIT_LOSS = 1, ERR_BIT_GRAD = 2, ERR_BIT_COMM = 4 };

// Programmatic dependent launch (PDL).  Kernels of the learner step are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization (launch_k), so a kernel's CTAs are scheduled
// while its predecessor in the stream is still draining; every such kernel starts with pdl_enter():
// griddepcontrol.wait (block until the predecessor grid has completed and its memory is visible --
// nothing of the predecessor's output is touched before it), then griddepcontrol.launch_dependents
// (let the successor be scheduled now).  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(const ddppo_ctx* ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = ctx->pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#define DDPPO_CUDA_TRY(ctx, expr)                                                 \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      if (ctx) (ctx)->last_error = std::string(#expr ": ") + cudaGetErrorString(_e); \
      return DDPPO_ERR_CUDA;                                                      \
    }                                                                             \
  } while (0)

#define DDPPO_NCCL_TRY(ctx, expr)                                                 \
  do {                                                                            \
    ncclResult_t _r = (expr);                                                     \
    if (_r != ncclSuccess) {                                                      \
      if (ctx) (ctx)->last_error = std::string(#expr ": ") + ncclGetErrorString(_r); \
      return DDPPO_ERR_COMM;                                                      \
    }                                                                             \
  } while (0)

#define DDPPO_REQUIRE(ctx, cond, msg)                                             \
  do {                                                                            \
    if (!(cond)) {                                                                \
      if (ctx) (ctx)->last_error = std::string("config: ") + (msg);               \
      return DDPPO_ERR_CONFIG;                                                    \
    }                                                                             \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ctx side streams (non-blocking, created on first use on the ctx's device)
inline ddppo_status ctx_side_streams(ddppo_ctx* ctx, cudaStream_t* a, cudaStream_t* b) {
  for (int i = 0; i < 2; ++i)
    if (!ctx->side[i]) DDPPO_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->side[i], cudaStreamNonBlocking));
  *a = ctx->side[0];
  *b = ctx->side[1];
  return DDPPO_OK;
}
// make `to` wait for all work enqueued so far on `from` (a recycled timing-free event)
inline cudaError_t fork_to(ddppo_ctx* ctx, cudaStream_t from, cudaStream_t to) {
  if (ctx->fork_events.size() < 64) {
    cudaEvent_t e;
    cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r != cudaSuccess) return r;
    ctx->fork_events.push_back(e);
  }
  cudaEvent_t e = ctx->fork_events[ctx->fork_next++ % ctx->fork_events.size()];
  cudaError_t r = cudaEventRecord(e, from);
  return r == cudaSuccess ? cudaStreamWaitEvent(to, e, 0) : r;
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One Adam element (PyTorch form; step_size = lr / (1 - b1^t), inv_sqrt_bc2 = 1 / sqrt(1 - b2^t))
__device__ __forceinline__ void adam_one(float& p, float& m, float& v, float g, float b1, float b2, float step_size,
                                         float inv_sqrt_bc2, float eps) {
  m = b1 * m + (1.f - b1) * g;
  v = b2 * v + (1.f - b2) * g * g;
  const float denom = sqrtf(v) * inv_sqrt_bc2 + eps;
  p = p - step_size * (m / denom);
}

// Deterministic block reduction of NV doubles per thread; result valid in thread 0.
// smem must hold NV * (blockDim/32) doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) smem[warp * NV + i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += smem[w * NV + i];
      v[i] = s;
    }
  }
  __syncthreads();
}

// "Last block done" pattern: the block reduces its threads' NV values (fixed order), thread 0
// writes them to partials[blockIdx*NV+i]; the last block to arrive sums the partials in block
// order (deterministic) into out[0..NV).  Every thread of every block must call it.  Returns
// true in the (whole) last block.  counter is reset for reuse.
template <int NV>
__device__ __forceinline__ bool last_block_reduce(double (&v)[NV], double* partials, unsigned int* counter,
                                                  double* out, double* smem) {
  __shared__ bool am_last;
  block_sum<NV>(v, smem);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) partials[blockIdx.x * NV + i] = v[i];
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  // fixed partition: thread t sums blocks t, t+bd, ... in order; then the ordered block_sum
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] += ((volatile double*)partials)[b * NV + i];
  }
  block_sum<NV>(acc, smem);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) out[i] = acc[i];
    *counter = 0u;
  }
  return true;
}

inline int grid_for(int n_items, int per_block, int max_blocks) {
  long long g = (n_items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

// ---------------------------------------------------------------- internal launchers
ddppo_status launch_gae(ddppo_ctx* ctx, const float* rew, const float* val, const uint8_t* done,
                        const int32_t* len, int E, int T, int ld, float gamma, float tau, float* adv,
                        float* ret, double* stats3, cudaStream_t st);
ddppo_status launch_adv_finalize(ddppo_ctx* ctx, const double* stats3, float eps, float* mean_invstd,
                                 cudaStream_t st);
ddppo_status launch_loss(ddppo_ctx* ctx, const float* logits, const float* values, const ddppo_batch& b,
                         const ddppo_loss_inputs& in, const float* mean_invstd, const ddppo_loss_cfg& cfg,
                         float* dlogits, float* dvalues, float* stats, cudaStream_t st);
// Adam's update count: host cfg.step (dstep == null) or device *dstep + step_add (learner runtime)
// frz_end: entries [0, frz_end) are frozen (a multiple of 4)
ddppo_status launch_clip_adam(ddppo_ctx* ctx, float* grad, float* params, float* m, float* v,
                              const uint8_t* freeze, int64_t P, const ddppo_adam_cfg& cfg, float inv_world,
                              float* grad_norm, cudaStream_t st, const int* dstep = nullptr, int step_add = 0,
                              int64_t frz_end = 0);

// bf16-operand implicit-GEMM (igemm.cu): operands read straight into UMMA canonical tiles.
enum { IG_DENSE_K = 0, IG_DENSE_MN = 1, IG_PIX_K = 2, IG_TAP_MN = 3 };
// Conv gather over an NHWC bf16 tensor x[F][SH][SW][SC] (the implicit-GEMM view of im2col): element
// (pixel q, column kk = (u*k + v)*SC + c) is, with q = (f*PH + i)*PW + j,
//   forward     : x[f][i*s - p + u][j*s - p + v][c]                          (0 outside)
//   transposed  : x[f][(i + p - u)/s][(j + p - v)/s][c] if both divisions are exact, else 0
struct IGather {
  const __nv_bfloat16* x;        // set from IgOperand::x
  int PH, PW, SH, SW, SC, k, s, p, transposed;
  int pw_log2, php_log2, sc_log2;  // filled by the launcher
};
struct IgOperand {
  int kind;                      // IG_*
  const __nv_bfloat16* x;
  int64_t ld;                    // dense kinds: leading dimension (elements)
  int64_t plane;                 // planes == 2: elements from the hi plane to the lo plane
  IGather g;                     // gather kinds
};
struct IGemm {                   // C[m][n] (+)= sum_k A(m,k) B(n,k), fp32 C
  IgOperand a, b;
  float* C;
  int64_t ldc;
  int M, N, K;
  int planes = 1;                // 1: bf16; 2: hi/lo planes, hi*hi + hi*lo + lo*hi
  int splits = 1;
  float* partial = nullptr;      // splits*M*N floats when splits > 1
  int accumulate = 0;
  int auto_split = 0;            // with `partial` (>= 16*M*N floats): split k when the tile grid is small
  // weight-gradient epilogue: C is [(u, v, c < wg_cp)][o] (M = k*k*wg_cp, N = Co); instead of C, the
  // split sum is written straight to wg_out in PyTorch order [o][c < wg_cr][u][v] (needs `partial`)
  float* wg_out = nullptr;
  int wg_cp = 0, wg_cr = 0, wg_kk = 0;
};
ddppo_status launch_igemm(ddppo_ctx* ctx, const IGemm& g, cudaStream_t st);
// C[m][n] (+)= sum_z part[z*zs + m*N + n] (split order); weight-gradient form: dw[o][c < Cr][tap] =
// sum_z part[z*zs + (tap*Cp + c)*N + o]
ddppo_status launch_splitk_reduce(ddppo_ctx* ctx, const float* part, int splits, int64_t zs, int M, int N, float* C,
                                  int64_t ldc, int accumulate, cudaStream_t st);
ddppo_status launch_splitk_reduce_wgrad(ddppo_ctx* ctx, const float* part, int splits, int64_t zs, int N, int Cp, int Cr,
                                        int kk, float* dw, cudaStream_t st);

// TMA-fed tcgen05 implicit-GEMM convolutions (tconv.cu): FPROP / stride-1 DGRAD (flip) and WGRAD over
// NHWC bf16 tensors; *splits_out > 1: the result is in `partial` ([splits][M][N]) for the reductions above
ddppo_status launch_tconv_fwd(ddppo_ctx* ctx, const __nv_bfloat16* x, int64_t xplane, int F, int H, int W, int C,
                              int k, int s, int p, int flip, const __nv_bfloat16* w, int64_t wplane, int N, int planes,
                              float* out, int64_t ldc, int accumulate, float* partial, int max_splits, int slot,
                              int* splits_out, cudaStream_t st, const float* res = nullptr,
                              const float* res_mask = nullptr);
ddppo_status launch_tconv_dgrad_s2(ddppo_ctx* ctx, const __nv_bfloat16* dy, int64_t dy_plane, int F, int Ho, int Wo,
                                   int Co, int H, int W, int Ci, int k, int p, const __nv_bfloat16* wd,
                                   int64_t wd_plane, int planes, float* dx, int accumulate, cudaStream_t st);
ddppo_status launch_tconv_wgrad(ddppo_ctx* ctx, const __nv_bfloat16* x, int F, int H, int W, int C, int k, int s,
                                int p, const __nv_bfloat16* dy, int N, float* dw, int Cr, float* partial, int max_splits,
                                int slot, int* splits_out, cudaStream_t st, int groups = 1);

// NVLink peer memory (peer.cu)
ddppo_status peer_exchange(ddppo_ctx* ctx, void* local, void** out);
ddppo_status peer_setup_flags(ddppo_ctx* ctx);
// sum of n <= kMaxCountVals int64 over the ranks (rank order) through the peer flag areas, on the
// context's own stream (host-blocking on that stream only)
ddppo_status peer_allreduce_counts(ddppo_ctx* ctx, int64_t* host_vals, int n);
// a8 of one minibatch over peer memory (ctx->a8_mode): peers[j] = rank j's gradient, pgs[j] = rank j's
// staged-shard buffer (both as mapped here); gsum scratch [P]; Adam step = *dstep + step_add
ddppo_status launch_peer_a8(ddppo_ctx* ctx, float* const* peers, float* const* pgs, float* gsum, float* params,
                            float* m, float* v, int64_t P, const ddppo_adam_cfg& cfg, const int* dstep, int step_add,
                            cudaStream_t st, const uint8_t* freeze = nullptr, int64_t frz_end = 0);
// Adam on an already summed gradient whose clip scale is in ctx->d_scalars[0] (adam.cu)
ddppo_status launch_adam_only(ddppo_ctx* ctx, const float* grad, float* params, float* m, float* v,
                              const uint8_t* freeze, int64_t P, const ddppo_adam_cfg& cfg, const int* dstep,
                              int step_add, cudaStream_t st, int64_t frz_end = 0);

// tcgen05 GEMM: C[m][n] (+)= sum_k A(m,k) B(n,k) over fp32 operands with generic strides (gemm_tc.cu)
struct GemmTC {
  const float* A;
  int64_t sam, sak;
  const float* B;
  int64_t sbn, sbk;
  float* C;
  int64_t ldc;
  int M, N, K;
  int splits = 1;            // split-K (> 1 needs `partial`, splits*M*N floats; summed in split order)
  float* partial = nullptr;
  int prec = 1;              // 1: bf16 operands; 3: bf16x3 (x = hi + lo, hi*hi + hi*lo + lo*hi), ~fp32 accuracy
  int accumulate = 0;        // C += result (else C = result)
};
ddppo_status launch_gemm_tc(ddppo_ctx* ctx, const GemmTC& g, cudaStream_t st);

// models
struct ModelLayout {
  int64_t P = 0;
  int n = 0;
  ddppo_tensor_info t[512];
};
ddppo_status build_layout(const ddppo_model_desc* d, ModelLayout* out);
int64_t layout_offset(const ModelLayout& L, const char* name);
// one past the last element of the visual encoder's tensors ("enc.*", which lead the layout); 0 if none
int64_t encoder_end(const ModelLayout& L);

size_t toy_workspace(int max_B, int T);
ddppo_status toy_fwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     float* logits, float* values, void* ws, cudaStream_t st);
ddppo_status toy_bwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     const float* dlogits, const float* dvalues, float* grad, void* ws, cudaStream_t st);

// Linear(H, A+1) head over Hs [S][H] (H = 512 or 1024)
ddppo_status launch_head_fwd(ddppo_ctx* ctx, const float* Wo, const float* bo, const float* Hs, int S, int H,
                             float* logits, float* values, cudaStream_t st);
ddppo_status launch_head_bwd(ddppo_ctx* ctx, const float* Wo, const float* Hs, const float* dlogits,
                             const float* dvalues, int S, int H, float* dH, float* dWo, float* dbo, cudaStream_t st);
ddppo_status launch_colsum(ddppo_ctx* ctx, const float* A, int lda, int S, int M, float* out, cudaStream_t st);

size_t depth_workspace(int arch, int hidden, int max_B, int T);
ddppo_status depth_fwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                       float* logits, float* values, void* ws, cudaStream_t st);
ddppo_status depth_bwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                       const float* dlogits, const float* dvalues, float* grad, void* ws, cudaStream_t st);

// LSTM-512 cluster recurrences (lstm.cu).  Sample s = b*T_run + t.
struct LstmPtrs {
  const float* Whh;    // [2048][512]
  const float* bih;    // [2048]
  const float* bhh;    // [2048]
  const float* GI;     // [S][2048]  W_ih x (no bias)
  const float* mask;   // [E][ld]
  const float* h0;     // [E][sld] (this layer's 512 entries at the pointer)
  const float* c0;     // [E][sld]
  const int32_t* env_idx;
  int B, T_run, ld;
  int sld;             // env stride of h0 / c0 (512 * layers)
  float* Hs;           // [S][512] h_t
  float* Hin;          // [S][512] mask_t h_{t-1}
  float* Cin;          // [S][512] mask_t c_{t-1}
  float* Cs;           // [S][512] c_t
  float4* IFGO;        // [S][512] gate activations (i, f, g, o)
  const float* dH;     // [S][512] dL/dh_t from above
  float* dG;           // [S][2048] dL/d(gate pre-activations)
  int H = 512;         // hidden size: 512 (lstm.cu, one cluster) or 1024 (lstm_wide.cu, 32 CTAs)
  // LSTM-1024 only: L2 exchange buffers (lstm_wide_exchange_bytes) and the device error word
  void* hx = nullptr;
  float* xpart = nullptr;
  unsigned* xcnt = nullptr;
  int* err = nullptr;
};
constexpr int kLstmWideCounters = 64;  // 4 forward group counters + 32 backward owner counters
size_t lstm_wide_exchange_bytes();
size_t lstm_wide_part_offset();  // byte offset of the backward's partials in the exchange buffer
ddppo_status launch_lstm1024_fwd(ddppo_ctx* ctx, const LstmPtrs& p, cudaStream_t st);
ddppo_status launch_lstm1024_bwd(ddppo_ctx* ctx, const LstmPtrs& p, cudaStream_t st);
ddppo_status launch_lstm_fwd(ddppo_ctx* ctx, const LstmPtrs& p, cudaStream_t st);
ddppo_status launch_lstm_bwd(ddppo_ctx* ctx, const LstmPtrs& p, cudaStream_t st);

size_t gps_workspace(int max_B, int T);
const float* gps_hidden_out(void* ws, int B, int T);
void depth_state_out(const ModelLayout& L, void* ws, int B, int T_run, int l, const float** Hs, const float** Cs);
ddppo_status gps_fwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     float* logits, float* values, void* ws, cudaStream_t st, bool skip_head = false);
ddppo_status gps_bwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     const float* dlogits, const float* dvalues, float* grad, void* ws, cudaStream_t st,
                     bool dh_ready = false);
// the recurrence + fused head / PPO loss / head input gradient (one launch; the learner runtime)
ddppo_status gps_fwd_loss(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                          const ddppo_loss_inputs& in, const float* mean_invstd, const ddppo_loss_cfg& cfg,
                          float* dlogits, float* dvalues, float* stats, void* ws, cudaStream_t st);

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
// the visual agents (a ResNet encoder over frames + LSTM policy) / those with RGB-D 256^2 input and a
// 2-layer LSTM
inline bool arch_rgbd(int a) {
  return a == DDPPO_ARCH_RGBD_R50_LSTM2 || a == DDPPO_ARCH_RGBD_SERX50_LSTM2 || a == DDPPO_ARCH_RGBD_SERX101_LSTM2;
}
inline bool arch_visual(int a) {
  return a == DDPPO_ARCH_DEPTH_R18_LSTM || arch_rgbd(a);
}
