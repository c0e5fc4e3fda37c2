// C-ABI entry points of libddppo.so (include/ddppo.h): context / NCCL plumbing, argument
// checking, the preemption protocol and the learner-step runtime that sequences the kernels.
#include <string.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

void destroy_graph_cache(ddppo_ctx* ctx);

extern "C" {

int ddppo_abi_version(void) { return DDPPO_ABI_VERSION; }

const char* ddppo_status_string(ddppo_status s) {
  switch (s) {
    case DDPPO_OK: return "ok";
    case DDPPO_ERR_CONFIG: return "config";
    case DDPPO_ERR_NUMERICAL: return "numerical";
    case DDPPO_ERR_PROTOCOL: return "protocol";
    case DDPPO_ERR_COMM: return "comm";
    case DDPPO_ERR_CUDA: return "cuda";
    case DDPPO_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown";
}

ddppo_status ddppo_get_unique_id(uint8_t host_id[128]) {
  if (!host_id) return DDPPO_ERR_CONFIG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return DDPPO_ERR_COMM;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(host_id, &id, 128);
  return DDPPO_OK;
}

ddppo_status ddppo_ctx_create(int rank, int world, const uint8_t* host_id, int device, ddppo_ctx** host_out) {
  if (!host_out || world < 1 || rank < 0 || rank >= world) return DDPPO_ERR_CONFIG;
  *host_out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return DDPPO_ERR_UNSUPPORTED;
  if (device < 0 || device >= ndev) return DDPPO_ERR_CONFIG;
  if (cudaSetDevice(device) != cudaSuccess) return DDPPO_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return DDPPO_ERR_CUDA;
  if (prop.major != 10 || prop.minor != 0) return DDPPO_ERR_UNSUPPORTED;  // built for sm_100a only
  ddppo_ctx* ctx = new ddppo_ctx();
  ctx->rank = rank;
  ctx->world = world;
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  bool ok = cudaMalloc(&ctx->d_err, sizeof(int)) == cudaSuccess &&
            cudaMalloc(&ctx->d_counters, CNT_NUM * sizeof(unsigned int)) == cudaSuccess &&
            cudaMalloc(&ctx->d_partials, kMaxPartials * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&ctx->d_scalars, 64 * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&ctx->d_i32, 64 * sizeof(int32_t)) == cudaSuccess &&
            cudaMalloc(&ctx->d_i64, kMaxCountVals * sizeof(int64_t)) == cudaSuccess &&
            cudaMalloc(&ctx->d_tile_cnt, kMaxTileCounters * sizeof(int)) == cudaSuccess;
  ok = ok && cudaMemset(ctx->d_err, 0, sizeof(int)) == cudaSuccess &&
       cudaMemset(ctx->d_counters, 0, CNT_NUM * sizeof(unsigned int)) == cudaSuccess &&
       cudaMemset(ctx->d_tile_cnt, 0, kMaxTileCounters * sizeof(int)) == cudaSuccess &&
       cudaDeviceSynchronize() == cudaSuccess;
  if (!ok) {
    ddppo_ctx_destroy(ctx);
    return DDPPO_ERR_CUDA;
  }
  if (world > 1) {
    if (!host_id) {
      ddppo_ctx_destroy(ctx);
      return DDPPO_ERR_CONFIG;
    }
    ncclUniqueId id;
    memcpy(&id, host_id, 128);
    if (ncclCommInitRank(&ctx->comm, world, id, rank) != ncclSuccess) {
      ctx->comm = nullptr;
      ddppo_ctx_destroy(ctx);
      return DDPPO_ERR_COMM;
    }
  }
  *host_out = ctx;
  return DDPPO_OK;
}

ddppo_status ddppo_ctx_destroy(ddppo_ctx* ctx) {
  if (!ctx) return DDPPO_OK;
  for (auto& r : ctx->pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ctx->pool) cudaEventDestroy(e);
  destroy_graph_cache(ctx);
  cudaFree(ctx->d_step);
  cudaFree(ctx->d_peer_epoch);
  for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
  for (auto e : ctx->fork_events) cudaEventDestroy(e);
  for (auto s : ctx->side)
    if (s) cudaStreamDestroy(s);
  cudaFree(ctx->own_flags);
  if (ctx->cnt_stream) cudaStreamDestroy(ctx->cnt_stream);
  if (ctx->h_cnt) cudaFreeHost(ctx->h_cnt);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_counters);
  cudaFree(ctx->d_partials);
  cudaFree(ctx->d_scalars);
  cudaFree(ctx->d_i32);
  cudaFree(ctx->d_i64);
  cudaFree(ctx->d_tile_cnt);
  delete ctx;
  return DDPPO_OK;
}

const char* ddppo_last_error(const ddppo_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null ctx"; }

ddppo_status ddppo_check(ddppo_ctx* ctx, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_CUDA_TRY(ctx, cudaStreamSynchronize(as_stream(stream)));
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  int err = 0;
  DDPPO_CUDA_TRY(ctx, cudaMemcpy(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err & ERR_BIT_COMM) {
    // the exchange left parameters untouched; counters of kernels that returned early are reset
    DDPPO_CUDA_TRY(ctx, cudaMemset(ctx->d_err, 0, sizeof(int)));
    DDPPO_CUDA_TRY(ctx, cudaMemset(ctx->d_counters, 0, CNT_NUM * sizeof(unsigned int)));
    ctx->last_error = "peer exchange timed out (a rank did not reach the gradient exchange)";
    return DDPPO_ERR_COMM;
  }
  if (err) {
    DDPPO_CUDA_TRY(ctx, cudaMemset(ctx->d_err, 0, sizeof(int)));
    ctx->last_error = std::string("non-finite value in ") + ((err & ERR_BIT_LOSS) ? "loss " : "") +
                      ((err & ERR_BIT_GRAD) ? "gradient" : "");
    return DDPPO_ERR_NUMERICAL;
  }
  return DDPPO_OK;
}

// ------------------------------------------------------------------ a2 / a3
ddppo_status ddppo_gae(ddppo_ctx* ctx, const float* rew, const float* val, const uint8_t* done, const int32_t* len,
                       int E, int T, int ld, float gamma, float tau, float* adv, float* ret, double* stats3,
                       void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, E == 0 || (rew && val && done && len && adv && ret), "gae: null pointer");
  return launch_gae(ctx, rew, val, done, len, E, T, ld, gamma, tau, adv, ret, stats3, as_stream(stream));
}

ddppo_status ddppo_adv_norm(ddppo_ctx* ctx, double* stats3, float eps, float* mean_invstd, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, stats3 && mean_invstd, "adv_norm: null pointer");
  cudaStream_t st = as_stream(stream);
  if (ctx->world > 1) {
    ProfScope ps(ctx, DDPPO_K_ALLREDUCE, st, 0);
    DDPPO_NCCL_TRY(ctx, ncclAllReduce(stats3, stats3, 3, ncclFloat64, ncclSum, ctx->comm, st));
  }
  return launch_adv_finalize(ctx, stats3, eps, mean_invstd, st);
}

// ------------------------------------------------------------------ model
ddppo_status ddppo_model_param_count(const ddppo_model_desc* host_desc, int64_t* host_P) {
  ModelLayout L;
  if (!host_P || build_layout(host_desc, &L) != DDPPO_OK) return DDPPO_ERR_CONFIG;
  *host_P = L.P;
  return DDPPO_OK;
}

ddppo_status ddppo_model_param_layout(const ddppo_model_desc* host_desc, ddppo_tensor_info* host_out, int cap,
                                      int* host_n) {
  ModelLayout L;
  if (!host_n || build_layout(host_desc, &L) != DDPPO_OK) return DDPPO_ERR_CONFIG;
  *host_n = L.n;
  if (host_out)
    for (int i = 0; i < L.n && i < cap; ++i) host_out[i] = L.t[i];
  return DDPPO_OK;
}

ddppo_status ddppo_workspace_size(const ddppo_model_desc* host_desc, int max_B, int T, size_t* host_bytes) {
  ModelLayout L;
  if (!host_bytes || build_layout(host_desc, &L) != DDPPO_OK || max_B < 1 || T < 1) return DDPPO_ERR_CONFIG;
  *host_bytes = host_desc->arch == DDPPO_ARCH_TOY_MLP   ? toy_workspace(max_B, T)
                : host_desc->arch == DDPPO_ARCH_GPS_GRU ? gps_workspace(max_B, T)
                                                        : depth_workspace(host_desc->arch, host_desc->hidden, max_B, T);
  return DDPPO_OK;
}

static ddppo_status check_batch(ddppo_ctx* ctx, const ddppo_batch* b) {
  DDPPO_REQUIRE(ctx, b != nullptr, "null batch");
  DDPPO_REQUIRE(ctx, b->B >= 1 && b->T >= 1 && b->T_run >= 1 && b->T_run <= b->T && b->ld >= b->T + 1 &&
                         b->E >= b->B,
                "batch: need 1 <= B <= E, 1 <= T_run <= T, ld >= T+1");
  DDPPO_REQUIRE(ctx, b->goal && b->len && b->env_idx, "batch: null pointer");
  return DDPPO_OK;
}

ddppo_status ddppo_policy_fwd(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, const float* params,
                              const ddppo_batch* host_batch, float* logits, float* values, void* ws, size_t ws_bytes,
                              void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  ModelLayout L;
  DDPPO_REQUIRE(ctx, build_layout(host_desc, &L) == DDPPO_OK, "bad model descriptor");
  ddppo_status s = check_batch(ctx, host_batch);
  if (s != DDPPO_OK) return s;
  size_t need = 0;
  ddppo_workspace_size(host_desc, host_batch->B, host_batch->T_run, &need);
  DDPPO_REQUIRE(ctx, ws && ws_bytes >= need, "workspace too small");
  if (host_desc->arch == DDPPO_ARCH_TOY_MLP)
    return toy_fwd(ctx, L, params, *host_batch, logits, values, ws, as_stream(stream));
  DDPPO_REQUIRE(ctx, host_batch->prev_action && host_batch->mask && host_batch->h0, "gps batch: null pointer");
  if (arch_visual(host_desc->arch)) {
    DDPPO_REQUIRE(ctx, host_batch->obs && host_batch->c0, "visual agent batch: obs and c0 required");
    return depth_fwd(ctx, L, params, *host_batch, logits, values, ws, as_stream(stream));
  }
  return gps_fwd(ctx, L, params, *host_batch, logits, values, ws, as_stream(stream));
}

ddppo_status ddppo_policy_bwd(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, const float* params,
                              const ddppo_batch* host_batch, const float* dlogits, const float* dvalues, float* grad,
                              void* ws, size_t ws_bytes, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  ModelLayout L;
  DDPPO_REQUIRE(ctx, build_layout(host_desc, &L) == DDPPO_OK, "bad model descriptor");
  ddppo_status s = check_batch(ctx, host_batch);
  if (s != DDPPO_OK) return s;
  size_t need = 0;
  ddppo_workspace_size(host_desc, host_batch->B, host_batch->T_run, &need);
  DDPPO_REQUIRE(ctx, ws && ws_bytes >= need, "workspace too small");
  if (host_desc->arch == DDPPO_ARCH_TOY_MLP)
    return toy_bwd(ctx, L, params, *host_batch, dlogits, dvalues, grad, ws, as_stream(stream));
  if (arch_visual(host_desc->arch))
    return depth_bwd(ctx, L, params, *host_batch, dlogits, dvalues, grad, ws, as_stream(stream));
  DDPPO_REQUIRE(ctx, host_batch->dgoal == nullptr, "policy_bwd: dgoal is produced by the visual agents only");
  return gps_bwd(ctx, L, params, *host_batch, dlogits, dvalues, grad, ws, as_stream(stream));
}

// ------------------------------------------------------------------ a6
ddppo_status ddppo_ppo_loss_grad(ddppo_ctx* ctx, const float* logits, const float* values,
                                 const ddppo_batch* host_batch, const ddppo_loss_inputs* host_in,
                                 const float* mean_invstd, const ddppo_loss_cfg* host_cfg, float* dlogits,
                                 float* dvalues, float* stats, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, host_batch && host_in && host_cfg && logits && values && dlogits && dvalues && stats,
                "loss: null pointer");
  DDPPO_REQUIRE(ctx, host_batch->env_idx && host_batch->len && host_batch->ld >= host_batch->T_run,
                "loss: bad batch");
  return launch_loss(ctx, logits, values, *host_batch, *host_in, mean_invstd, *host_cfg, dlogits, dvalues, stats,
                     as_stream(stream));
}

// ------------------------------------------------------------------ a8
ddppo_status ddppo_grad_allreduce_step(ddppo_ctx* ctx, float* grad, float* params, float* m, float* v,
                                       const uint8_t* freeze_mask, int64_t P, const ddppo_adam_cfg* host_cfg,
                                       float* grad_norm, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, grad && params && m && v && host_cfg && P >= 1, "grad_allreduce_step: bad arguments");
  cudaStream_t st = as_stream(stream);
  if (ctx->world > 1) {
    ProfScope ps(ctx, DDPPO_K_ALLREDUCE, st, 0);
    DDPPO_NCCL_TRY(ctx, ncclAllReduce(grad, grad, (size_t)P, ncclFloat32, ncclSum, ctx->comm, st));
  }
  return launch_clip_adam(ctx, grad, params, m, v, freeze_mask, P, *host_cfg, 1.f / (float)ctx->world, grad_norm,
                          st);
}

// ------------------------------------------------------------------ a9 / a10
ddppo_status ddppo_preempt_threshold(const ddppo_preempt_cfg* c, int world, int* host_K, int* host_min_steps) {
  if (!c || world < 1 || c->T < 1 || c->p_percent < 1 || c->p_percent > 100) return DDPPO_ERR_CONFIG;
  const int base = c->other_workers ? world - 1 : world;
  int K = (c->p_percent * base + 99) / 100;
  if (K < 1) K = 1;
  if (host_K) *host_K = K;
  if (host_min_steps) *host_min_steps = c->min_steps > 0 ? c->min_steps : (c->T + 3) / 4;
  return DDPPO_OK;
}

ddppo_status ddppo_preempt_decide(const ddppo_preempt_cfg* c, int world, int my_steps, int finished_count,
                                  int* host_should_stop) {
  int K = 0, ms = 0;
  ddppo_status s = ddppo_preempt_threshold(c, world, &K, &ms);
  if (s != DDPPO_OK || !host_should_stop) return DDPPO_ERR_CONFIG;
  *host_should_stop = (my_steps >= c->T) || (my_steps >= ms && finished_count >= K);
  return DDPPO_OK;
}

ddppo_status ddppo_preempt_poll(ddppo_ctx* ctx, int my_steps, int finished, int active,
                                const ddppo_preempt_cfg* host_cfg, int* host_should_stop, int* host_finished_count,
                                int* host_active_count) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  int32_t h[2] = {finished ? 1 : 0, active ? 1 : 0};
  if (ctx->world > 1) {
    if (ctx->peer_flags[ctx->rank]) {
      // a registered learner's NVLink peer areas: one exchange kernel on the context's own stream
      int64_t v[2] = {h[0], h[1]};
      ddppo_status s = peer_allreduce_counts(ctx, v, 2);
      if (s != DDPPO_OK) return s;
      h[0] = (int32_t)v[0];
      h[1] = (int32_t)v[1];
    } else {
      // NCCL on the context's own non-blocking stream (not queued behind the caller's work)
      if (!ctx->cnt_stream) {
        DDPPO_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->cnt_stream, cudaStreamNonBlocking));
        DDPPO_CUDA_TRY(ctx, cudaMallocHost(&ctx->h_cnt, kMaxCountVals * sizeof(int64_t)));
      }
      int32_t* hp = reinterpret_cast<int32_t*>(ctx->h_cnt);
      hp[0] = h[0];
      hp[1] = h[1];
      DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_i32, hp, sizeof(h), cudaMemcpyHostToDevice, ctx->cnt_stream));
      DDPPO_NCCL_TRY(ctx, ncclAllReduce(ctx->d_i32, ctx->d_i32, 2, ncclInt32, ncclSum, ctx->comm, ctx->cnt_stream));
      DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(hp, ctx->d_i32, sizeof(h), cudaMemcpyDeviceToHost, ctx->cnt_stream));
      DDPPO_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->cnt_stream));
      h[0] = hp[0];
      h[1] = hp[1];
    }
  }
  if (host_finished_count) *host_finished_count = h[0];
  if (host_active_count) *host_active_count = h[1];
  int stop = 0;
  ddppo_status s = ddppo_preempt_decide(host_cfg, ctx->world, my_steps, h[0], &stop);
  if (s != DDPPO_OK) {
    ctx->last_error = "preempt: bad cfg";
    return s;
  }
  if (host_should_stop) *host_should_stop = stop;
  return DDPPO_OK;
}

ddppo_status ddppo_rollout_steps(const int32_t* host_len, int E, int T, int64_t* host_steps) {
  if (!host_len || !host_steps || E < 1 || T < 1) return DDPPO_ERR_CONFIG;
  int64_t n = 0;
  for (int e = 0; e < E; ++e) {
    if (host_len[e] < 0) return DDPPO_ERR_CONFIG;
    n += host_len[e] < T ? host_len[e] : T;
  }
  *host_steps = n;
  return DDPPO_OK;
}

ddppo_status ddppo_allreduce_counts(ddppo_ctx* ctx, int64_t* host_vals, int n) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, host_vals && n >= 0 && n <= kMaxCountVals, "allreduce_counts: 0 <= n <= 64");
  if (ctx->world == 1 || n == 0) return DDPPO_OK;
  // with the NVLink peer areas set up (a registered learner): an exchange on the context's own
  // stream, so the host does not wait behind the learner work queued on the caller's stream
  if (ctx->peer_flags[ctx->rank]) return peer_allreduce_counts(ctx, host_vals, n);
  if (!ctx->cnt_stream) {
    DDPPO_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->cnt_stream, cudaStreamNonBlocking));
    DDPPO_CUDA_TRY(ctx, cudaMallocHost(&ctx->h_cnt, kMaxCountVals * sizeof(int64_t)));
  }
  for (int i = 0; i < n; ++i) ctx->h_cnt[i] = host_vals[i];
  DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_i64, ctx->h_cnt, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                                      ctx->cnt_stream));
  DDPPO_NCCL_TRY(ctx, ncclAllReduce(ctx->d_i64, ctx->d_i64, n, ncclInt64, ncclSum, ctx->comm, ctx->cnt_stream));
  DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_cnt, ctx->d_i64, n * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                      ctx->cnt_stream));
  DDPPO_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->cnt_stream));
  for (int i = 0; i < n; ++i) host_vals[i] = ctx->h_cnt[i];
  return DDPPO_OK;
}

// ------------------------------------------------------------------ learner step runtime
namespace {
struct LearnerWs {
  double* stats3;
  float* mean_invstd;
  float* logits;
  float* values;
  float* dlogits;
  float* dvalues;
  float* grad;      // this minibatch's gradient (one of grad2[], by minibatch parity when peers are used)
  float* grad2[2];
  float* gsum;      // rank-ordered sum of all ranks' gradients (peer path)
  float* pgather;   // this rank's updated parameter shard, read by the peers (sharded a8)
  float* grad_norm;
  float* stats;     // [epochs*minibatches][8] loss statistics (copied to the caller's stats_out after the step)
  void* model_ws;
  size_t model_bytes;
};
size_t carve_learner(const ddppo_model_desc* d, int E, int T, int mb, int epochs, void* base, LearnerWs* w) {
  int64_t P = 0;
  ddppo_model_param_count(d, &P);
  const int B = E / mb;
  size_t model_bytes = 0;
  ddppo_workspace_size(d, B, T, &model_bytes);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? reinterpret_cast<char*>(base) + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  };
  LearnerWs t;
  t.stats3 = (double*)take(4 * sizeof(double));
  t.mean_invstd = (float*)take(4 * sizeof(float));
  t.logits = (float*)take((size_t)B * T * 4 * sizeof(float));
  t.values = (float*)take((size_t)B * T * sizeof(float));
  t.dlogits = (float*)take((size_t)B * T * 4 * sizeof(float));
  t.dvalues = (float*)take((size_t)B * T * sizeof(float));
  t.grad2[0] = (float*)take((size_t)P * sizeof(float));
  t.grad2[1] = (float*)take((size_t)P * sizeof(float));
  t.grad = t.grad2[0];
  t.gsum = (float*)take((size_t)P * sizeof(float));
  t.pgather = (float*)take((size_t)P * sizeof(float));
  t.grad_norm = (float*)take(8 * sizeof(float));
  t.stats = (float*)take((size_t)epochs * mb * 8 * sizeof(float));
  t.model_ws = take(model_bytes);
  t.model_bytes = model_bytes;
  if (w) *w = t;
  return off;
}
}  // namespace

ddppo_status ddppo_learner_workspace_size(const ddppo_model_desc* host_desc, int E, int T, int ld, int minibatches,
                                          int epochs, size_t* host_bytes) {
  ModelLayout L;
  if (!host_bytes || build_layout(host_desc, &L) != DDPPO_OK || minibatches < 1 || E % minibatches || T < 1 ||
      ld < T + 1 || epochs < 1)
    return DDPPO_ERR_CONFIG;
  *host_bytes = carve_learner(host_desc, E, T, minibatches, epochs, nullptr, nullptr);
  return DDPPO_OK;
}

ddppo_status ddppo_layout_hash(const ddppo_model_desc* host_desc, int E, int T, int ld, int minibatches, int epochs,
                               uint64_t* host_hash) {
  ModelLayout L;
  if (!host_hash || build_layout(host_desc, &L) != DDPPO_OK) return DDPPO_ERR_CONFIG;
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* c = reinterpret_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
  };
  for (int i = 0; i < L.n; ++i) {
    const ddppo_tensor_info& t = L.t[i];
    mix(t.name, strnlen(t.name, sizeof(t.name)));
    mix(&t.offset, sizeof(t.offset));
    mix(&t.numel, sizeof(t.numel));
    mix(&t.ndim, sizeof(t.ndim));
    mix(t.shape, sizeof(int64_t) * (size_t)t.ndim);
  }
  const int32_t geo[5] = {E, T, ld, minibatches, epochs};
  mix(geo, sizeof(geo));
  *host_hash = h;
  return DDPPO_OK;
}

ddppo_status ddppo_layout_check(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, int E, int T, int ld,
                                int minibatches, int epochs) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  uint64_t h = 0;
  DDPPO_REQUIRE(ctx, ddppo_layout_hash(host_desc, E, T, ld, minibatches, epochs, &h) == DDPPO_OK,
                "layout_check: bad model descriptor");
  if (ctx->world == 1) return DDPPO_OK;
  uint64_t* d = nullptr;
  DDPPO_CUDA_TRY(ctx, cudaMalloc(&d, sizeof(uint64_t) * ctx->world));
  std::vector<uint64_t> all(ctx->world);
  ncclResult_t nr = ncclSuccess;
  cudaError_t ce = cudaMemcpy(d + ctx->rank, &h, sizeof(h), cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) nr = ncclAllGather(d + ctx->rank, d, 1, ncclUint64, ctx->comm, 0);
  if (ce == cudaSuccess && nr == ncclSuccess)
    ce = cudaMemcpy(all.data(), d, sizeof(uint64_t) * ctx->world, cudaMemcpyDeviceToHost);
  cudaFree(d);
  DDPPO_CUDA_TRY(ctx, ce);
  DDPPO_NCCL_TRY(ctx, nr);
  std::string bad;
  for (int r = 0; r < ctx->world; ++r)
    if (all[r] != all[0]) bad += " " + std::to_string(r);
  if (!bad.empty()) {
    ctx->last_error = "layout hash differs from rank 0's on rank(s)" + bad;
    return DDPPO_ERR_PROTOCOL;
  }
  return DDPPO_OK;
}

ddppo_status ddppo_learner_register(ddppo_ctx* ctx, void* ws, size_t ws_bytes) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, ws && ws_bytes > 0, "learner_register: null workspace");
  if (ctx->world == 1) return DDPPO_OK;  // nothing to share
  DDPPO_REQUIRE(ctx, ctx->world <= kMaxPeers, "learner_register: at most 8 ranks");
  DDPPO_REQUIRE(ctx, ctx->peer_ws == nullptr, "learner_register: a workspace is already registered");
  ddppo_status s = peer_setup_flags(ctx);
  if (s != DDPPO_OK) return s;
  void* out[kMaxPeers] = {};
  s = peer_exchange(ctx, ws, out);
  if (s != DDPPO_OK) return s;
  for (int r = 0; r < ctx->world; ++r) ctx->peer_ws_base[r] = reinterpret_cast<char*>(out[r]);
  ctx->peer_ws = ws;
  ctx->peer_mb = 0;
  return DDPPO_OK;
}

}  // extern "C"

namespace {
__global__ void set_int_kernel(int* p, int v) { *p = v; }
__global__ void add_int_kernel(int* p, int v) { *p += v; }

struct MbShape {
  int T_run, n_valid;
};

// a2..a8 for one rollout, every host-side value fixed by (config, pointers, mbs): replayable as a
// CUDA graph.  Adam's update count is read on the device (*ctx->d_step + k + 1 for minibatch k).
ddppo_status learner_body(ddppo_ctx* ctx, const ModelLayout& L, const ddppo_model_desc* host_desc,
                          const ddppo_rollout* ro, const ddppo_learner_cfg* cfg, float* params, float* m, float* v,
                          float* adv, float* ret, float* stats_out, void* ws, LearnerWs& w, cudaStream_t st,
                          const std::vector<MbShape>& mbs, bool use_peers, uint64_t peer_mb0) {
  const bool visual = arch_visual(host_desc->arch);
  // a2 GAE (+ local adv stats), a3 global normalisation statistics
  ddppo_status s = launch_gae(ctx, ro->rew, ro->val, ro->done, ro->len, ro->E, ro->T, ro->ld, cfg->gamma, cfg->tau,
                              adv, ret, w.stats3, st);
  if (s != DDPPO_OK) return s;
  if (cfg->normalize_adv) {
    s = ddppo_adv_norm(ctx, w.stats3, cfg->adv_eps, w.mean_invstd, st);
    if (s != DDPPO_OK) return s;
  }
  const int B = ro->E / cfg->minibatches;
  ddppo_loss_inputs li = {ro->action, ro->logp_old, ro->val, ret, adv};
  // a frozen visual encoder (NEXT-4): its tensors lead the layout; Adam leaves [0, frz_end) untouched
  const int64_t frz_end = (cfg->freeze_encoder && visual) ? encoder_end(L) : 0;
  const ddppo_adam_cfg acfg = cfg->adam;
  int k = 0;
  for (int e = 0; e < cfg->epochs; ++e) {
    for (int j = 0; j < cfg->minibatches; ++j, ++k) {
      ddppo_batch b;
      b.goal = ro->goal;
      b.prev_action = ro->prev_action;
      b.mask = ro->mask;
      b.h0 = ro->h0;
      b.len = ro->len;
      b.env_idx = ro->perms + (size_t)e * ro->E + (size_t)j * B;
      b.E = ro->E;
      b.T = ro->T;
      b.ld = ro->ld;
      b.B = B;
      b.T_run = mbs[k].T_run;  // a4: the minibatch runs to its longest env
      b.n_valid = mbs[k].n_valid;
      b.obs = ro->obs;
      b.obs_rgb = ro->obs_rgb;
      b.dgoal = nullptr;
      b.flags = cfg->freeze_encoder ? DDPPO_BATCH_FREEZE_ENCODER : 0;
      b.reserved_flags = 0;
      b.c0 = ro->c0;
      float* st_out = w.stats + (size_t)k * 8;
      const float* mis = cfg->normalize_adv ? w.mean_invstd : nullptr;
      if (host_desc->arch == DDPPO_ARCH_TOY_MLP)
        s = toy_fwd(ctx, L, params, b, w.logits, w.values, w.model_ws, st);
      else if (visual)
        s = depth_fwd(ctx, L, params, b, w.logits, w.values, w.model_ws, st);
      else  // GPS: the recurrence with head + PPO loss + head input gradient in its epilogue, one launch
        s = gps_fwd_loss(ctx, L, params, b, li, mis, cfg->loss, w.dlogits, w.dvalues, st_out, w.model_ws, st);
      if (s != DDPPO_OK) return s;
      if (host_desc->arch != DDPPO_ARCH_GPS_GRU)
        s = launch_loss(ctx, w.logits, w.values, b, li, mis, cfg->loss, w.dlogits, w.dvalues, st_out, st);
      if (s != DDPPO_OK) return s;
      w.grad = use_peers ? w.grad2[(peer_mb0 + k) & 1] : w.grad2[0];
      if (host_desc->arch == DDPPO_ARCH_TOY_MLP)
        s = toy_bwd(ctx, L, params, b, w.dlogits, w.dvalues, w.grad, w.model_ws, st);
      else if (visual)
        s = depth_bwd(ctx, L, params, b, w.dlogits, w.dvalues, w.grad, w.model_ws, st);
      else
        s = gps_bwd(ctx, L, params, b, w.dlogits, w.dvalues, w.grad, w.model_ws, st, /*dh_ready=*/true);
      if (s != DDPPO_OK) return s;
      if (use_peers) {  // a8 over NVLink peer memory: rank-ordered sum + clip norm, then Adam
        ProfScope ps(ctx, DDPPO_K_ALLREDUCE, st, 0);
        float* peers[kMaxPeers];
        float* pgs[kMaxPeers];
        const size_t off = (size_t)((char*)w.grad - (char*)ws), off_pg = (size_t)((char*)w.pgather - (char*)ws);
        for (int r = 0; r < ctx->world; ++r) {
          peers[r] = reinterpret_cast<float*>(ctx->peer_ws_base[r] + off);
          pgs[r] = reinterpret_cast<float*>(ctx->peer_ws_base[r] + off_pg);
        }
        s = launch_peer_a8(ctx, peers, pgs, w.gsum, params, m, v, L.P, acfg, ctx->d_step, k + 1, st, cfg->freeze_mask,
                           frz_end);
      } else {
        if (ctx->world > 1) {
          ProfScope ps(ctx, DDPPO_K_ALLREDUCE, st, 0);
          DDPPO_NCCL_TRY(ctx, ncclAllReduce(w.grad, w.grad, (size_t)L.P, ncclFloat32, ncclSum, ctx->comm, st));
        }
        s = launch_clip_adam(ctx, w.grad, params, m, v, cfg->freeze_mask, L.P, acfg, 1.f / (float)ctx->world, nullptr,
                             st, ctx->d_step, k + 1, frz_end);
      }
      if (s != DDPPO_OK) return s;
    }
  }
  add_int_kernel<<<1, 1, 0, st>>>(ctx->d_step, k);  // the device update count advances with the step
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

template <typename T>
void key_put(std::vector<unsigned char>& key, const T& v) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(&v);
  key.insert(key.end(), p, p + sizeof(T));
}
}  // namespace

struct ddppo_ctx::GraphCache {
  struct Entry {
    std::vector<unsigned char> key;
    cudaGraphExec_t exec = nullptr;
    int64_t launches[DDPPO_K_COUNT] = {};
    uint64_t used = 0;
  };
  static constexpr size_t kMaxEntries = 4;  // e.g. double-buffered outputs: a few live keys
  std::vector<Entry> entries;
  // keys run eagerly so far (most recent last, a few kept): a key is captured when it repeats (its
  // lazy setup is done) -- also when keys alternate (e.g. double-buffered statistics)
  std::vector<std::vector<unsigned char>> seen;
  uint64_t clock = 0;
  cudaStream_t stream = nullptr;    // capture / replay stream (non-blocking; the caller's may be legacy)
};

void destroy_graph_cache(ddppo_ctx* ctx) {
  if (!ctx->graph) return;
  for (auto& e : ctx->graph->entries)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  if (ctx->graph->stream) cudaStreamDestroy(ctx->graph->stream);
  delete ctx->graph;
  ctx->graph = nullptr;
}

extern "C" {

ddppo_status ddppo_set_a8_mode(ddppo_ctx* ctx, int mode) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, mode == DDPPO_A8_SHARDED || mode == DDPPO_A8_ALLREAD || mode == DDPPO_A8_AUTO,
                "set_a8_mode: unknown mode");
  ctx->a8_mode = mode;
  return DDPPO_OK;
}

ddppo_status ddppo_set_conv_engine(ddppo_ctx* ctx, int engine) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, engine == DDPPO_CONV_TMA || engine == DDPPO_CONV_CPASYNC, "set_conv_engine: unknown engine");
  ctx->conv_engine = engine;
  return DDPPO_OK;
}

ddppo_status ddppo_set_fwd_planes(ddppo_ctx* ctx, int planes) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, planes == 1 || planes == 2, "set_fwd_planes: 1 or 2");
  ctx->fwd_planes = planes;
  return DDPPO_OK;
}

ddppo_status ddppo_set_graphs(ddppo_ctx* ctx, int enable) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  ctx->graphs = enable != 0;
  return DDPPO_OK;
}

ddppo_status ddppo_learner_step(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, const ddppo_rollout* ro,
                                const ddppo_learner_cfg* cfg, float* params, float* m, float* v, float* adv,
                                float* ret, float* stats_out, void* ws, size_t ws_bytes, int32_t* host_step_out,
                                void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  ModelLayout L;
  DDPPO_REQUIRE(ctx, build_layout(host_desc, &L) == DDPPO_OK, "bad model descriptor");
  DDPPO_REQUIRE(ctx, ro && cfg && params && m && v && adv && ret && ws, "learner_step: null pointer");
  DDPPO_REQUIRE(ctx, ro->host_len && ro->host_perms && ro->perms, "learner_step: lengths/perms required");
  DDPPO_REQUIRE(ctx, cfg->minibatches >= 1 && ro->E % cfg->minibatches == 0 && cfg->epochs >= 1,
                "learner_step: minibatches must divide E (S:L155)");
  DDPPO_REQUIRE(ctx, cfg->adam.step >= 0, "learner_step: adam.step must be >= 0");
  DDPPO_REQUIRE(ctx, cfg->freeze_mask == nullptr || ((uintptr_t)cfg->freeze_mask & 3) == 0,
                "learner_step: freeze_mask must be 4-byte aligned");
  DDPPO_REQUIRE(ctx, (cfg->normalize_adv != 0) == (cfg->loss.normalize_adv != 0),
                "learner_step: normalize_adv and loss.normalize_adv must agree");
  const bool visual = arch_visual(host_desc->arch);
  DDPPO_REQUIRE(ctx, !visual || (ro->obs && ro->c0), "learner_step: the visual agents need obs and c0");
  DDPPO_REQUIRE(ctx, !arch_rgbd(host_desc->arch) || ro->obs_rgb, "learner_step: RGB-D needs obs_rgb");
  size_t need = 0;
  ddppo_status s =
      ddppo_learner_workspace_size(host_desc, ro->E, ro->T, ro->ld, cfg->minibatches, cfg->epochs, &need);
  DDPPO_REQUIRE(ctx, s == DDPPO_OK, "learner_step: bad rollout geometry (ld >= T + 1, minibatches | E)");
  DDPPO_REQUIRE(ctx, ws_bytes >= need, "learner_step: workspace too small");
  LearnerWs w;
  carve_learner(host_desc, ro->E, ro->T, cfg->minibatches, cfg->epochs, ws, &w);
  cudaStream_t st = as_stream(stream);
  const bool use_peers = ctx->world > 1 && ctx->peer_ws == ws;  // ddppo_learner_register'ed workspace
  // a4 on the host: every minibatch's T_run / n_valid from the host copies of lengths and perms
  const int B = ro->E / cfg->minibatches;
  int L_max = 0;
  for (int n = 0; n < ro->E; ++n) L_max = std::max(L_max, std::min(ro->host_len[n], ro->T));
  DDPPO_REQUIRE(ctx, L_max >= 1, "learner_step: empty rollout");
  std::vector<MbShape> mbs;
  for (int e = 0; e < cfg->epochs; ++e)
    for (int j = 0; j < cfg->minibatches; ++j) {
      MbShape sh = {0, 0};
      for (int q = 0; q < B; ++q) {
        const int n = ro->host_perms[(size_t)e * ro->E + (size_t)j * B + q];
        DDPPO_REQUIRE(ctx, n >= 0 && n < ro->E, "learner_step: perms must hold env ids");
        const int Ln = std::min(ro->host_len[n], ro->T);
        sh.T_run = std::max(sh.T_run, Ln);
        sh.n_valid += Ln;
      }
      mbs.push_back(sh);
    }
  const int n_mb = (int)mbs.size();
  // Adam's update count lives on the device; (re)seed it when the caller's count differs
  if (!ctx->d_step) DDPPO_CUDA_TRY(ctx, cudaMalloc(&ctx->d_step, sizeof(int)));
  if ((int64_t)cfg->adam.step != ctx->step_expected) {
    set_int_kernel<<<1, 1, 0, st>>>(ctx->d_step, cfg->adam.step);
    ctx->count(1);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  }
  const uint64_t mb0 = ctx->peer_mb;
  const bool graph = ctx->graphs && !ctx->prof;  // per-family profiling needs per-launch events
  if (!graph) {
    s = learner_body(ctx, L, host_desc, ro, cfg, params, m, v, adv, ret, stats_out, ws, w, st, mbs, use_peers, mb0);
  } else {
    // the whole step as one CUDA graph, captured once per (configuration, buffers, minibatch shapes)
    std::vector<unsigned char> key;
    key_put(key, *host_desc);
    ddppo_rollout rk = *ro;
    rk.host_len = nullptr;
    rk.host_perms = nullptr;
    key_put(key, rk);
    ddppo_learner_cfg ck = *cfg;
    ck.adam.step = 0;
    key_put(key, ck);
    // (stats_out is not part of the key: the graph writes the workspace's statistics, copied out below)
    for (const void* p : {(const void*)params, (const void*)m, (const void*)v, (const void*)adv, (const void*)ret,
                          (const void*)ws})
      key_put(key, p);
    key_put(key, use_peers);
    key_put(key, ctx->a8_mode);
    key_put(key, ctx->conv_engine);
    key_put(key, ctx->fwd_planes);
    key_put(key, (int)(mb0 & 1));
    for (const MbShape& sh : mbs) key_put(key, sh);
    if (!ctx->graph) {
      ctx->graph = new ddppo_ctx::GraphCache();
      // the critical path (the capture / replay stream) at the highest priority: work forked to the
      // side streams (weight gradients) only fills SMs the chain of input gradients leaves idle
      int lo = 0, hi = 0;
      DDPPO_CUDA_TRY(ctx, cudaDeviceGetStreamPriorityRange(&lo, &hi));
      DDPPO_CUDA_TRY(ctx, cudaStreamCreateWithPriority(&ctx->graph->stream, cudaStreamNonBlocking, hi));
    }
    ddppo_ctx::GraphCache& gc = *ctx->graph;
    cudaStream_t gs = gc.stream;
    ddppo_ctx::GraphCache::Entry* hit = nullptr;
    for (auto& e : gc.entries)
      if (e.key == key) hit = &e;
    bool seen_before = false;
    for (const auto& k : gc.seen) seen_before = seen_before || k == key;
    if (!hit && !seen_before) {
      // first time with this configuration: run eagerly (lazy allocations, attribute setup), capture
      // when it repeats
      gc.seen.push_back(key);
      if (gc.seen.size() > 2 * ddppo_ctx::GraphCache::kMaxEntries) gc.seen.erase(gc.seen.begin());
      DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, gs));
      s = learner_body(ctx, L, host_desc, ro, cfg, params, m, v, adv, ret, stats_out, ws, w, gs, mbs, use_peers,
                       mb0);
      if (s != DDPPO_OK) return s;
      DDPPO_CUDA_TRY(ctx, fork_to(ctx, gs, st));
      if (stats_out)
        DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(stats_out, w.stats, (size_t)n_mb * 8 * sizeof(float),
                                            cudaMemcpyDeviceToDevice, st));
      ctx->step_expected = (int64_t)cfg->adam.step + n_mb;
      ctx->peer_mb = mb0 + (uint64_t)n_mb;
      if (host_step_out) *host_step_out = cfg->adam.step + n_mb;
      return DDPPO_OK;
    }
    if (!hit) {
      if (gc.entries.size() >= ddppo_ctx::GraphCache::kMaxEntries) {  // evict the least recently used
        size_t lru = 0;
        for (size_t i = 1; i < gc.entries.size(); ++i)
          if (gc.entries[i].used < gc.entries[lru].used) lru = i;
        cudaGraphExecDestroy(gc.entries[lru].exec);
        gc.entries.erase(gc.entries.begin() + (long)lru);
      }
      int64_t before[DDPPO_K_COUNT];
      memcpy(before, ctx->launches, sizeof(before));
      DDPPO_CUDA_TRY(ctx, cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
      s = learner_body(ctx, L, host_desc, ro, cfg, params, m, v, adv, ret, stats_out, ws, w, gs, mbs, use_peers,
                       mb0);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(gs, &g);
      if (s != DDPPO_OK || ce != cudaSuccess || !g) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        memcpy(ctx->launches, before, sizeof(before));
        if (s != DDPPO_OK) return s;
        ctx->last_error = std::string("learner_step: graph capture failed: ") + cudaGetErrorString(ce);
        return DDPPO_ERR_CUDA;
      }
      ddppo_ctx::GraphCache::Entry e;
      const cudaError_t ie = cudaGraphInstantiate(&e.exec, g, 0);
      cudaGraphDestroy(g);
      DDPPO_CUDA_TRY(ctx, ie);
      e.key = key;
      for (int i = 0; i < DDPPO_K_COUNT; ++i) e.launches[i] = ctx->launches[i] - before[i];
      memcpy(ctx->launches, before, sizeof(before));
      gc.entries.push_back(std::move(e));
      hit = &gc.entries.back();
    }
    hit->used = ++gc.clock;
    DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, gs));
    DDPPO_CUDA_TRY(ctx, cudaGraphLaunch(hit->exec, gs));
    DDPPO_CUDA_TRY(ctx, fork_to(ctx, gs, st));
    for (int i = 0; i < DDPPO_K_COUNT; ++i) ctx->launches[i] += hit->launches[i];
  }
  if (s != DDPPO_OK) return s;
  if (stats_out)  // outside the graph: the caller may alternate statistics buffers without new captures
    DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(stats_out, w.stats, (size_t)n_mb * 8 * sizeof(float),
                                        cudaMemcpyDeviceToDevice, st));
  ctx->step_expected = (int64_t)cfg->adam.step + n_mb;
  ctx->peer_mb = mb0 + (uint64_t)n_mb;
  if (host_step_out) *host_step_out = cfg->adam.step + n_mb;
  return DDPPO_OK;
}

// ------------------------------------------------------------------ measurement
ddppo_status ddppo_profile_enable(ddppo_ctx* ctx, int enable) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  ctx->prof = enable != 0;
  return DDPPO_OK;
}

ddppo_status ddppo_profile_flops(ddppo_ctx* ctx, double* host_flops, int reset) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  for (int i = 0; i < DDPPO_K_COUNT; ++i) {
    if (host_flops) host_flops[i] = ctx->flops[i];
    if (reset) ctx->flops[i] = 0.0;
  }
  return DDPPO_OK;
}

ddppo_status ddppo_profile_smem_bytes(ddppo_ctx* ctx, double* host_bytes, int reset) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  for (int i = 0; i < DDPPO_K_COUNT; ++i) {
    if (host_bytes) host_bytes[i] = ctx->smem_bytes[i];
    if (reset) ctx->smem_bytes[i] = 0.0;
  }
  return DDPPO_OK;
}

ddppo_status ddppo_profile_read(ddppo_ctx* ctx, double* host_ms, int64_t* host_launches, int reset) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  for (auto& r : ctx->pending) {
    DDPPO_CUDA_TRY(ctx, cudaEventSynchronize(r.b));
    float ms = 0.f;
    DDPPO_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, r.a, r.b));
    ctx->ms[r.fam] += ms;
    ctx->pool.push_back(r.a);
    ctx->pool.push_back(r.b);
  }
  ctx->pending.clear();
  for (int i = 0; i < DDPPO_K_COUNT; ++i) {
    if (host_ms) host_ms[i] = ctx->ms[i];
    if (host_launches) host_launches[i] = ctx->launches[i];
    if (reset) {
      ctx->ms[i] = 0.0;
      ctx->launches[i] = 0;
    }
  }
  return DDPPO_OK;
}

}  // extern "C"
