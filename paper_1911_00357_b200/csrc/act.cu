// Collection side (NEXT-1): batched single-step policy inference with action sampling
// (include/ddppo.h ddppo_policy_act).  P:L163 "each worker collects experience with pi_theta";
// P:L461 one batched forward per GPU over its environments.  The step runs the agent's own forward
// kernels on a T_run = 1 slice of the rollout (<= 8 envs per launch group, the recurrences' limit),
// reads the new recurrent state out of their workspace, then one thread per env samples an action
// from the logits with the documented counter-based generator.
#include "common.cuh"

namespace {

constexpr int kGroup = 8;  // envs per forward launch (the GRU / LSTM cluster kernels hold <= 8)

__device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void iota_kernel(int32_t* p, int n, int32_t* ones) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    p[i] = i;
    ones[i] = 1;
  }
}

// one thread per env: categorical sample (or argmax) from 4 logits
__global__ void sample_kernel(const float* __restrict__ logits, int E, int A, uint64_t seed, int64_t counter,
                              int greedy, int32_t* __restrict__ actions, float* __restrict__ logp) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const float* z = logits + (size_t)e * A;
  float m = z[0];
  int amax = 0;
  for (int a = 1; a < A; ++a)
    if (z[a] > m) {
      m = z[a];
      amax = a;
    }
  float w[8];
  float S = 0.f;
  for (int a = 0; a < A; ++a) {
    w[a] = expf(z[a] - m);
    S += w[a];
  }
  int act = A - 1;
  if (greedy) {
    act = amax;
  } else {
    const uint64_t r = splitmix64_d(seed * 0x9E3779B97F4A7C15ull + (uint64_t)counter * 0xD1B54A32D192ED03ull +
                                    (uint64_t)e) >> 40;
    const float target = ((float)r * 0x1p-24f) * S;
    float c = 0.f;
    for (int a = 0; a < A; ++a) {
      c += w[a];
      if (c > target) {
        act = a;
        break;
      }
    }
  }
  actions[e] = act;
  logp[e] = (z[act] - m) - logf(S);
}

__global__ void copy_rows_kernel(const float* __restrict__ src, int rows, int cols, float* __restrict__ dst, int ld_dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * cols; i += gridDim.x * blockDim.x) {
    const int r = i / cols, c = i - r * cols;
    dst[(size_t)r * ld_dst + c] = src[i];
  }
}

struct ActWs {
  int32_t* env_idx;
  int32_t* len;
  float* logits;
  float* values;
  void* model;
  size_t model_bytes;
};
size_t carve_act(const ddppo_model_desc* d, int E, void* base, ActWs* w) {
  size_t mb = 0;
  ddppo_workspace_size(d, std::min(E, kGroup), 1, &mb);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? reinterpret_cast<char*>(base) + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  };
  ActWs t;
  t.env_idx = (int32_t*)take((size_t)E * 4);
  t.len = (int32_t*)take((size_t)E * 4);
  t.logits = (float*)take((size_t)E * 8 * 4);
  t.values = (float*)take((size_t)E * 4);
  t.model = take(mb);
  t.model_bytes = mb;
  if (w) *w = t;
  return off;
}

}  // namespace

extern "C" ddppo_status ddppo_act_workspace_size(const ddppo_model_desc* host_desc, int E, size_t* host_bytes) {
  ModelLayout L;
  if (!host_bytes || E < 1 || build_layout(host_desc, &L) != DDPPO_OK) return DDPPO_ERR_CONFIG;
  *host_bytes = carve_act(host_desc, E, nullptr, nullptr);
  return DDPPO_OK;
}

extern "C" ddppo_status ddppo_policy_act(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, const float* params,
                                         const ddppo_act_batch* a, int32_t* actions, float* logp, float* values,
                                         float* logits, void* ws, size_t ws_bytes, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  ModelLayout L;
  DDPPO_REQUIRE(ctx, build_layout(host_desc, &L) == DDPPO_OK, "act: bad model descriptor");
  DDPPO_REQUIRE(ctx, a && params && actions && logp && values && ws, "act: null pointer");
  DDPPO_REQUIRE(ctx, a->E >= 1 && a->T >= 1 && a->t >= 0 && a->t < a->T && a->ld >= a->T + 1, "act: bad geometry");
  DDPPO_REQUIRE(ctx, a->goal && a->prev_action && a->mask && a->h_in && a->h_out, "act: null input");
  const int arch = host_desc->arch;
  const bool visual = arch_visual(arch);
  DDPPO_REQUIRE(ctx, arch != DDPPO_ARCH_TOY_MLP, "act: the toy MLP has no recurrent policy (use ddppo_policy_fwd)");
  DDPPO_REQUIRE(ctx, !visual || (a->obs && a->c_in && a->c_out), "act: the visual agents need obs and c_in / c_out");
  const size_t need = carve_act(host_desc, a->E, nullptr, nullptr);
  DDPPO_REQUIRE(ctx, ws_bytes >= need, "act: workspace too small (ddppo_act_workspace_size)");
  ActWs w;
  carve_act(host_desc, a->E, ws, &w);
  cudaStream_t st = as_stream(stream);
  const int A = host_desc->num_actions, layers = arch_rgbd(arch) ? 2 : 1;
  const int H = host_desc->hidden, sld = layers * H;
  iota_kernel<<<1, 256, 0, st>>>(w.env_idx, a->E, w.len);
  ctx->count(1);
  const int64_t HW = arch_rgbd(arch) ? 256 * 256 : 64 * 64;
  for (int e0 = 0; e0 < a->E; e0 += kGroup) {
    const int B = std::min(kGroup, a->E - e0);
    ddppo_batch b = {};
    b.goal = a->goal + (size_t)a->t * 3;  // column t of [E][T][3]: element (env, 0) -> (env, t)
    b.prev_action = a->prev_action + a->t;
    b.mask = a->mask + a->t;
    b.h0 = a->h_in;
    b.len = w.len;
    b.env_idx = w.env_idx + e0;
    b.E = a->E;
    b.T = a->T;
    b.ld = a->ld;
    b.B = B;
    b.T_run = 1;
    b.n_valid = B;
    if (visual) {
      b.obs = a->obs + (size_t)a->t * HW;
      b.obs_rgb = a->obs_rgb ? a->obs_rgb + (size_t)a->t * 3 * HW : nullptr;
      b.c0 = a->c_in;
    }
    float* lg = w.logits + (size_t)e0 * A;
    float* vl = w.values + e0;
    ddppo_status s = visual ? depth_fwd(ctx, L, params, b, lg, vl, w.model, st)
                            : gps_fwd(ctx, L, params, b, lg, vl, w.model, st);
    if (s != DDPPO_OK) return s;
    // the new recurrent state (sample b*1 + 0 of each layer) -> h_out / c_out rows e0..e0+B
    for (int l = 0; l < layers; ++l) {
      const float *Hs = nullptr, *Cs = nullptr;
      if (visual) depth_state_out(L, w.model, B, 1, l, &Hs, &Cs);
      else Hs = gps_hidden_out(w.model, B, 1);
      copy_rows_kernel<<<grid_for(B * H, 256, 64), 256, 0, st>>>(Hs, B, H, a->h_out + (size_t)e0 * sld + l * H, sld);
      if (visual)
        copy_rows_kernel<<<grid_for(B * H, 256, 64), 256, 0, st>>>(Cs, B, H, a->c_out + (size_t)e0 * sld + l * H, sld);
      ctx->count(visual ? 2 : 1);
    }
  }
  sample_kernel<<<grid_for(a->E, 128, 1024), 128, 0, st>>>(w.logits, a->E, A, a->seed, a->counter, a->greedy, actions,
                                                          logp);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(values, w.values, (size_t)a->E * 4, cudaMemcpyDeviceToDevice, st));
  if (logits) DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(logits, w.logits, (size_t)a->E * A * 4, cudaMemcpyDeviceToDevice, st));
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
