// a8 (after the NCCL sum): fused 1/N scale + global-L2 clip + Adam (K16 v1).
//
// P:L150-158 (Eq. 3) ParamUpdate(theta, (1/N) sum_i grad_i); P:L219 Adam lr 2.5e-4; readings
// Z14/Z15: beta 0.9/0.999, eps 1e-8, PyTorch bias-corrected form, clip 0.5 on the
// averaged gradient with coef = min(1, max_norm/(||g|| + 1e-6)).
// Two launches: (1) sum of squares of g/N in fp64 per block -> last block -> coef (device
// scalar, so the update needs no host round trip); (2) the elementwise update, float4.
// HBM traffic 4P (pass 1) + 28P (pass 2: read g, p, m, v; write p, m, v) bytes.
#include <string.h>

#include "common.cuh"

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
grad_norm_kernel(const float* __restrict__ g, int64_t P, float inv_world, float max_norm, double* partials,
                 unsigned int* counter, float* scalars, float* grad_norm_out, int* err) {
  pdl_enter();
  __shared__ double red[kThreads / 32];
  __shared__ double fin[1];
  double acc[1] = {0.0};
  const int64_t P4 = P / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float s = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P4; i += stride) {
    const float4 x = reinterpret_cast<const float4*>(g)[i];
    const float a = x.x * inv_world, b = x.y * inv_world, c = x.z * inv_world, d = x.w * inv_world;
    s += a * a + b * b + c * c + d * d;
  }
  for (int64_t i = P4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    const float a = g[i] * inv_world;
    s += a * a;
  }
  acc[0] = (double)s;
  if (last_block_reduce<1>(acc, partials, counter, fin, red)) {
    if (threadIdx.x == 0) {
      const double total = sqrt(fin[0]);
      double coef = 1.0;
      if (max_norm > 0.f) coef = fmin(1.0, (double)max_norm / (total + 1e-6));
      scalars[0] = (float)coef * inv_world;  // combined scale applied to the summed gradient
      scalars[1] = (float)total;
      if (grad_norm_out) grad_norm_out[0] = (float)total;
      if (!isfinite(total)) atomicOr(err, ERR_BIT_GRAD);
    }
  }
}


// step = (dstep ? *dstep : 0) + step_add (the learner runtime keeps the update count on the device, so
// a captured CUDA graph needs no host-side scalar); bias corrections in fp64 once per block
__global__ void __launch_bounds__(kThreads)
adam_kernel(const float* __restrict__ g, float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
            const uint8_t* __restrict__ freeze, int64_t P, const float* __restrict__ scalars, float b1, float b2,
            float lr, const int* __restrict__ dstep, int step_add, float eps, const int* err, int64_t frz_end) {
  pdl_enter();
  __shared__ float sbc[2];
  // a failed peer exchange (ERR_BIT_COMM) or a non-finite gradient norm (ERR_BIT_GRAD) leaves
  // the parameters untouched until ddppo_check reports it
  if (err && (*(volatile const int*)err & (ERR_BIT_COMM | ERR_BIT_GRAD))) return;
  if (threadIdx.x == 0) {
    const int step = (dstep ? *dstep : 0) + step_add;
    const double bc1 = 1.0 - pow((double)b1, (double)step), bc2 = 1.0 - pow((double)b2, (double)step);
    sbc[0] = (float)((double)lr / bc1);
    sbc[1] = (float)(1.0 / sqrt(bc2));
  }
  __syncthreads();
  const float step_size = sbc[0], inv_sqrt_bc2 = sbc[1];
  const float scale = scalars[0];
  const int64_t P4 = P / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // entries [0, frz_end) are frozen (the visual encoder of a transfer task: a multiple of 4 in the layout)
  for (int64_t i = frz_end / 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P4; i += stride) {
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    float4 pp = reinterpret_cast<float4*>(p)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    uint32_t fr = 0;
    if (freeze) fr = reinterpret_cast<const uint32_t*>(freeze)[i];
    float4 po = pp, mo = mm, vo = vv;
    adam_one(pp.x, mm.x, vv.x, gg.x * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
    adam_one(pp.y, mm.y, vv.y, gg.y * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
    adam_one(pp.z, mm.z, vv.z, gg.z * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
    adam_one(pp.w, mm.w, vv.w, gg.w * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
    if (fr) {
      if (fr & 0xffu) { pp.x = po.x; mm.x = mo.x; vv.x = vo.x; }
      if (fr & 0xff00u) { pp.y = po.y; mm.y = mo.y; vv.y = vo.y; }
      if (fr & 0xff0000u) { pp.z = po.z; mm.z = mo.z; vv.z = vo.z; }
      if (fr & 0xff000000u) { pp.w = po.w; mm.w = mo.w; vv.w = vo.w; }
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
  }
  for (int64_t i = P4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    if (freeze && freeze[i]) continue;
    float pp = p[i], mm = m[i], vv = v[i];
    adam_one(pp, mm, vv, g[i] * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
  }
}

}  // namespace

ddppo_status launch_adam_only(ddppo_ctx* ctx, const float* grad, float* params, float* m, float* v,
                              const uint8_t* freeze, int64_t P, const ddppo_adam_cfg& cfg, const int* dstep,
                              int step_add, cudaStream_t st, int64_t frz_end) {
  DDPPO_REQUIRE(ctx, P >= 1 && (dstep || step_add >= 1), "adam: need P >= 1 and step >= 1");
  DDPPO_REQUIRE(ctx, frz_end % 4 == 0 && frz_end <= P, "adam: frozen prefix must be a multiple of 4");
  const int blocks = grid_for((int)std::min<int64_t>((P + 3) / 4, 1 << 30), kThreads, ctx->sm_count * 4);
  ProfScope ps(ctx, DDPPO_K_ADAM, st, 1);
  launch_k(ctx, adam_kernel, blocks, kThreads, 0, st, grad, params, m, v, freeze, P, ctx->d_scalars, cfg.beta1,
           cfg.beta2,
                                           cfg.lr, dstep, step_add, cfg.eps, ctx->d_err, frz_end);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status launch_clip_adam(ddppo_ctx* ctx, float* grad, float* params, float* m, float* v,
                              const uint8_t* freeze, int64_t P, const ddppo_adam_cfg& cfg, float inv_world,
                              float* grad_norm, cudaStream_t st, const int* dstep, int step_add, int64_t frz_end) {
  if (!dstep) step_add = cfg.step;
  DDPPO_REQUIRE(ctx, P >= 1 && (dstep || step_add >= 1), "adam: need P >= 1 and step >= 1");
  DDPPO_REQUIRE(ctx, (uintptr_t)grad % 16 == 0 && (uintptr_t)params % 16 == 0 && (uintptr_t)m % 16 == 0 &&
                         (uintptr_t)v % 16 == 0 && (freeze == nullptr || (uintptr_t)freeze % 4 == 0),
                "adam: buffers must be 16-byte aligned");
  DDPPO_REQUIRE(ctx, frz_end % 4 == 0 && frz_end <= P, "adam: frozen prefix must be a multiple of 4");
  const int blocks = grid_for((int)std::min<int64_t>((P + 3) / 4, 1 << 30), kThreads, ctx->sm_count * 4);
  ProfScope ps(ctx, DDPPO_K_ADAM, st, 2);
  launch_k(ctx, grad_norm_kernel, blocks, kThreads, 0, st, grad, P, inv_world, cfg.max_grad_norm, ctx->d_partials,
                                                ctx->d_counters + CNT_NORM, ctx->d_scalars, grad_norm, ctx->d_err);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  launch_k(ctx, adam_kernel, blocks, kThreads, 0, st, grad, params, m, v, freeze, P, ctx->d_scalars, cfg.beta1,
           cfg.beta2,
                                           cfg.lr, dstep, step_add, cfg.eps, ctx->d_err, frz_end);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

// ---------------------------------------------------------------- critic re-initialisation (NEXT-4)
namespace {
__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void reinit_critic_kernel(float* __restrict__ w_row, float* __restrict__ b_elem, float* __restrict__ mw,
                                     float* __restrict__ vw, float* __restrict__ mb, float* __restrict__ vb, int fan_in,
                                     uint64_t seed) {
  pdl_enter();
  const float bound = 1.0f / sqrtf((float)fan_in);
  for (int i = threadIdx.x; i <= fan_in; i += blockDim.x) {
    const uint64_t u = splitmix64(seed * 0x9E3779B97F4A7C15ull + (uint64_t)i) >> 40;  // 24 random bits
    const float val = ((float)u * 0x1p-23f - 1.0f) * bound;
    if (i < fan_in) {
      w_row[i] = val;
      mw[i] = 0.f;
      vw[i] = 0.f;
    } else {
      *b_elem = val;
      *mb = 0.f;
      *vb = 0.f;
    }
  }
}
}  // namespace

extern "C" ddppo_status ddppo_reinit_critic(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, float* params, float* m,
                                            float* v, uint64_t seed, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  ModelLayout L;
  DDPPO_REQUIRE(ctx, build_layout(host_desc, &L) == DDPPO_OK, "reinit_critic: bad model descriptor");
  DDPPO_REQUIRE(ctx, params && m && v, "reinit_critic: null pointer");
  const int64_t hw = layout_offset(L, "head.weight"), hb = layout_offset(L, "head.bias");
  DDPPO_REQUIRE(ctx, hw >= 0 && hb >= 0, "reinit_critic: model has no head");
  int fan_in = 0, A = host_desc->num_actions;
  for (int i = 0; i < L.n; ++i)
    if (strcmp(L.t[i].name, "head.weight") == 0) fan_in = (int)L.t[i].shape[1];
  const int64_t row = hw + (int64_t)A * fan_in, bi = hb + A;
  cudaStream_t st = as_stream(stream);
  launch_k(ctx, reinit_critic_kernel, 1, 256, 0, st, params + row, params + bi, m + row, v + row, m + bi, v + bi,
           fan_in, seed);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
