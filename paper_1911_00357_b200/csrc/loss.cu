// a6 fused PPO loss + gradient (K3).
//
// P:L129-138 (Eq. 2): min(r A, clip(r, 1-eps, 1+eps) A), r = pi/pi_old; value term
// with PPO2 value clipping and an entropy bonus (readings Z3/Z4); per-worker mean
// over the valid samples (P:L171 equal weighting).  One thread per sample (A = 4: one float4
// of logits), grid-stride; reads 16 (logits) + 4 (value) + 4 (action) + 4*4 (lp_old, V_old,
// R, A) = 40 B and writes 16 + 4 = 20 B per sample.  Loss statistics are reduced in fp64 in
// fixed block order (last-block pattern) -- bit-reproducible, no float atomics.
// Gradient (closed form, torch tie conventions; derivation in oracle/ppo.py):
//   dL/dz_j = -(1/n) A rho [u <= c] (1[j=a] - p_j) + (c_e/n) p_j (log p_j + H)
//   dL/dv   =  (c_v/n) * (e1 if e1^2 > e2^2 ; e2*[|v-v_old| <= eps_v] if e1^2 < e2^2 ; average if =)
#include "common.cuh"

namespace {

constexpr int kThreads = 256;

struct SampleOut {
  float4 dz;
  float dv;
  float surr, lv, H, clipped, kl;
};

// one valid sample: logits z, value v, action a, lp_old, V_old, R, normalised A (Eq. 2 + Z3-Z5)
__device__ __forceinline__ SampleOut ppo_sample(float4 z, float v, int a, float lpo, float vo, float R, float A,
                                                float inv_n, float eps, float vclip_eps, float c_v, float c_e,
                                                int use_vclip) {
  SampleOut o;
  const float zmax = fmaxf(fmaxf(z.x, z.y), fmaxf(z.z, z.w));
  const float e0 = __expf(z.x - zmax), e1 = __expf(z.y - zmax), e2 = __expf(z.z - zmax), e3 = __expf(z.w - zmax);
  const float se = e0 + e1 + e2 + e3;
  const float lse = zmax + __logf(se);
  const float lp0 = z.x - lse, lp1 = z.y - lse, lp2 = z.z - lse, lp3 = z.w - lse;
  const float inv_se = 1.f / se;
  const float p0 = e0 * inv_se, p1 = e1 * inv_se, p2 = e2 * inv_se, p3 = e3 * inv_se;
  const float za = a == 0 ? z.x : a == 1 ? z.y : a == 2 ? z.z : z.w;
  const float lp = za - lse;
  const float rho = __expf(lp - lpo);
  const float u = rho * A;
  const float rc = fminf(fmaxf(rho, 1.f - eps), 1.f + eps);
  const float c = rc * A;
  o.surr = fminf(u, c);
  o.H = -(p0 * lp0 + p1 * lp1 + p2 * lp2 + p3 * lp3);
  // value loss
  const float e1v = v - R;
  float gv;
  if (use_vclip) {
    const float d = v - vo;
    const float vc = vo + fminf(fmaxf(d, -vclip_eps), vclip_eps);
    const float e2v = vc - R;
    const float s1 = e1v * e1v, s2 = e2v * e2v;
    o.lv = 0.5f * fmaxf(s1, s2);
    const float inside = (fabsf(d) <= vclip_eps) ? 1.f : 0.f;
    gv = s1 > s2 ? e1v : (s1 < s2 ? e2v * inside : 0.5f * e1v + 0.5f * e2v * inside);
  } else {
    o.lv = 0.5f * e1v * e1v;
    gv = e1v;
  }
  // policy gradient wrt log pi(a): -(1/n) * dmin/drho * A * rho
  const float gu = u < c ? 1.f : (u == c ? 0.5f : 0.f);
  const float inside_r = (rho >= 1.f - eps && rho <= 1.f + eps) ? 1.f : 0.f;
  const float dlp = -inv_n * (gu * A + (1.f - gu) * A * inside_r) * rho;
  const float ce = c_e * inv_n;
  o.dz.x = dlp * ((a == 0 ? 1.f : 0.f) - p0) + ce * p0 * (lp0 + o.H);
  o.dz.y = dlp * ((a == 1 ? 1.f : 0.f) - p1) + ce * p1 * (lp1 + o.H);
  o.dz.z = dlp * ((a == 2 ? 1.f : 0.f) - p2) + ce * p2 * (lp2 + o.H);
  o.dz.w = dlp * ((a == 3 ? 1.f : 0.f) - p3) + ce * p3 * (lp3 + o.H);
  o.dv = c_v * inv_n * gv;
  o.clipped = (fabsf(rho - 1.f) > eps) ? 1.f : 0.f;
  o.kl = lpo - lp;
  return o;
}

__device__ __forceinline__ void write_stats(const double (&fin)[6], float inv_n, float c_v, float c_e, float n_valid,
                                            float* stats_out, int* err) {
  const double in = (double)inv_n;
  stats_out[0] = (float)(-fin[0] * in);
  stats_out[1] = (float)(fin[1] * in);
  stats_out[2] = (float)(fin[2] * in);
  stats_out[3] = (float)(fin[3] * in);
  stats_out[4] = (float)(fin[4] * in);
  const float tot = (float)(-fin[0] * in + (double)c_v * fin[1] * in - (double)c_e * fin[2] * in);
  stats_out[5] = tot;
  stats_out[6] = n_valid;
  stats_out[7] = 0.f;
  if (!isfinite(tot)) atomicOr(err, ERR_BIT_LOSS);
}

__global__ void __launch_bounds__(kThreads)
ppo_loss_kernel(const float* __restrict__ logits, const float* __restrict__ values,
                const int32_t* __restrict__ env_idx, const int32_t* __restrict__ len, int B, int T_run, int ld,
                const int32_t* __restrict__ action, const float* __restrict__ logp_old,
                const float* __restrict__ value_old, const float* __restrict__ ret, const float* __restrict__ adv,
                const float* __restrict__ mean_invstd, float inv_n, float eps, float vclip_eps, float c_v, float c_e,
                int use_vclip, float* __restrict__ dlogits, float* __restrict__ dvalues, double* partials,
                unsigned int* counter, float* stats_out, int* err, float n_valid) {
  __shared__ double red[6 * (kThreads / 32)];
  __shared__ double fin[6];
  double acc[6] = {0, 0, 0, 0, 0, 0};
  float mu = 0.f, invstd = 1.f;
  if (mean_invstd) {
    mu = mean_invstd[0];
    invstd = mean_invstd[1];
  }
  const int M = B * T_run;
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < M; m += gridDim.x * blockDim.x) {
    const int b = m / T_run, t = m - b * T_run;
    const int n = env_idx[b];
    float4 dz = make_float4(0.f, 0.f, 0.f, 0.f);
    float dv = 0.f;
    if (t < len[n]) {
      const size_t s = (size_t)n * ld + t;
      const float A = mean_invstd ? (adv[s] - mu) * invstd : adv[s];
      const SampleOut o = ppo_sample(*reinterpret_cast<const float4*>(logits + (size_t)m * 4), values[m], action[s],
                                     logp_old[s], value_old[s], ret[s], A, inv_n, eps, vclip_eps, c_v, c_e, use_vclip);
      dz = o.dz;
      dv = o.dv;
      acc[0] += (double)o.surr;
      acc[1] += (double)o.lv;
      acc[2] += (double)o.H;
      acc[3] += (double)o.clipped;
      acc[4] += (double)o.kl;
    }
    *reinterpret_cast<float4*>(dlogits + (size_t)m * 4) = dz;
    dvalues[m] = dv;
  }
  if (last_block_reduce<6>(acc, partials, counter, fin, red)) {
    if (threadIdx.x == 0) write_stats(fin, inv_n, c_v, c_e, n_valid, stats_out, err);
  }
}

// The head, the loss and the head's input gradient of one minibatch in one pass (learner runtime):
// warp per sample: logits / value = W_o h + b_o (h = Hs[s], 512), the sample's loss gradient
// (ppo_sample), then dH[s] = W_o^T [dlogits; dvalue]; dlogits / dvalues are stored for the head's
// weight gradient; loss statistics reduced as in ppo_loss_kernel (fixed order).
constexpr int kHid = 512;
__global__ void __launch_bounds__(kThreads)
head_loss_kernel(const float* __restrict__ Wo, const float* __restrict__ bo, const float* __restrict__ Hs,
                 const int32_t* __restrict__ env_idx, const int32_t* __restrict__ len, int B, int T_run, int ld,
                 const int32_t* __restrict__ action, const float* __restrict__ logp_old,
                 const float* __restrict__ value_old, const float* __restrict__ ret, const float* __restrict__ adv,
                 const float* __restrict__ mean_invstd, float inv_n, float eps, float vclip_eps, float c_v, float c_e,
                 int use_vclip, float* __restrict__ dlogits, float* __restrict__ dvalues, float* __restrict__ dH,
                 double* partials, unsigned int* counter, float* stats_out, int* err, float n_valid) {
  __shared__ double red[6 * (kThreads / 32)];
  __shared__ double fin[6];
  __shared__ float wo[5 * kHid];
  for (int i = threadIdx.x; i < 5 * kHid; i += blockDim.x) wo[i] = Wo[i];
  __syncthreads();
  double acc[6] = {0, 0, 0, 0, 0, 0};
  float mu = 0.f, invstd = 1.f;
  if (mean_invstd) {
    mu = mean_invstd[0];
    invstd = mean_invstd[1];
  }
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31, M = B * T_run;
  for (int m = blockIdx.x * warps + (threadIdx.x >> 5); m < M; m += gridDim.x * warps) {
    const int b = m / T_run, t = m - b * T_run;
    const int n = env_idx[b];
    const float* h = Hs + (size_t)m * kHid;
    float hv[kHid / 32];
    float out[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < kHid / 32; ++i) {
      hv[i] = h[lane + 32 * i];
#pragma unroll
      for (int o = 0; o < 5; ++o) out[o] += wo[o * kHid + lane + 32 * i] * hv[i];
    }
#pragma unroll
    for (int o = 0; o < 5; ++o) out[o] = warp_sum(out[o]) + bo[o];
    float4 dz = make_float4(0.f, 0.f, 0.f, 0.f);
    float dv = 0.f;
    if (t < len[n]) {  // (warp-uniform)
      const size_t s = (size_t)n * ld + t;
      const float A = mean_invstd ? (adv[s] - mu) * invstd : adv[s];
      const SampleOut o = ppo_sample(make_float4(out[0], out[1], out[2], out[3]), out[4], action[s], logp_old[s],
                                     value_old[s], ret[s], A, inv_n, eps, vclip_eps, c_v, c_e, use_vclip);
      dz = o.dz;
      dv = o.dv;
      if (lane == 0) {
        acc[0] += (double)o.surr;
        acc[1] += (double)o.lv;
        acc[2] += (double)o.H;
        acc[3] += (double)o.clipped;
        acc[4] += (double)o.kl;
      }
    }
    if (lane == 0) {
      *reinterpret_cast<float4*>(dlogits + (size_t)m * 4) = dz;
      dvalues[m] = dv;
    }
    float* dh = dH + (size_t)m * kHid;
#pragma unroll
    for (int i = 0; i < kHid / 32; ++i) {
      const int k = lane + 32 * i;
      dh[k] = wo[k] * dz.x + wo[kHid + k] * dz.y + wo[2 * kHid + k] * dz.z + wo[3 * kHid + k] * dz.w +
              wo[4 * kHid + k] * dv;
    }
  }
  if (last_block_reduce<6>(acc, partials, counter, fin, red)) {
    if (threadIdx.x == 0) write_stats(fin, inv_n, c_v, c_e, n_valid, stats_out, err);
  }
}

}  // namespace

ddppo_status launch_head_loss(ddppo_ctx* ctx, const float* Wo, const float* bo, const float* Hs, const ddppo_batch& b,
                              const ddppo_loss_inputs& in, const float* mean_invstd, const ddppo_loss_cfg& cfg,
                              float* dlogits, float* dvalues, float* dH, float* stats, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.T_run >= 1 && b.n_valid >= 1, "loss: need B, T_run, n_valid >= 1");
  DDPPO_REQUIRE(ctx, !cfg.normalize_adv || mean_invstd, "loss: normalize_adv needs mean_invstd");
  const int M = b.B * b.T_run;
  const int blocks = grid_for(M, kThreads / 32, ctx->sm_count * 2);
  ProfScope ps(ctx, DDPPO_K_LOSS, st, 1);
  head_loss_kernel<<<blocks, kThreads, 0, st>>>(
      Wo, bo, Hs, b.env_idx, b.len, b.B, b.T_run, b.ld, in.action, in.logp_old, in.value_old, in.ret, in.adv,
      cfg.normalize_adv ? mean_invstd : nullptr, 1.f / (float)b.n_valid, cfg.clip_eps, cfg.vclip_eps, cfg.c_v,
      cfg.c_e, cfg.use_value_clip, dlogits, dvalues, dH, ctx->d_partials, ctx->d_counters + CNT_LOSS, stats,
      ctx->d_err, (float)b.n_valid);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status launch_loss(ddppo_ctx* ctx, const float* logits, const float* values, const ddppo_batch& b,
                         const ddppo_loss_inputs& in, const float* mean_invstd, const ddppo_loss_cfg& cfg,
                         float* dlogits, float* dvalues, float* stats, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.T_run >= 1 && b.n_valid >= 1, "loss: need B, T_run, n_valid >= 1");
  DDPPO_REQUIRE(ctx, (uintptr_t)logits % 16 == 0 && (uintptr_t)dlogits % 16 == 0, "loss: logits must be 16B aligned");
  DDPPO_REQUIRE(ctx, !cfg.normalize_adv || mean_invstd, "loss: normalize_adv needs mean_invstd");
  const int M = b.B * b.T_run;
  const int blocks = grid_for(M, kThreads, ctx->sm_count * 8);
  ProfScope ps(ctx, DDPPO_K_LOSS, st, 1);
  ppo_loss_kernel<<<blocks, kThreads, 0, st>>>(
      logits, values, b.env_idx, b.len, b.B, b.T_run, b.ld, in.action, in.logp_old, in.value_old, in.ret, in.adv,
      cfg.normalize_adv ? mean_invstd : nullptr, 1.f / (float)b.n_valid, cfg.clip_eps, cfg.vclip_eps, cfg.c_v,
      cfg.c_e, cfg.use_value_clip, dlogits, dvalues, ctx->d_partials, ctx->d_counters + CNT_LOSS, stats,
      ctx->d_err, (float)b.n_valid);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
