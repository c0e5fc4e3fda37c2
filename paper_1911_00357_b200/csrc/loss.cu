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
#include "ppo_sample.cuh"

namespace {

constexpr int kThreads = 256;


__global__ void __launch_bounds__(kThreads)
ppo_loss_kernel(const float* __restrict__ logits, const float* __restrict__ values,
                const int32_t* __restrict__ env_idx, const int32_t* __restrict__ len, int B, int T_run, int ld,
                const int32_t* __restrict__ action, const float* __restrict__ logp_old,
                const float* __restrict__ value_old, const float* __restrict__ ret, const float* __restrict__ adv,
                const float* __restrict__ mean_invstd, float inv_n, float eps, float vclip_eps, float c_v, float c_e,
                int use_vclip, float* __restrict__ dlogits, float* __restrict__ dvalues, double* partials,
                unsigned int* counter, float* stats_out, int* err, float n_valid) {
  pdl_enter();
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

}  // namespace

ddppo_status launch_loss(ddppo_ctx* ctx, const float* logits, const float* values, const ddppo_batch& b,
                         const ddppo_loss_inputs& in, const float* mean_invstd, const ddppo_loss_cfg& cfg,
                         float* dlogits, float* dvalues, float* stats, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.T_run >= 1 && b.n_valid >= 1, "loss: need B, T_run, n_valid >= 1");
  DDPPO_REQUIRE(ctx, (uintptr_t)logits % 16 == 0 && (uintptr_t)dlogits % 16 == 0, "loss: logits must be 16B aligned");
  DDPPO_REQUIRE(ctx, !cfg.normalize_adv || mean_invstd, "loss: normalize_adv needs mean_invstd");
  const int M = b.B * b.T_run;
  const int blocks = grid_for(M, kThreads, ctx->sm_count * 8);
  ProfScope ps(ctx, DDPPO_K_LOSS, st, 1);
  launch_k(ctx, ppo_loss_kernel, blocks, kThreads, 0, st, 
      logits, values, b.env_idx, b.len, b.B, b.T_run, b.ld, in.action, in.logp_old, in.value_old, in.ret, in.adv,
      cfg.normalize_adv ? mean_invstd : nullptr, 1.f / (float)b.n_valid, cfg.clip_eps, cfg.vclip_eps, cfg.c_v,
      cfg.c_e, cfg.use_value_clip, dlogits, dvalues, ctx->d_partials, ctx->d_counters + CNT_LOSS, stats,
      ctx->d_err, (float)b.n_valid);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
