// Per-sample PPO loss math shared by the loss kernels (loss.cu) and the GRU forward kernel's fused
// head + loss epilogue (gps.cu).  P:L129-138 (Eq. 2), readings Z3-Z5; the gradient
// derivation is in oracle/ppo.py.
#pragma once
#include "common.cuh"

namespace {

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

}  // namespace
