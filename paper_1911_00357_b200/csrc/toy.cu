// Flat parameter layouts (include/ddppo.h) and the toy MLP actor-critic (configs[0]).
//
// Toy: goal [d, cos th, sin th] -> Linear(3,64) -> tanh -> Linear(64, A+1).  Samples
// are independent; M = B*T_run is tiny (8 in configs[0]), so one CTA does the forward and one
// CTA per hidden unit group does the backward with fixed-order sums (deterministic).
#include <string.h>

#include "common.cuh"

static void add_tensor(ModelLayout* L, const char* name, int ndim, const int64_t* shape, int fan_in) {
  ddppo_tensor_info& t = L->t[L->n++];
  memset(&t, 0, sizeof(t));
  strncpy(t.name, name, sizeof(t.name) - 1);
  t.ndim = ndim;
  t.numel = 1;
  for (int i = 0; i < ndim; ++i) {
    t.shape[i] = shape[i];
    t.numel *= shape[i];
  }
  t.fan_in = fan_in;
  t.offset = (L->P + 3) / 4 * 4;
  L->P = t.offset + t.numel;
}

ddppo_status build_layout(const ddppo_model_desc* d, ModelLayout* out) {
  if (!d || d->num_actions != 4) return DDPPO_ERR_CONFIG;
  ModelLayout L;
  const int64_t A1 = d->num_actions + 1;
  if (d->arch == DDPPO_ARCH_TOY_MLP) {
    if (d->hidden != 64) return DDPPO_ERR_CONFIG;
    const int64_t h = 64;
    int64_t s0[2] = {h, 3}, s1[1] = {h}, s2[2] = {A1, h}, s3[1] = {A1};
    add_tensor(&L, "fc1.weight", 2, s0, 3);
    add_tensor(&L, "fc1.bias", 1, s1, 3);
    add_tensor(&L, "head.weight", 2, s2, (int)h);
    add_tensor(&L, "head.bias", 1, s3, (int)h);
  } else if (d->arch == DDPPO_ARCH_GPS_GRU) {
    if (d->hidden != 512) return DDPPO_ERR_CONFIG;
    const int64_t H = d->hidden, G = 3 * H;
    int64_t a[2] = {32, 3}, b[1] = {32}, c[2] = {A1, 32}, wi[2] = {G, 64}, wh[2] = {G, H}, bg[1] = {G},
            hw[2] = {A1, H}, hb[1] = {A1};
    add_tensor(&L, "goal_fc.weight", 2, a, 3);
    add_tensor(&L, "goal_fc.bias", 1, b, 3);
    add_tensor(&L, "act_embed.weight", 2, c, 1);
    add_tensor(&L, "rnn.weight_ih", 2, wi, (int)H);
    add_tensor(&L, "rnn.weight_hh", 2, wh, (int)H);
    add_tensor(&L, "rnn.bias_ih", 1, bg, (int)H);
    add_tensor(&L, "rnn.bias_hh", 1, bg, (int)H);
    add_tensor(&L, "head.weight", 2, hw, (int)H);
    add_tensor(&L, "head.bias", 1, hb, (int)H);
  } else if (d->arch == DDPPO_ARCH_DEPTH_R18_LSTM || d->arch == DDPPO_ARCH_RGBD_R50_LSTM2 ||
             d->arch == DDPPO_ARCH_RGBD_SERX50_LSTM2 || d->arch == DDPPO_ARCH_RGBD_SERX101_LSTM2) {
    // LSTM 512 (one 16-CTA cluster, lstm.cu) or 1024 ("512-dimensional or 1024-dimensional",
    // 32 CTAs exchanging through L2, lstm_wide.cu)
    if (d->hidden != 512 && d->hidden != 1024) return DDPPO_ERR_CONFIG;
    const bool serx = d->arch == DDPPO_ARCH_RGBD_SERX50_LSTM2 || d->arch == DDPPO_ARCH_RGBD_SERX101_LSTM2;
    const bool r101 = d->arch == DDPPO_ARCH_RGBD_SERX101_LSTM2;
    const bool rgbd = d->arch == DDPPO_ARCH_RGBD_R50_LSTM2 || serx;
    (void)r101;
    const int64_t H = d->hidden, G = 4 * H;
    char name[48];
    // conv weight [Co][Ci][k][k] (fan_in Ci*k*k), GroupNorm gamma (ones: fan_in 0) / beta (zeros: -1)
    auto conv = [&](const char* pre, int64_t co, int64_t ci, int64_t k) {
      int64_t s[4] = {co, ci, k, k};
      snprintf(name, sizeof(name), "%s.weight", pre);
      add_tensor(&L, name, 4, s, (int)(ci * k * k));
    };
    auto gn = [&](const char* pre, int64_t c) {
      int64_t s[1] = {c};
      snprintf(name, sizeof(name), "%s.weight", pre);
      add_tensor(&L, name, 1, s, 0);
      snprintf(name, sizeof(name), "%s.bias", pre);
      add_tensor(&L, name, 1, s, -1);
    };
    conv("enc.stem.conv", 32, rgbd ? 4 : 1, 7);
    gn("enc.stem.gn", 32);
    const int64_t widths[4] = {32, 64, 128, 256};
    int64_t cin = 32;
    char pre[40], sub[48];
    if (rgbd) {  // half-width ResNet50: bottlenecks [3, 4, 6, 3], outputs 4 x width
      const int nblocks[4] = {3, 4, r101 ? 23 : 6, 3};
      for (int li = 0; li < 4; ++li)
        for (int bi = 0; bi < nblocks[li]; ++bi) {
          const int64_t w = widths[li];
          const bool down = (bi == 0 && li > 0) || cin != 4 * w;
          snprintf(pre, sizeof(pre), "enc.layer%d.%d", li + 1, bi);
          // SE-ResNeXt (R9): inner width 2w, the 3x3 grouped (16 groups: weight [2w][2w/16][3][3])
          const int64_t wi = serx ? 2 * w : w, gi = serx ? wi / 16 : wi;
          const int64_t cis[3] = {cin, gi, wi}, cos_[3] = {wi, wi, 4 * w}, ks[3] = {1, 3, 1};
          for (int j = 0; j < 3; ++j) {
            snprintf(sub, sizeof(sub), "%s.conv%d", pre, j + 1);
            conv(sub, cos_[j], cis[j], ks[j]);
            snprintf(sub, sizeof(sub), "%s.gn%d", pre, j + 1);
            gn(sub, cos_[j]);
          }
          if (serx) {  // squeeze-excitation: fc1 [4w/16][4w], fc2 [4w][4w/16] with biases (default init)
            const int64_t co = 4 * w, r = co / 16;
            int64_t w1[2] = {r, co}, b1[1] = {r}, w2[2] = {co, r}, b2[1] = {co};
            snprintf(sub, sizeof(sub), "%s.se.fc1.weight", pre);
            add_tensor(&L, sub, 2, w1, (int)co);
            snprintf(sub, sizeof(sub), "%s.se.fc1.bias", pre);
            add_tensor(&L, sub, 1, b1, (int)co);
            snprintf(sub, sizeof(sub), "%s.se.fc2.weight", pre);
            add_tensor(&L, sub, 2, w2, (int)r);
            snprintf(sub, sizeof(sub), "%s.se.fc2.bias", pre);
            add_tensor(&L, sub, 1, b2, (int)r);
          }
          if (down) {
            snprintf(sub, sizeof(sub), "%s.down.conv", pre);
            conv(sub, 4 * w, cin, 1);
            snprintf(sub, sizeof(sub), "%s.down.gn", pre);
            gn(sub, 4 * w);
          }
          cin = 4 * w;
        }
    }
    for (int li = 0; li < 4 && !rgbd; ++li)
      for (int bi = 0; bi < 2; ++bi) {
        const int64_t c = widths[li];
        const bool down = (bi == 0 && li > 0) || cin != c;
        snprintf(pre, sizeof(pre), "enc.layer%d.%d", li + 1, bi);
        snprintf(sub, sizeof(sub), "%s.conv1", pre);
        conv(sub, c, cin, 3);
        snprintf(sub, sizeof(sub), "%s.gn1", pre);
        gn(sub, c);
        snprintf(sub, sizeof(sub), "%s.conv2", pre);
        conv(sub, c, c, 3);
        snprintf(sub, sizeof(sub), "%s.gn2", pre);
        gn(sub, c);
        if (down) {
          snprintf(sub, sizeof(sub), "%s.down.conv", pre);
          conv(sub, c, cin, 1);
          snprintf(sub, sizeof(sub), "%s.down.gn", pre);
          gn(sub, c);
        }
        cin = c;
      }
    conv("enc.compress.conv", 128, rgbd ? 1024 : 256, 3);
    gn("enc.compress.gn", 128);
    const int64_t fin = rgbd ? 2048 : 512;  // 128 x 4 x 4 / 128 x 2 x 2
    int64_t vw[2] = {512, fin}, vb[1] = {512}, a[2] = {32, 3}, b[1] = {32}, e[2] = {A1, 32}, wi[2] = {G, 576},
            wi1[2] = {G, H}, wh[2] = {G, H}, bg[1] = {G}, hw[2] = {A1, H}, hb[1] = {A1};
    add_tensor(&L, "visual_fc.weight", 2, vw, (int)fin);
    add_tensor(&L, "visual_fc.bias", 1, vb, (int)fin);
    add_tensor(&L, "goal_fc.weight", 2, a, 3);
    add_tensor(&L, "goal_fc.bias", 1, b, 3);
    add_tensor(&L, "act_embed.weight", 2, e, 1);
    if (!rgbd) {
      add_tensor(&L, "rnn.weight_ih", 2, wi, (int)H);
      add_tensor(&L, "rnn.weight_hh", 2, wh, (int)H);
      add_tensor(&L, "rnn.bias_ih", 1, bg, (int)H);
      add_tensor(&L, "rnn.bias_hh", 1, bg, (int)H);
    } else {
      for (int l = 0; l < 2; ++l) {
        snprintf(name, sizeof(name), "rnn.weight_ih_l%d", l);
        add_tensor(&L, name, 2, l == 0 ? wi : wi1, (int)H);
        snprintf(name, sizeof(name), "rnn.weight_hh_l%d", l);
        add_tensor(&L, name, 2, wh, (int)H);
        snprintf(name, sizeof(name), "rnn.bias_ih_l%d", l);
        add_tensor(&L, name, 1, bg, (int)H);
        snprintf(name, sizeof(name), "rnn.bias_hh_l%d", l);
        add_tensor(&L, name, 1, bg, (int)H);
      }
    }
    add_tensor(&L, "head.weight", 2, hw, (int)H);
    add_tensor(&L, "head.bias", 1, hb, (int)H);
  } else {
    return DDPPO_ERR_CONFIG;
  }
  *out = L;
  return DDPPO_OK;
}

int64_t layout_offset(const ModelLayout& L, const char* name) {
  for (int i = 0; i < L.n; ++i)
    if (strcmp(L.t[i].name, name) == 0) return L.t[i].offset;
  return -1;
}

int64_t encoder_end(const ModelLayout& L) {
  int64_t end = 0;
  for (int i = 0; i < L.n && strncmp(L.t[i].name, "enc.", 4) == 0; ++i) end = L.t[i].offset + L.t[i].numel;
  return (end + 3) / 4 * 4;
}

namespace {
constexpr int kH = 64, kA1 = 5;

// one thread per sample: h = tanh(W1 g + b1) (saved), out = W2 h + b2
__global__ void toy_fwd_kernel(const float* __restrict__ W1, const float* __restrict__ b1,
                               const float* __restrict__ W2, const float* __restrict__ b2,
                               const float* __restrict__ goal, const int32_t* __restrict__ env_idx, int T,
                               int T_run, int M, float* __restrict__ hsave, float* __restrict__ logits,
                               float* __restrict__ values) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < M; m += gridDim.x * blockDim.x) {
    const int b = m / T_run, t = m - b * T_run;
    const float* g = goal + ((size_t)env_idx[b] * T + t) * 3;
    const float g0 = g[0], g1 = g[1], g2 = g[2];
    float out[kA1];
    for (int o = 0; o < kA1; ++o) out[o] = b2[o];
    for (int j = 0; j < kH; ++j) {
      const float h = tanhf(W1[j * 3 + 0] * g0 + W1[j * 3 + 1] * g1 + W1[j * 3 + 2] * g2 + b1[j]);
      hsave[(size_t)m * kH + j] = h;
      for (int o = 0; o < kA1; ++o) out[o] += W2[o * kH + j] * h;
    }
    for (int o = 0; o < 4; ++o) logits[(size_t)m * 4 + o] = out[o];
    values[m] = out[4];
  }
}

// thread j (hidden unit) accumulates its own gradient rows over all samples in order
__global__ void toy_bwd_kernel(const float* __restrict__ W2, const float* __restrict__ goal,
                               const int32_t* __restrict__ env_idx, int T, int T_run, int M,
                               const float* __restrict__ hsave, const float* __restrict__ dlogits,
                               const float* __restrict__ dvalues, float* __restrict__ gW1, float* __restrict__ gb1,
                               float* __restrict__ gW2, float* __restrict__ gb2) {
  const int j = threadIdx.x;
  if (j < kH) {
    float w2[kA1];
    for (int o = 0; o < kA1; ++o) w2[o] = W2[o * kH + j];
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, ab = 0.f, d2[kA1] = {0.f, 0.f, 0.f, 0.f, 0.f};
    for (int m = 0; m < M; ++m) {
      const int b = m / T_run, t = m - b * T_run;
      const float* g = goal + ((size_t)env_idx[b] * T + t) * 3;
      const float h = hsave[(size_t)m * kH + j];
      float dout[kA1];
      for (int o = 0; o < 4; ++o) dout[o] = dlogits[(size_t)m * 4 + o];
      dout[4] = dvalues[m];
      float dh = 0.f;
      for (int o = 0; o < kA1; ++o) {
        dh += w2[o] * dout[o];
        d2[o] += dout[o] * h;
      }
      const float dpre = dh * (1.f - h * h);
      a0 += dpre * g[0];
      a1 += dpre * g[1];
      a2 += dpre * g[2];
      ab += dpre;
    }
    gW1[j * 3 + 0] = a0;
    gW1[j * 3 + 1] = a1;
    gW1[j * 3 + 2] = a2;
    gb1[j] = ab;
    for (int o = 0; o < kA1; ++o) gW2[o * kH + j] = d2[o];
  } else if (j < kH + kA1) {
    const int o = j - kH;
    float s = 0.f;
    for (int m = 0; m < M; ++m) s += o < 4 ? dlogits[(size_t)m * 4 + o] : dvalues[m];
    gb2[o] = s;
  }
}
}  // namespace

size_t toy_workspace(int max_B, int T) { return align_up((size_t)max_B * T * kH * sizeof(float), 256); }

ddppo_status toy_fwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     float* logits, float* values, void* ws, cudaStream_t st) {
  const int M = b.B * b.T_run;
  ProfScope ps(ctx, DDPPO_K_NET_FWD, st, 1);
  toy_fwd_kernel<<<grid_for(M, 128, ctx->sm_count * 4), 128, 0, st>>>(
      params + layout_offset(L, "fc1.weight"), params + layout_offset(L, "fc1.bias"),
      params + layout_offset(L, "head.weight"), params + layout_offset(L, "head.bias"), b.goal, b.env_idx, b.T,
      b.T_run, M, (float*)ws, logits, values);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status toy_bwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     const float* dlogits, const float* dvalues, float* grad, void* ws, cudaStream_t st) {
  const int M = b.B * b.T_run;
  ProfScope ps(ctx, DDPPO_K_NET_BWD, st, 1);
  toy_bwd_kernel<<<1, 96, 0, st>>>(params + layout_offset(L, "head.weight"), b.goal, b.env_idx, b.T, b.T_run, M,
                                   (const float*)ws, dlogits, dvalues, grad + layout_offset(L, "fc1.weight"),
                                   grad + layout_offset(L, "fc1.bias"), grad + layout_offset(L, "head.weight"),
                                   grad + layout_offset(L, "head.bias"));
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
