/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU restatement of the reference's memory-efficient dense-block path
 * (denseplan, /root/reference/proj/include/denseplan).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.
 *
 * This file is included twice by dp_oracle.c, once with R=float and once
 * with R=double; FN(x) suffixes every symbol with _f32 / _f64.
 *
 * Every function restates one reference routine with the SAME loop order,
 * the SAME summation order and the SAME expression association, so that for
 * identical inputs it is bit-identical to the reference compiled with the
 * same compiler flags (no FMA contraction).  Layout is the reference's NCHW:
 * element (i,c,y,x) of a tensor with per-sample stride S lives at
 * p[i*S + (c*h + y)*w + x]   (dp/tensor.hpp:102-108).
 */

/* ---- batch statistics: dp/ops.hpp:138-162 (two-pass, biased) ---------- */
void FN(batch_statistics)(const R* x, int64_t xs, int64_t n, int64_t c,
                          int64_t h, int64_t w, R* mean, R* var) {
  const R count = (R)(n * h * w);
  for (int64_t ch = 0; ch < c; ++ch) {
    R sum = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t y = 0; y < h; ++y)
        for (int64_t xx = 0; xx < w; ++xx) sum += x[i * xs + (ch * h + y) * w + xx];
    const R m = sum / count;
    R sq = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t y = 0; y < h; ++y)
        for (int64_t xx = 0; xx < w; ++xx) {
          const R d = x[i * xs + (ch * h + y) * w + xx] - m;
          sq += d * d;
        }
    mean[ch] = m;
    var[ch] = sq / count;
  }
}

/* ---- batchnorm_apply: dp/ops.hpp:115-134 ------------------------------ */
/* y = gamma * (x - mean) * inv + beta, inv = 1/sqrt(var + eps), evaluated
 * left to right exactly as the reference's expression. */
void FN(batchnorm_apply)(const R* x, int64_t xs, int64_t n, int64_t c, int64_t h,
                         int64_t w, const R* gamma, const R* beta,
                         const R* mean, const R* var, R eps, R* dst,
                         int64_t ds) {
  for (int64_t ch = 0; ch < c; ++ch) {
    const R g = gamma[ch];
    const R b = beta[ch];
    const R inv = (R)1 / SQRT(var[ch] + eps);
    const R mu = mean[ch];
    for (int64_t i = 0; i < n; ++i)
      for (int64_t y = 0; y < h; ++y)
        for (int64_t xx = 0; xx < w; ++xx) {
          const int64_t o = (ch * h + y) * w + xx;
          dst[i * ds + o] = g * (x[i * xs + o] - mu) * inv + b;
        }
  }
}

/* ---- running-statistics update: dp/ops.hpp:185-194 --------------------- */
/* rm = (1-m)*rm + m*mean ; rv = (1-m)*rv + m*var_biased (F5). */
void FN(running_update)(int64_t c, const R* mean, const R* var, R momentum,
                        R* rm, R* rv) {
  for (int64_t ch = 0; ch < c; ++ch) {
    rm[ch] = ((R)1 - momentum) * rm[ch] + momentum * mean[ch];
    rv[ch] = ((R)1 - momentum) * rv[ch] + momentum * var[ch];
  }
}

/* ---- batchnorm_backward: dp/ops.hpp:206-243 ---------------------------- */
void FN(batchnorm_backward)(const R* gy, int64_t gys, const R* x, int64_t xs,
                            int64_t n, int64_t c, int64_t h, int64_t w,
                            const R* gamma, const R* mean, const R* var, R eps,
                            R* gx, int64_t gxs, R* dgamma, R* dbeta) {
  const R count = (R)(n * h * w);
  for (int64_t ch = 0; ch < c; ++ch) {
    const R g = gamma[ch];
    const R mu = mean[ch];
    const R inv = (R)1 / SQRT(var[ch] + eps);
    R sum_g = 0;
    R sum_gx = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t y = 0; y < h; ++y)
        for (int64_t xx = 0; xx < w; ++xx) {
          const int64_t o = (ch * h + y) * w + xx;
          const R gv = gy[i * gys + o];
          const R xh = (x[i * xs + o] - mu) * inv;
          sum_g += gv;
          sum_gx += gv * xh;
        }
    dgamma[ch] = sum_gx;
    dbeta[ch] = sum_g;
    const R mg = sum_g / count;
    const R mgx = sum_gx / count;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t y = 0; y < h; ++y)
        for (int64_t xx = 0; xx < w; ++xx) {
          const int64_t o = (ch * h + y) * w + xx;
          const R gv = gy[i * gys + o];
          const R xh = (x[i * xs + o] - mu) * inv;
          gx[i * gxs + o] = g * inv * (gv - mg - xh * mgx);
        }
  }
}

/* ---- relu: dp/ops.hpp:248-287 ------------------------------------------ */
void FN(relu_inplace)(R* t, int64_t ts, int64_t n, int64_t per_sample) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < per_sample; ++j) {
      const R v = t[i * ts + j];
      t[i * ts + j] = v > (R)0 ? v : (R)0;
    }
}

/* grad = ref > 0 ? grad : 0 (subgradient at 0 is 0), dp/ops.hpp:268-287 */
void FN(relu_backward_inplace)(R* g, int64_t gs, const R* ref, int64_t rs,
                               int64_t n, int64_t per_sample) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < per_sample; ++j)
      g[i * gs + j] = ref[i * rs + j] > (R)0 ? g[i * gs + j] : (R)0;
}

/* ---- conv2d_forward: dp/ops.hpp:315-342 (cross-correlation) ------------ */
/* weights (oc, ic, kh, kw) contiguous; output spatial = (in+2p-k)/s+1. */
void FN(conv2d_forward)(const R* x, int64_t xs, int64_t n, int64_t cin,
                        int64_t h, int64_t w, const R* wt, int64_t cout,
                        int64_t kh, int64_t kw, int64_t stride, int64_t pad,
                        R* dst, int64_t ds) {
  const int64_t oh = (h + 2 * pad - kh) / stride + 1;
  const int64_t ow = (w + 2 * pad - kw) / stride + 1;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t oc = 0; oc < cout; ++oc)
      for (int64_t oy = 0; oy < oh; ++oy)
        for (int64_t ox = 0; ox < ow; ++ox) {
          R acc = 0;
          for (int64_t ic = 0; ic < cin; ++ic)
            for (int64_t ky = 0; ky < kh; ++ky) {
              const int64_t iy = oy * stride - pad + ky;
              if (iy < 0 || iy >= h) continue;
              for (int64_t kx = 0; kx < kw; ++kx) {
                const int64_t ix = ox * stride - pad + kx;
                if (ix < 0 || ix >= w) continue;
                acc += x[i * xs + (ic * h + iy) * w + ix] *
                       wt[((oc * cin + ic) * kh + ky) * kw + kx];
              }
            }
          dst[i * ds + (oc * oh + oy) * ow + ox] = acc;
        }
}

/* ---- conv2d_backward: dp/ops.hpp:346-387 ------------------------------- */
/* grad_w and grad_x are zero-filled then scattered in loop order
 * i, oc, oy, ox, ic, ky, kx.  gx may be NULL (stem). */
void FN(conv2d_backward)(const R* gy, int64_t gys, const R* x, int64_t xs,
                         int64_t n, int64_t cin, int64_t h, int64_t w,
                         const R* wt, int64_t cout, int64_t kh, int64_t kw,
                         int64_t stride, int64_t pad, R* gx, int64_t gxs,
                         R* gw) {
  const int64_t oh = (h + 2 * pad - kh) / stride + 1;
  const int64_t ow = (w + 2 * pad - kw) / stride + 1;
  for (int64_t j = 0; j < cout * cin * kh * kw; ++j) gw[j] = 0;
  if (gx)
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < cin * h * w; ++j) gx[i * gxs + j] = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t oc = 0; oc < cout; ++oc)
      for (int64_t oy = 0; oy < oh; ++oy)
        for (int64_t ox = 0; ox < ow; ++ox) {
          const R g = gy[i * gys + (oc * oh + oy) * ow + ox];
          for (int64_t ic = 0; ic < cin; ++ic)
            for (int64_t ky = 0; ky < kh; ++ky) {
              const int64_t iy = oy * stride - pad + ky;
              if (iy < 0 || iy >= h) continue;
              for (int64_t kx = 0; kx < kw; ++kx) {
                const int64_t ix = ox * stride - pad + kx;
                if (ix < 0 || ix >= w) continue;
                const int64_t wi = ((oc * cin + ic) * kh + ky) * kw + kx;
                gw[wi] += g * x[i * xs + (ic * h + iy) * w + ix];
                if (gx) gx[i * gxs + (ic * h + iy) * w + ix] += g * wt[wi];
              }
            }
        }
}

/* ---- dense block forward (pre-activation, bottleneck) -------------------
 * Restates GraphPlan::forward_layer, dp/graph.hpp:618-670 + 722, for every
 * layer of one block (dp/graph.hpp:750-755), SharedAll strategy.
 *
 *   feats : (n, c_out, h, w) with c_out = c0 + m*k.  On entry channels
 *           [0, c0) hold the block input; on return channels c0+l*k..+k hold
 *           layer l's output y_l (the block-output concat of graph.hpp:756).
 *   z     : m * (n, bk, h, w)      retained bottleneck outputs conv_a_out.
 *   params: flat per-layer layout (see dp_oracle.c header).
 *   stats : flat per-layer [mean_a(c_l) var_a(c_l) mean_b(bk) var_b(bk)].
 *   running: same layout as stats; updated in place when update_running.
 * Returns 0, or 9 (DegenerateBatchError) when n*h*w < 2 (ops.hpp:180-183).
 */
int FN(block_forward)(int64_t n, int64_t h, int64_t w, int64_t c0, int64_t m,
                      int64_t k, int64_t bk, const R* params, R* feats, R* z,
                      R* stats, R* running, int update_running) {
  const R eps = (R)1e-5;
  const R momentum = (R)0.1;
  if (n * h * w < 2) return 9;
  const int64_t hw = h * w;
  const int64_t c_out = c0 + m * k;
  const int64_t fs = c_out * hw; /* feats per-sample stride */
  R* act_a = (R*)malloc(sizeof(R) * (size_t)(n * (c_out + bk) * hw));
  R* act_b = act_a; /* act_b lives after act_a in Shared2 (graph.hpp:646) */
  int64_t po = 0, so = 0;
  for (int64_t l = 0; l < m; ++l) {
    const int64_t c = c0 + l * k;
    const R* ga = params + po;
    const R* ba = ga + c;
    const R* w1 = ba + c;
    const R* gb = w1 + bk * c;
    const R* bb = gb + bk;
    const R* w2 = bb + bk;
    po += 2 * c + bk * c + 2 * bk + 9 * k * bk;
    R* mean_a = stats + so;
    R* var_a = mean_a + c;
    R* mean_b = var_a + c;
    R* var_b = mean_b + bk;
    R* rm_a = running + so;
    R* rv_a = rm_a + c;
    R* rm_b = rv_a + c;
    R* rv_b = rm_b + bk;
    so += 2 * c + 2 * bk;
    /* cat = channel prefix [0, c) of feats (zero-copy view of the concat). */
    FN(batch_statistics)(feats, fs, n, c, h, w, mean_a, var_a);
    if (update_running) FN(running_update)(c, mean_a, var_a, momentum, rm_a, rv_a);
    FN(batchnorm_apply)(feats, fs, n, c, h, w, ga, ba, mean_a, var_a, eps, act_a,
                        c * hw);
    FN(relu_inplace)(act_a, c * hw, n, c * hw);
    R* zl = z + l * n * bk * hw;
    FN(conv2d_forward)(act_a, c * hw, n, c, h, w, w1, bk, 1, 1, 1, 0, zl, bk * hw);
    act_b = act_a + n * c * hw;
    FN(batch_statistics)(zl, bk * hw, n, bk, h, w, mean_b, var_b);
    if (update_running) FN(running_update)(bk, mean_b, var_b, momentum, rm_b, rv_b);
    FN(batchnorm_apply)(zl, bk * hw, n, bk, h, w, gb, bb, mean_b, var_b, eps,
                        act_b, bk * hw);
    FN(relu_inplace)(act_b, bk * hw, n, bk * hw);
    FN(conv2d_forward)(act_b, bk * hw, n, bk, h, w, w2, k, 3, 3, 1, 1,
                       feats + c * hw, fs);
  }
  free(act_a);
  return 0;
}

/* ---- dense block backward -------------------------------------------------
 * Restates GraphPlan::backward_block + backward_layer pre-act bottleneck
 * branch (dp/graph.hpp:1054-1063, 856-945) including the rematerialization
 * of concat/BN_a/ReLU and BN_b/ReLU from the SAVED statistics
 * (graph.hpp:831-854, 884-901).
 *
 *   acc   : (n, c_out, h, w) block-gradient accumulator, pre-filled by the
 *           consumer (head/transition BN backward).  On return its prefix
 *           [0, c0) is the gradient w.r.t. the block input and every slice
 *           holds the full gradient of that feature.
 *   grads : flat per-layer layout identical to params (dgamma_a, dbeta_a,
 *           dW1, dgamma_b, dbeta_b, dW2) — written, not accumulated.
 */
int FN(block_backward)(int64_t n, int64_t h, int64_t w, int64_t c0, int64_t m,
                       int64_t k, int64_t bk, const R* params, const R* feats,
                       const R* z, const R* stats, R* acc, R* grads) {
  const R eps = (R)1e-5;
  const int64_t hw = h * w;
  const int64_t c_out = c0 + m * k;
  const int64_t fs = c_out * hw;
  const int64_t cmax = c0 + (m - 1) * k;
  /* Shared2 (act_a then act_b) and the two transient gradient slots. */
  R* act_a = (R*)malloc(sizeof(R) * (size_t)(n * (cmax + bk) * hw));
  R* slot0 = (R*)malloc(sizeof(R) * (size_t)(n * (cmax > bk ? cmax : bk) * hw));
  R* slot1 = (R*)malloc(sizeof(R) * (size_t)(n * (cmax > bk ? cmax : bk) * hw));
  int64_t* poffs = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  int64_t* soffs = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  int64_t po = 0, so = 0;
  for (int64_t l = 0; l < m; ++l) {
    const int64_t c = c0 + l * k;
    poffs[l] = po;
    soffs[l] = so;
    po += 2 * c + bk * c + 2 * bk + 9 * k * bk;
    so += 2 * c + 2 * bk;
  }
  for (int64_t l = m - 1; l >= 0; --l) {
    const int64_t c = c0 + l * k;
    const R* ga = params + poffs[l];
    const R* ba = ga + c;
    const R* w1 = ba + c;
    const R* gb = w1 + bk * c;
    const R* bb = gb + bk;
    const R* w2 = bb + bk;
    R* dga = grads + poffs[l];
    R* dba = dga + c;
    R* dw1 = dba + c;
    R* dgb = dw1 + bk * c;
    R* dbb = dgb + bk;
    R* dw2 = dbb + bk;
    const R* mean_a = stats + soffs[l];
    const R* var_a = mean_a + c;
    const R* mean_b = var_a + c;
    const R* var_b = mean_b + bk;
    const R* zl = z + l * n * bk * hw;
    /* grad_out = acc.channel_view(c_in + l*k, k)  (graph.hpp:869-870) */
    const R* grad_out = acc + c * hw;
    /* rematerialize: cat = feats prefix; act_a = relu(bn_a(cat)) */
    FN(batchnorm_apply)(feats, fs, n, c, h, w, ga, ba, mean_a, var_a, eps, act_a,
                        c * hw);
    FN(relu_inplace)(act_a, c * hw, n, c * hw);
    R* act_b = act_a + n * c * hw;
    FN(batchnorm_apply)(zl, bk * hw, n, bk, h, w, gb, bb, mean_b, var_b, eps,
                        act_b, bk * hw);
    FN(relu_inplace)(act_b, bk * hw, n, bk * hw);
    /* t0 = dX of conv_b; dW2  (graph.hpp:905-907) */
    R* t0 = slot0;
    FN(conv2d_backward)(grad_out, fs, act_b, bk * hw, n, bk, h, w, w2, k, 3, 3, 1,
                        1, t0, bk * hw, dw2);
    FN(relu_backward_inplace)(t0, bk * hw, act_b, bk * hw, n, bk * hw);
    /* t1 = BN_b backward (graph.hpp:913-916) */
    R* t1 = slot1;
    FN(batchnorm_backward)(t0, bk * hw, zl, bk * hw, n, bk, h, w, gb, mean_b,
                           var_b, eps, t1, bk * hw, dgb, dbb);
    /* t2 = dX of conv_a; dW1 (graph.hpp:920-922) */
    R* t2 = slot0;
    FN(conv2d_backward)(t1, bk * hw, act_a, c * hw, n, c, h, w, w1, bk, 1, 1, 1, 0,
                        t2, c * hw, dw1);
    FN(relu_backward_inplace)(t2, c * hw, act_a, c * hw, n, c * hw);
    /* t3 = BN_a backward against the recomputed cat (graph.hpp:929-932) */
    R* t3 = slot1;
    FN(batchnorm_backward)(t2, c * hw, feats, fs, n, c, h, w, ga, mean_a, var_a,
                           eps, t3, c * hw, dga, dba);
    /* acc[:, :c] += t3 (graph.hpp:936-941) */
    for (int64_t ch = 0; ch < c; ++ch)
      for (int64_t i = 0; i < n; ++i)
        for (int64_t y = 0; y < h; ++y)
          for (int64_t xx = 0; xx < w; ++xx) {
            const int64_t o = (ch * h + y) * w + xx;
            acc[i * fs + o] += t3[i * c * hw + o];
          }
  }
  free(act_a);
  free(slot0);
  free(slot1);
  free(poffs);
  free(soffs);
  return 0;
}
