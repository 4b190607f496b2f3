/*
 * prnet_oracle.c -- plain, slow, single-threaded CPU oracle of the PRNet
 * pattern-attention forward.  TEST INFRASTRUCTURE ONLY (see prnet_oracle.h):
 * nothing on the product path includes, links or calls this file.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (abstract P:18-23,
 * conclusion P:44-47); "Def k" = SURVEY.md §8(c) "Definition" step k; "Ax" =
 * SURVEY.md §8(c) ambiguity register entry x (restated in DESIGN.md §3).
 *
 * Every function below follows its definition step literally: plain loops in
 * the order the definition writes them, fp64 arithmetic, no blocking, no
 * fusion, no reordering, no reuse of one step's loop for another.
 */
#include "prnet_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Def 6: epsilon inside the seasonal (Pearson) normaliser.  A4. */
static const double ORACLE_EPS_S = 1e-12;
/* Def 7: epsilon added to the series variance in the trend normaliser.  A5. */
static const double ORACLE_EPS_T = 1e-5;

/* Def 1: N = floor(L/S) (N >= 1 needs L >= S), r = L - N*S, M = ceil(H/S).
 * A1 (S is an input), A2 (drop the oldest r points), A3 (M = ceil). */
int oracle_dims(int32_t L, int32_t S, int32_t H, int32_t* N, int32_t* r, int32_t* M) {
  if (S < 2 || L < S || H < 1) return -1;
  *N = L / S;
  *r = L - (*N) * S;
  *M = (H + S - 1) / S;
  return 0;
}

/* Def 2: segment n holds x[r + n*S + t], t = 0..S-1; n = 0 is the oldest
 * segment (A2, A16).  P:21 "similarity between segments". */
static void oracle_segment(const float* x, int N, int S, int r, double* X) {
  for (int n = 0; n < N; n++)
    for (int t = 0; t < S; t++)
      X[n * S + t] = (double)x[r + n * S + t];
}

/* Def 3-4: mu_n = (1/S) sum_t X_n[t];  z_n = X_n - mu_n;  nu2_n = sum_t z_n[t]^2;
 * kappa_n = sum_t ttilde_t z_n[t] / V with ttilde_t = t - (S-1)/2 and
 * V = sum_t ttilde_t^2 = S(S^2-1)/12.  (A4 seasonal descriptors, A5 trend
 * descriptors; kappa_n is the least-squares slope of segment n.) */
static void oracle_descriptors(const double* X, int N, int S, double* mu, double* z,
                               double* nu2, double* kappa) {
  double V = 0.0;
  for (int t = 0; t < S; t++) {
    double tt = (double)t - 0.5 * (double)(S - 1);
    V += tt * tt;
  }
  for (int n = 0; n < N; n++) {
    double s = 0.0;
    for (int t = 0; t < S; t++) s += X[n * S + t];
    mu[n] = s / (double)S;
    for (int t = 0; t < S; t++) z[n * S + t] = X[n * S + t] - mu[n];
    double q = 0.0;
    for (int t = 0; t < S; t++) q += z[n * S + t] * z[n * S + t];
    nu2[n] = q;
    double k = 0.0;
    for (int t = 0; t < S; t++) {
      double tt = (double)t - 0.5 * (double)(S - 1);
      k += tt * z[n * S + t];
    }
    kappa[n] = k / V;
  }
}

/* SURVEY §8(f) f3, A4 variant "linear detrending before the correlation"
 * (metric_variant bit 1): the seasonal metric sees the residual of each segment
 * about its least-squares line, e_n[t] = z_n[t] - kappa_n ttilde_t, and its
 * squared norm; Def 6 is then applied to (e, |e|^2) in place of (z, nu2). */
static void oracle_detrend(const double* z, const double* kappa, int N, int S, double* e,
                           double* e2) {
  for (int n = 0; n < N; n++) {
    double q = 0.0;
    for (int t = 0; t < S; t++) {
      double tt = (double)t - 0.5 * (double)(S - 1);
      e[n * S + t] = z[n * S + t] - kappa[n] * tt;
      q += e[n * S + t] * e[n * S + t];
    }
    e2[n] = q;
  }
}

/* SURVEY §8(f) f1 (RevIN-style instance normalisation, reading R-f1 in DESIGN.md
 * §3): statistics of the N*S segmented points the method consumes,
 *   mu_r = (1/(N S)) sum X,  var_r = (1/(N S)) sum (X - mu_r)^2,
 * Xhat = (X - mu_r) / sqrt(var_r + eps_r); the forecast is de-normalised as
 * y = yhat sqrt(var_r + eps_r) + mu_r. */
static void oracle_instance_stats(const double* X, int N, int S, double* mu_r, double* var_r) {
  double s = 0.0;
  for (int k = 0; k < N * S; k++) s += X[k];
  *mu_r = s / ((double)N * (double)S);
  double q = 0.0;
  for (int k = 0; k < N * S; k++) q += (X[k] - *mu_r) * (X[k] - *mu_r);
  *var_r = q / ((double)N * (double)S);
}

/* Def 5: sigma^2 = (1/(N S)) sum_n [nu2_n + S (mu_n - mubar)^2], mubar = mean_n mu_n:
 * the population variance of the N*S segmented points (A5 normaliser). */
static double oracle_series_variance(const double* mu, const double* nu2, int N, int S) {
  double mbar = 0.0;
  for (int n = 0; n < N; n++) mbar += mu[n];
  mbar /= (double)N;
  double acc = 0.0;
  for (int n = 0; n < N; n++) acc += nu2[n] + (double)S * (mu[n] - mbar) * (mu[n] - mbar);
  return acc / ((double)N * (double)S);
}

/* Def 6 (seasonal metric, "two metrics ... seasonal"; A4):
 * rho_ij = <z_i, z_j> / sqrt((nu2_i + eps_s)(nu2_j + eps_s)). */
static void oracle_seasonal_similarity(const double* z, const double* nu2, int N, int S,
                                       double* rho) {
  for (int i = 0; i < N; i++)
    for (int j = 0; j < N; j++) {
      double g = 0.0;
      for (int t = 0; t < S; t++) g += z[i * S + t] * z[j * S + t];
      rho[i * N + j] = g / sqrt((nu2[i] + ORACLE_EPS_S) * (nu2[j] + ORACLE_EPS_S));
    }
}

/* Def 7 (trend metric, "... or trend"; A5):
 * D_ij = (mu_i - mu_j)^2 + ((S^2-1)/12) (kappa_i - kappa_j)^2,
 * which equals (1/S) ||T_i - T_j||^2 for the least-squares lines
 * T_n[t] = mu_n + kappa_n ttilde_t. */
static void oracle_trend_distance(const double* mu, const double* kappa, int N, int S,
                                  int level_only, double* D) {
  /* level_only (metric_variant bit 0, SURVEY §8(f) f3 / A5 variant "level only"):
   * D_ij = (mu_i - mu_j)^2 */
  double c = level_only ? 0.0 : ((double)S * (double)S - 1.0) / 12.0;
  for (int i = 0; i < N; i++)
    for (int j = 0; j < N; j++) {
      double dm = mu[i] - mu[j];
      double dk = kappa[i] - kappa[j];
      D[i * N + j] = dm * dm + c * dk * dk;
    }
}

/* Def 8 (pattern attention weights, "pattern attention mechanism"; A6, A9):
 * A[i][j] = exp(l_ij - max_k l_ik) / sum_k exp(l_ik - max_k l_ik), dense over all
 * j including j = i, where l_ij = sign * m_ij / tau. */
static void oracle_softmax_rows(const double* m, int N, double sign, double scale_inv,
                                double* A) {
  for (int i = 0; i < N; i++) {
    double mx = -INFINITY;
    for (int j = 0; j < N; j++) {
      double l = sign * m[i * N + j] * scale_inv;
      if (l > mx) mx = l;
    }
    double s = 0.0;
    for (int j = 0; j < N; j++) s += exp(sign * m[i * N + j] * scale_inv - mx);
    for (int j = 0; j < N; j++) A[i * N + j] = exp(sign * m[i * N + j] * scale_inv - mx) / s;
  }
}

/* Def 9 (aggregation into patterns, "aggregates similar segments to
 * extract patterns"; A10): P = A X, (N x N)(N x S). */
static void oracle_aggregate(const double* A, const double* X, int N, int S, double* P) {
  for (int i = 0; i < N; i++)
    for (int t = 0; t < S; t++) {
      double s = 0.0;
      for (int j = 0; j < N; j++) s += A[i * N + j] * X[j * S + t];
      P[i * S + t] = s;
    }
}

/* SURVEY §8(f) f3 / A10 variant "each branch aggregates its component (T_n or z_n)"
 * (metric_variant bit 2, reading R-f4 in DESIGN.md §3): the values each branch
 * aggregates are the component its metric measures,
 *   seasonal  Vs_n[t] = z_n[t]                      (plain, bit 1 = 0)
 *             Vs_n[t] = z_n[t] - kappa_n ttilde_t   (detrended metric, bit 1 = 1)
 *   trend     Vt_n[t] = mu_n + kappa_n ttilde_t     (the least-squares line T_n, bit 0 = 0)
 *             Vt_n[t] = mu_n                        (level-only trend metric, bit 0 = 1)
 * and Def 9 becomes P_s = A_s Vs, P_t = A_t Vt. */
static void oracle_components(const double* z, const double* mu, const double* kappa, int N,
                              int S, int level_only, int detrended, double* Vs, double* Vt) {
  for (int n = 0; n < N; n++)
    for (int t = 0; t < S; t++) {
      double tt = (double)t - 0.5 * (double)(S - 1);
      Vs[n * S + t] = detrended ? z[n * S + t] - kappa[n] * tt : z[n * S + t];
      Vt[n * S + t] = level_only ? mu[n] : mu[n] + kappa[n] * tt;
    }
}

/* Def 10-11 (linear head, NS "the per-channel linear head maps to the
 * forecast horizon"; A7, A8, A11, A3):
 * Y[m][t] = sum_n ws[m][n] P_s[n][t] + wt[m][n] P_t[n][t];
 * y[h] = Y[h div S][h mod S] + b[h], h = 0..H-1. */
static void oracle_head(const double* Ps, const double* Pt, const float* ws, const float* wt,
                        const float* bias, int N, int S, int M, int H, double* Yfull,
                        double* y) {
  for (int m = 0; m < M; m++)
    for (int t = 0; t < S; t++) {
      double s = 0.0;
      for (int n = 0; n < N; n++)
        s += (double)ws[m * N + n] * Ps[n * S + t] + (double)wt[m * N + n] * Pt[n * S + t];
      Yfull[m * S + t] = s;
    }
  for (int h = 0; h < H; h++) y[h] = Yfull[(h / S) * S + (h % S)] + (double)bias[h];
}

/* SURVEY §8(f) f3 "moving-average seasonal/trend decomposition feeding each branch"
 * (reading R-f5 in DESIGN.md §3; the series decomposition of the decomposition-based LTSF
 * models): over the N*S segmented points p_0..p_{NS-1} (after RevIN when on), with an
 * odd kernel k = 2h + 1 and the ends padded by repeating the first / last point,
 *   trend_i = (1/k) sum_{d=-h..h} p_{clamp(i+d, 0, NS-1)},   seasonal_i = p_i - trend_i. */
static void oracle_decompose(const double* X, int NS, int k, double* Xs, double* Xt) {
  int h = (k - 1) / 2;
  for (int i = 0; i < NS; i++) {
    double s = 0.0;
    for (int d = -h; d <= h; d++) {
      int j = i + d;
      if (j < 0) j = 0;
      if (j > NS - 1) j = NS - 1;
      s += X[j];
    }
    Xt[i] = s / (double)k;
    Xs[i] = X[i] - Xt[i];
  }
}

int oracle_series(const float* x, int32_t L, int32_t S, int32_t H, const float* ws,
                  const float* wt, const float* bias, double tau_s, double tau_t, double* y,
                  const oracle_debug* dbg) {
  return oracle_series_ex(x, L, S, H, ws, wt, bias, tau_s, tau_t, 0, 0, 0.0, 0, y, dbg);
}

int oracle_series_ex(const float* x, int32_t L, int32_t S, int32_t H, const float* ws,
                     const float* wt, const float* bias, double tau_s, double tau_t,
                     int32_t metric_variant, int32_t instance_norm, double eps_r,
                     int32_t ma_kernel, double* y, const oracle_debug* dbg) {
  int32_t N, r, M;
  if (oracle_dims(L, S, H, &N, &r, &M) != 0) return -1;
  if (!(tau_s > 0.0) || !(tau_t > 0.0)) return -1;
  if (metric_variant < 0 || metric_variant > 7 || !(eps_r >= 0.0)) return -1;
  if (ma_kernel < 0 || (ma_kernel > 0 && ma_kernel % 2 == 0)) return -1;
  size_t nS = (size_t)N * S, nN = (size_t)N * N, mS = (size_t)M * S;
  double* X = (double*)malloc(nS * sizeof(double));
  double* Xs = (double*)malloc(nS * sizeof(double));   /* seasonal branch input */
  double* Xt = (double*)malloc(nS * sizeof(double));   /* trend branch input    */
  double* zs = (double*)malloc(nS * sizeof(double));
  double* zt = (double*)malloc(nS * sizeof(double));
  double* mus = (double*)malloc(N * sizeof(double));
  double* nu2s = (double*)malloc(N * sizeof(double));
  double* kaps = (double*)malloc(N * sizeof(double));
  double* mut = (double*)malloc(N * sizeof(double));
  double* nu2t = (double*)malloc(N * sizeof(double));
  double* kapt = (double*)malloc(N * sizeof(double));
  double* rho = (double*)malloc(nN * sizeof(double));
  double* D = (double*)malloc(nN * sizeof(double));
  double* Dh = (double*)malloc(nN * sizeof(double));
  double* As = (double*)malloc(nN * sizeof(double));
  double* At = (double*)malloc(nN * sizeof(double));
  double* Ps = (double*)malloc(nS * sizeof(double));
  double* Pt = (double*)malloc(nS * sizeof(double));
  double* Yf = (double*)malloc(mS * sizeof(double));

  oracle_segment(x, N, S, r, X);                                   /* Def 2   */
  double mu_r = 0.0, s_r = 1.0;
  if (instance_norm) {                                             /* f1      */
    double var_r;
    oracle_instance_stats(X, N, S, &mu_r, &var_r);
    s_r = sqrt(var_r + eps_r);
    for (size_t k = 0; k < nS; k++) X[k] = (X[k] - mu_r) / s_r;
  }
  if (ma_kernel > 0) {                                             /* f3, R-f5 */
    oracle_decompose(X, (int)nS, ma_kernel, Xs, Xt);
  } else {                                    /* both branches see the segments */
    memcpy(Xs, X, nS * sizeof(double));
    memcpy(Xt, X, nS * sizeof(double));
  }
  oracle_descriptors(Xs, N, S, mus, zs, nu2s, kaps);               /* Def 3-4, seasonal */
  oracle_descriptors(Xt, N, S, mut, zt, nu2t, kapt);               /* Def 3-4, trend    */
  double sigma2 = oracle_series_variance(mut, nu2t, N, S);         /* Def 5   */
  if (metric_variant & 2) {                                        /* f3      */
    double* e = (double*)malloc(nS * sizeof(double));
    double* e2 = (double*)malloc(N * sizeof(double));
    oracle_detrend(zs, kaps, N, S, e, e2);
    oracle_seasonal_similarity(e, e2, N, S, rho);                  /* Def 6 on e */
    free(e);
    free(e2);
  } else {
    oracle_seasonal_similarity(zs, nu2s, N, S, rho);               /* Def 6   */
  }
  oracle_trend_distance(mut, kapt, N, S, metric_variant & 1, D);   /* Def 7   */
  for (size_t k = 0; k < nN; k++) Dh[k] = D[k] / (sigma2 + ORACLE_EPS_T);
  oracle_softmax_rows(rho, N, +1.0, 1.0 / tau_s, As);              /* Def 8   */
  oracle_softmax_rows(Dh, N, -1.0, 1.0 / tau_t, At);               /* Def 8   */
  if (metric_variant & 4) {                                        /* f3, A10 */
    double* Vs = (double*)malloc(nS * sizeof(double));
    double* Vt = (double*)malloc(nS * sizeof(double));
    double* dummy = (double*)malloc(nS * sizeof(double));
    /* seasonal component of the seasonal input, trend component of the trend input */
    oracle_components(zs, mus, kaps, N, S, metric_variant & 1, metric_variant & 2, Vs, dummy);
    oracle_components(zt, mut, kapt, N, S, metric_variant & 1, metric_variant & 2, dummy, Vt);
    oracle_aggregate(As, Vs, N, S, Ps);                            /* Def 9 on Vs */
    oracle_aggregate(At, Vt, N, S, Pt);                            /* Def 9 on Vt */
    free(Vs);
    free(Vt);
    free(dummy);
  } else {
    oracle_aggregate(As, Xs, N, S, Ps);                            /* Def 9   */
    oracle_aggregate(At, Xt, N, S, Pt);                            /* Def 9   */
  }
  oracle_head(Ps, Pt, ws, wt, bias, N, S, M, H, Yf, y);            /* Def 10-11 */
  if (instance_norm)                                               /* f1      */
    for (int32_t h = 0; h < H; h++) y[h] = y[h] * s_r + mu_r;

  if (dbg) {
    if (dbg->seg) memcpy(dbg->seg, X, nS * sizeof(double));
    if (dbg->mu) memcpy(dbg->mu, mut, N * sizeof(double));
    if (dbg->nu2) memcpy(dbg->nu2, nu2s, N * sizeof(double));
    if (dbg->kappa) memcpy(dbg->kappa, kapt, N * sizeof(double));
    if (dbg->sigma2) dbg->sigma2[0] = sigma2;
    if (dbg->rho) memcpy(dbg->rho, rho, nN * sizeof(double));
    if (dbg->dist) memcpy(dbg->dist, D, nN * sizeof(double));
    if (dbg->a_s) memcpy(dbg->a_s, As, nN * sizeof(double));
    if (dbg->a_t) memcpy(dbg->a_t, At, nN * sizeof(double));
    if (dbg->p_s) memcpy(dbg->p_s, Ps, nS * sizeof(double));
    if (dbg->p_t) memcpy(dbg->p_t, Pt, nS * sizeof(double));
    if (dbg->y_full) memcpy(dbg->y_full, Yf, mS * sizeof(double));
  }
  free(X); free(Xs); free(Xt); free(zs); free(zt); free(mus); free(nu2s); free(kaps);
  free(mut); free(nu2t); free(kapt); free(rho); free(D); free(Dh);
  free(As); free(At); free(Ps); free(Pt); free(Yf);
  return 0;
}

int oracle_forward(const float* x, int64_t B, int32_t C, int32_t L, int32_t S, int32_t H,
                   const float* ws, const float* wt, const float* bias,
                   int32_t head_per_channel, double tau_s, double tau_t, float* y,
                   double* y64) {
  return oracle_forward_ex(x, B, C, L, S, H, ws, wt, bias, head_per_channel, tau_s, tau_t, 0, 0,
                           0.0, 0, y, y64);
}

int oracle_forward_ex(const float* x, int64_t B, int32_t C, int32_t L, int32_t S, int32_t H,
                      const float* ws, const float* wt, const float* bias,
                      int32_t head_per_channel, double tau_s, double tau_t,
                      int32_t metric_variant, int32_t instance_norm, double eps_r,
                      int32_t ma_kernel, float* y, double* y64) {
  int32_t N, r, M;
  if (B < 0 || C < 1 || oracle_dims(L, S, H, &N, &r, &M) != 0) return -1;
  double* yy = (double*)malloc((size_t)H * sizeof(double));
  for (int64_t b = 0; b < B; b++)
    for (int32_t c = 0; c < C; c++) {
      int64_t cw = head_per_channel ? c : 0;
      const float* xs = x + (b * C + c) * (int64_t)L;
      if (oracle_series_ex(xs, L, S, H, ws + cw * M * N, wt + cw * M * N, bias + cw * H,
                           tau_s, tau_t, metric_variant, instance_norm, eps_r, ma_kernel, yy,
                           NULL) != 0) {
        free(yy);
        return -1;
      }
      for (int32_t h = 0; h < H; h++) {
        int64_t o = (b * C + c) * (int64_t)H + h;
        if (y) y[o] = (float)yy[h];
        if (y64) y64[o] = yy[h];
      }
    }
  free(yy);
  return 0;
}

void oracle_error_sums(const float* y, const float* target, int64_t n, double* out3) {
  double sse = 0.0, sae = 0.0;
  for (int64_t i = 0; i < n; i++) {
    double d = (double)y[i] - (double)target[i];
    sse += d * d;
    sae += fabs(d);
  }
  out3[0] = sse;
  out3[1] = sae;
  out3[2] = (double)n;
}

/* SURVEY §8(f) f4, the backward pass of the head (reading R-f6 in DESIGN.md §3): for an
 * upstream gradient dy = dL/dy of one series, with y[h] = (Y[h div S][h mod S] + b[h]) s_r
 * + mu_r (s_r = 1, mu_r = 0 without instance_norm) and Def 10
 * Y[m][t] = sum_n ws[m][n] P_s[n][t] + wt[m][n] P_t[n][t]:
 *   dY[m][t] = dy[m S + t] s_r  (0 for m S + t >= H),
 *   dws[m][n] += sum_t dY[m][t] P_s[n][t],   dwt[m][n] += sum_t dY[m][t] P_t[n][t],
 *   db[h] += dy[h] s_r.
 * The patterns P_s, P_t come from oracle_series_ex (Def 2-9 with every widening flag). */
int oracle_backward_head_ex(const float* x, int64_t B, int32_t C, int32_t L, int32_t S,
                            int32_t H, const float* ws, const float* wt, const float* bias,
                            int32_t head_per_channel, double tau_s, double tau_t,
                            int32_t metric_variant, int32_t instance_norm, double eps_r,
                            int32_t ma_kernel, const float* dy, double* dws, double* dwt,
                            double* db) {
  int32_t N, r, M;
  if (B < 0 || C < 1 || oracle_dims(L, S, H, &N, &r, &M) != 0) return -1;
  int32_t Cw = head_per_channel ? C : 1;
  memset(dws, 0, (size_t)Cw * M * N * sizeof(double));
  memset(dwt, 0, (size_t)Cw * M * N * sizeof(double));
  memset(db, 0, (size_t)Cw * H * sizeof(double));
  size_t nS = (size_t)N * S;
  double* Ps = (double*)malloc(nS * sizeof(double));
  double* Pt = (double*)malloc(nS * sizeof(double));
  double* X = (double*)malloc(nS * sizeof(double));
  double* yy = (double*)malloc((size_t)H * sizeof(double));
  int rc = 0;
  for (int64_t b = 0; b < B && rc == 0; b++)
    for (int32_t c = 0; c < C; c++) {
      int64_t cw = head_per_channel ? c : 0;
      const float* xs = x + (b * C + c) * (int64_t)L;
      oracle_debug dbg;
      memset(&dbg, 0, sizeof(dbg));
      dbg.p_s = Ps;
      dbg.p_t = Pt;
      if (oracle_series_ex(xs, L, S, H, ws + cw * M * N, wt + cw * M * N, bias + cw * H,
                           tau_s, tau_t, metric_variant, instance_norm, eps_r, ma_kernel, yy,
                           &dbg) != 0) {
        rc = -1;
        break;
      }
      double s_r = 1.0;
      if (instance_norm) {                                         /* f1 scale */
        double mu_r, var_r;
        oracle_segment(xs, N, S, r, X);
        oracle_instance_stats(X, N, S, &mu_r, &var_r);
        s_r = sqrt(var_r + eps_r);
      }
      const float* g = dy + (b * C + c) * (int64_t)H;
      for (int32_t m = 0; m < M; m++)
        for (int32_t n = 0; n < N; n++) {
          double as = 0.0, at = 0.0;
          for (int32_t t = 0; t < S; t++) {
            int32_t h = m * S + t;
            double dY = h < H ? (double)g[h] * s_r : 0.0;
            as += dY * Ps[n * S + t];
            at += dY * Pt[n * S + t];
          }
          dws[(cw * M + m) * N + n] += as;
          dwt[(cw * M + m) * N + n] += at;
        }
      for (int32_t h = 0; h < H; h++) db[cw * H + h] += (double)g[h] * s_r;
    }
  free(Ps); free(Pt); free(X); free(yy);
  return rc;
}

/* ------------------------------------------------------------------------------------------
 * SURVEY §8(f) f4, the full backward (reading R-f7 in DESIGN.md §3): gradients of
 * L = sum_h dy[h] y[h] with respect to the input x, the head (ws, wt, bias) and the
 * temperatures tau_s, tau_t, for the base reading (metric_variant bit 0, the level-only
 * trend, allowed: it only zeroes the kappa weight of Def 7).  Each step below is the
 * adjoint of one forward Definition step, applied in reverse order (Def 11 back to Def 2);
 * the forward quantities come from the forward functions above, recomputed in fp64.
 * ------------------------------------------------------------------------------------------ */

/* adjoint of Def 10-11: dY[m][t] = dy[m S + t] (0 past H); db[h] += dy[h];
 * dws[m][n] += sum_t dY[m][t] P_s[n][t] (dwt likewise);
 * dP_s[n][t] = sum_m ws[m][n] dY[m][t] (dP_t likewise). */
static void oracle_head_adj(const double* Ps, const double* Pt, const float* ws, const float* wt,
                            const float* dy, int N, int S, int M, int H, double* dws,
                            double* dwt, double* db, double* dPs, double* dPt) {
  for (int h = 0; h < H; h++) db[h] += (double)dy[h];
  for (int m = 0; m < M; m++)
    for (int n = 0; n < N; n++) {
      double as = 0.0, at = 0.0;
      for (int t = 0; t < S; t++) {
        int h = m * S + t;
        double dY = h < H ? (double)dy[h] : 0.0;
        as += dY * Ps[n * S + t];
        at += dY * Pt[n * S + t];
      }
      dws[m * N + n] += as;
      dwt[m * N + n] += at;
    }
  for (int n = 0; n < N; n++)
    for (int t = 0; t < S; t++) {
      double gs = 0.0, gt = 0.0;
      for (int m = 0; m < M; m++) {
        int h = m * S + t;
        double dY = h < H ? (double)dy[h] : 0.0;
        gs += (double)ws[m * N + n] * dY;
        gt += (double)wt[m * N + n] * dY;
      }
      dPs[n * S + t] = gs;
      dPt[n * S + t] = gt;
    }
}

/* adjoint of Def 9 (P = A X): dA[i][j] = sum_t dP[i][t] X[j][t];
 * dX[j][t] += sum_i A[i][j] dP[i][t]. */
static void oracle_aggregate_adj(const double* A, const double* X, const double* dP, int N, int S,
                                 double* dA, double* dX) {
  for (int i = 0; i < N; i++)
    for (int j = 0; j < N; j++) {
      double s = 0.0;
      for (int t = 0; t < S; t++) s += dP[i * S + t] * X[j * S + t];
      dA[i * N + j] = s;
    }
  for (int j = 0; j < N; j++)
    for (int t = 0; t < S; t++) {
      double s = 0.0;
      for (int i = 0; i < N; i++) s += A[i * N + j] * dP[i * S + t];
      dX[j * S + t] += s;
    }
}

/* adjoint of one row softmax of Def 8 (A = softmax_j(l)): dl[i][j] = A[i][j] (dA[i][j] -
 * sum_k A[i][k] dA[i][k]). */
static void oracle_softmax_adj(const double* A, const double* dA, int N, double* dl) {
  for (int i = 0; i < N; i++) {
    double s = 0.0;
    for (int k = 0; k < N; k++) s += A[i * N + k] * dA[i * N + k];
    for (int j = 0; j < N; j++) dl[i * N + j] = A[i * N + j] * (dA[i * N + j] - s);
  }
}

/* adjoint of Def 7 with its normalisation Dhat = D / (sigma2 + eps_t) and the trend logits
 * l_t = -Dhat / tau_t: dDhat = -dl_t / tau_t; dtau_t += sum dl_t Dhat / tau_t^2;
 * dD = dDhat / (sigma2 + eps_t); dsigma2 += -sum dDhat D / (sigma2 + eps_t)^2;
 * D_ij = (mu_i - mu_j)^2 + w (kappa_i - kappa_j)^2 (w = (S^2 - 1)/12, 0 for bit 0):
 * dmu_i += 2 (mu_i - mu_j) dD_ij, dmu_j -= 2 (mu_i - mu_j) dD_ij (kappa likewise with w). */
static void oracle_trend_adj(const double* mu, const double* kappa, const double* D,
                             double sigma2, const double* dlt, int N, int S, int level_only,
                             double tau_t, double* dmu, double* dkappa, double* dsigma2,
                             double* dtau_t) {
  double w = level_only ? 0.0 : ((double)S * (double)S - 1.0) / 12.0;
  double den = sigma2 + ORACLE_EPS_T;
  for (int i = 0; i < N; i++)
    for (int j = 0; j < N; j++) {
      double Dh = D[i * N + j] / den;
      double dDh = -dlt[i * N + j] / tau_t;
      *dtau_t += dlt[i * N + j] * Dh / (tau_t * tau_t);
      double dD = dDh / den;
      *dsigma2 += -dDh * D[i * N + j] / (den * den);
      double gm = 2.0 * (mu[i] - mu[j]) * dD;
      double gk = 2.0 * w * (kappa[i] - kappa[j]) * dD;
      dmu[i] += gm;
      dmu[j] -= gm;
      dkappa[i] += gk;
      dkappa[j] -= gk;
    }
}

/* adjoint of Def 6 with the seasonal logits l_s = rho / tau_s: drho = dl_s / tau_s;
 * dtau_s += -sum dl_s rho / tau_s^2; rho_ij = <z_i, z_j> g_i g_j with
 * g_n = (nu2_n + eps_s)^(-1/2):
 *   dz_i[t] += sum_j drho_ij g_i g_j z_j[t],  dz_j[t] += sum_i drho_ij g_i g_j z_i[t],
 *   dg_i += sum_j drho_ij <z_i, z_j> g_j,     dg_j += sum_i drho_ij <z_i, z_j> g_i,
 *   dnu2_n += dg_n (-1/2) (nu2_n + eps_s)^(-3/2). */
static void oracle_seasonal_adj(const double* z, const double* nu2, const double* rho,
                                const double* dls, int N, int S, double tau_s, double* dz,
                                double* dnu2, double* dtau_s) {
  double* g = (double*)malloc(N * sizeof(double));
  double* dg = (double*)calloc(N, sizeof(double));
  for (int n = 0; n < N; n++) g[n] = 1.0 / sqrt(nu2[n] + ORACLE_EPS_S);
  for (int i = 0; i < N; i++)
    for (int j = 0; j < N; j++) {
      double drho = dls[i * N + j] / tau_s;
      *dtau_s += -dls[i * N + j] * rho[i * N + j] / (tau_s * tau_s);
      double G = 0.0;
      for (int t = 0; t < S; t++) G += z[i * S + t] * z[j * S + t];
      for (int t = 0; t < S; t++) {
        dz[i * S + t] += drho * g[i] * g[j] * z[j * S + t];
        dz[j * S + t] += drho * g[i] * g[j] * z[i * S + t];
      }
      dg[i] += drho * G * g[j];
      dg[j] += drho * G * g[i];
    }
  for (int n = 0; n < N; n++)
    dnu2[n] += dg[n] * (-0.5) * pow(nu2[n] + ORACLE_EPS_S, -1.5);
  free(g);
  free(dg);
}

/* adjoint of Def 5: sigma2 = (1/(N S)) sum_n [nu2_n + S (mu_n - mubar)^2]:
 * dnu2_n += dsigma2 / (N S);  dmu_n += dsigma2 2 (mu_n - mubar) / N
 * (the mubar path contributes sum_n (mu_n - mubar) = 0). */
static void oracle_series_variance_adj(const double* mu, int N, int S, double dsigma2,
                                       double* dnu2, double* dmu) {
  double mbar = 0.0;
  for (int n = 0; n < N; n++) mbar += mu[n];
  mbar /= (double)N;
  for (int n = 0; n < N; n++) {
    dnu2[n] += dsigma2 / ((double)N * (double)S);
    dmu[n] += dsigma2 * 2.0 * (mu[n] - mbar) / (double)N;
  }
}

/* adjoint of Def 3-4: nu2_n = sum_t z_n[t]^2 -> dz_n[t] += 2 z_n[t] dnu2_n;
 * kappa_n = sum_t ttilde_t z_n[t] / V -> dz_n[t] += ttilde_t dkappa_n / V;
 * z_n = X_n - mu_n -> dX_n[t] += dz_n[t], dmu_n -= sum_t dz_n[t];
 * mu_n = (1/S) sum_t X_n[t] -> dX_n[t] += dmu_n / S. */
static void oracle_descriptors_adj(const double* z, int N, int S, const double* dnu2,
                                   const double* dkappa, double* dz, double* dmu, double* dX) {
  double V = 0.0;
  for (int t = 0; t < S; t++) {
    double tt = (double)t - 0.5 * (double)(S - 1);
    V += tt * tt;
  }
  for (int n = 0; n < N; n++) {
    for (int t = 0; t < S; t++) {
      double tt = (double)t - 0.5 * (double)(S - 1);
      dz[n * S + t] += 2.0 * z[n * S + t] * dnu2[n] + tt * dkappa[n] / V;
    }
    double s = 0.0;
    for (int t = 0; t < S; t++) {
      dX[n * S + t] += dz[n * S + t];
      s += dz[n * S + t];
    }
    dmu[n] -= s;
    for (int t = 0; t < S; t++) dX[n * S + t] += dmu[n] / (double)S;
  }
}

/* One series: the adjoint chain Def 11 -> Def 2.  dx (L doubles) is overwritten (0 for the
 * r dropped points); dws/dwt ([M][N]), db ([H]) and dtau ([2]: tau_s, tau_t) accumulate. */
int oracle_backward_series(const float* x, int32_t L, int32_t S, int32_t H, const float* ws,
                           const float* wt, const float* bias, double tau_s, double tau_t,
                           int32_t metric_variant, const float* dy, double* dx, double* dws,
                           double* dwt, double* db, double* dtau) {
  int32_t N, r, M;
  if (oracle_dims(L, S, H, &N, &r, &M) != 0 || !(tau_s > 0.0) || !(tau_t > 0.0) ||
      (metric_variant & ~1) != 0)
    return -1;
  size_t nS = (size_t)N * S, nN = (size_t)N * N;
  double* X = (double*)malloc(nS * sizeof(double));
  double* mu = (double*)malloc(N * sizeof(double));
  double* z = (double*)malloc(nS * sizeof(double));
  double* nu2 = (double*)malloc(N * sizeof(double));
  double* kappa = (double*)malloc(N * sizeof(double));
  double* rho = (double*)malloc(nN * sizeof(double));
  double* D = (double*)malloc(nN * sizeof(double));
  double* Dh = (double*)malloc(nN * sizeof(double));
  double* As = (double*)malloc(nN * sizeof(double));
  double* At = (double*)malloc(nN * sizeof(double));
  double* Ps = (double*)malloc(nS * sizeof(double));
  double* Pt = (double*)malloc(nS * sizeof(double));
  double* dPs = (double*)malloc(nS * sizeof(double));
  double* dPt = (double*)malloc(nS * sizeof(double));
  double* dAs = (double*)malloc(nN * sizeof(double));
  double* dAt = (double*)malloc(nN * sizeof(double));
  double* dls = (double*)malloc(nN * sizeof(double));
  double* dlt = (double*)malloc(nN * sizeof(double));
  double* dX = (double*)calloc(nS, sizeof(double));
  double* dz = (double*)calloc(nS, sizeof(double));
  double* dmu = (double*)calloc(N, sizeof(double));
  double* dkappa = (double*)calloc(N, sizeof(double));
  double* dnu2 = (double*)calloc(N, sizeof(double));

  /* forward, Def 2-9 (the functions above) */
  oracle_segment(x, N, S, r, X);
  oracle_descriptors(X, N, S, mu, z, nu2, kappa);
  double sigma2 = oracle_series_variance(mu, nu2, N, S);
  oracle_seasonal_similarity(z, nu2, N, S, rho);
  oracle_trend_distance(mu, kappa, N, S, metric_variant & 1, D);
  for (size_t k = 0; k < nN; k++) Dh[k] = D[k] / (sigma2 + ORACLE_EPS_T);
  oracle_softmax_rows(rho, N, +1.0, 1.0 / tau_s, As);
  oracle_softmax_rows(Dh, N, -1.0, 1.0 / tau_t, At);
  oracle_aggregate(As, X, N, S, Ps);
  oracle_aggregate(At, X, N, S, Pt);
  (void)bias;   /* y = Y + b: the bias enters the gradient only as db */

  /* adjoints, Def 11 -> Def 2 */
  oracle_head_adj(Ps, Pt, ws, wt, dy, N, S, M, H, dws, dwt, db, dPs, dPt);   /* Def 10-11 */
  oracle_aggregate_adj(As, X, dPs, N, S, dAs, dX);                          /* Def 9 (s) */
  oracle_aggregate_adj(At, X, dPt, N, S, dAt, dX);                          /* Def 9 (t) */
  oracle_softmax_adj(As, dAs, N, dls);                                      /* Def 8 (s) */
  oracle_softmax_adj(At, dAt, N, dlt);                                      /* Def 8 (t) */
  double dsigma2 = 0.0;
  oracle_trend_adj(mu, kappa, D, sigma2, dlt, N, S, metric_variant & 1, tau_t, dmu, dkappa,
                   &dsigma2, &dtau[1]);                                     /* Def 7     */
  oracle_seasonal_adj(z, nu2, rho, dls, N, S, tau_s, dz, dnu2, &dtau[0]);   /* Def 6     */
  oracle_series_variance_adj(mu, N, S, dsigma2, dnu2, dmu);                 /* Def 5     */
  oracle_descriptors_adj(z, N, S, dnu2, dkappa, dz, dmu, dX);               /* Def 3-4   */
  for (int32_t k = 0; k < L; k++) dx[k] = 0.0;                              /* Def 2     */
  for (int n = 0; n < N; n++)
    for (int t = 0; t < S; t++) dx[r + n * S + t] = dX[n * S + t];

  free(X); free(mu); free(z); free(nu2); free(kappa); free(rho); free(D); free(Dh);
  free(As); free(At); free(Ps); free(Pt); free(dPs); free(dPt); free(dAs); free(dAt);
  free(dls); free(dlt); free(dX); free(dz); free(dmu); free(dkappa); free(dnu2);
  return 0;
}

int oracle_backward(const float* x, int64_t B, int32_t C, int32_t L, int32_t S, int32_t H,
                    const float* ws, const float* wt, const float* bias,
                    int32_t head_per_channel, double tau_s, double tau_t,
                    int32_t metric_variant, const float* dy, double* dx, double* dws,
                    double* dwt, double* db, double* dtau) {
  int32_t N, r, M;
  if (B < 0 || C < 1 || oracle_dims(L, S, H, &N, &r, &M) != 0) return -1;
  int32_t Cw = head_per_channel ? C : 1;
  memset(dws, 0, (size_t)Cw * M * N * sizeof(double));
  memset(dwt, 0, (size_t)Cw * M * N * sizeof(double));
  memset(db, 0, (size_t)Cw * H * sizeof(double));
  dtau[0] = dtau[1] = 0.0;
  for (int64_t b = 0; b < B; b++)
    for (int32_t c = 0; c < C; c++) {
      int64_t cw = head_per_channel ? c : 0;
      int64_t o = b * C + c;
      if (oracle_backward_series(x + o * L, L, S, H, ws + cw * M * N, wt + cw * M * N,
                                 bias + cw * H, tau_s, tau_t, metric_variant, dy + o * H,
                                 dx + o * L, dws + cw * M * N, dwt + cw * M * N, db + cw * H,
                                 dtau) != 0)
        return -1;
    }
  return 0;
}
