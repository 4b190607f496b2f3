/*
 * prnet_oracle.h -- CPU ORACLE for the PRNet pattern-attention forward.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this code.  The
 * product path (paper_2404_02445_b200/, libprnet.so) never includes, links or
 * calls it, and shares no header, helper or constant with it.
 *
 * What it computes (one (window, channel) series x in R^L at a time):
 *   PAPER.md:19-22 (abstract): segments, "two metrics to evaluate the similarity
 *   between segments which contain different dominant patterns (seasonal or
 *   trend)", "a pattern attention mechanism, which aggregates similar segments
 *   to extract patterns for forecasting"; PAPER.md:45 (conclusion).  The
 *   method sections (\subfile lines) have no body, so every
 *   formula is the reading fixed in SURVEY.md §8(c) "Definition" steps 1-11
 *   and ambiguity register A1-A18, restated in DESIGN.md §3.
 *
 * Arithmetic: inputs are fp32 (as the C-ABI receives them); every quantity is
 * computed in IEEE double, single-threaded, in the order the definition
 * states; the output is rounded once to fp32 (plus an fp64 copy for tests).
 *
 * Parity status of each function: see the comment above it in
 * prnet_oracle.c and DESIGN.md §4 (pins).  The formulas themselves are
 * "parity unpinned" against the paper's own equations (absent from the
 * reference); they are pinned against the closed forms,
 * invariants, limits and worked examples listed there.
 */
#ifndef PRNET_ORACLE_H
#define PRNET_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Per-series intermediates (all caller-allocated; any pointer may be NULL).
 * Sizes: seg N*S, mu/nu2/kappa N, rho/dist/a_s/a_t N*N, p_s/p_t N*S,
 * y_full M*S, y H. Row-major. */
typedef struct {
  double* seg;     /* X[n][t]                      (Definition step 2)  */
  double* mu;      /* mu_n                          (step 4)             */
  double* nu2;     /* nu^2_n                        (step 4)             */
  double* kappa;   /* kappa_n                       (step 4)             */
  double* sigma2;  /* [1] sigma^2                   (step 5)             */
  double* rho;     /* rho_ij                        (step 6)             */
  double* dist;    /* D_ij (unnormalised)           (step 7)             */
  double* a_s;     /* A_s                           (step 8)             */
  double* a_t;     /* A_t                           (step 8)             */
  double* p_s;     /* P_s = A_s X                   (step 9)             */
  double* p_t;     /* P_t = A_t X                   (step 9)             */
  double* y_full;  /* Y[m][t] before truncation     (step 10)            */
} oracle_debug;

/* Derived sizes (Definition step 1).  Returns 0 on success, -1 if S < 2,
 * L < S or H < 1. */
int oracle_dims(int32_t L, int32_t S, int32_t H, int32_t* N, int32_t* r, int32_t* M);

/* One series.  x: L fp32 values; ws, wt: M*N (row m = future segment m,
 * column n = pattern n); bias: H.  y: H doubles.  dbg may be NULL.
 * Returns 0, or -1 on invalid dims / tau <= 0. */
int oracle_series(const float* x, int32_t L, int32_t S, int32_t H,
                  const float* ws, const float* wt, const float* bias,
                  double tau_s, double tau_t, double* y, const oracle_debug* dbg);

/* As oracle_series, with the SURVEY §8(f) widening (DESIGN.md §3 readings R-f1, R-f3):
 * metric_variant bit 0: level-only trend distance D_ij = (mu_i - mu_j)^2;
 * metric_variant bit 1: seasonal metric on the residuals about each segment's
 *                       least-squares line;
 * metric_variant bit 2: component values (A10 variant, reading R-f4): the seasonal
 *                       branch aggregates z_n (bit 1: z_n - kappa_n ttilde), the trend
 *                       branch the line T_n (bit 0: the level mu_n);
 * instance_norm != 0:   RevIN-style normalisation of the segmented points with
 *                       eps_r, de-normalised forecast;
 * ma_kernel = k > 0:    moving-average decomposition (odd k, edge-replicate padding) of
 *                       the segmented points (reading R-f5): the seasonal branch (Def 3-4,
 *                       6, 9) runs on x - MA(x), the trend branch (Def 3-5, 7, 9) on MA(x).
 *                       dbg->mu, kappa, sigma2 are then the trend branch's, dbg->nu2 the
 *                       seasonal branch's, dbg->seg the segments before the split.
 * Returns -1 also for metric_variant outside [0, 7], eps_r < 0, ma_kernel < 0 or even. */
int oracle_series_ex(const float* x, int32_t L, int32_t S, int32_t H,
                     const float* ws, const float* wt, const float* bias,
                     double tau_s, double tau_t, int32_t metric_variant,
                     int32_t instance_norm, double eps_r, int32_t ma_kernel, double* y,
                     const oracle_debug* dbg);

/* A batch x[B][C][L] -> y[B][C][H] (fp32, rounded from the fp64 result) and
 * optionally y64 (fp64).  head_per_channel: 1 -> ws/wt are [C][M][N], bias
 * [C][H]; 0 -> [1][M][N], [1][H].  Series are processed in (b, c) order,
 * one after the other.  Returns 0 or -1. */
int oracle_forward(const float* x, int64_t B, int32_t C, int32_t L, int32_t S,
                   int32_t H, const float* ws, const float* wt, const float* bias,
                   int32_t head_per_channel, double tau_s, double tau_t,
                   float* y, double* y64);

int oracle_forward_ex(const float* x, int64_t B, int32_t C, int32_t L, int32_t S,
                      int32_t H, const float* ws, const float* wt, const float* bias,
                      int32_t head_per_channel, double tau_s, double tau_t,
                      int32_t metric_variant, int32_t instance_norm, double eps_r,
                      int32_t ma_kernel, float* y, double* y64);

/* SURVEY §8(f) f4 (reading R-f6): gradients of L = sum dy * y with respect to the head
 * (ws, wt: [Cw][M][N]; bias: [Cw][H]) for the upstream gradient dy [B][C][H], summed over
 * the batch (and over the channels when head_per_channel = 0).  Outputs are fp64 and
 * overwritten.  Returns 0 or -1. */
int oracle_backward_head_ex(const float* x, int64_t B, int32_t C, int32_t L, int32_t S,
                            int32_t H, const float* ws, const float* wt, const float* bias,
                            int32_t head_per_channel, double tau_s, double tau_t,
                            int32_t metric_variant, int32_t instance_norm, double eps_r,
                            int32_t ma_kernel, const float* dy, double* dws, double* dwt,
                            double* db);

/* SURVEY §8(f) f4, the full backward (reading R-f7): gradients of L = sum dy * y with
 * respect to the input x (dx [B][C][L], 0 at the r dropped points), the head (dws, dwt
 * [Cw][M][N], db [Cw][H], summed over the batch) and the temperatures (dtau[0] = dL/dtau_s,
 * dtau[1] = dL/dtau_t, summed over every series), for the base reading (metric_variant 0
 * or 1).  The adjoint of each Definition step is its own function, applied Def 11 -> Def 2.
 * Outputs are fp64 and overwritten.  Returns 0 or -1. */
int oracle_backward(const float* x, int64_t B, int32_t C, int32_t L, int32_t S, int32_t H,
                    const float* ws, const float* wt, const float* bias,
                    int32_t head_per_channel, double tau_s, double tau_t,
                    int32_t metric_variant, const float* dy, double* dx, double* dws,
                    double* dwt, double* db, double* dtau);
/* one series (dws, dwt, db, dtau accumulate; dx [L] overwritten) */
int oracle_backward_series(const float* x, int32_t L, int32_t S, int32_t H, const float* ws,
                           const float* wt, const float* bias, double tau_s, double tau_t,
                           int32_t metric_variant, const float* dy, double* dx, double* dws,
                           double* dwt, double* db, double* dtau);

/* Sum of squared and absolute errors of y against target (n values), fp64,
 * in index order: out[0] = SSE, out[1] = SAE, out[2] = n.  (Bench metric,
 * PAPER.md:22 "accuracy"; MSE = SSE/n, MAE = SAE/n.) */
void oracle_error_sums(const float* y, const float* target, int64_t n, double* out3);

#ifdef __cplusplus
}
#endif
#endif
