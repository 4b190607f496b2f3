/* abi_caller.c -- a plain C99 caller of the PRNet C ABI (include/prnet.h), test
 * infrastructure.  Built by tests/test_abi_c.py with gcc against the header and linked
 * against libprnet.so; it uses no CUDA API (the host-buffer entry point owns the device
 * side), so it exercises exactly what a C user sees.
 *
 *   abi_caller layout           -> JSON: sizeof / offsetof of prnet_config, ABI version
 *   abi_caller nodevice         -> prnet_create on a machine without a GPU: status + message
 *   abi_caller run OUT.bin      -> create / load_params / forward_host / destroy on a fixed
 *                                  C = 3, L = 720, S = 24, H = 96 problem; writes x, params
 *                                  and y (float32) to OUT.bin for the Python side to check
 */
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "prnet.h"

#define FIELD(f) printf("  \"%s\": %zu,\n", #f, offsetof(prnet_config, f))

static float lcg(uint32_t* s) { /* deterministic values in [-1, 1) */
  *s = *s * 1664525u + 1013904223u;
  return (float)((*s >> 8) & 0xFFFFFF) / 8388608.0f - 1.0f;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  if (strcmp(argv[1], "layout") == 0) {
    printf("{\n  \"sizeof\": %zu,\n", sizeof(prnet_config));
    FIELD(abi_version); FIELD(channels); FIELD(lookback); FIELD(seg_len); FIELD(horizon);
    FIELD(head_per_channel); FIELD(metric_variant); FIELD(tau_seasonal); FIELD(tau_trend);
    FIELD(device); FIELD(instance_norm); FIELD(ma_kernel);
    printf("  \"abi\": %d\n}\n", PRNET_ABI_VERSION);
    return 0;
  }
  prnet_config cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.abi_version = PRNET_ABI_VERSION;
  cfg.channels = 3; cfg.lookback = 720; cfg.seg_len = 24; cfg.horizon = 96;
  cfg.head_per_channel = 1; cfg.tau_seasonal = 1.0f; cfg.tau_trend = 1.0f; cfg.device = 0;
  prnet_handle* h = NULL;
  prnet_status st = prnet_create(&cfg, &h);
  if (strcmp(argv[1], "nodevice") == 0) {
    printf("%d %s\n", (int)st, prnet_last_error(NULL));
    return h == NULL ? 0 : 1;
  }
  if (strcmp(argv[1], "run") != 0 || argc < 3) return 2;
  if (st != PRNET_OK) { fprintf(stderr, "create: %d %s\n", st, prnet_last_error(NULL)); return 3; }
  int32_t N, M, r;
  if (prnet_get_dims(h, &N, &M, &r) != PRNET_OK || N != 30 || M != 4 || r != 0) return 4;
  const int B = 5, C = 3, L = 720, H = 96;
  const size_t nx = (size_t)B * C * L, ny = (size_t)B * C * H, nw = (size_t)C * M * N, nb = (size_t)C * H;
  float* x = malloc(nx * 4); float* y = malloc(ny * 4);
  float* ws = malloc(nw * 4); float* wt = malloc(nw * 4); float* b = malloc(nb * 4);
  uint32_t seed = 12345u;
  for (size_t k = 0; k < nx; k++) x[k] = lcg(&seed) + 0.5f * (float)((k % L) % 24) / 24.0f;
  for (size_t k = 0; k < nw; k++) { ws[k] = 0.2f * lcg(&seed); wt[k] = 0.2f * lcg(&seed); }
  for (size_t k = 0; k < nb; k++) b[k] = 0.1f * lcg(&seed);
  if ((st = prnet_load_params(h, ws, wt, b, (int64_t)nw, (int64_t)nb)) != PRNET_OK) return 5;
  /* a rejected call: wrong parameter count -> INVALID_ARG, nothing written */
  if (prnet_load_params(h, ws, wt, b, (int64_t)nw - 1, (int64_t)nb) != PRNET_ERR_INVALID_ARG) return 6;
  if ((st = prnet_forward_host(h, x, B, y)) != PRNET_OK) {
    fprintf(stderr, "forward_host: %d %s\n", st, prnet_last_error(h)); return 7;
  }
  prnet_destroy(h);
  FILE* f = fopen(argv[2], "wb");
  if (!f) return 8;
  fwrite(x, 4, nx, f); fwrite(ws, 4, nw, f); fwrite(wt, 4, nw, f); fwrite(b, 4, nb, f);
  fwrite(y, 4, ny, f);
  fclose(f);
  free(x); free(y); free(ws); free(wt); free(b);
  return 0;
}
