/* The FLCE through the C ABI from plain C: cudaMalloc'd buffers, one lk_flce_forward_backward
 * call (fp32 inputs: the split-operand tcgen05 path), checked against a float64 loop
 * restatement of Liger's FLCE (MEAN over non-ignored rows, ignored rows zero).  This is what
 * a non-Python caller of the reference's operator would do.  Built and run
 * by tests/test_capi_c.py on the GPU. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "liger_b200.h"

enum { BT = 96, H = 128, V = 1000 };

static unsigned long long lcg = 12345;
static double urand(void) { /* uniform in [-1, 1) */
  lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
  return (double)(lcg >> 11) / (double)(1ull << 53) * 2.0 - 1.0;
}

#define CU(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));              \
      return 2;                                                                \
    }                                                                          \
  } while (0)

int main(void) {
  static float x[BT * H], w[V * H], gx[BT * H], gw[V * H];
  static int64_t t[BT];
  static double z[V], dz[BT * V], rgx[BT * H], rgw[V * H];
  for (int i = 0; i < BT * H; ++i) x[i] = (float)urand();
  for (int i = 0; i < V * H; ++i) w[i] = (float)(urand() * 3.0 / sqrt((double)H));
  for (int i = 0; i < BT; ++i) t[i] = (i % 7 == 3) ? -100 : (int64_t)((urand() + 1.0) * 0.5 * (V - 1));

  /* float64 restatement: loss = mean over valid rows of lse - z_t; dZ = (softmax - onehot) / n */
  int n_valid = 0;
  for (int i = 0; i < BT; ++i) n_valid += t[i] != -100;
  double loss = 0.0;
  memset(dz, 0, sizeof(dz));
  for (int i = 0; i < BT; ++i) {
    if (t[i] == -100) continue;
    double m = -INFINITY, s = 0.0;
    for (int v = 0; v < V; ++v) {
      double a = 0.0;
      for (int k = 0; k < H; ++k) a += (double)x[i * H + k] * (double)w[v * H + k];
      z[v] = a;
      if (a > m) m = a;
    }
    for (int v = 0; v < V; ++v) s += exp(z[v] - m);
    const double lse = m + log(s);
    loss += (lse - z[t[i]]) / n_valid;
    for (int v = 0; v < V; ++v) dz[i * V + v] = (exp(z[v] - lse) - (v == t[i] ? 1.0 : 0.0)) / n_valid;
  }
  for (int i = 0; i < BT; ++i)
    for (int k = 0; k < H; ++k) {
      double a = 0.0;
      for (int v = 0; v < V; ++v) a += dz[i * V + v] * (double)w[v * H + k];
      rgx[i * H + k] = a;
    }
  for (int v = 0; v < V; ++v)
    for (int k = 0; k < H; ++k) {
      double a = 0.0;
      for (int i = 0; i < BT; ++i) a += dz[i * V + v] * (double)x[i * H + k];
      rgw[v * H + k] = a;
    }

  float *dx, *dw, *dgx, *dgw, *dloss_rows, *dloss;
  int64_t *dt, *dstats;
  CU(cudaMalloc((void**)&dx, sizeof(x)));
  CU(cudaMalloc((void**)&dw, sizeof(w)));
  CU(cudaMalloc((void**)&dgx, sizeof(gx)));
  CU(cudaMalloc((void**)&dgw, sizeof(gw)));
  CU(cudaMalloc((void**)&dloss_rows, BT * sizeof(float)));
  CU(cudaMalloc((void**)&dloss, sizeof(float)));
  CU(cudaMalloc((void**)&dt, sizeof(t)));
  CU(cudaMalloc((void**)&dstats, 2 * sizeof(int64_t)));
  CU(cudaMemcpy(dx, x, sizeof(x), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(dw, w, sizeof(w), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(dt, t, sizeof(t), cudaMemcpyHostToDevice));

  lk_flce_args a;
  memset(&a, 0, sizeof(a));
  a.x = dx; a.weight = dw; a.target = dt;
  a.bt = BT; a.hidden = H; a.vocab = V; a.dtype = LK_F32;
  a.ignore_index = -100; a.reduction = LK_REDUCTION_MEAN;
  a.loss_rows = dloss_rows; a.loss_sum = dloss; a.grad_x = dgx; a.grad_w = dgw; a.target_stats = dstats;
  a.workspace_bytes = lk_flce_workspace_bytes_for(&a);
  CU(cudaMalloc(&a.workspace, a.workspace_bytes));
  const int rc = lk_flce_forward_backward(&a);
  if (rc != LK_OK) {
    fprintf(stderr, "lk_flce_forward_backward: %d %s\n", rc, lk_last_error());
    return 1;
  }
  CU(cudaDeviceSynchronize());
  float got_loss = 0.f;
  int64_t stats[2];
  CU(cudaMemcpy(&got_loss, dloss, sizeof(float), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(gx, dgx, sizeof(gx), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(gw, dgw, sizeof(gw), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(stats, dstats, sizeof(stats), cudaMemcpyDeviceToHost));

  /* fp32 tolerance (north star): |a - b| <= 1e-4 (|b| + max|b|) */
  double mx = 0.0, mw = 0.0, ex = 0.0, ew = 0.0;
  for (int i = 0; i < BT * H; ++i) mx = fmax(mx, fabs(rgx[i]));
  for (int i = 0; i < V * H; ++i) mw = fmax(mw, fabs(rgw[i]));
  for (int i = 0; i < BT * H; ++i) ex = fmax(ex, fabs(gx[i] - rgx[i]) / (fabs(rgx[i]) + mx));
  for (int i = 0; i < V * H; ++i) ew = fmax(ew, fabs(gw[i] - rgw[i]) / (fabs(rgw[i]) + mw));
  const double el = fabs(got_loss - loss) / fabs(loss);
  int zero_rows = 1;
  for (int i = 0; i < BT; ++i)
    if (t[i] == -100)
      for (int k = 0; k < H; ++k) zero_rows &= gx[i * H + k] == 0.f;
  printf("loss %.7f (f64 %.7f) rel %.2e; grad_x %.2e; grad_w %.2e; n_valid %lld/%d; ignored rows zero %d\n",
         got_loss, loss, el, ex, ew, (long long)stats[0], n_valid, zero_rows);
  if (el > 1e-4 || ex > 1e-4 || ew > 1e-4 || stats[0] != n_valid || stats[1] != 0 || !zero_rows) return 1;
  printf("c flce ok\n");
  return 0;
}
