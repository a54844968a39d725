/* Plain-C consumer of include/liger_b200.h: the header compiles as C99 and the library's
 * host-only entry points (version, plan, workspace queries, argument validation) answer
 * without a GPU.  Built and run by tests/test_capi_c.py. */
#include <stdio.h>
#include <string.h>

#include "liger_b200.h"

#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      fprintf(stderr, "check failed: %s (line %d)\n", #cond, __LINE__); \
      return 1;                                                       \
    }                                                                 \
  } while (0)

int main(void) {
  const char* v = lk_version();
  CHECK(v != NULL && strstr(v, "sm_100a") != NULL);
  int64_t c = 0, n = 0;
  CHECK(lk_flce_plan(8192, 4096, 128256, LK_BF16, &c, &n) == LK_OK);
  CHECK(c == 2816 && n == 3);
  CHECK(lk_flce_plan(0, 4096, 128256, LK_BF16, &c, &n) == LK_SIZE_MISMATCH);
  lk_flce_args a;
  memset(&a, 0, sizeof(a));
  a.bt = 8192;
  a.hidden = 4096;
  a.vocab = 128256;
  a.dtype = LK_BF16;
  a.grad_x = (void*)16;
  a.grad_w = (void*)16;
  const size_t ws = lk_flce_workspace_bytes_for(&a);
  CHECK(ws > (size_t)2816 * 128256 * 2);
  a.x_row_index = (const int64_t*)16; /* kept-row gather: one more chunk-sized X buffer */
  CHECK(lk_flce_workspace_bytes_for(&a) > ws);
  CHECK(lk_flce_forward_backward(NULL) == LK_INVALID_ARGUMENT);
  CHECK(lk_compact_rows(NULL, -1, -100, NULL, NULL, NULL, NULL) == LK_INVALID_ARGUMENT);
  CHECK(lk_gather_rows(NULL, 4, 3, NULL, 4, NULL, 0, NULL) == LK_INVALID_ARGUMENT);
  CHECK(lk_peer_allreduce(NULL, 2, 0, LK_PEER_CTL_BYTES, 8, LK_BF16, 1, 0, NULL) == LK_INVALID_ARGUMENT);
  CHECK(lk_test_select_path(LK_PATH_DW_ACCUM16, 2) == -1);
  printf("c abi ok: %s, plan %lld x %lld, workspace %zu bytes\n", v, (long long)c, (long long)n, ws);
  return 0;
}
