/* A plain-C consumer of the drop-in boundary (include/rsr_b200.h): what a C / cgo / JNI host
 * binding of the reference's multiply path calls.  It preprocesses a random ternary matrix on
 * the GPU, multiplies an integer vector through a host-buffer session (the reference's calling
 * convention: host fp64 in, fresh host fp64 out) and checks every column against a naive CPU
 * product.  No torch, no Python: only the CUDA runtime for device buffers.
 *
 *   gcc -O2 -std=c11 -I include integration/c_example.c -L paper_2411_06360_b200/lib -lrsr_b200 \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2411_06360_b200/lib -o c_example
 *   ./c_example [rows cols k]      (needs a GPU; tests/test_integration_stub.py builds and runs it)
 */
#include <cuda_runtime_api.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "rsr_b200.h"

#define CK(x)                                                                   \
  do {                                                                          \
    if ((x) != RSR_OK) {                                                        \
      fprintf(stderr, "%s failed: %s\n", #x, rsr_b200_last_error());           \
      return 1;                                                                 \
    }                                                                           \
  } while (0)
#define CU(x)                                                                   \
  do {                                                                          \
    if ((x) != cudaSuccess) {                                                   \
      fprintf(stderr, "%s failed\n", #x);                                       \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 3000, cols = argc > 2 ? atoll(argv[2]) : 777;
  const int32_t k = argc > 3 ? atoi(argv[3]) : 8;
  if (rsr_b200_abi_version() != RSR_B200_ABI_VERSION) {
    fprintf(stderr, "ABI mismatch\n");
    return 1;
  }
  int8_t* A = (int8_t*)malloc((size_t)(rows * cols));
  double* v = (double*)malloc(sizeof(double) * (size_t)rows);
  double* out = (double*)malloc(sizeof(double) * (size_t)cols);
  uint32_t s = 12345;
  for (int64_t i = 0; i < rows * cols; ++i) {
    s = s * 1664525u + 1013904223u;
    A[i] = (int8_t)((int)(s >> 24) % 3 - 1);
  }
  for (int64_t r = 0; r < rows; ++r) {
    s = s * 1664525u + 1013904223u;
    v[r] = (double)((int)(s >> 24) % 201 - 100);  /* integer-valued fp64: exact on the int32 kernel */
  }
  /* index layout + device arrays (rsr_index_layout fills the descriptor's sizes) */
  rsr_index_desc d;
  size_t perm_b, seg_b, key_b;
  CK(rsr_index_layout(rows, cols, k, 2, &d, &perm_b, &seg_b, &key_b));
  for (int h = 0; h < 2; ++h) {
    CU(cudaMalloc(&d.half[h].perm, perm_b));
    CU(cudaMalloc((void**)&d.half[h].seg, seg_b));
    CU(cudaMalloc((void**)&d.half[h].bucket, key_b));
  }
  int8_t* dA;
  CU(cudaMalloc((void**)&dA, (size_t)(rows * cols)));
  CU(cudaMemcpy(dA, A, (size_t)(rows * cols), cudaMemcpyHostToDevice));
  const size_t ws_b = rsr_preprocess_workspace_bytes(&d);
  void* ws;
  int32_t* bad;
  CU(cudaMalloc(&ws, ws_b));
  CU(cudaMalloc((void**)&bad, 4));
  CU(cudaMemset(bad, 0, 4));
  CK(rsr_preprocess_ternary(dA, cols, &d, bad, ws, ws_b, NULL));
  CU(cudaDeviceSynchronize());
  /* the reference's calling convention through a session: host fp64 in, host fp64 out */
  rsr_host_session* sess;
  CK(rsr_host_session_create(&d, &sess));
  for (int call = 0; call < 3; ++call) {
    CK(rsr_host_session_multiply(sess, v, RSR_F64, sizeof(double) * (size_t)rows, out, RSR_F64,
                                 sizeof(double) * (size_t)cols, RSR_VARIANT_RSRPP, NULL));
    for (int64_t c = 0; c < cols; ++c) {
      double ref = 0;
      for (int64_t r = 0; r < rows; ++r) ref += v[r] * (double)A[r * cols + c];
      if (ref != out[c]) {
        fprintf(stderr, "mismatch at column %lld: %f vs %f\n", (long long)c, out[c], ref);
        return 1;
      }
    }
  }
  rsr_host_session_destroy(sess);
  printf("c_example ok: %lld x %lld, k = %d, 3 session calls bit-exact\n", (long long)rows, (long long)cols, k);
  return 0;
}
