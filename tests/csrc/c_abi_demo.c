/* c_abi_demo.c -- a plain-C (C11) consumer of include/mpfk.h: proves the
 * header is valid C and that libmpfk links without C++ on the caller side.
 * Run without a GPU it must report MPFK_ENODEV for compute calls (no CPU
 * fallback); with a GPU it multiplies two small DD matrices. */
#include <stdio.h>
#include <string.h>

#include "mpfk.h"

int main(void) {
  double a[2 * 2 * 4], b[2 * 2 * 4], c[2 * 2 * 4];
  memset(a, 0, sizeof a);
  memset(b, 0, sizeof b);
  memset(c, 0, sizeof c);
  /* A = B = I (2x2, stride 4, 2 planes) */
  a[0] = a[5] = b[0] = b[5] = 1.0;
  mpfk_mat A = {a, 2, 2, 4, 0}, B = {b, 2, 2, 4, 0}, C = {c, 2, 2, 4, 0};
  printf("abi %d devices %d\n", mpfk_abi_version(), mpfk_device_count());
  mpfk_mat bad = {c, 3, 2, 4, 0};
  int rc = mpfk_matmul_block_into(2, &bad, &A, &B, 32, MPFK_NORMAL);
  printf("shape check rc=%d msg=%s\n", rc, mpfk_last_error());
  if (rc != MPFK_EINVAL) return 1;
  rc = mpfk_matmul_block_parallel_into(2, &C, &A, &B, 32, MPFK_SIMD_LOADSTORE, 1);
  if (mpfk_device_count() == 0) {
    printf("no device rc=%d msg=%s\n", rc, mpfk_last_error());
    return rc == MPFK_ENODEV ? 0 : 1;
  }
  printf("gemm rc=%d c00=%g c11=%g c01=%g\n", rc, c[0], c[5], c[1]);
  return (rc == MPFK_OK && c[0] == 1.0 && c[5] == 1.0 && c[1] == 0.0) ? 0 : 1;
}
