/*
 * oracle_common.h — index helpers shared by the two C files of the CPU oracle (oracle/ only).
 *
 * TEST INFRASTRUCTURE ONLY (see prony_oracle.c). Not included by, and not including, anything under
 * paper_2012_11430_b200/.
 *
 * Conventions (readings R1, R2):
 *   grid : f~(k) for k in the box {-n..n+1}^d, L = 2n+2 values per axis, lexicographic
 *          with the LAST coordinate fastest: box index of k = sum_i (k_i+n) L^(d-1-i).
 *   I_n  : {0..n}^d, same lexicographic order; row r <-> multi-index digits of r base n+1.
 */
#ifndef PRONY_ORACLE_COMMON_H
#define PRONY_ORACLE_COMMON_H

#include <complex.h>
#include <stdint.h>

typedef double complex cplx;

#define ORACLE_MAX_D 16

/* multi-index of element r of I_n (digits base n+1, last coordinate fastest) */
static inline void index_of(int d, int n, int64_t r, int* k) {
  for (int i = d - 1; i >= 0; --i) {
    k[i] = (int)(r % (n + 1));
    r /= (n + 1);
  }
}

/* box index of the integer point v in {-n..n+1}^d; -1 if outside the box */
static inline int64_t box_index(int d, int n, const int* v) {
  const int64_t L = 2 * (int64_t)n + 2;
  int64_t idx = 0;
  for (int i = 0; i < d; ++i) {
    int b = v[i] + n;
    if (b < 0 || b >= L) return -1;
    idx = idx * L + b;
  }
  return idx;
}

static inline int64_t count_N(int d, int n) {
  int64_t N = 1;
  for (int i = 0; i < d; ++i) N *= (n + 1);
  return N;
}

#endif
