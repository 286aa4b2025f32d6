/* Test driver (not part of the oracle): runs the oracle's C entry points on small
 * seeded inputs under -fsanitize=address,undefined (tests/test_oracle_pins.py) and checks
 * them against each other -- Algorithm 4 (both senses) against minimax / widest
 * Floyd-Warshall and brute force, the row windows against the full matrix, the points
 * path against Algorithm 4 on its own R1 weights.  Prints "ok" and exits 0 on success. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t writes, traversed;
  double t_mst, t_sort, t_copy;
} oracle_stats;

int oracle_appd_weights(const float* W, int64_t n, int sense, float* M, oracle_stats* st);
int oracle_appd_weights_rows(const float* W, int64_t n, int64_t r0, int64_t R, float* M, oracle_stats* st);
int oracle_appd_points(const float* X, int64_t n, int64_t d, float* M, oracle_stats* st);
int oracle_appd_points_rows(const float* X, int64_t n, int64_t d, int64_t r0, int64_t R, float* M, oracle_stats* st);
int oracle_appd_points_metric(const float* X, int64_t n, int64_t d, int metric, float* M, oracle_stats* st);
void oracle_points_weights(const float* X, int64_t n, int64_t d, int64_t r0, int64_t R, float* Wblk);
int oracle_floyd(const float* W, int64_t n, int sense, float* M);
int oracle_brute(const float* W, int64_t n, int sense, float* M);
int oracle_mst_path(const float* W, int64_t n, float* M);

static uint64_t state = 12345;
static uint64_t next(void) {
  uint64_t z = (state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static int same(const float* a, const float* b, int64_t cnt) { return memcmp(a, b, sizeof(float) * cnt) == 0; }

static void weights(float* W, int64_t n, int levels) {
  for (int64_t i = 0; i < n; i++) {
    W[i * n + i] = 0.0f;
    for (int64_t j = i + 1; j < n; j++) {
      float w = levels ? (float)(1 + next() % (uint64_t)levels) : (float)((next() >> 40) * 0x1p-24) + 0x1p-25f;
      W[i * n + j] = W[j * n + i] = w;
    }
  }
}

int main(void) {
  oracle_stats st;
  for (int t = 0; t < 60; t++) {
    const int64_t n = 1 + (int64_t)(next() % 40);
    const int levels = t % 3 == 0 ? 0 : (t % 3 == 1 ? 3 : 255);
    float* W = malloc(sizeof(float) * n * n);
    float* A = malloc(sizeof(float) * n * n);
    float* B = malloc(sizeof(float) * n * n);
    weights(W, n, levels);
    for (int sense = 1; sense >= -1; sense -= 2) {
      if (oracle_appd_weights(W, n, sense, A, &st) || oracle_floyd(W, n, sense, B) || !same(A, B, n * n)) {
        printf("Algorithm 4 != Floyd (n %lld sense %d)\n", (long long)n, sense);
        return 1;
      }
      if (n <= 7 && (oracle_brute(W, n, sense, B) || !same(A, B, n * n))) {
        printf("Algorithm 4 != brute force (n %lld)\n", (long long)n);
        return 1;
      }
    }
    oracle_appd_weights(W, n, 1, A, &st);
    if (oracle_mst_path(W, n, B) || !same(A, B, n * n)) {
      printf("Algorithm 4 != MST path (n %lld)\n", (long long)n);
      return 1;
    }
    const int64_t r0 = n / 3, R = n - n / 3;
    if (oracle_appd_weights_rows(W, n, r0, R, B, &st) || !same(A + r0 * n, B, R * n)) {
      printf("row window != full (n %lld)\n", (long long)n);
      return 1;
    }
    free(W);
    free(A);
    free(B);
  }
  for (int t = 0; t < 20; t++) {
    const int64_t n = 1 + (int64_t)(next() % 30), d = 1 + (int64_t)(next() % 6);
    float* X = malloc(sizeof(float) * n * d);
    float* W = malloc(sizeof(float) * n * n);
    float* A = malloc(sizeof(float) * n * n);
    float* B = malloc(sizeof(float) * n * n);
    for (int64_t e = 0; e < n * d; e++) X[e] = (float)((next() >> 40) * 0x1p-24);
    oracle_points_weights(X, n, d, 0, n, W);
    if (oracle_appd_points(X, n, d, A, &st) || oracle_appd_weights(W, n, 1, B, &st) || !same(A, B, n * n)) {
      printf("points != weights on R1 (n %lld)\n", (long long)n);
      return 1;
    }
    if (oracle_appd_points_rows(X, n, d, 1 < n ? 1 : 0, n - (1 < n ? 1 : 0), B, &st) ||
        !same(A + (1 < n ? 1 : 0) * n, B, (n - (1 < n ? 1 : 0)) * n)) {
      printf("points row window != full (n %lld)\n", (long long)n);
      return 1;
    }
    for (int metric = 1; metric <= 2; metric++)
      if (oracle_appd_points_metric(X, n, d, metric, A, &st)) {
        printf("metric %d failed\n", metric);
        return 1;
      }
    free(X);
    free(W);
    free(A);
    free(B);
  }
  printf("ok\n");
  return 0;
}
