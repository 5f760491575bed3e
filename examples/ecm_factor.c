/* ecm_factor.c — plain C client of libecmgpu (include/ecmgpu.h): ECM stage 1 on the GPU for a
 * hexadecimal N, host buffers in and out (ECM_HOST_BUFFERS), no Python, no torch.
 *
 *   gcc -O2 -I include examples/ecm_factor.c -L paper_1310_3809_b200 -lecmgpu \
 *       -Wl,-rpath,$PWD/paper_1310_3809_b200 -o ecm_factor
 *   ./ecm_factor <hex N> [B1=2000] [curves=256] [seed=1]
 * Prints every proper factor found (checked by the library's gcd; status 1) and exits 0, or 2
 * when none is found, 1 on bad input.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ecmgpu.h"

static uint64_t splitmix(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* big-endian hex -> little-endian 32-bit limbs; returns bit length or -1 */
static int parse_hex(const char *h, uint32_t *w, int cap) {
  memset(w, 0, sizeof(uint32_t) * cap);
  if (h[0] == '0' && (h[1] == 'x' || h[1] == 'X')) h += 2;
  int n = (int)strlen(h), bit = 0;
  for (int i = n - 1; i >= 0; --i, bit += 4) {
    char c = h[i];
    int v = (c >= '0' && c <= '9') ? c - '0' : (c >= 'a' && c <= 'f') ? c - 'a' + 10 : (c >= 'A' && c <= 'F') ? c - 'A' + 10 : -1;
    if (v < 0 || bit / 32 >= cap) return -1;
    w[bit / 32] |= (uint32_t)v << (bit % 32);
  }
  int bl = 0;
  for (int i = cap - 1; i >= 0 && !bl; --i)
    if (w[i]) bl = 32 * i + 32 - __builtin_clz(w[i]);
  return bl;
}

static void print_hex(const uint32_t *w, int L) {
  int i = L - 1;
  while (i > 0 && !w[i]) --i;
  printf("0x%x", w[i]);
  for (--i; i >= 0; --i) printf("%08x", w[i]);
}

int main(int argc, char **argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s <hex N> [B1] [curves] [seed]\n", argv[0]);
    return 1;
  }
  uint32_t N[16];
  const int bl = parse_hex(argv[1], N, 16);
  const uint64_t B1 = argc > 2 ? strtoull(argv[2], 0, 10) : 2000;
  const size_t curves = argc > 3 ? strtoull(argv[3], 0, 10) : 256;
  uint64_t seed = argc > 4 ? strtoull(argv[4], 0, 10) : 1;
  int L = 0;
  static const int widths[] = {4, 6, 8, 12, 16};
  for (int j = 0; j < 5 && !L; ++j)
    if (bl > 0 && bl <= 32 * widths[j] - 2) L = widths[j];
  if (!L || curves == 0) {
    fprintf(stderr, "bad input\n");
    return 1;
  }
  uint64_t *sig = malloc(curves * sizeof(uint64_t));
  uint32_t *g = malloc(curves * L * sizeof(uint32_t));
  uint8_t *st = malloc(curves);
  for (size_t i = 0; i < curves; ++i) sig[i] = 6 + (splitmix(&seed) >> 2);
  ecm_status s = ecm_stage1_batch(N, L, B1, sig, curves, NULL, NULL, g, st, NULL,
                                  ECM_HOST_BUFFERS | ECM_NO_XAFF, NULL);
  if (s != ECM_OK) {
    fprintf(stderr, "ecm_stage1_batch: %s\n", ecm_strerror(s));
    return 1;
  }
  int found = 0;
  for (size_t i = 0; i < curves; ++i) {
    if (st[i] == ECM_CURVE_FACTOR || st[i] == ECM_CURVE_SETUP_FACTOR) {
      printf("factor ");
      print_hex(g + i * L, L);
      printf(" curve %zu sigma %llu\n", i, (unsigned long long)sig[i]);
      found = 1;
    }
  }
  if (!found) printf("no factor found (%zu curves, B1 = %llu)\n", curves, (unsigned long long)B1);
  printf("%s\n", ecm_version());
  free(sig);
  free(g);
  free(st);
  return found ? 0 : 2;
}
