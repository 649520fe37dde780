// Host check of the tag classifier (csrc/common.cuh: classify16 / classify16b)
// against the per-byte definition (R2: bytes other than 1, 2, 3 are leaves).
#include "common.cuh"
#include <cstdio>
#include <random>
#include <cstring>
using namespace tb;
static void ref(const uint8_t* b, uint32_t& o, uint32_t& c, uint32_t& bl) {
  o = c = bl = 0;
  for (int i = 0; i < 16; i++) {
    if (b[i] == 1 || b[i] == 2) o |= 1u << i;
    if (b[i] == 3) c |= 1u << i;
    if (b[i] == 2) bl |= 1u << i;
  }
}
int main() {
  std::mt19937 g(1);
  long bad = 0, n = 0;
  uint8_t b[16];
  for (int it = 0; it < 4000000; it++) {
    for (int i = 0; i < 16; i++) {
      uint32_t r = g();
      b[i] = (r & 3) == 0 ? (uint8_t)(r >> 8) : (uint8_t)((r >> 8) & 3);
    }
    if (it < 256 * 16) { for (int i = 0; i < 16; i++) b[i] = g() & 3; b[it / 256] = it & 255; }
    uint4 w; memcpy(&w, b, 16);
    uint32_t o, c, bl, o2, c2, bl2, o3, c3;
    ref(b, o, c, bl);
    classify16b(w, o2, c2, bl2);
    classify16(w, o3, c3);
    n++;
    if (o != o2 || c != c2 || bl != bl2 || o != o3 || c != c3) { if (bad++ < 5) printf("mismatch it %d\n", it); }
  }
  printf("%ld cases, %ld bad\n", n, bad);
  return bad != 0;
}
