// Pin helper: runs the CUDA toolkit's own Philox4x32-10 (curand_philox4x32_x.h, host branch of
// mulhilo32) on the CPU and prints outputs for counters read from stdin:
//   input lines:  c0 c1 c2 c3 k0 k1   (decimal u32)
//   output lines: x0 x1 x2 x3
// It is an independent implementation used only to pin oracle/rid_oracle.c (tests/).
#include <cstdio>
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%u %u %u %u %u %u", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = {c0, c1, c2, c3};
    uint2 k = {k0, k1};
    uint4 r = curand_Philox4x32_10(c, k);
    std::printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
  return 0;
}
