// Independent Philox4x32-10 reference for the oracle pin: NVIDIA cuRAND's
// curand_Philox4x32_10 (curand_philox4x32_x.h), compiled for the HOST.
// Reads lines "c0 c1 c2 c3 k0 k1" (decimal) from stdin, prints "x0 x1 x2 x3".
#include <cstdio>
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main() {
  unsigned a[6];
  while (std::scanf("%u %u %u %u %u %u", &a[0], &a[1], &a[2], &a[3], &a[4], &a[5]) == 6) {
    uint4 c = {a[0], a[1], a[2], a[3]};
    uint2 k = {a[4], a[5]};
    uint4 r = curand_Philox4x32_10(c, k);
    std::printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
  return 0;
}
