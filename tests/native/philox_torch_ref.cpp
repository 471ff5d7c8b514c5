// Independent Philox4x32-10 reference for the oracle pin test: PyTorch's
// at::philox_engine (ATen/core/PhiloxRNGEngine.h), a third-party
// implementation shipped in this image. Reads "c0 c1 c2 c3 k0 k1" lines
// (decimal) on stdin and prints the four output words. The engine's counter
// is {offset lo, offset hi, subsequence lo, subsequence hi} and its key is
// the 64-bit seed split lo/hi.
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
#include <cstdint>

int main() {
  unsigned long long c0, c1, c2, c3, k0, k1;
  while (std::scanf("%llu %llu %llu %llu %llu %llu", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint64_t seed = (uint64_t)k0 | ((uint64_t)k1 << 32);
    uint64_t subseq = (uint64_t)c2 | ((uint64_t)c3 << 32);
    uint64_t offset = (uint64_t)c0 | ((uint64_t)c1 << 32);
    at::philox_engine e(seed, subseq, 0);
    e.set_offset(offset);
    uint32_t r0 = e(), r1 = e(), r2 = e(), r3 = e();
    std::printf("%u %u %u %u\n", r0, r1, r2, r3);
  }
  return 0;
}
