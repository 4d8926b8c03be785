// Host-only check of the tcgen05 engine's K-split choice (mma_launch.cuh) on the
// bench shapes; prints "name splits" per line (tests/test_split_model.py).
#include <cstdio>
#include "../../paper_2510_03631_b200/csrc/mma_launch.cuh"
using qpir::mma_choose_splits;
int main() {
  const uint32_t sms = 148;
  // tiles, K-blocks, min splits, output bytes, wave bytes (2 panels x 16 KB x 148), hbm-bound
  const double wb = 2.0 * 16384.0 * sms;
  std::printf("c2_b4 %u\n", mma_choose_splits(480, 64, sms, 0, 1, 4.0 * 122880 * 4, wb, true));
  std::printf("c2_b64 %u\n", mma_choose_splits(480, 64, sms, 0, 1, 64.0 * 122880 * 4, wb, false));
  std::printf("c4_b64 %u\n", mma_choose_splits(480, 512, sms, 0, 1, 64.0 * 122880 * 4, wb, false));
  std::printf("c4_b256 %u\n", mma_choose_splits(1920, 512, sms, 0, 1, 256.0 * 122880 * 4, wb, false));
  std::printf("c5 %u\n", mma_choose_splits(960, 2048, sms, 0, 1, 15360.0 * 1024 * 4, wb, false));
  std::printf("ftr %u\n", mma_choose_splits(12, 2560, sms, 0, 5, 128.0 * 3072 * 8, wb, false));
  std::printf("forced %u\n", mma_choose_splits(12, 2560, sms, 7, 5, 0.0, wb, false));
  std::printf("forced_min %u\n", mma_choose_splits(12, 2560, sms, 2, 5, 0.0, wb, false));
  return 0;
}
