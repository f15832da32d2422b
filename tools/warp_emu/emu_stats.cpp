#define PAAM_EMU_STATS 1
#include "../../paper_2404_06452_b200/csrc/fused.cu"
extern "C" void emu_fused_stats(const paam_batch* b, uint32_t* wide_list, uint32_t* wide_count, uint64_t* stats) {
  gridDim.x = 1;
  for (int i = 0; i < 8; i++) paam::emu_stats[i] = 0;
  emu::launch_block(0, paam::FW * 32, [&]() { paam::fused_kernel<false>(*b, wide_list, wide_count, wide_count + 1, nullptr, nullptr, nullptr, nullptr); });
  for (int i = 0; i < 8; i++) stats[i] = paam::emu_stats[i];
}
