#include "../../paper_2404_06452_b200/csrc/fused.cu"
// c32: b carries a compact batch (paam_batch32 pointers, as paam_pack_analyze32 builds it)
extern "C" void emu_fused(const paam_batch* b, uint32_t* wide_list, uint32_t* wide_count, int32_t* status, uint64_t* wcrt,
                          uint8_t* sched, int64_t* bins, int c32) {
  gridDim.x = 1;
  emu::launch_block(0, paam::FW * 32, [&]() {
    if (c32) paam::fused_kernel<true>(*b, wide_list, wide_count, wide_count + 1, status, wcrt, sched, bins);
    else paam::fused_kernel<false>(*b, wide_list, wide_count, wide_count + 1, status, wcrt, sched, bins);
  });
}
