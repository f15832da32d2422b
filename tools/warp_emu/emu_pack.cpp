#include "../../paper_2404_06452_b200/csrc/pack.cu"
extern "C" void emu_pack(const paam_batch* b, paam::Record* rec, int32_t* status, uint32_t* wide_list, uint32_t* wide_count) {
  gridDim.x = 1;
  emu::launch_block(0, paam::WARPS * 32, [&]() { paam::pack_kernel(*b, rec, status, wide_list, wide_count, wide_count + 1); });
}
