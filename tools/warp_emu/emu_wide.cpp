#include "../../paper_2404_06452_b200/csrc/wide.cu"
extern "C" void emu_wide(const paam_batch* b, const uint32_t* list, const uint32_t* count, int32_t* status, uint64_t* wcrt,
                         uint8_t* sched, int64_t* bins, int32_t* fail, int c32) {
  gridDim.x = 1;
  blockDim.x = 32;
  emu::launch_block(0, 32, [&]() {
    if (c32) paam::wide_kernel<true>(*b, list, count, status, wcrt, sched, bins, fail);
    else paam::wide_kernel<false>(*b, list, count, status, wcrt, sched, bins, fail);
  });
}
