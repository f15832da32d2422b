#include "../../paper_2404_06452_b200/csrc/analyze.cu"
extern "C" void emu_analyze(const paam::Record* rec, uint32_t n, uint64_t comm, uint32_t flags, uint32_t n_bins,
                            uint64_t* wcrt, uint8_t* sched, int64_t* bins) {
  gridDim.x = 1;
  static unsigned int ticket;
  ticket = 0;
  emu::launch_block(0, paam::AW * 32, [&]() { paam::analyze_kernel(rec, n, comm, flags, n_bins, wcrt, sched, bins, nullptr, &ticket); });
}
