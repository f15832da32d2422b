#include "../../paper_2404_06452_b200/csrc/simulate.cu"
extern "C" void emu_simulate(const paam_batch* b, const paam::Record* rec, uint32_t n, uint64_t horizon, uint64_t seed,
                             uint64_t first, uint32_t simf, const paam_sim_out* out) {
  gridDim.x = 1;
  static unsigned int ticket;
  static uint4 evbuf[paam::SW * paam::EVCAP];
  ticket = 0;
  emu::launch_block(0, paam::SW * 32, [&]() {
    paam::simulate_kernel(*b, rec, n, horizon, seed, first, simf, *out, &ticket, evbuf);
  });
}
extern "C" unsigned emu_record_bytes() { return sizeof(paam::Record); }
