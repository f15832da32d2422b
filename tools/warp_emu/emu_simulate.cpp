#include "../../paper_2404_06452_b200/csrc/simulate.cu"
extern "C" void emu_simulate(const paam_batch* b, const paam::Record* rec, uint32_t n, uint64_t horizon, uint64_t seed,
                             uint64_t first, uint32_t simf, const paam_sim_out* out) {
  gridDim.x = 1;
  static unsigned int tickets[3];
  static uint32_t big[1 << 16];
  tickets[0] = tickets[1] = tickets[2] = 0;
  emu::launch_block(0, paam::SW * 32, [&]() {
    paam::simulate_kernel<16>(*b, rec, n, horizon, seed, first, simf, *out, &tickets[0], nullptr, nullptr, big, &tickets[2]);
  });
  emu::launch_block(0, paam::SW * 32, [&]() {
    paam::simulate_kernel<32>(*b, rec, n, horizon, seed, first, simf, *out, &tickets[1], big, &tickets[2], nullptr, nullptr);
  });
}
extern "C" unsigned emu_record_bytes() { return sizeof(paam::Record); }
