// simulate.cu -- §8(a) steps 7-8 (placeholder until the DES kernel lands).
#include "common.cuh"
using namespace paam;
extern "C" int paam_simulate(const paam_sets* sets, uint32_t n, uint64_t horizon, uint64_t seed, uint64_t* out_resp,
                             uint64_t* out_digest, const uint64_t* bound, int64_t* out_violations,
                             paam_stream_t stream) {
  return fail(PAAM_EINVAL, "paam_simulate: not implemented yet");
}
