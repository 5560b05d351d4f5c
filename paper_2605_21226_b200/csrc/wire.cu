// wire.cu — device-side checks of OCTO v1 records (unpack_keys padding
// rules, codec.hpp:440-462): every padding bit of the direction stream, the
// norm stream and (for dim % 8 != 0) the QJL sign bytes must be zero.
// One thread per record; records are read bytewise (rec_bytes is odd in
// general), so this is a cheap latency-bound pass used only on untrusted
// input.
#include "common.cuh"
#include "kernels.h"

namespace oqd {

__global__ void validate_records_kernel(OqCodecParams p, const uint8_t* __restrict__ recs,
                                        size_t n, int* bad) {
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    const uint8_t* r = recs + v * p.rec_bytes;
    int flags = 0;
    const uint32_t dbits = 2 * p.nt * p.b_dir, nbits = p.nt * p.b_nrm;
    if (dbits & 7) {
      const uint8_t last = r[4 + p.dir_bytes - 1];
      if (last >> (dbits & 7)) flags |= 1;
    }
    if (nbits & 7) {
      const uint8_t last = r[4 + p.dir_bytes + p.nrm_bytes - 1];
      if (last >> (nbits & 7)) flags |= 2;
    }
    if (p.qjl && (p.dim & 7)) {
      const uint8_t last = r[p.rec_bytes - 1];
      if (last >> (p.dim & 7)) flags |= 4;
    }
    if (flags) atomicOr(bad, flags);
  }
}

cudaError_t launch_validate_records(const OqCodecParams& p, const uint8_t* recs, size_t n,
                                    int* bad, cudaStream_t st, int num_sms) {
  size_t blocks = (n + 255) / 256;
  if (blocks > (size_t)num_sms * 8) blocks = (size_t)num_sms * 8;
  validate_records_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, recs, n, bad);
  return cudaGetLastError();
}

}  // namespace oqd
