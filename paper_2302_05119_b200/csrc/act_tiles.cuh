// Tiles of the ACTIVE blocks split evenly over a persistent grid (shared by
// the ALS streaming kernels: xslab5.cu, xoz.cu).
#pragma once

namespace cb {

// The CTA's share of the tiles of the ACTIVE blocks (ALS: converged blocks
// drop out): tiles are numbered over active blocks only and split evenly
// over the grid, so the last sweeps (few blocks left) still use every SM.
// Every role of a CTA walks the same sequence.
struct ActTiles {
  int s;            // current block
  long long t;      // tile within the block
  long long left;   // tiles left for this CTA
};

template <typename NT>
__device__ __forceinline__ ActTiles act_tiles_begin(const int* active, int S, NT ntiles) {
  long long A = 0;
  for (int s = 0; s < S; ++s)
    if (!active || active[s]) A += ntiles(s);
  const long long G = gridDim.x;
  const long long q0 = (long long)blockIdx.x * A / G, q1 = (long long)(blockIdx.x + 1) * A / G;
  ActTiles it{0, 0, q1 - q0};
  long long off = 0;
  for (; it.s < S; ++it.s) {
    if (active && !active[it.s]) continue;
    const long long n = ntiles(it.s);
    if (q0 < off + n) break;
    off += n;
  }
  it.t = q0 - off;
  return it;
}

template <typename NT>
__device__ __forceinline__ void act_tiles_next(ActTiles& it, const int* active, int S, NT ntiles) {
  --it.left;
  if (++it.t >= ntiles(it.s)) {
    it.t = 0;
    do { ++it.s; } while (it.s < S && active && !active[it.s]);
  }
}

}  // namespace cb
