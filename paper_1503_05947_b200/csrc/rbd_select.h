// rbd_select.h — the winner rule of the multi-GPU record exchange, shared by
// the device kernels (rbd_persistent.cuh: k_shard_pack / k_shard_select) and the
// host (rbd_shard_pick in the C ABI, driven by the gloo world-2 test).
//
// Every rank contributes a 16-byte record {best residual, GLOBAL column index}
// of its shard (index -1: no candidate). The winner is the largest residual,
// ties to the smallest global index — the reference's strict '>' scan from
// j = 0 (workspace.cpp:107-113) survives any column sharding, because every
// rank's record is already its shard's first maximum.
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define RBD_HD __host__ __device__ __forceinline__
#else
#define RBD_HD inline
#endif

namespace rbdsel {

RBD_HD long long index_bits(double v) {
  long long j;
  memcpy(&j, &v, sizeof(j));
  return j;
}

RBD_HD double index_as_double(long long j) {
  double v;
  memcpy(&v, &j, sizeof(v));
  return v;
}

// recs[r * stride + 0] = value, recs[r * stride + 1] = index bits. Returns the
// owner rank (or -1 when no rank has a candidate) and the winning record.
RBD_HD int pick(const double* recs, int nranks, int stride, double* best_v, long long* best_j) {
  double bv = -1.0;
  long long bj = 0x7fffffffffffffffLL;
  int br = -1;
  for (int r = 0; r < nranks; ++r) {
    const double v = recs[(long long)r * stride];
    const long long j = index_bits(recs[(long long)r * stride + 1]);
    if (j < 0) continue;
    if (v > bv || (v == bv && j < bj)) {
      bv = v;
      bj = j;
      br = r;
    }
  }
  *best_v = bv;
  *best_j = bj;
  return br;
}

}  // namespace rbdsel
