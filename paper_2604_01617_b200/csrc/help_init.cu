// help_init.cu — the random initial HELP graph on the device (reference graph.py:120-129):
//   rng = default_rng(seed)
//   ids = rng.integers(0, n - 1, size=(n, gamma)); ids += ids >= arange(n)[:, None]
// reproduced exactly and in parallel.  NumPy fills an int64 array with range < 2^32 by
// Lemire's method on 32-bit draws taken low half first from each 64-bit PCG64 output
// (buffered_bounded_lemire_uint32); whether a 32-bit draw is accepted depends on that draw
// alone, so the stream splits into independent blocks: thread t jumps the PCG64 state ahead
// by t * kInitBlock outputs (128-bit LCG advance), classifies its draws, and an exclusive
// scan of accepted counts places every value.  The host then redraws rows holding a repeated
// id with the same generator advanced past the consumed outputs (graph.py keeps that part).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "rng.cuh"
#include "sb_internal.h"

namespace sb {

constexpr int kInitBlock = 32;  // 64-bit PCG64 outputs per thread

// state after `delta` steps: s' = A^delta s + c (A^(delta-1) + ... + 1), by squaring
SB_HD sbrng::U128 pcg_advance_state(sbrng::U128 s, sbrng::U128 inc, uint64_t delta) {
  sbrng::U128 cur_mult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
  sbrng::U128 cur_plus = inc;
  sbrng::U128 acc_mult = {0, 1}, acc_plus = {0, 0};
  while (delta > 0) {
    if (delta & 1) {
      acc_mult = sbrng::mul128(acc_mult, cur_mult);
      acc_plus = sbrng::add128(sbrng::mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = sbrng::mul128(sbrng::add128(cur_mult, {0, 1}), cur_plus);
    cur_mult = sbrng::mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return sbrng::add128(sbrng::mul128(acc_mult, s), acc_plus);
}

SB_DEV uint64_t pcg_out(sbrng::U128 s) {
  uint64_t x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct InitArgs {
  sbrng::U128 s0, inc;      // generator state before the draw
  uint32_t excl;            // n - 1 (values in [0, n - 2])
  uint32_t thr;             // Lemire rejection threshold
  int64_t need;             // n * gamma accepted values
  int64_t threads;
  int g;
  int32_t* ids;             // n x gamma
  int64_t* cnt;             // per-thread accepted counts -> exclusive offsets
  int64_t* consumed;        // [0]: raw 32-bit draws consumed, [1]: the unused high half
};

SB_DEV bool lemire_accept(uint32_t x, uint32_t excl, uint32_t thr, uint32_t* val) {
  const uint64_t mm = (uint64_t)x * excl;
  *val = (uint32_t)(mm >> 32);
  return (uint32_t)mm >= thr;  // leftover >= excl implies >= thr
}

__global__ void init_count_kernel(InitArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.threads) return;
  sbrng::U128 s = pcg_advance_state(a.s0, a.inc, (uint64_t)t * kInitBlock);
  int c = 0;
  for (int i = 0; i < kInitBlock; ++i) {
    s = sbrng::add128(sbrng::mul128(s, {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull}), a.inc);
    const uint64_t v = pcg_out(s);
    uint32_t val;
    c += lemire_accept((uint32_t)v, a.excl, a.thr, &val);
    c += lemire_accept((uint32_t)(v >> 32), a.excl, a.thr, &val);
  }
  a.cnt[t] = c;
}

__global__ void init_write_kernel(InitArgs a, const int64_t* off) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.threads) return;
  int64_t pos = off[t];
  if (pos >= a.need) return;
  sbrng::U128 s = pcg_advance_state(a.s0, a.inc, (uint64_t)t * kInitBlock);
  for (int i = 0; i < kInitBlock && pos < a.need; ++i) {
    s = sbrng::add128(sbrng::mul128(s, {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull}), a.inc);
    const uint64_t v = pcg_out(s);
    for (int h = 0; h < 2 && pos < a.need; ++h) {
      uint32_t val;
      if (lemire_accept((uint32_t)(h ? v >> 32 : v), a.excl, a.thr, &val)) {
        const int64_t row = pos / a.g;
        a.ids[pos] = (int32_t)(val + (val >= (uint32_t)row ? 1u : 0u));
        if (pos == a.need - 1) {
          a.consumed[0] = ((int64_t)t * kInitBlock + i) * 2 + h + 1;
          a.consumed[1] = (int64_t)(uint32_t)(v >> 32);  // buffered by NumPy when h == 0
        }
        ++pos;
      }
    }
  }
}

// rows holding a repeated id (warp per row: bitonic sort of the row in shared memory)
__global__ void init_dup_rows_kernel(const int32_t* ids, int64_t n, int g, int gpad,
                                     int64_t* bad, unsigned long long* nbad) {
  extern __shared__ int32_t sh[];
  const int wpb = blockDim.x >> 5;
  int32_t* row = sh + warp_id() * gpad;
  const int64_t r = (int64_t)blockIdx.x * wpb + warp_id();
  if (r >= n) return;
  for (int t = lane_id(); t < gpad; t += 32) row[t] = t < g ? ids[r * g + t] : 0x7FFFFFFF;
  __syncwarp();
  for (int k = 2; k <= gpad; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane_id(); i < gpad; i += 32) {
        const int p = i ^ j;
        if (p > i) {
          const int32_t x = row[i], y = row[p];
          if ((x > y) == ((i & k) == 0)) { row[i] = y; row[p] = x; }
        }
      }
      __syncwarp();
    }
  bool dup = false;
  for (int t = lane_id() + 1; t < g; t += 32) dup = dup || row[t] == row[t - 1];
  if (__any_sync(0xFFFFFFFFu, dup) && lane_id() == 0) {
    const unsigned long long k = atomicAdd(nbad, 1ull);
    bad[k] = r;
  }
}

int launch_init_random_ids(uint64_t seed, int64_t n, int g, int32_t* ids, int64_t* scratch,
                           int64_t scratch_slots, int64_t* consumed, int64_t* bad,
                           unsigned long long* nbad, cudaStream_t st) {
  sbrng::Pcg64 gen;
  {
    uint32_t w[8];
    uint32_t ent[4];
    int ne = sbrng::int_words(seed, ent);
    // SeedSequence(entropy=seed).generate_state(8): one-integer entropy
    uint32_t pool[4];
    uint32_t hc = sbrng::kInitA;
    for (int i = 0; i < 4; ++i) pool[i] = sbrng::hashmix(i < ne ? ent[i] : 0u, &hc);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = sbrng::mix(pool[d], sbrng::hashmix(pool[s], &hc));
    for (int s = 4; s < ne; ++s)
      for (int d = 0; d < 4; ++d) pool[d] = sbrng::mix(pool[d], sbrng::hashmix(ent[s], &hc));
    uint32_t hb = sbrng::kInitB;
    for (int i = 0; i < 8; ++i) {
      uint32_t v = pool[i & 3];
      v ^= hb;
      hb *= sbrng::kMultB;
      v *= hb;
      v ^= v >> 16;
      w[i] = v;
    }
    sbrng::pcg_seed_words(&gen, w);
  }
  InitArgs a;
  a.s0 = gen.s;
  a.inc = gen.inc;
  const uint32_t r = (uint32_t)(n - 2);  // inclusive range of rng.integers(0, n - 1)
  a.excl = r + 1u;
  a.thr = (0xFFFFFFFFu - r) % a.excl;
  a.need = n * (int64_t)g;
  a.g = g;
  a.ids = ids;
  a.consumed = consumed;
  // raw draws: the values plus a generous margin for rejections (rate < excl / 2^32)
  const int64_t raw = a.need + a.need / 256 + 4096;
  a.threads = (raw / 2 + kInitBlock - 1) / kInitBlock;
  if (a.threads + 1 > scratch_slots) return (int)cudaErrorInvalidValue;
  a.cnt = scratch;
  int64_t* off = scratch + a.threads + 1;
  const unsigned blocks = (unsigned)((a.threads + 255) / 256);
  init_count_kernel<<<blocks, 256, 0, st>>>(a);
  int e = exclusive_scan(a.cnt, off, a.threads, scratch + 2 * (a.threads + 1), st);
  if (e) return e;
  cudaMemsetAsync(consumed, 0xFF, 2 * sizeof(int64_t), st);
  init_write_kernel<<<blocks, 256, 0, st>>>(a, off);
  const int gpad = next_pow2(g);
  cudaMemsetAsync(nbad, 0, sizeof(unsigned long long), st);
  init_dup_rows_kernel<<<(unsigned)((n + 7) / 8), 256, 8 * gpad * sizeof(int32_t), st>>>(
      ids, n, g, gpad, bad, nbad);
  return (int)cudaGetLastError();
}

int64_t init_random_ids_scratch_slots(int64_t n, int g) {
  const int64_t need = n * (int64_t)g;
  const int64_t raw = need + need / 256 + 4096;
  const int64_t threads = (raw / 2 + kInitBlock - 1) / kInitBlock;
  return 2 * (threads + 1) + scan_tmp_slots(threads);
}

}  // namespace sb
