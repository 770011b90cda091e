// Host-side property check of the balanced persistent schedule (csrc/common.cuh Balance /
// balance_items / balance_item, mode 0 hand-off): over many (units, chunks, ranges, N) it checks
// that the ranges cover every (unit, chunk) exactly once, that every published head is consumed
// by the next range's tail of the same unit at the same token, and the no-stall ordering (a
// range runs at least as many chunks before its tail as the previous range spent on its head;
// the last, clipped range may wait for at most that head, which its predecessor runs first).
// Built and run by tests/test_schedule_native.py; exit code 0 = all properties hold.
#include <cstdio>
#include <vector>

#include "../../paper_2501_02573_b200/csrc/common.cuh"

using namespace linattn;

static int check(int units, int nc, int ranges, int chunk, int ragged, int ntiles) {
  const int N = nc * chunk - ragged;
  Balance P;
  P.on = 1;
  P.units = units;
  P.nc = nc;
  P.w = (int)(((long long)units * nc + ranges - 1) / ranges);
  P.ntiles = ntiles;
  P.chunk = chunk;
  P.tile = 128;
  if (P.w < nc) return 0;                              // mode 0 needs ranges of >= one unit
  std::vector<int> seen((size_t)units * nc, 0);
  std::vector<int> head_unit(ranges + 1, -1), head_hi(ranges + 1, -1), head_chunks(ranges + 1, 0);
  for (int t = 0; t <= ranges; ++t) {
    long long a = 0, b = 0;
    const int n = balance_items(P, t, a, b);
    int before_tail = 0;
    for (int k = 0; k < n; ++k) {
      const WorkItem w = balance_item(P, N, t, k, a, b);
      const int u = w.bh * ntiles + w.j0 / P.tile;
      if (w.lo % chunk != 0 || w.hi <= w.lo || w.hi > N || u < 0 || u >= units) {
        printf("bad item t=%d k=%d u=%d lo=%d hi=%d\n", t, k, u, w.lo, w.hi);
        return 1;
      }
      const int c0 = w.lo / chunk, c1 = (w.hi + chunk - 1) / chunk;
      for (int c = c0; c < c1; ++c) ++seen[(size_t)u * nc + c];
      if (w.out_slot >= 0) {                           // head: first item, publishes slot t
        if (k != 0 || w.out_slot != t || w.lo != 0) { printf("head order t=%d k=%d\n", t, k); return 1; }
        head_unit[t] = u;
        head_hi[t] = w.hi;
        head_chunks[t] = c1 - c0;
      }
      if (w.in_slot >= 0) {                            // tail: last item, consumes slot t-1
        if (k != n - 1 || w.in_slot != t - 1 || w.hi != N) { printf("tail order t=%d k=%d\n", t, k); return 1; }
        if (head_unit[t - 1] != u || head_hi[t - 1] != w.lo) {
          printf("hand-off mismatch t=%d: head (u=%d, hi=%d) tail (u=%d, lo=%d)\n", t, head_unit[t - 1],
                 head_hi[t - 1], u, w.lo);
          return 1;
        }
        // no stall: the previous range has finished its head (run first) by the time this range
        // reaches its tail -- except the last, clipped range, which waits at most that head
        const bool last = b == (long long)units * nc && b - a < P.w;
        if (!last && before_tail < head_chunks[t - 1]) { printf("stall t=%d\n", t); return 1; }
      }
      before_tail += c1 - c0;
    }
  }
  for (size_t i = 0; i < seen.size(); ++i)
    if (seen[i] != 1) { printf("chunk %zu covered %d times\n", i, seen[i]); return 1; }
  return 0;
}

int main() {
  int cases = 0;
  const int units_list[] = {1, 2, 5, 149, 150, 160, 256, 300, 512, 1000};
  const int nc_list[] = {1, 2, 3, 17, 64, 128, 257};
  const int ranges_list[] = {1, 2, 7, 74, 148, 296};
  for (int units : units_list)
    for (int nc : nc_list)
      for (int ranges : ranges_list)
        for (int chunk : {32, 64})
          for (int ragged : {0, 1, chunk - 1})
            for (int ntiles : {1, 2}) {
              if (units % ntiles != 0) continue;
              if (check(units, nc, ranges, chunk, ragged, ntiles)) {
                printf("FAILED units=%d nc=%d ranges=%d chunk=%d ragged=%d ntiles=%d\n", units, nc, ranges,
                       chunk, ragged, ntiles);
                return 1;
              }
              ++cases;
            }
  printf("balance schedule: %d configurations OK\n", cases);
  return 0;
}
