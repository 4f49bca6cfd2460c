// Register-pass plan of the tiled NTT, shared by the kernels (ntt.cu) and the
// host-side table builder (context.cu).
#pragma once

#ifndef FHE_NTT_MAXE
#define FHE_NTT_MAXE 5
#endif
// pass radix limit of the whole-row tiles (ntt_tiles.cuh RowsTile)
#ifndef FHE_ROW_MAXE
#define FHE_ROW_MAXE FHE_NTT_MAXE
#endif

// A local transform of 2^log_s points runs npass register passes of radix
// 2^pass_e; pass p starts at local stage pass_r0.
// (maxe: largest pass radix exponent; tiles may lower it, see tile_maxe)
constexpr int npass(int log_s, int maxe = FHE_NTT_MAXE) { return (log_s + maxe - 1) / maxe; }
constexpr int pass_e(int log_s, int p, int maxe = FHE_NTT_MAXE) {
  return log_s / npass(log_s, maxe) + (p < log_s % npass(log_s, maxe) ? 1 : 0);
}
constexpr int pass_r0(int log_s, int p, int maxe = FHE_NTT_MAXE) {
  int r = 0;
  for (int i = 0; i < p; ++i) r += pass_e(log_s, i, maxe);
  return r;
}

// Four-step split N = N1 * N2 used for log N >= 13 (column stages first).
constexpr int split_log_n1(int log_n) { return log_n >= 16 ? 8 : (log_n >= 14 ? 7 : 6); }

// Staged twiddle order.  Stage s of a local transform reads 2^s twiddles
// (per chunk); they are kept at (1 << s) + perm(s, j).  Stages of the last
// register pass (s >= p_last) hold pair j = (g << rr) | blk (rr = s - p_last,
// g the thread's group) at (blk << p_last) | g, so the groups of a warp read
// consecutive pairs.
constexpr int staged_perm(int log_s, int s, int j, int maxe = FHE_NTT_MAXE) {
  const int pl = pass_r0(log_s, npass(log_s, maxe) - 1, maxe);
  if (s < pl) return j;
  const int rr = s - pl;
  return ((j & ((1 << rr) - 1)) << pl) | (j >> rr);
}
