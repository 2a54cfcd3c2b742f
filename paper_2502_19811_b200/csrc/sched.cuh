// Unit schedule of the persistent layer kernel: which (layer, pair, n-block,
// half, K slice) the g-th claim of a launch runs.  Host+device so the
// sequence properties (coverage, H-group and fold ordering) are tested on the
// CPU (tests/sched_harness.cu).
#pragma once

#include <cstdint>

#include "layers.cuh"

#define COMET_HD __host__ __device__ __forceinline__

namespace comet {

constexpr uint32_t kHalfN = kBlockN / 2;  // 256 columns per UMMA / accumulator

struct Unit {
  int layer, pair, nb;
  int half;  // -1: full 512-column unit; 0/1: one 256-column half
  int ks;    // K slice (split-K): k-blocks [kb0, kb1) of S slices
  int kb0, kb1;  // contraction k-blocks of this unit (whole K or one slice)
  int np;        // slices of this output tile (1: no fp32 partials)
};

// Uneven two-slice tail of layer1 (STREAMK): when layer1 has fewer output
// tiles U than pairs but more than half as many (one partial round, e.g.
// Mixtral EP=8 M=8192: 64 tiles of K = 14336 on 74 pairs, 10 pairs idle for
// a whole ~150 us unit), every tile is cut into a head [0, c) and a tail
// [c, KB).  The U heads are claimed first (U pairs in lockstep over the same
// k-blocks, as whole units would be: the weight and H blocks stay shared in
// L2); the idle pairs claim the tails (again in lockstep, consecutive tiles)
// and the head pairs take the rest when they finish.  c balances the two:
// U * (KB - c + o) = (pairs - U) * c, o = a tail's fixed cost (TMEM drain +
// fp32 partial) in k-blocks.  The last slice to land reduces head + tail in
// slice order (deterministic).  Contiguous stream-K ranges over the tiles'
// concatenated k-blocks were tried first: every pair at a different k offset
// lost the L2 reuse and ran HBM-bound (MX EP=8 0.41 -> 0.51 ms).  Heads
// before tails is not the per-n-block ascending order fold chains need, so
// shapes with fold chains keep whole units.
constexpr int kTailCostKb = 6;

// A layer's unit sequence: units [0, full) are full 512-column units; unit
// full + v is half (v & 1) of full unit full + v/2.  Layer0 alone cuts a
// mostly idle last round into halves (the tail takes half a unit time); layer1
// splits its last `split_units` units (the end of the launch in modes 1/2).
struct Sched {
  int full;   // full units before the split tail
  int total;  // units in the sequence (full + halves)
  int S;      // K slices per output tile (split-K; 1 = off)
  int c;      // S == 2 uneven tail split: head k-blocks (0 = even slices, consecutive per tile)
  int c_late;   // head k-blocks of tiles whose pair's H rows complete late (pair >= late_lo)
  int late_lo;
};
COMET_HD Sched make_sched(int U, int n_split, int S = 1) {
  n_split = S > 1 ? 0 : max(0, min(U, n_split));
  return {U * S - n_split, U * S + n_split, S, 0, 0, 1 << 30};
}
// Split-K when a layer has too few output tiles to fill the pairs (small M
// per rank, e.g. Mixtral EP=8 at 1K tokens: 8 layer1 tiles of K = 14336 on
// 74 pairs): S slices of >= 4 k-blocks, S * tiles <= pairs, S <= 8.
COMET_HD int ksplit_for(const LayerArgs& p, int P, int n_pairs) {
  if (!p.ksplit_max || P == 0) return 1;
  const int tiles = P * p.n_blocks;
  return max(1, min(min(p.ksplit_max, p.k_blocks / 4), n_pairs / tiles));
}
COMET_HD int layer0_split(int U, int n_pairs) {
  const int rem = U % n_pairs;
  return (rem > 0 && 2 * rem <= n_pairs) ? rem : 0;
}

// Unit u -> (pair, n-block), L2-aware rasters.
//  layer0: groups of G pairs; inside a group n-block middle, pair inner (the
//          group's A rows stay in L2 across all n-blocks; each weight block is
//          read once per group).
//  layer1: waves of W n-blocks (the reference's column waves, resolver.py:
//          273-296, at wave granularity: a wave's reduce chunks complete
//          together); inside a wave, groups of G2 pairs, n-block middle,
//          pair inner.
//  raster 2 (layer1 inside the fused launch): groups of G2 pairs outer (the
//          layer0 groups, so a group's layer1 units become ready together),
//          then waves of G n-blocks, n-block, pair inner.  For a fixed
//          n-block pairs still ascend, which the fused combine's fold needs.
COMET_HD Unit decode_unit(int u, int layer, int raster, int P, int NB, int G, int G2) {
  Unit r;
  r.layer = layer;
  if (raster == 0) {
    const int per_group = G * NB;
    const int g = u / per_group;
    const int base = g * G;
    const int ge = min(G, P - base);
    const int rem = u - g * per_group;
    r.nb = rem / ge;
    r.pair = base + rem % ge;
  } else if (raster == 1) {
    const int per_wave = P * G;
    const int w = u / per_wave;
    const int nb0 = w * G;
    const int we = min(G, NB - nb0);
    const int rem = u - w * per_wave;
    const int per_group = G2 * we;
    const int g = rem / per_group;
    const int base = g * G2;
    const int ge = min(G2, P - base);
    const int rem2 = rem - g * per_group;
    r.nb = nb0 + rem2 / ge;
    r.pair = base + rem2 % ge;
  } else {
    const int per_group = G2 * NB;
    const int g = u / per_group;
    const int base = g * G2;
    const int ge = min(G2, P - base);
    const int rem = u - g * per_group;
    const int per_wave = ge * G;
    const int w = rem / per_wave;
    const int nb0 = w * G;
    const int rem2 = rem - w * per_wave;
    r.nb = nb0 + rem2 / ge;
    r.pair = base + rem2 % ge;
  }
  return r;
}

// The last n-block of a layer holds <= 256 real columns.
COMET_HD bool narrow_block(const LayerArgs& p, int nb) {
  const int cols = p.out_ld - nb * static_cast<int>(kBlockN);
  return cols > 0 && cols <= static_cast<int>(kHalfN);
}
// 256-column halves a 128-row tile collects over all n-blocks of a layer.
COMET_HD uint32_t tile_halves(const LayerArgs& p) {
  return 2u * static_cast<uint32_t>(p.n_blocks) - (narrow_block(p, p.n_blocks - 1) ? 1u : 0u);
}

// Fused-combine fold chains: the epilogue of a token's last hosted row waits
// for its earlier hosted rows (same n-block, earlier pairs).  Those waits
// need, per n-block, pairs claimed in ascending order with every slice of a
// tile claimed before any slice of a later tile (else a pair blocked in a
// fold wait may hold the claim its predecessor tile is waiting for).
COMET_HD bool fold_chains(const LayerArgs& p) {
  return p.fuse_combine && p.experts_per_group > 1 && p.topk > 1;
}

COMET_HD int seq_total(const KernelArgs& f, int P, int n_pairs, Sched& s0, Sched& s1) {
  s0 = make_sched(0, 0);
  s1 = make_sched(0, 0);
  if (f.mode != 1) {
    const int U0 = P * f.l[0].n_blocks;
    s0 = make_sched(U0, f.l[0].split_tail ? layer0_split(U0, n_pairs) : 0, ksplit_for(f.l[0], P, n_pairs));
  }
  if (f.mode != 0) {
    const int U1 = P * f.l[1].n_blocks;
    // split_units < 0: automatic -- a layer1 of 1-4 rounds ends its last 16
    // units in halves (the partial last round balances better), else none
    const int split1 = f.l[1].split_units >= 0 ? f.l[1].split_units
                       : (U1 > n_pairs && U1 < 4 * n_pairs) ? 16 : 0;
    s1 = make_sched(U1, split1, ksplit_for(f.l[1], P, n_pairs));
    if (f.l[1].streamk && f.interleave == 0 && s1.S == 1 && 2 * U1 > n_pairs && U1 + 2 <= n_pairs &&
        !fold_chains(f.l[1])) {
      const int KB = f.l[1].k_blocks;
      // Fused launch: layer0's leftover units (U0 mod pairs; run as halves
      // when they are few) complete their pairs' H rows ~delta k-blocks after
      // the others -- those pairs are the last of layer0's last group (raster
      // 0: n-block major, pair inner).  Their heads are shortened by delta and
      // the work moves to the tails.
      int late_lo = 1 << 30, L = 0, delta = 0;
      if (f.mode == 2 && s0.S == 1) {
        const int U0 = s0.full + (s0.total - s0.full) / 2;
        const int rem0 = U0 % n_pairs;
        if (rem0 > 0 && f.l[0].raster == 0) {
          const int G = max(1, f.l[0].order_group);
          const int ge = P - ((P - 1) / G) * G;
          late_lo = P - min(rem0, ge);
          L = (P - late_lo) * f.l[1].n_blocks;
          // a 256-column half runs ~1.35x slower per FLOP: ~0.67 unit
          delta = s0.total > s0.full ? (f.l[0].k_blocks * 27) / 40 : f.l[0].k_blocks;
        }
      }
      const int c = min(KB - 4, max(KB / 2, (U1 * (KB + kTailCostKb) + L * delta + n_pairs - 1) / n_pairs));
      const int c_late = c - delta;
      if (c > 0 && c < KB) s1 = {2 * U1, 2 * U1, 2, c, c_late >= KB / 4 ? c_late : c, late_lo};
    }
  }
  return s0.total + s1.total;
}

// Claimed sequence index -> (layer, pair, n-block, half).
COMET_HD Unit unit_at(const KernelArgs& f, int g, int P, const Sched& s0, const Sched& s1) {
  if (f.interleave > 0) {
    // Interleaved fused sequence (layer1 pairs in the layer0 pair order, both
    // in groups of G pairs, no split tails / split-K): layer0 group k, then
    // layer1 group k - L.  Layer1 work becomes claimable while layer0 still
    // waits for its input (zero-copy forward: PCIe-paced dispatch), and its
    // H rows are L groups old when claimed.  A layer1 unit's fold
    // predecessors (earlier experts' rows) sit in earlier layer1 groups.
    const int G = f.l[0].order_group, L = f.interleave;
    const int NB0 = f.l[0].n_blocks, NB1 = f.l[1].n_blocks;
    const int n_g = (P + G - 1) / G;
    int layer = 0, u = 0;
    for (int k = 0; k < n_g + L; ++k) {
      if (k < n_g) {
        const int sz = min(G, P - k * G) * NB0;
        if (g < sz) { layer = 0; u = k * G * NB0 + g; break; }
        g -= sz;
      }
      if (k >= L) {
        const int j = k - L;
        const int sz = min(G, P - j * G) * NB1;
        if (g < sz) { layer = 1; u = j * G * NB1 + g; break; }
        g -= sz;
      }
    }
    const LayerArgs& p = f.l[layer];
    Unit w = decode_unit(u, layer, p.raster, P, p.n_blocks, p.order_group, p.order_group2);
    w.ks = 0;
    w.half = narrow_block(p, w.nb) ? 0 : -1;
    w.kb0 = 0;
    w.kb1 = p.k_blocks;
    w.np = 1;
    return w;
  }
  int layer = 0;
  Sched s = s0;
  if (g >= s0.total) {
    g -= s0.total;
    layer = 1;
    s = s1;
  }
  const LayerArgs& p = f.l[layer];
  Unit w;
  if (g < s.full) {
    // the K slices of one output tile are consecutive claims (they finish
    // together; the last one reduces) -- or, for the uneven tail split, all
    // heads and then all tails
    const int U = s.full / s.S;
    const int u = s.c > 0 ? g % U : g / s.S;
    w = decode_unit(u, layer, p.raster, P, p.n_blocks, p.order_group, p.order_group2);
    w.ks = s.c > 0 ? g / U : g % s.S;
    // a ragged last n-block of <= 256 columns (e.g. K/tp = 3200) runs as a
    // half unit: one 256-wide UMMA instead of two over mostly padding
    w.half = narrow_block(p, w.nb) ? 0 : -1;
  } else {
    const int v = g - s.full;
    w = decode_unit(s.full + (v >> 1), layer, p.raster, P, p.n_blocks, p.order_group, p.order_group2);
    w.half = v & 1;
    w.ks = 0;
  }
  if (s.c > 0) {
    const int c = w.pair >= s.late_lo ? s.c_late : s.c;
    w.kb0 = w.ks ? c : 0;
    w.kb1 = w.ks ? p.k_blocks : c;
  } else {
    w.kb0 = w.ks * p.k_blocks / s.S;
    w.kb1 = (w.ks + 1) * p.k_blocks / s.S;
  }
  w.np = s.S;
  return w;
}

}  // namespace comet
