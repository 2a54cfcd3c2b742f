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
  int ks;    // K slice (split-K): k-blocks [ks*KB/S, (ks+1)*KB/S) of S slices
};

// A layer's unit sequence: units [0, full) are full 512-column units; unit
// full + v is half (v & 1) of full unit full + v/2.  Layer0 alone cuts a
// mostly idle last round into halves (the tail takes half a unit time); layer1
// splits its last `split_units` units (the end of the launch in modes 1/2).
struct Sched {
  int full;   // full units before the split tail
  int total;  // units in the sequence (full + halves)
  int S;      // K slices per output tile (split-K; 1 = off)
};
COMET_HD Sched make_sched(int U, int n_split, int S = 1) {
  n_split = S > 1 ? 0 : max(0, min(U, n_split));
  return {U * S - n_split, U * S + n_split, S};
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

COMET_HD int seq_total(const KernelArgs& f, int P, int n_pairs, Sched& s0, Sched& s1) {
  s0 = {0, 0};
  s1 = {0, 0};
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
    // together; the last one reduces)
    w = decode_unit(g / s.S, layer, p.raster, P, p.n_blocks, p.order_group, p.order_group2);
    w.ks = g % s.S;
    // a ragged last n-block of <= 256 columns (e.g. K/tp = 3200) runs as a
    // half unit: one 256-wide UMMA instead of two over mostly padding
    w.half = narrow_block(p, w.nb) ? 0 : -1;
  } else {
    const int v = g - s.full;
    w = decode_unit(s.full + (v >> 1), layer, p.raster, P, p.n_blocks, p.order_group, p.order_group2);
    w.half = v & 1;
    w.ks = 0;
  }
  return w;
}

COMET_HD int slices_of(const Unit& w, const Sched& s0, const Sched& s1) {
  return w.layer ? s1.S : s0.S;
}

}  // namespace comet
