// Host test of the layer kernel's unit schedule (csrc/sched.cuh), run by
// tests/test_sched_host.py: for random shapes and knob sets, the claim
// sequence of a fused launch (mode 2) must
//   (1) cover every (layer, pair, n-block) exactly once -- one full unit, or
//       both 256-column halves, or every K slice once;
//   (2) put every layer0 unit of a pair before any layer1 unit of that pair
//       (a layer1 unit waits for its H rows; an earlier claim never waits on
//       a later one, so the persistent grid cannot deadlock);
//   (3) keep, for each layer1 n-block, pairs in ascending order when the
//       fused combine has fold chains (a token's last hosted row reads rows
//       of earlier pairs at the same columns);
//   (4) give the K slices of a split tile contraction ranges [kb0, kb1)
//       that partition [0, KB) (even split-K and the uneven head / tail split
//       of layer1's partial round).
// Prints "OK <cases>" or the first violation.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <random>
#include <tuple>
#include <vector>

#include "../paper_2502_19811_b200/csrc/sched.cuh"

using namespace comet;

static int check(const KernelArgs& f, int P, int n_pairs, const char* tag) {
  Sched s0, s1;
  const int total = seq_total(f, P, n_pairs, s0, s1);
  std::map<std::tuple<int, int, int>, std::vector<std::pair<int, int>>> seen;  // (layer,pair,nb) -> (half,ks)
  std::map<std::tuple<int, int, int>, std::vector<std::pair<int, int>>> kr;    // -> (kb0, kb1) per slice
  std::vector<int> l0_last(P, -1), l1_first(P, 1 << 30);
  std::map<int, int> last_pair_at_nb;  // layer1: nb*2+half -> last pair seen
  for (int g = 0; g < total; ++g) {
    const Unit w = unit_at(f, g, P, s0, s1);
    if (w.pair < 0 || w.pair >= P || w.nb < 0 || w.nb >= f.l[w.layer].n_blocks) {
      printf("FAIL %s: g=%d decodes out of range (layer %d pair %d nb %d)\n", tag, g, w.layer, w.pair, w.nb);
      return 1;
    }
    seen[{w.layer, w.pair, w.nb}].push_back({w.half, w.ks});
    kr[{w.layer, w.pair, w.nb}].push_back({w.kb0, w.kb1});
    if (w.np != (w.layer ? s1.S : s0.S)) {
      printf("FAIL %s: g=%d slice count %d != S\n", tag, g, w.np);
      return 1;
    }
    if (w.layer == 0) l0_last[w.pair] = g;
    else {
      if (g < l1_first[w.pair]) l1_first[w.pair] = g;
      for (int h = 0; h < 2; ++h) {
        if (w.half >= 0 && w.half != h) continue;
        const int key = w.nb * 2 + h;
        auto it = last_pair_at_nb.find(key);
        if (it != last_pair_at_nb.end() && it->second > w.pair && fold_chains(f.l[1])) {
          printf("FAIL %s: layer1 nb %d half %d visits pair %d after pair %d (g=%d)\n", tag, w.nb, h, w.pair,
                 it->second, g);
          return 1;
        }
        last_pair_at_nb[key] = w.pair;
      }
    }
  }
  for (int layer = 0; layer < 2; ++layer) {
    const Sched& s = layer ? s1 : s0;
    for (int pr = 0; pr < P; ++pr)
      for (int nb = 0; nb < f.l[layer].n_blocks; ++nb) {
        auto it = seen.find({layer, pr, nb});
        if (it == seen.end()) {
          printf("FAIL %s: layer %d pair %d nb %d never claimed\n", tag, layer, pr, nb);
          return 1;
        }
        std::vector<std::pair<int, int>> v = it->second;
        bool ok = false;
        if (s.S > 1) {
          ok = (int)v.size() == s.S;
          for (int k = 0; k < s.S && ok; ++k) {
            int c = 0;
            for (auto& e : v) c += e.second == k && (e.first < 0 || (e.first == 0 && narrow_block(f.l[layer], nb)));
            ok = c == 1;
          }
        } else if (v.size() == 1) {
          ok = v[0].second == 0 && (v[0].first == -1 || (v[0].first == 0 && narrow_block(f.l[layer], nb)));
        } else if (v.size() == 2) {
          ok = v[0].second == 0 && v[1].second == 0 && v[0].first + v[1].first == 1 && v[0].first >= 0 &&
               v[1].first >= 0;
        }
        if (!ok) {
          printf("FAIL %s: layer %d pair %d nb %d claimed %zu times (bad halves/slices)\n", tag, layer, pr, nb,
                 v.size());
          return 1;
        }
        std::vector<std::pair<int, int>> r = kr[{layer, pr, nb}];
        std::sort(r.begin(), r.end());
        const int KB = f.l[layer].k_blocks;
        bool kok = true;
        if (s.S > 1) {
          kok = r.front().first == 0 && r.back().second == KB;
          for (size_t i = 0; i < r.size() && kok; ++i) kok = r[i].second > r[i].first && (i == 0 || r[i].first == r[i - 1].second);
        } else {
          for (auto& e : r) kok = kok && e.first == 0 && e.second == KB;
        }
        if (!kok) {
          printf("FAIL %s: layer %d pair %d nb %d K slices do not partition [0, %d)\n", tag, layer, pr, nb, KB);
          return 1;
        }
      }
  }
  for (int pr = 0; pr < P; ++pr)
    if (l1_first[pr] < l0_last[pr]) {
      printf("FAIL %s: pair %d layer1 claimed at %d before its last layer0 unit at %d\n", tag, pr, l1_first[pr],
             l0_last[pr]);
      return 1;
    }
  return 0;
}

int main(int argc, char** argv) {
  const int n_cases = argc > 1 ? atoi(argv[1]) : 3000;
  std::mt19937 rng(12345);
  auto pick = [&](int lo, int hi) { return lo + static_cast<int>(rng() % static_cast<unsigned>(hi - lo + 1)); };
  for (int c = 0; c < n_cases; ++c) {
    KernelArgs f{};
    f.mode = 2;
    const int P = pick(1, 80);
    const int n_pairs = std::vector<int>{2, 8, 37, 66, 74}[pick(0, 4)];
    LayerArgs& a = f.l[0];
    LayerArgs& b = f.l[1];
    a.n_blocks = pick(1, 30);
    b.n_blocks = pick(1, 12);
    a.out_ld = a.n_blocks * 512 - (pick(0, 1) ? pick(0, 400) : 0);
    b.out_ld = b.n_blocks * 512 - (pick(0, 1) ? pick(0, 400) : 0);
    a.k_blocks = pick(1, 230);
    b.k_blocks = pick(1, 230);
    a.raster = 0;
    b.raster = 2;
    a.order_group = pick(1, 10);
    b.order_group = pick(1, 8);
    b.order_group2 = pick(0, 1) ? a.order_group : pick(1, 10);
    f.interleave = pick(0, 2) ? 0 : pick(1, 4);
    if (f.interleave > 0) {  // as comet_forward_zerocopy sets it up
      b.order_group2 = a.order_group;
    } else {
      a.split_tail = pick(0, 1);
      a.ksplit_max = pick(0, 1) ? 8 : 0;
      b.ksplit_max = pick(0, 1) ? 8 : 0;
      b.split_units = std::vector<int>{0, 0, 5, 55, 74, 1000}[pick(0, 5)];
      b.streamk = pick(0, 2) != 0;
      b.fuse_combine = pick(0, 1);
      b.experts_per_group = pick(1, 8);
      b.topk = pick(1, 8);
    }
    char tag[160];
    snprintf(tag, sizeof tag, "case %d (P=%d pairs=%d NB0=%d NB1=%d KB1=%d G=%d G2=%d ilv=%d split0=%d split1=%d ks=%d/%d sk=%d)", c,
             P, n_pairs, a.n_blocks, b.n_blocks, b.k_blocks, a.order_group, b.order_group2, f.interleave,
             a.split_tail, b.split_units, a.ksplit_max, b.ksplit_max, b.streamk);
    if (check(f, P, n_pairs, tag)) return 1;
  }
  printf("OK %d\n", n_cases);
  return 0;
}
