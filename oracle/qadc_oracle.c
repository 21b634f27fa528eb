/*
 * qadc_oracle.c -- TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's Quick ADC distance and selection steps, for oracle checks at
 * the BASELINE sizes (cfg4: 1e9 codes per query), where the numpy oracle
 * (oracle/pqscan_oracle.py) would take ~45 s per query.  Only tests/ use it
 * (through ctypes); the product library never links it.
 *
 * Restated functions (reference /root/reference/pkg/src/pqscan):
 *   quantized_distances  quickadc.py:87-101  acc = min(acc + t[j][c_j], 127)
 *                                            per component, int16 semantics
 *   _select_best         scan.py:142-154     the r smallest (distance, id)
 *                                            pairs, ascending, ties by id
 * on PQL1 nibble-packed 4-bit codes (scan.py:293-316: component 2j in the low
 * nibble of byte j, 2j+1 in the high nibble).  Pinned against the golden
 * fixtures of the real reference and the numpy oracle
 * (tests/test_oracle_c.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BINS 127

/* one code's saturated sum, quickadc.py:87-101 (clamp after every add) */
static inline int qdist1(const uint8_t* row, int m, const uint8_t* qt) {
  int acc = 0;
  for (int j = 0; j < m; j += 2) {
    const uint8_t b = row[j >> 1];
    acc += qt[j * 16 + (b & 15)];
    if (acc > BINS) acc = BINS;
    acc += qt[(j + 1) * 16 + (b >> 4)];
    if (acc > BINS) acc = BINS;
  }
  return acc;
}

/* quantized_distances over n packed codes (m even) -> out[n] */
void pqo_qdist_packed(const uint8_t* packed, int64_t n, int m, const uint8_t* qt, uint8_t* out) {
  const int rb = m / 2;
  for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)qdist1(packed + i * rb, m, qt);
}

/* quantized_distances + _select_best with ids = id_base + i (ascending with
 * the storage position, CodeList default ids scan.py:170-171): the r smallest
 * (bin, id) pairs in ascending order.  Counting selection: the cut bin b* is
 * the smallest bin whose cumulative count reaches min(r, n); every code with
 * bin < b* is kept, and the first (in id order) codes with bin == b* fill
 * up -- exactly lexsort((ids, bins))[:r] on the partition's candidates.
 * Returns the number written (min(r, n)).  bins_scratch: n bytes or NULL
 * (then the sums are recomputed in the second pass). */
int64_t pqo_qadc_topr_packed(const uint8_t* packed, int64_t n, int m, const uint8_t* qt, int64_t id_base, int r,
                             uint8_t* bins_scratch, uint8_t* out_bins, int64_t* out_ids) {
  const int rb = m / 2;
  int64_t hist[BINS + 1];
  memset(hist, 0, sizeof(hist));
  for (int64_t i = 0; i < n; ++i) {
    const int b = qdist1(packed + i * rb, m, qt);
    if (bins_scratch) bins_scratch[i] = (uint8_t)b;
    ++hist[b];
  }
  const int64_t r_eff = (int64_t)r < n ? (int64_t)r : n;
  if (r_eff <= 0) return 0;
  int cut = 0;
  int64_t below = 0; /* codes with bin < cut */
  while (below + hist[cut] < r_eff) below += hist[cut++];
  /* output offsets per bin (counting sort of the kept codes) */
  int64_t start[BINS + 1];
  int64_t acc = 0;
  for (int b = 0; b <= BINS; ++b) {
    start[b] = acc;
    if (b < cut) acc += hist[b];
  }
  int64_t need_cut = r_eff - below, taken_cut = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int b = bins_scratch ? bins_scratch[i] : qdist1(packed + i * rb, m, qt);
    if (b < cut) {
      const int64_t p = start[b]++;
      out_bins[p] = (uint8_t)b;
      out_ids[p] = id_base + i;
    } else if (b == cut && taken_cut < need_cut) {
      const int64_t p = below + taken_cut++;
      out_bins[p] = (uint8_t)b;
      out_ids[p] = id_base + i;
    }
  }
  return r_eff;
}

/* merge of per-shard top-r lists by (bin, id) -- NeighborSet.push semantics
 * (scan.py:109-118): G sorted lists of counts[g] entries -> the r smallest */
int64_t pqo_merge_topr(int G, const uint8_t* bins, const int64_t* ids, const int64_t* counts, int64_t stride, int r,
                       uint8_t* out_bins, int64_t* out_ids) {
  int64_t* pos = (int64_t*)calloc((size_t)G, sizeof(int64_t));
  int64_t k = 0;
  while (k < r) {
    int best = -1;
    for (int g = 0; g < G; ++g) {
      if (pos[g] >= counts[g]) continue;
      const uint8_t b = bins[g * stride + pos[g]];
      const int64_t id = ids[g * stride + pos[g]];
      if (best < 0 || b < bins[best * stride + pos[best]] ||
          (b == bins[best * stride + pos[best]] && id < ids[best * stride + pos[best]]))
        best = g;
    }
    if (best < 0) break;
    out_bins[k] = bins[best * stride + pos[best]];
    out_ids[k] = ids[best * stride + pos[best]];
    ++pos[best];
    ++k;
  }
  free(pos);
  return k;
}
