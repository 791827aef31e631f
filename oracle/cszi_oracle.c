/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the cuSZ-i ("ebcomp") hot path.
 *
 * A plain-C restatement of the reference algorithm, used exclusively by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm as the CHECKER.  Nothing in the product package links or calls this.
 *
 * Each function cites the reference file:line it restates (paths relative
 * to the reference package, pkg/src/ebcomp/).  Parity is pinned against the
 * reference itself (imported in the build container) and against the golden
 * fixtures under tests/golden/ (see tests/golden/make_golden.py).
 *
 * Build: oracle/Makefile  (-O2 -fopenmp -ffp-contract=off, no -ffast-math:
 * every double operation must round exactly like numpy's float64 ufuncs).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Status codes shared with oracle.py (names follow ebcomp/errors.py). */
enum {
  ORC_OK = 0,
  ORC_LENGTH_OVERFLOW = -1,
  ORC_EMPTY_HISTOGRAM = -2,
  ORC_TRUNCATED = -3,
  ORC_CORRUPT = -4,
  ORC_UNKNOWN_SYMBOL = -5,
  ORC_OUT_OF_RANGE = -6,
  ORC_NOMEM = -7,
};

/* predictor.py:62-69 — weight vectors over offsets (-3s, -s, +s, +3s). */
static const double W_CUBIC[2][4] = {
    {-1.0 / 16.0, 9.0 / 16.0, 9.0 / 16.0, -1.0 / 16.0},
    {-3.0 / 40.0, 23.0 / 40.0, 23.0 / 40.0, -3.0 / 40.0},
};
static const double W_QUAD_L[4] = {-1.0 / 8.0, 6.0 / 8.0, 3.0 / 8.0, 0.0};
static const double W_QUAD_R[4] = {0.0, 3.0 / 8.0, 6.0 / 8.0, -1.0 / 8.0};
static const double W_LINEAR[4] = {0.0, 0.5, 0.5, 0.0};
static const double W_COPY[4] = {0.0, 1.0, 0.0, 0.0};

/* predictor.py:230-235 — multiples of stride, closed with extent-1. */
static int64_t anchor_axis(int64_t extent, int64_t stride, int64_t *out) {
  int64_t k = 0;
  for (int64_t c = 0; c < extent; c += stride) out[k++] = c;
  if (out[k - 1] != extent - 1) out[k++] = extent - 1;
  return k;
}

int64_t orc_count_anchor_axis(int64_t extent, int64_t stride) {
  int64_t k = (extent + stride - 1) / stride;
  if ((k - 1) * stride != extent - 1) k++;
  return k;
}

/*
 * One (level, dimension) pass — predictor.py:283-344 (_run_pass), applied to
 * the point lattice built in predictor.py:379-390 (interpolate_level).
 * Grids are handled as 3D; a rank-r grid is padded with leading extent-1
 * axes, which carry no pass points and a single anchor coordinate.
 */
typedef struct {
  int64_t ext[3];
  int64_t tile[3];
  int64_t radius;
  int variant[3];
} orc_geom;

static void run_pass(const orc_geom *g, int mode, int d, int64_t s, double level_eb,
                     const int passed[3], float *recon, const float *src, int32_t *codes,
                     uint8_t *is_out, const float *outval, int threads) {
  const int64_t e0 = g->ext[0], e1 = g->ext[1], e2x = g->ext[2];
  int64_t lo[3], step[3];
  for (int a = 0; a < 3; ++a) {
    if (a == d) {
      lo[a] = s;
      step[a] = 2 * s;
    } else if (passed[a]) {
      lo[a] = 0;
      step[a] = s;
    } else {
      lo[a] = 0;
      step[a] = 2 * s;
    }
  }
  const int64_t stride_d = (d == 0) ? e1 * e2x : (d == 1 ? e2x : 1);
  const int64_t extent = g->ext[d];
  const int64_t tile = g->tile[d];
  const double *wc = W_CUBIC[g->variant[d]];
  const double e2 = 2.0 * level_eb;
  const int64_t R = g->radius;
  int64_t n0 = (e0 - lo[0] + step[0] - 1) / step[0];
  if (n0 < 0) n0 = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
#endif
  for (int64_t i0 = 0; i0 < n0; ++i0) {
    int64_t c[3];
    c[0] = lo[0] + i0 * step[0];
    for (c[1] = lo[1]; c[1] < e1; c[1] += step[1]) {
      for (c[2] = lo[2]; c[2] < e2x; c[2] += step[2]) {
        const int64_t pd = c[d];
        const int64_t offset = pd % tile;
        /* predictor.py:297-306 — availability masks and the case table */
        const int m3 = offset >= 3 * s;
        const int p1 = pd + s <= extent - 1;
        const int p3 = (offset <= tile - 3 * s) && (pd + 3 * s <= extent - 1);
        const double *w;
        int av[4];
        if (m3 && p1 && p3) {
          w = wc; av[0] = 1; av[1] = 1; av[2] = 1; av[3] = 1;
        } else if (m3 && p1 && !p3) {
          w = W_QUAD_L; av[0] = 1; av[1] = 1; av[2] = 1; av[3] = 0;
        } else if (!m3 && p1 && p3) {
          w = W_QUAD_R; av[0] = 0; av[1] = 1; av[2] = 1; av[3] = 1;
        } else if (!m3 && p1 && !p3) {
          w = W_LINEAR; av[0] = 0; av[1] = 1; av[2] = 1; av[3] = 0;
        } else {
          w = W_COPY; av[0] = 0; av[1] = 1; av[2] = 0; av[3] = 0;
        }
        const int64_t idx = (c[0] * e1 + c[1]) * e2x + c[2];
        const int64_t offs[4] = {-3 * s, -s, s, 3 * s};
        double t4[4];
        for (int k = 0; k < 4; ++k)
          t4[k] = av[k] ? (double)recon[idx + offs[k] * stride_d] : 0.0;
        /* predictor.py:325 — one fixed four-term expression shape */
        const double pred = ((w[0] * t4[0] + w[1] * t4[1]) + w[2] * t4[2]) + w[3] * t4[3];
        if (mode == 0) {
          /* predictor.py:327-339 — synchronized quantization */
          const float o32 = src[idx];
          const double o = (double)o32;
          const double t = (o - pred) / e2;
          const double qf = trunc(t + copysign(0.5, t));
          const int big = fabs(qf) >= (double)R;
          const double qsel = big ? 0.0 : qf;
          const int32_t q = (int32_t)qsel;
          const float rec = (float)(pred + e2 * (double)q);
          const int bad = big || (fabs((double)rec - o) > level_eb);
          recon[idx] = bad ? o32 : rec;
          codes[idx] = bad ? 0 : q;
          is_out[idx] = (uint8_t)bad;
        } else {
          /* predictor.py:340-344 — replay from codes */
          const double q = (double)codes[idx];
          const float rec = (float)(pred + e2 * q);
          recon[idx] = is_out[idx] ? outval[idx] : rec;
        }
      }
    }
  }
}

/*
 * compress_predict / decompress_predict core — predictor.py:395-465 with the
 * level loop of predictor.py:367-392.  level_eb[] holds eb/alpha**(level-1)
 * for the levels coarse->fine, computed by the Python caller exactly as
 * plan_levels does (predictor.py:122-136).  order[] lists the padded-3D axis
 * ids of the rank's dim_order.
 *
 * mode 0 (compress): src = original data; fills recon, codes, is_out.
 * mode 1 (decompress): recon must hold zeros; anchors[] holds the anchor
 * block in lattice order; codes/is_out/outval drive the replay.
 */
int orc_predict(int mode, const int64_t ext[3], int64_t S, const int64_t tile[3],
                const double *level_eb, int nlev, const int variant[3], const int *order,
                int norder, int64_t radius, const float *src, float *recon, int32_t *codes,
                uint8_t *is_out, const float *outval, const float *anchors_in, int threads) {
  orc_geom g;
  for (int a = 0; a < 3; ++a) {
    g.ext[a] = ext[a];
    g.tile[a] = tile[a];
    g.variant[a] = variant[a];
  }
  g.radius = radius;
  int64_t *ax[3];
  int64_t na[3];
  for (int a = 0; a < 3; ++a) {
    ax[a] = (int64_t *)malloc(sizeof(int64_t) * (ext[a] / S + 3));
    if (!ax[a]) return ORC_NOMEM;
    na[a] = anchor_axis(ext[a], S, ax[a]);
  }
  const int64_t nanch = na[0] * na[1] * na[2];
  int64_t *aidx = (int64_t *)malloc(sizeof(int64_t) * nanch);
  float *aval = (float *)malloc(sizeof(float) * nanch);
  if (!aidx || !aval) return ORC_NOMEM;
  int64_t k = 0;
  for (int64_t i = 0; i < na[0]; ++i)
    for (int64_t j = 0; j < na[1]; ++j)
      for (int64_t l = 0; l < na[2]; ++l) {
        const int64_t idx = (ax[0][i] * ext[1] + ax[1][j]) * ext[2] + ax[2][l];
        aidx[k] = idx;
        aval[k] = (mode == 0) ? src[idx] : anchors_in[k];
        k++;
      }
  /* predictor.py:401-403 / :446-447 — seed the anchor block */
  for (int64_t i = 0; i < nanch; ++i) recon[aidx[i]] = aval[i];
  int64_t s = S / 2;
  for (int lv = 0; lv < nlev && s >= 1; ++lv, s /= 2) {
    int passed[3] = {0, 0, 0};
    for (int oi = 0; oi < norder; ++oi) {
      const int d = order[oi];
      if (s < ext[d]) {
        run_pass(&g, mode, d, s, level_eb[lv], passed, recon, src, codes, is_out, outval,
                 threads);
        /* predictor.py:391 — restore anchors predicted over by the pass */
        for (int64_t i = 0; i < nanch; ++i) recon[aidx[i]] = aval[i];
      }
      passed[d] = 1;
    }
  }
  if (mode == 0) {
    /* predictor.py:414-415 — anchors carry code 0 and are never outliers */
    for (int64_t i = 0; i < nanch; ++i) {
      codes[aidx[i]] = 0;
      is_out[aidx[i]] = 0;
    }
  }
  for (int a = 0; a < 3; ++a) free(ax[a]);
  free(aidx);
  free(aval);
  return ORC_OK;
}

/* huffman.py:60-74 — histogram of codes shifted by +R. */
int orc_histogram(const int32_t *codes, int64_t n, int64_t radius, int64_t *counts) {
  memset(counts, 0, sizeof(int64_t) * 2 * radius);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t c = codes[i];
    if (c <= -radius || c >= radius) return ORC_OUT_OF_RANGE;
    counts[c + radius]++;
  }
  return ORC_OK;
}

/*
 * huffman.py:77-102 — code lengths from a binary min-heap keyed by
 * (frequency, smallest contained symbol); a symbol's length is the number of
 * merges its node takes part in, i.e. its depth in the merge tree.
 */
typedef struct {
  int64_t f;
  int64_t m;
  int32_t node;
} heap_item;

static int item_less(const heap_item *a, const heap_item *b) {
  return a->f < b->f || (a->f == b->f && a->m < b->m);
}
static void sift_down(heap_item *h, int64_t n, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && item_less(&h[l], &h[m])) m = l;
    if (r < n && item_less(&h[r], &h[m])) m = r;
    if (m == i) return;
    heap_item t = h[i];
    h[i] = h[m];
    h[m] = t;
    i = m;
  }
}
static void sift_up(heap_item *h, int64_t i) {
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!item_less(&h[i], &h[p])) return;
    heap_item t = h[i];
    h[i] = h[p];
    h[p] = t;
    i = p;
  }
}

int orc_code_lengths(const int64_t *counts, int64_t nbins, uint8_t *lengths) {
  memset(lengths, 0, (size_t)nbins);
  int64_t alive = 0;
  for (int64_t s = 0; s < nbins; ++s) alive += counts[s] != 0;
  if (alive == 0) return ORC_EMPTY_HISTOGRAM;
  if (alive == 1) {
    for (int64_t s = 0; s < nbins; ++s)
      if (counts[s]) lengths[s] = 1;
    return ORC_OK;
  }
  heap_item *h = (heap_item *)malloc(sizeof(heap_item) * alive);
  int32_t *parent = (int32_t *)malloc(sizeof(int32_t) * 2 * alive);
  int32_t *leaf_sym = (int32_t *)malloc(sizeof(int32_t) * alive);
  if (!h || !parent || !leaf_sym) return ORC_NOMEM;
  int64_t n = 0;
  for (int64_t s = 0; s < nbins; ++s)
    if (counts[s]) {
      h[n].f = counts[s];
      h[n].m = s;
      h[n].node = (int32_t)n;
      leaf_sym[n] = (int32_t)s;
      n++;
    }
  for (int64_t i = n / 2 - 1; i >= 0; --i) sift_down(h, n, i);
  int32_t next_node = (int32_t)alive;
  while (n > 1) {
    heap_item a = h[0];
    h[0] = h[--n];
    sift_down(h, n, 0);
    heap_item b = h[0];
    h[0] = h[--n];
    sift_down(h, n, 0);
    parent[a.node] = next_node;
    parent[b.node] = next_node;
    heap_item c;
    c.f = a.f + b.f;
    c.m = a.m < b.m ? a.m : b.m;
    c.node = next_node++;
    h[n++] = c;
    sift_up(h, n - 1);
  }
  const int32_t root = next_node - 1;
  int32_t *depth = (int32_t *)calloc((size_t)next_node, sizeof(int32_t));
  int rc = ORC_OK;
  /* internal nodes are numbered in creation order: parents come later */
  for (int32_t v = root - 1; v >= 0; --v) depth[v] = depth[parent[v]] + 1;
  for (int64_t i = 0; i < alive; ++i) {
    if (depth[i] > 32) rc = ORC_LENGTH_OVERFLOW;
    lengths[leaf_sym[i]] = (uint8_t)(depth[i] > 255 ? 255 : depth[i]);
  }
  free(h);
  free(parent);
  free(leaf_sym);
  free(depth);
  return rc;
}

/*
 * huffman.py:128-160 — canonical codes in (length, symbol) order plus the
 * first_code / first_index / count tables of the decoder.
 */
int orc_canonical(const uint8_t *lengths, int64_t nbins, uint32_t *words, int64_t *first_code,
                  int64_t *first_index, int64_t *length_counts, int64_t *sorted_syms,
                  int64_t *ncoded) {
  for (int64_t s = 0; s < nbins; ++s)
    if (lengths[s] > 32) return ORC_LENGTH_OVERFLOW;
  memset(words, 0, sizeof(uint32_t) * nbins);
  memset(first_code, 0, sizeof(int64_t) * 33);
  memset(first_index, 0, sizeof(int64_t) * 33);
  memset(length_counts, 0, sizeof(int64_t) * 33);
  int64_t idx = 0;
  for (int ln = 1; ln <= 32; ++ln)
    for (int64_t s = 0; s < nbins; ++s)
      if (lengths[s] == ln) sorted_syms[idx++] = s;
  *ncoded = idx;
  uint64_t code = 0;
  int prev = 0;
  for (int64_t i = 0; i < idx; ++i) {
    const int64_t sym = sorted_syms[i];
    const int ln = lengths[sym];
    code <<= (ln - prev);
    if (ln != prev) {
      first_code[ln] = (int64_t)code;
      first_index[ln] = i;
    }
    length_counts[ln]++;
    words[sym] = (uint32_t)code;
    code += 1;
    prev = ln;
  }
  return ORC_OK;
}

/* _kernels.py:36-60 — MSB-first packing; returns bytes written. */
int64_t orc_huffman_encode(const int32_t *codes, int64_t n, int64_t radius,
                           const uint8_t *lengths, const uint32_t *words, uint8_t *out,
                           uint64_t *bit_count) {
  uint64_t acc = 0;
  int nbits = 0;
  int64_t pos = 0;
  uint64_t bits = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t s = (int64_t)codes[i] + radius;
    if (s < 0 || s >= 2 * radius || lengths[s] == 0) return -(i + 1);
    const int ln = lengths[s];
    acc = (acc << ln) | (uint64_t)words[s];
    nbits += ln;
    bits += (uint64_t)ln;
    while (nbits >= 8) {
      out[pos++] = (uint8_t)((acc >> (nbits - 8)) & 0xFF);
      nbits -= 8;
    }
  }
  if (nbits > 0) out[pos++] = (uint8_t)((acc << (8 - nbits)) & 0xFF);
  *bit_count = bits;
  return pos;
}

/* _kernels.py:63-92 — bit-at-a-time canonical decoder (codes = sym - R). */
int orc_huffman_decode(const uint8_t *stream, int64_t nbytes, int64_t n, int64_t radius,
                       const int64_t *first_code, const int64_t *first_index,
                       const int64_t *counts, const int64_t *sorted_syms, int32_t *out) {
  uint64_t bitpos = 0;
  const uint64_t total = (uint64_t)nbytes * 8;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t cur = 0;
    int ln = 0;
    for (;;) {
      if (bitpos >= total) return ORC_TRUNCATED;
      const uint8_t byte = stream[bitpos >> 3];
      const uint32_t bit = (byte >> (7 - (bitpos & 7))) & 1u;
      cur = (cur << 1) | bit;
      bitpos++;
      ln++;
      if (ln > 32) return ORC_TRUNCATED;
      if (counts[ln] > 0) {
        const int64_t off = (int64_t)cur - first_code[ln];
        if (off >= 0 && off < counts[ln]) {
          out[i] = (int32_t)(sorted_syms[first_index[ln] + off] - radius);
          break;
        }
      }
    }
  }
  return ORC_OK;
}

/* pass2.py:30-67 — zero-run codec id 0; returns encoded length. */
int64_t orc_pass2_encode(const uint8_t *in, int64_t n, uint8_t *out) {
  int64_t o = 0, cursor = 0, i = 0;
  while (i < n) {
    if (in[i] == 0 && i + 1 < n && in[i + 1] == 0) {
      int64_t e = i;
      while (e < n && in[e] == 0) e++;
      /* literals before the run: pass2.py:40-47 */
      for (int64_t p = cursor; p < i;) {
        int64_t take = (i - p) < 128 ? (i - p) : 128;
        out[o++] = (uint8_t)(take - 1);
        memcpy(out + o, in + p, (size_t)take);
        o += take;
        p += take;
      }
      for (int64_t run = e - i; run > 0;) {
        int64_t take = run < 128 ? run : 128;
        out[o++] = (uint8_t)(127 + take);
        run -= take;
      }
      cursor = e;
      i = e;
    } else {
      i++;
    }
  }
  for (int64_t p = cursor; p < n;) {
    int64_t take = (n - p) < 128 ? (n - p) : 128;
    out[o++] = (uint8_t)(take - 1);
    memcpy(out + o, in + p, (size_t)take);
    o += take;
    p += take;
  }
  return o;
}

/* pass2.py:70-86 — decode; returns decoded length or ORC_CORRUPT.  With
 * out == NULL only the decoded length is computed. */
int64_t orc_pass2_decode(const uint8_t *in, int64_t n, uint8_t *out, int64_t cap) {
  int64_t pos = 0, o = 0;
  while (pos < n) {
    const uint8_t c = in[pos++];
    if (c < 128) {
      const int64_t take = (int64_t)c + 1;
      if (pos + take > n) return ORC_CORRUPT;
      if (out) {
        if (o + take > cap) return ORC_CORRUPT;
        memcpy(out + o, in + pos, (size_t)take);
      }
      o += take;
      pos += take;
    } else {
      const int64_t z = (int64_t)c - 127;
      if (out) {
        if (o + z > cap) return ORC_CORRUPT;
        memset(out + o, 0, (size_t)z);
      }
      o += z;
    }
  }
  return o;
}

/* grid.py:104-108 + grid.py:60-62 — min/max and the first non-finite index. */
int64_t orc_range(const float *x, int64_t n, float *lo, float *hi) {
  float a = INFINITY, b = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    const float v = x[i];
    if (!isfinite(v)) return i;
    if (v < a) a = v;
    if (v > b) b = v;
  }
  *lo = a;
  *hi = b;
  return -1;
}

/*
 * Lorenzo predictor — _kernels.py:104-215 (lorenzo_1d/2d/3d), driven by
 * lorenzo.py:22-53.  Rank-r grids are padded to 3D with leading extent-1
 * axes; each rank keeps the reference's own expression (the 1D / 2D sums
 * are not rewritten as the 3D one).  compress != 0: quantize `orig` into
 * codes / is_out and write the reconstruction; else replay codes / is_out /
 * outval into recon.
 */
int orc_lorenzo(int compress, int rank, const int64_t ext[3], const float *orig, float *recon,
                int32_t *codes, uint8_t *is_out, const float *outval, double e2, int64_t radius,
                double bound) {
  const int64_t nz = ext[0], ny = ext[1], nx = ext[2];
  for (int64_t z = 0; z < nz; ++z)
    for (int64_t y = 0; y < ny; ++y)
      for (int64_t x = 0; x < nx; ++x) {
        const int64_t i = (z * ny + y) * nx + x;
        double pred;
        if (rank == 1) {
          pred = x > 0 ? (double)recon[i - 1] : 0.0;
        } else if (rank == 2) {
          const double a = y > 0 ? (double)recon[i - nx] : 0.0;
          const double b = x > 0 ? (double)recon[i - 1] : 0.0;
          const double c = (y > 0 && x > 0) ? (double)recon[i - nx - 1] : 0.0;
          pred = a + b - c;
        } else {
          const int64_t pz = ny * nx;
          const double a1 = z > 0 ? (double)recon[i - pz] : 0.0;
          const double a2 = y > 0 ? (double)recon[i - nx] : 0.0;
          const double a3 = x > 0 ? (double)recon[i - 1] : 0.0;
          const double a4 = (y > 0 && x > 0) ? (double)recon[i - nx - 1] : 0.0;
          const double a5 = (z > 0 && x > 0) ? (double)recon[i - pz - 1] : 0.0;
          const double a6 = (z > 0 && y > 0) ? (double)recon[i - pz - nx] : 0.0;
          const double a7 = (z > 0 && y > 0 && x > 0) ? (double)recon[i - pz - nx - 1] : 0.0;
          pred = a1 + a2 + a3 - a4 - a5 - a6 + a7;
        }
        if (compress) {
          const double o = (double)orig[i];
          const double t = (o - pred) / e2;
          int64_t q = 0;
          float r = 0.0f;
          int outlier = 1;
          if (fabs(t) < (double)radius - 0.5) {
            q = (int64_t)trunc(t + copysign(0.5, t));
            if (llabs(q) < radius) {
              r = (float)(pred + e2 * (double)q);
              if (fabs((double)r - o) <= bound) outlier = 0;
            }
          }
          if (outlier) {
            codes[i] = 0;
            is_out[i] = 1;
            recon[i] = orig[i];
          } else {
            codes[i] = (int32_t)q;
            recon[i] = r;
          }
        } else {
          if (is_out[i]) recon[i] = outval[i];
          else recon[i] = (float)(pred + e2 * (double)codes[i]);
        }
      }
  return ORC_OK;
}
