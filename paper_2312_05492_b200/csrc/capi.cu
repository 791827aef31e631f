// extern "C" entry points of libcszi.so (see include/cszi.h) and the
// stream-ordered orchestration of the compress / decompress paths
// (pipeline.py:66-204).  No exceptions cross the ABI; no host sync inside.
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <initializer_list>
#include <tuple>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace cszi {
int launch_ctl_init(cszi_ctl *ctl, cudaStream_t st);
int launch_range(const float *x, uint64_t n, cszi_ctl *ctl, cudaStream_t st);
int launch_tune(const float *x, const cszi_geom *g, const cszi_params *p, cszi_ctl *ctl,
                int32_t *vals, cudaStream_t st, bool reset_outputs = false,
                u64 *zero_hist = nullptr, int nzero = 0);
int launch_sample_gather(const float *x, const cszi_geom *g, int32_t *vals, cudaStream_t st,
                         cszi_ctl *reset_ctl = nullptr);
int launch_tune_from_samples(const int32_t *vals, const cszi_geom *g, const cszi_params *p,
                             cszi_ctl *ctl, cudaStream_t st, u64 *zero_hist = nullptr,
                             int nzero = 0);
uint64_t slab_anchor_count(const cszi_geom *g);
int launch_concat_bits(uint8_t *dst, u64 dst_bit, const uint8_t *src, u64 nbits,
                       cudaStream_t st);
int launch_pack_outliers(const u64 *idx, const float *val, u64 k, uint8_t *out,
                         cudaStream_t st);
int launch_predict(const float *x, const cszi_geom *g, int32_t radius, const cszi_ctl *ctl,
                   uint16_t *sym, u64 *hist, bool exact, cudaStream_t st,
                   uint32_t *nzmap = nullptr, bool *nz_done = nullptr);
int launch_reconstruct(const uint16_t *sym, const float *anchors, const u64 *oidx,
                       const float *oval, u64 nout, const u64 *nout_dev, const cszi_geom *g,
                       int32_t radius,
                       const double *leb, int nlev, const int32_t variant[3],
                       const int32_t order[3], float *y, cudaStream_t st);
int launch_gather_anchors(const float *x, const cszi_geom *g, float *out, cudaStream_t st);
int launch_interp_level(float *recon, const float *source, int32_t *codes, uint8_t *is_out,
                        const float *oval, const float *anchor_block, const cszi_geom *g,
                        int64_t s, double leb, const int32_t variant[3], const int32_t order[3],
                        int32_t R, int32_t mode, cudaStream_t st);
int launch_hist_i32(const int32_t *codes, u64 n, int R, u64 *hist, cszi_ctl *ctl,
                    cudaStream_t st);
int launch_codebook(const u64 *hist, int nbins, uint8_t *lengths, uint32_t *words,
                    cszi_ctl *ctl, cudaStream_t st, bool set_bits = false);
size_t dec_tables_bytes(int nbins);
int launch_canonical(const uint8_t *lengths, int nbins, uint32_t *words, void *dec_tables,
                     cszi_ctl *ctl, cudaStream_t st,
                     u64 expect_raw_len = 0);
u64 enc_scratch_bytes(u64 n);
int launch_encode(int mode, const void *src, u64 n, int R, const uint8_t *lengths,
                  const uint32_t *words, uint32_t *out, u64 cap_bytes, const float *xval,
                  u64 *o_idx, float *o_val, u64 o_cap, void *scratch, cszi_ctl *ctl,
                  cudaStream_t st, u64 idx_offset, uint32_t bit_base = 0,
                  const uint32_t *nzmap = nullptr, const u64 *hist = nullptr,
                  bool bits_known = false);
u64 dec_scratch_bytes(u64 nbytes, int table_mode);
int launch_decode(const uint8_t *bytes, u64 nbytes, u64 n, int R, const void *dec_tables,
                  void *out, int out_kind, void *scratch, cszi_ctl *ctl, cudaStream_t st,
                  int table_mode, int lmax, u64 w0, u64 w1);
u64 huff_chunks(u64 nbytes);
u64 p2d_chunks(u64 n);
u64 p2d_resolve_scratch_bytes(u64 n);
int launch_p2d_tables_range(const uint8_t *in, u64 n, u64 c0, u64 c1, uint8_t *tab,
                            uint32_t *ctab, cudaStream_t st);
int launch_p2d_resolve(const uint8_t *tab, const uint32_t *ctab, u64 n, uint8_t *E,
                       uint32_t *cnt, u64 *off, void *scratch, cszi_ctl *ctl, cudaStream_t st);
int launch_p2d_expand_range(const uint8_t *in, u64 n, const uint8_t *E, const u64 *off,
                            const uint32_t *cnt, u64 c0, u64 c1, uint8_t *out, u64 cap,
                            cszi_ctl *ctl, cudaStream_t st);
int launch_huff_sync_range(const uint8_t *bytes, u64 nbytes, const void *dec_tables, u64 h0,
                           u64 h1, u64 entry, u64 *X, uint32_t *K, uint8_t *D, u64 *entry_used,
                           void *scratch, cszi_ctl *ctl, cudaStream_t st);
int launch_huff_write_window(const uint8_t *bytes, u64 nbytes, u64 n, int R,
                             const void *dec_tables, const u64 *X, uint32_t *K, const uint8_t *D,
                             u64 w0, u64 w1, uint16_t *out, void *scratch, cszi_ctl *ctl,
                             cudaStream_t st);
u64 p2enc_scratch_bytes(u64 n);
int launch_pass2_encode(const uint8_t *in, const u64 *Np, u64 cap_n, uint8_t *out,
                        void *scratch, cszi_ctl *ctl, cudaStream_t st);
u64 p2dec_scratch_bytes(u64 n);
int launch_pass2_decode(const uint8_t *in, u64 n, uint8_t *out, u64 cap, void *scratch,
                        cszi_ctl *ctl, cudaStream_t st, int expand);

int launch_lorenzo(int mode, const float *x, float *rec, uint16_t *sym, const cszi_geom *g,
                   const cszi_ctl *ctl, double e2, int R, const u64 *oidx, const float *oval,
                   const u64 *nout_dev, u64 nout_host, cudaStream_t st);
int launch_lorenzo_eb(cszi_ctl *ctl, double eb, int rel, int R, cudaStream_t st);
int launch_hist_sym(const uint16_t *sym, u64 n, int R, u64 *hist, cudaStream_t st);

// ---------------------------------------------------------------------------
// small device helpers of the pipeline
// ---------------------------------------------------------------------------
// Reset the output fields of ctl, keeping the range of a prior cszi_range.


// Sections after the anchors and codebook: bitstream bytes, then the
// outlier section (archive.py:184-189: u64 count + packed (u64, f32)).
// oval == nullptr: the values are gathered from the field x (the bitmap
// encode lists only the outlier indices)
__global__ void k_assemble(uint8_t *raw, u64 head, const uint8_t *bits, const u64 *oidx,
                           const float *oval, const float *x, u64 raw_cap, u64 bits_cap,
                           u64 o_cap, cszi_ctl *ctl, int is_payload, int bits_in_place) {
  const u64 nbits = ctl->bits;
  const u64 k = ctl->n_outliers;
  const u64 nbytes = (nbits + 7) / 8;
  const u64 total = head + nbytes + 8 + 12 * k;
  if (total > raw_cap || nbytes > bits_cap || k > o_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctl->flags, (uint32_t)CSZI_F_CAPACITY);
    return;
  }
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  const u64 nthr = (u64)gridDim.x * blockDim.x;
  // bitstream: 16-byte chunks where possible
  uint8_t *dst = raw + head;
  if (!bits_in_place)
    for (u64 i = tid; i < nbytes; i += nthr) dst[i] = bits[i];
  uint8_t *os = raw + head + nbytes;
  if (tid < 8) os[tid] = (uint8_t)(k >> (8 * tid));
  for (u64 r = tid; r < k; r += nthr) {
    uint8_t *q = os + 8 + 12 * r;
    const u64 ix = oidx[r];
    const uint32_t vb = __float_as_uint(oval ? oval[r] : x[ix]);
#pragma unroll
    for (int b = 0; b < 8; ++b) q[b] = (uint8_t)(ix >> (8 * b));
#pragma unroll
    for (int b = 0; b < 4; ++b) q[8 + b] = (uint8_t)(vb >> (8 * b));
  }
  if (tid == 0) {
    ctl->raw_len = total;
    if (is_payload) ctl->payload_len = total;
  }
}

// Decompress: parse + validate the outlier section (archive.py:192-206) and
// mark outlier points with the 0xFFFF sentinel in the symbol array.
__global__ void k_outliers_parse(const uint8_t *sec, u64 sec_len, u64 n, u64 *oidx, float *oval,
                                 uint16_t *sym, cszi_ctl *ctl) {
  if (sec_len < 8) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctl->flags, (uint32_t)CSZI_F_OUTLIER_COUNT);
    return;
  }
  u64 k = 0;
  for (int b = 0; b < 8; ++b) k |= (u64)sec[b] << (8 * b);
  if (k > (sec_len - 8) / 12 || 8 + 12 * k != sec_len) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctl->flags, (uint32_t)CSZI_F_OUTLIER_COUNT);
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->n_outliers = k;
  for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < k;
       r += (u64)gridDim.x * blockDim.x) {
    const uint8_t *q = sec + 8 + 12 * r;
    u64 ix = 0;
    uint32_t vb = 0;
    for (int b = 0; b < 8; ++b) ix |= (u64)q[b] << (8 * b);
    for (int b = 0; b < 4; ++b) vb |= (uint32_t)q[8 + b] << (8 * b);
    oidx[r] = ix;
    oval[r] = __uint_as_float(vb);
    if (r > 0) {
      const uint8_t *pq = q - 12;
      u64 pi = 0;
      for (int b = 0; b < 8; ++b) pi |= (u64)pq[b] << (8 * b);
      if (!(ix > pi)) atomicOr(&ctl->flags, (uint32_t)CSZI_F_OUTLIER_ORDER);
    }
    if (ix >= n) atomicOr(&ctl->flags, (uint32_t)CSZI_F_OUTLIER_INDEX);
  }
}
// sym holds the window [w0, w1) of the symbol array ([0, n) for a grid)
__global__ void k_outliers_mark(const u64 *oidx, const cszi_ctl *ctl, u64 n, uint16_t *sym,
                                u64 w0, u64 w1) {
  if (ctl->flags & (CSZI_F_OUTLIER_COUNT | CSZI_F_OUTLIER_ORDER | CSZI_F_OUTLIER_INDEX)) return;
  const u64 k = ctl->n_outliers;
  for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < k;
       r += (u64)gridDim.x * blockDim.x) {
    const u64 ix = oidx[r];
    if (ix < n && ix >= w0 && ix < w1) sym[ix - w0] = 0xFFFFu;
  }
}


// ---------------------------------------------------------------------------
// sharded compress glue (distributed.py): one launch per step instead of a
// chain of host-side tensor ops per slab
// ---------------------------------------------------------------------------
// range keys of a slab for the MIN all-reduce: (vmin key, -vmax key, first
// non-finite global flat index or INT64_MAX)
__global__ void k_shard_keys(const cszi_ctl *ctl, u64 flat0, int64_t *keys) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  keys[0] = (int64_t)ctl->vmin_key;
  keys[1] = -(int64_t)ctl->vmax_key;
  const u64 f = ctl->first_nonfinite;
  keys[2] = (f == ~0ull) ? INT64_MAX : (int64_t)(f + flat0);
}
// the all-reduced keys back into a slab's ctl
__global__ void k_shard_set_range(cszi_ctl *ctl, const int64_t *keys) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  ctl->vmin_key = (uint32_t)keys[0];
  ctl->vmax_key = (uint32_t)(-keys[1]);
  ctl->first_nonfinite = (keys[2] == INT64_MAX) ? ~0ull : (u64)keys[2];
}
// bits of a slab's Huffman piece: local histogram . code lengths (outliers
// and anchors are counted as R, which is how they are coded)
__global__ void k_shard_piece_bits(const u64 *hist, const uint8_t *lengths, int nbins,
                                   int64_t *out) {
  __shared__ u64 part[32];
  u64 v = 0;
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) v += hist[i] * (u64)lengths[i];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CSZI_FULL, v, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    *out = (int64_t)t;
  }
}
// (bit count, outlier count) of an encoded slab piece
__global__ void k_shard_counts(const cszi_ctl *ctl, int64_t *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  out[0] = (int64_t)ctl->bits;
  out[1] = (int64_t)ctl->n_outliers;
}

// root assembly of a sharded archive (cszi_shard_assemble)
__global__ void k_or_words(uint32_t *dst, const uint32_t *src, u64 nw) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nw; i += (u64)gridDim.x * blockDim.x)
    dst[i] |= src[i];
}
__global__ void k_shard_records(const u64 *idx, const float *val, u64 k, uint8_t *out) {
  for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < k;
       r += (u64)gridDim.x * blockDim.x) {
    uint8_t *q = out + 12 * r;
    const u64 ix = idx[r];
    const uint32_t vb = __float_as_uint(val[r]);
#pragma unroll
    for (int b = 0; b < 8; ++b) q[b] = (uint8_t)(ix >> (8 * b));
#pragma unroll
    for (int b = 0; b < 4; ++b) q[8 + b] = (uint8_t)(vb >> (8 * b));
  }
}
__global__ void k_shard_tail(uint8_t *count_at, u64 k, u64 raw_len, int is_payload,
                             cszi_ctl *ctl) {
  if (blockIdx.x != 0) return;
  if (threadIdx.x < 8) count_at[threadIdx.x] = (uint8_t)(k >> (8 * threadIdx.x));
  if (threadIdx.x == 0) {
    ctl->raw_len = raw_len;
    if (is_payload) ctl->payload_len = raw_len;
  }
}

// Cut points for the distributed pass-2 encode: positions i in [lo + 2, hi)
// where a run of >= 2 zero bytes ends (b[i-2] == b[i-1] == 0, b[i] != 0):
// the zero-run codec's segmentation has a boundary there whatever precedes
// the run (pass2.py:30-67), so the stream can be encoded piecewise.
__global__ void k_find_cuts(const uint8_t *__restrict__ b, u64 lo, u64 hi,
                            unsigned long long *first, unsigned long long *last) {
  for (u64 i = lo + 2 + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < hi;
       i += (u64)gridDim.x * blockDim.x) {
    if (b[i] != 0 && b[i - 1] == 0 && b[i - 2] == 0) {
      atomicMin(first, (unsigned long long)i);
      atomicMax(last, (unsigned long long)i);
    }
  }
}
__global__ void k_cuts_out(const unsigned long long *fl, int64_t *out) {
  out[0] = fl[0] == ~0ull ? -1 : (int64_t)fl[0];
  out[1] = fl[1] == 0 ? -1 : (int64_t)fl[1];
}

// ---------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------
static inline u64 al(u64 b) { return (b + 255) & ~(u64)255; }

struct Carver {
  unsigned char *p;
  u64 used;
  unsigned char *take(u64 b) {
    unsigned char *r = p ? p + used : nullptr;
    used += al(b);
    return r;
  }
};

static u64 grid_n(const cszi_geom *g) { return (u64)g->ext[0] * g->ext[1] * g->ext[2]; }
static u64 anchors_count(const cszi_geom *g) {
  u64 c = 1;
  for (int a = 0; a < 3; ++a) {
    const int64_t e = g->ext[a], S = g->stride;
    c *= (u64)((e - 1) / S + 1 + (((e - 1) % S) ? 1 : 0));
  }
  return c;
}
static u64 raw_capacity(const cszi_geom *g, int32_t R, const cszi_caps *caps) {
  return 4 * anchors_count(g) + 2 * (u64)R + caps->bits_cap + 8 + 12 * caps->outlier_cap;
}

struct CompressWS {
  int32_t *samples;
  uint16_t *sym;
  uint32_t *nzmap;  // non-R bit per symbol (t3 predictor -> sparse encoder)
  u64 *hist;
  uint32_t *words;
  uint32_t *bits;
  u64 *oidx;
  float *oval;
  uint8_t *raw;
  void *enc_scratch;
  void *p2_scratch;
};

static u64 layout_compress(const cszi_geom *g, int32_t R, const cszi_caps *caps, void *base,
                           CompressWS *W) {
  const u64 n = grid_n(g);
  Carver c{reinterpret_cast<unsigned char *>(base), 0};
  CompressWS w;
  w.samples = reinterpret_cast<int32_t *>(c.take(4 * CSZI_SAMPLE_WORDS));
  w.sym = reinterpret_cast<uint16_t *>(c.take(2 * n + 32));
  w.nzmap = reinterpret_cast<uint32_t *>(c.take(n / 8 + 16));
  w.hist = reinterpret_cast<u64 *>(c.take(8 * 2 * (u64)R));
  w.words = reinterpret_cast<uint32_t *>(c.take(4 * 2 * (u64)R));
  w.bits = reinterpret_cast<uint32_t *>(c.take(caps->bits_cap + 16));
  w.oidx = reinterpret_cast<u64 *>(c.take(8 * caps->outlier_cap + 8));
  w.oval = reinterpret_cast<float *>(c.take(4 * caps->outlier_cap + 4));
  w.raw = reinterpret_cast<uint8_t *>(c.take(raw_capacity(g, R, caps) + 16));
  w.enc_scratch = c.take(enc_scratch_bytes(n));
  w.p2_scratch = c.take(p2enc_scratch_bytes(raw_capacity(g, R, caps)));
  if (W) *W = w;
  return c.used;
}

// Lorenzo compress: the interp layout (no anchors are written) plus the
// float reconstruction the recurrence reads back across tiles
static u64 layout_compress_lz(const cszi_geom *g, int32_t R, const cszi_caps *caps, void *base,
                              CompressWS *W, float **rec) {
  const u64 used = layout_compress(g, R, caps, base, W);
  if (rec) *rec = base ? reinterpret_cast<float *>(reinterpret_cast<unsigned char *>(base) + used)
                       : nullptr;
  return used + al(4 * grid_n(g) + 16);
}

struct DecompressWS {
  uint8_t *raw;
  void *p2_scratch;
  void *dec_tables;
  uint16_t *sym;
  u64 *oidx;
  float *oval;
  void *dec_scratch;
};

// symbols a decompress needs: the whole grid, or for a z-slab shard
// [z0, z1) its planes plus the closing halo plane: [z0, min(z1 + 1, nz))
static u64 sym_window(const cszi_geom *g, u64 *w0) {
  const u64 plane = (u64)g->ext[1] * g->ext[2];
  if (g->slab[1] > g->slab[0]) {
    const u64 z0 = (u64)g->slab[0];
    const u64 z1 = std::min<u64>((u64)g->slab[1] + 1, (u64)g->ext[0]);
    if (w0) *w0 = z0 * plane;
    return (z1 - z0) * plane;
  }
  if (w0) *w0 = 0;
  return grid_n(g);
}

static u64 layout_decompress(const cszi_geom *g, int32_t R, const u64 sec[4], u64 payload_len,
                             int table_mode, void *base, DecompressWS *W) {
  const u64 n = grid_n(g);
  const u64 raw = sec[0] + sec[1] + sec[2] + sec[3];
  const u64 kmax = sec[3] >= 8 ? (sec[3] - 8) / 12 + 1 : 1;
  Carver c{reinterpret_cast<unsigned char *>(base), 0};
  DecompressWS w;
  w.raw = c.take(raw + 64);
  w.p2_scratch = c.take(p2dec_scratch_bytes(payload_len));
  w.dec_tables = c.take(dec_tables_bytes(2 * R));
  w.sym = reinterpret_cast<uint16_t *>(c.take(2 * sym_window(g, nullptr) + 32));
  w.oidx = reinterpret_cast<u64 *>(c.take(8 * kmax));
  w.oval = reinterpret_cast<float *>(c.take(4 * kmax));
  w.dec_scratch = c.take(dec_scratch_bytes(sec[2], table_mode));
  if (W) *W = w;
  return c.used;
}

static int grid_for(u64 work) {
  const int sms = sm_count();
  u64 b = (work + 255) / 256;
  if (b > (u64)sms * 8) b = (u64)sms * 8;
  if (b < 1) b = 1;
  return (int)b;
}

#define CK(x)                   \
  do {                          \
    const int rc_ = (x);        \
    if (rc_ != CSZI_OK) return rc_; \
  } while (0)

static int check_geom(const cszi_geom *g, int32_t R) {
  if (!g || g->rank < 1 || g->rank > 3) return CSZI_E_INVALID_ARG;
  if (g->stride < 2 || (g->stride & (g->stride - 1))) return CSZI_E_INVALID_ARG;
  for (int a = 0; a < 3; ++a)
    if (g->ext[a] < 1 || g->tile[a] < 1) return CSZI_E_INVALID_ARG;
  if (R < 2) return CSZI_E_INVALID_ARG;
  if (2 * (int64_t)R > 16384) return CSZI_E_UNSUPPORTED;  // uint16 symbols + codebook kernel
  return CSZI_OK;
}

static std::mutex g_cache_mu;
static int g_sms[64];
static std::map<std::pair<int, const void *>, size_t> g_smem_set;
static std::map<std::tuple<int, const void *, int, size_t>, int> g_occ;

int sm_count() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && g_sms[dev]) return g_sms[dev];
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) g_sms[dev] = sms;
  return sms;
}

void ensure_smem(const void *fn, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  size_t &cur = g_smem_set[{dev, fn}];
  if (smem > cur || cur == 0) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (smem > cur) cur = smem;
  }
}

int occupancy(const void *fn, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  const auto key = std::make_tuple(dev, fn, threads, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  int per = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem) != cudaSuccess ||
      per < 1)
    per = 1;
  g_occ[key] = per;
  return per;
}

static std::atomic<unsigned long long> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

// ---------------------------------------------------------------------------
// CUDA-graph replay of the whole-path entry points.  A compress / decompress
// call is a fixed, data-independent launch sequence (every data-dependent
// decision is a device predicate), so it is captured once per distinct
// argument set (pointers, geometry, parameters, stream, device, env
// switches) and replayed with one cudaGraphLaunch: the GPU no longer waits
// on the host issuing ~20 launches, and the host issues one.  Captures run
// on a private stream (the caller's may be the legacy default stream, which
// cannot be captured); the executable graph is launched on the caller's.
// CSZI_NO_GRAPH=1 launches directly.
// ---------------------------------------------------------------------------
struct GraphEntry {
  std::string key;
  cudaGraphExec_t exec;
  unsigned long long launches;
};
static std::mutex g_graph_mu;
static std::vector<GraphEntry> g_graphs;  // most recently used last
constexpr size_t GRAPH_CACHE = 64;  // batches of snapshots cycle through (x, payload) pairs

// side stream of the current device for forked branches inside a call
static cudaStream_t side_stream() {
  static cudaStream_t ss[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!ss[dev]) cudaStreamCreateWithFlags(&ss[dev], cudaStreamNonBlocking);
  return ss[dev];
}

static cudaStream_t capture_stream(int dev) {
  static cudaStream_t cs[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  if (!cs[dev]) cudaStreamCreateWithFlags(&cs[dev], cudaStreamNonBlocking);
  return cs[dev];
}

template <class F>
static int run_graphed(std::string key, cudaStream_t st, F &&body) {
  if (getenv("CSZI_NO_GRAPH")) return body(st);
  int dev = 0;
  cudaGetDevice(&dev);
  const void *sp = st;
  key.append(reinterpret_cast<const char *>(&sp), sizeof(sp));
  key.append(reinterpret_cast<const char *>(&dev), sizeof(dev));
  for (const char *e : {"CSZI_NO_TMA", "CSZI_NO_NZ"}) key.push_back(getenv(e) ? '1' : '0');
  std::lock_guard<std::mutex> lk(g_graph_mu);
  for (size_t i = 0; i < g_graphs.size(); ++i) {
    if (g_graphs[i].key == key) {
      GraphEntry e = g_graphs[i];
      g_graphs.erase(g_graphs.begin() + i);
      g_graphs.push_back(e);
      if (cudaGraphLaunch(e.exec, st) != cudaSuccess) return CSZI_E_CUDA;
      note_launch((int)e.launches);
      return CSZI_OK;
    }
  }
  cudaStream_t cs = capture_stream(dev);
  if (!cs) return body(st);
  const unsigned long long l0 = g_launches.load();
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaGetLastError();
    return body(st);
  }
  const int rc = body(cs);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
  const unsigned long long nl = g_launches.load() - l0;
  g_launches.fetch_sub(nl);  // captured, not executed
  if (rc != CSZI_OK || ec != cudaSuccess || !graph) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return rc != CSZI_OK ? rc : CSZI_E_CUDA;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) return CSZI_E_CUDA;
  if (g_graphs.size() >= GRAPH_CACHE) {
    cudaGraphExecDestroy(g_graphs.front().exec);
    g_graphs.erase(g_graphs.begin());
  }
  g_graphs.push_back({key, exec, nl});
  if (cudaGraphLaunch(exec, st) != cudaSuccess) return CSZI_E_CUDA;
  note_launch((int)nl);
  return CSZI_OK;
}

template <class T>
static void key_add(std::string &k, const T &v) {
  k.append(reinterpret_cast<const char *>(&v), sizeof(T));
}

}  // namespace cszi

using namespace cszi;

static double dmul_host(double a, double b) { return a * b; }  // exact (x2)

extern "C" {

const char *cszi_version(void) {
  return "libcszi 0.1 sm_100a (fp64 RN, no FMA contraction; decoupled look-back)";
}

uint64_t cszi_compress_workspace_size(const cszi_geom *g, int32_t radius, const cszi_caps *caps) {
  return layout_compress(g, radius, caps, nullptr, nullptr) + 256;
}

uint64_t cszi_payload_capacity(const cszi_geom *g, int32_t radius, const cszi_caps *caps) {
  const u64 raw = raw_capacity(g, radius, caps);
  return raw + raw / 128 + 64;
}

static int compress_body(const float *x, const cszi_geom *g, const cszi_params *p,
                         const cszi_caps *caps, int32_t pass2, int32_t range_done,
                         uint8_t *payload, void *workspace, uint64_t ws_bytes, cszi_ctl *ctl,
                         cudaStream_t st) {
  const int32_t R = p->radius;
  CK(check_geom(g, R));
  CompressWS W;
  const u64 need = layout_compress(g, R, caps, workspace, &W);
  if (ws_bytes < need) return CSZI_E_CAPACITY;
  const u64 n = grid_n(g);
  const u64 nbins = 2 * (u64)R;
  const u64 na = anchors_count(g);
  const u64 raw_cap = raw_capacity(g, R, caps);
  uint8_t *raw = pass2 ? W.raw : payload;
  bool anchors_done = false;
  if (!range_done) {
    CK(launch_ctl_init(ctl, st));
    // the sample gather and the anchor gather read only x: they run on a
    // side stream beside the range scan (a fork / join in the captured
    // graph), the decision waits for both
    cudaStream_t side = side_stream();
    cudaEvent_t fork = nullptr, join = nullptr;
    if (side) {
      cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    }
    if (side && fork && join) {
      cudaEventRecord(fork, st);
      cudaStreamWaitEvent(side, fork, 0);
      CK(launch_sample_gather(x, g, W.samples, side));
      CK(launch_gather_anchors(x, g, reinterpret_cast<float *>(raw), side));
      anchors_done = true;
      cudaEventRecord(join, side);
      CK(launch_range(x, n, ctl, st));
      cudaStreamWaitEvent(st, join, 0);
    } else {
      CK(launch_range(x, n, ctl, st));
      CK(launch_sample_gather(x, g, W.samples, st));
    }
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    CK(launch_tune_from_samples(W.samples, g, p, ctl, st, W.hist, (int)nbins));
  } else {
    // a prior range scan is kept; its output fields are reset by the sample gather
    CK(launch_tune(x, g, p, ctl, W.samples, st, true, W.hist, (int)nbins));
  }
  bool nz = false;
  CK(launch_predict(x, g, R, ctl, W.sym, W.hist, p->exact != 0, st, W.nzmap, &nz));
  if (!anchors_done) CK(launch_gather_anchors(x, g, reinterpret_cast<float *>(raw), st));
  uint8_t *lengths = raw + 4 * na;  // the codebook section is the length table
  CK(launch_codebook(W.hist, (int)nbins, lengths, W.words, ctl, st, true));
  const u64 head = 4 * na + nbins;
  // the bitstream is packed straight into its section when the section is
  // word-aligned (R even); otherwise into W.bits and copied by k_assemble
  const bool in_place = ((reinterpret_cast<uintptr_t>(raw) + head) & 3) == 0;
  uint32_t *bits_out = in_place ? reinterpret_cast<uint32_t *>(raw + head) : W.bits;
  CK(launch_encode(0, W.sym, n, R, lengths, W.words, bits_out, caps->bits_cap, x, W.oidx, W.oval,
                   caps->outlier_cap, W.enc_scratch, ctl, st, 0, 0, nz ? W.nzmap : nullptr,
                   W.hist, true));  // k_codebook already set ctl->bits
  k_assemble<<<grid_for(n / 16), 256, 0, st>>>(raw, head, reinterpret_cast<uint8_t *>(W.bits),
                                                W.oidx, nz ? nullptr : W.oval, x, raw_cap,
                                                caps->bits_cap,
                                                caps->outlier_cap, ctl, pass2 ? 0 : 1,
                                                in_place ? 1 : 0);
  note_launch();
  if (pass2) CK(launch_pass2_encode(raw, reinterpret_cast<const u64 *>(&ctl->raw_len), raw_cap, payload, W.p2_scratch, ctl, st));
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int cszi_compress(const float *x, const cszi_geom *g, const cszi_params *p,
                  const cszi_caps *caps, int32_t pass2, int32_t range_done, uint8_t *payload,
                  void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, void *stream) {
  if (!x || !g || !p || !caps || !ctl) return CSZI_E_INVALID_ARG;
  std::string k("C");
  for (const void *q : {(const void *)x, (const void *)payload, (const void *)workspace, (const void *)ctl})
    key_add(k, q);
  key_add(k, *g);
  key_add(k, *p);
  key_add(k, *caps);
  key_add(k, pass2);
  key_add(k, range_done);
  key_add(k, ws_bytes);
  return run_graphed(std::move(k), reinterpret_cast<cudaStream_t>(stream), [&](cudaStream_t st) {
    return compress_body(x, g, p, caps, pass2, range_done, payload, workspace, ws_bytes, ctl, st);
  });
}

uint64_t cszi_decompress_workspace_size(const cszi_geom *g, int32_t radius,
                                        const uint64_t sec_len[4], uint64_t payload_len) {
  return layout_decompress(g, radius, reinterpret_cast<const u64 *>(sec_len), payload_len, 1,
                           nullptr, nullptr) + 256;
}

static int decompress_body(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                           const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                           const double *level_eb, int32_t nlev, const int32_t variant[3],
                           const int32_t order[3], int32_t table_mode, float *y,
                           void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, cudaStream_t st) {
  CK(check_geom(g, radius));
  DecompressWS W;
  const u64 need = layout_decompress(g, radius, reinterpret_cast<const u64 *>(sec_len),
                                     payload_len, 1, workspace, &W);
  if (ws_bytes < need) return CSZI_E_CAPACITY;
  const u64 n = grid_n(g);
  const u64 nbins = 2 * (u64)radius;
  const u64 raw_len = sec_len[0] + sec_len[1] + sec_len[2] + sec_len[3];
  CK(launch_ctl_init(ctl, st));
  const uint8_t *raw = payload;
  if (pass2) {
    CK(launch_pass2_decode(payload, payload_len, W.raw, raw_len, W.p2_scratch, ctl, st, 1));
    raw = W.raw;
  }
  if (sec_len[1] != nbins) return CSZI_E_MALFORMED;
  const uint8_t *anchors = raw;
  const uint8_t *lengths = raw + sec_len[0];
  const uint8_t *bits = lengths + sec_len[1];
  const uint8_t *outl = bits + sec_len[2];
  // (the pass-2 raw-length check runs inside k_canonical)
  CK(launch_canonical(lengths, (int)nbins, nullptr, W.dec_tables, ctl, st, pass2 ? raw_len : 0));
  u64 w0 = 0;
  const u64 wn = sym_window(g, &w0);  // z-slab shard: only its symbol window
  CK(launch_decode(bits, sec_len[2], n, radius, W.dec_tables, W.sym, 0, W.dec_scratch, ctl, st,
                   table_mode, 32, w0, w0 + wn));
  const u64 kmax = sec_len[3] >= 8 ? (sec_len[3] - 8) / 12 : 0;
  k_outliers_parse<<<grid_for(kmax), 256, 0, st>>>(outl, sec_len[3], n, W.oidx, W.oval, W.sym,
                                                   ctl);
  note_launch();
  k_outliers_mark<<<grid_for(kmax), 256, 0, st>>>(W.oidx, ctl, n, W.sym, w0, w0 + wn);
  note_launch();
  // the anchor section is 4-byte aligned inside the decoded payload
  const float *anc = reinterpret_cast<const float *>(anchors);
  // the outlier count is device-resident (ctl->n_outliers, set by the parse)
  CK(launch_reconstruct(W.sym, anc, W.oidx, W.oval, kmax,
                        reinterpret_cast<const u64 *>(&ctl->n_outliers), g, radius, level_eb,
                        nlev, variant, order, y, st));
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int cszi_decompress(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                    const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                    const double *level_eb, int32_t nlev, const int32_t variant[3],
                    const int32_t order[3], int32_t table_mode, float *y, void *workspace,
                    uint64_t ws_bytes, cszi_ctl *ctl, void *stream) {
  if (!payload || !sec_len || !g || !level_eb || !variant || !order || !ctl || nlev < 0 ||
      nlev > CSZI_MAX_LEVELS)
    return CSZI_E_INVALID_ARG;
  std::string k("D");
  for (const void *q : {(const void *)payload, (const void *)y, (const void *)workspace, (const void *)ctl})
    key_add(k, q);
  key_add(k, payload_len);
  key_add(k, pass2);
  k.append(reinterpret_cast<const char *>(sec_len), 4 * sizeof(uint64_t));
  key_add(k, *g);
  key_add(k, radius);
  k.append(reinterpret_cast<const char *>(level_eb), nlev * sizeof(double));
  key_add(k, nlev);
  k.append(reinterpret_cast<const char *>(variant), 3 * sizeof(int32_t));
  k.append(reinterpret_cast<const char *>(order), 3 * sizeof(int32_t));
  key_add(k, table_mode);
  key_add(k, ws_bytes);
  return run_graphed(std::move(k), reinterpret_cast<cudaStream_t>(stream), [&](cudaStream_t st) {
    return decompress_body(payload, payload_len, pass2, sec_len, g, radius, level_eb, nlev,
                           variant, order, table_mode, y, workspace, ws_bytes, ctl, st);
  });
}

// ---- sharded decompress split by Huffman chunk ranges (distributed.py) ------
// The stages of cszi_decompress over one workspace (cszi_decompress_workspace_
// size): prologue (pass-2 decode + code tables), sync of a chunk range (the
// caller all-gathers X / K / D between ranks), write of the z-slab's symbol
// window, epilogue (outliers + reconstruction of the slab).
static const uint8_t *split_raw(const uint8_t *payload, int32_t pass2, const DecompressWS &W) {
  return pass2 ? W.raw : payload;
}

int cszi_decompress_prologue(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                             const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                             void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, void *stream) {
  if (!payload || !sec_len || !g || !ctl) return CSZI_E_INVALID_ARG;
  CK(check_geom(g, radius));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DecompressWS W;
  if (ws_bytes < layout_decompress(g, radius, reinterpret_cast<const u64 *>(sec_len), payload_len,
                                   1, workspace, &W))
    return CSZI_E_CAPACITY;
  const u64 nbins = 2 * (u64)radius;
  const u64 raw_len = sec_len[0] + sec_len[1] + sec_len[2] + sec_len[3];
  CK(launch_ctl_init(ctl, st));
  if (pass2) CK(launch_pass2_decode(payload, payload_len, W.raw, raw_len, W.p2_scratch, ctl, st, 1));
  if (sec_len[1] != nbins) return CSZI_E_MALFORMED;
  const uint8_t *lengths = split_raw(payload, pass2, W) + sec_len[0];
  CK(launch_canonical(lengths, (int)nbins, nullptr, W.dec_tables, ctl, st, pass2 ? raw_len : 0));
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

uint64_t cszi_huff_chunks(uint64_t nbytes) { return huff_chunks(nbytes); }

// the prologue for a raw payload already expanded into the workspace (the
// pass-2 decode split across ranks): ctl reset + code tables
int cszi_decompress_prologue_raw(uint64_t payload_len, const uint64_t sec_len[4],
                                 const cszi_geom *g, int32_t radius, void *workspace,
                                 uint64_t ws_bytes, cszi_ctl *ctl, void *stream) {
  if (!sec_len || !g || !ctl) return CSZI_E_INVALID_ARG;
  CK(check_geom(g, radius));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DecompressWS W;
  if (ws_bytes < layout_decompress(g, radius, reinterpret_cast<const u64 *>(sec_len), payload_len,
                                   1, workspace, &W))
    return CSZI_E_CAPACITY;
  const u64 nbins = 2 * (u64)radius;
  if (sec_len[1] != nbins) return CSZI_E_MALFORMED;
  CK(launch_ctl_init(ctl, st));
  CK(launch_canonical(W.raw + sec_len[0], (int)nbins, nullptr, W.dec_tables, ctl, st, 0));
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

uint64_t cszi_decompress_raw_offset(const cszi_geom *g, int32_t radius,
                                    const uint64_t sec_len[4], uint64_t payload_len) {
  DecompressWS W;
  unsigned char *base = reinterpret_cast<unsigned char *>((uintptr_t)4096);
  layout_decompress(g, radius, reinterpret_cast<const u64 *>(sec_len), payload_len, 1, base, &W);
  return (uint64_t)(W.raw - base);
}

uint64_t cszi_p2d_chunks(uint64_t n) { return p2d_chunks(n); }
uint64_t cszi_p2d_resolve_scratch_size(uint64_t n) { return p2d_resolve_scratch_bytes(n); }

int cszi_p2d_tables(const uint8_t *in, uint64_t n, uint64_t c0, uint64_t c1, uint8_t *tab,
                    uint32_t *ctab, void *stream) {
  if (!in || !tab || !ctab) return CSZI_E_INVALID_ARG;
  return launch_p2d_tables_range(in, n, c0, c1, tab, ctab, reinterpret_cast<cudaStream_t>(stream));
}

int cszi_p2d_resolve(const uint8_t *tab, const uint32_t *ctab, uint64_t n, uint8_t *E,
                     uint32_t *cnt, uint64_t *off, void *scratch, cszi_ctl *ctl, void *stream) {
  if (!tab || !ctab || !E || !cnt || !off || !scratch || !ctl) return CSZI_E_INVALID_ARG;
  return launch_p2d_resolve(tab, ctab, n, E, cnt, reinterpret_cast<u64 *>(off), scratch, ctl,
                            reinterpret_cast<cudaStream_t>(stream));
}

int cszi_p2d_expand(const uint8_t *in, uint64_t n, const uint8_t *E, const uint64_t *off,
                    const uint32_t *cnt, uint64_t c0, uint64_t c1, uint8_t *out, uint64_t cap,
                    cszi_ctl *ctl, void *stream) {
  if (!in || !E || !off || !cnt || !out || !ctl) return CSZI_E_INVALID_ARG;
  return launch_p2d_expand_range(in, n, E, reinterpret_cast<const u64 *>(off), cnt, c0, c1, out,
                                 cap, ctl, reinterpret_cast<cudaStream_t>(stream));
}

int cszi_decompress_sync_range(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                               const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                               uint64_t h0, uint64_t h1, uint64_t entry, uint64_t *X,
                               uint32_t *K, uint8_t *D, uint64_t *entry_used, void *workspace,
                               uint64_t ws_bytes, cszi_ctl *ctl, void *stream) {
  if (!payload || !sec_len || !g || !X || !K || !D || !ctl) return CSZI_E_INVALID_ARG;
  DecompressWS W;
  if (ws_bytes < layout_decompress(g, radius, reinterpret_cast<const u64 *>(sec_len), payload_len,
                                   1, workspace, &W))
    return CSZI_E_CAPACITY;
  const uint8_t *bits = split_raw(payload, pass2, W) + sec_len[0] + sec_len[1];
  return launch_huff_sync_range(bits, sec_len[2], W.dec_tables, h0, h1, entry,
                                reinterpret_cast<u64 *>(X), K, D,
                                reinterpret_cast<u64 *>(entry_used), W.dec_scratch, ctl,
                                reinterpret_cast<cudaStream_t>(stream));
}

int cszi_decompress_write_window(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                                 const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                                 const uint64_t *X, uint32_t *K, const uint8_t *D,
                                 void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, void *stream) {
  if (!payload || !sec_len || !g || !X || !K || !D || !ctl) return CSZI_E_INVALID_ARG;
  DecompressWS W;
  if (ws_bytes < layout_decompress(g, radius, reinterpret_cast<const u64 *>(sec_len), payload_len,
                                   1, workspace, &W))
    return CSZI_E_CAPACITY;
  const uint8_t *bits = split_raw(payload, pass2, W) + sec_len[0] + sec_len[1];
  u64 w0 = 0;
  const u64 wn = sym_window(g, &w0);
  return launch_huff_write_window(bits, sec_len[2], grid_n(g), radius, W.dec_tables,
                                  reinterpret_cast<const u64 *>(X), K, D, w0, w0 + wn, W.sym,
                                  W.dec_scratch, ctl, reinterpret_cast<cudaStream_t>(stream));
}

int cszi_decompress_epilogue(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                             const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                             const double *level_eb, int32_t nlev, const int32_t variant[3],
                             const int32_t order[3], float *y, void *workspace, uint64_t ws_bytes,
                             cszi_ctl *ctl, void *stream) {
  if (!payload || !sec_len || !g || !level_eb || !variant || !order || !y || !ctl)
    return CSZI_E_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DecompressWS W;
  if (ws_bytes < layout_decompress(g, radius, reinterpret_cast<const u64 *>(sec_len), payload_len,
                                   1, workspace, &W))
    return CSZI_E_CAPACITY;
  const uint8_t *raw = split_raw(payload, pass2, W);
  const uint8_t *outl = raw + sec_len[0] + sec_len[1] + sec_len[2];
  const u64 n = grid_n(g);
  u64 w0 = 0;
  const u64 wn = sym_window(g, &w0);
  const u64 kmax = sec_len[3] >= 8 ? (sec_len[3] - 8) / 12 : 0;
  k_outliers_parse<<<grid_for(kmax), 256, 0, st>>>(outl, sec_len[3], n, W.oidx, W.oval, W.sym,
                                                   ctl);
  note_launch();
  k_outliers_mark<<<grid_for(kmax), 256, 0, st>>>(W.oidx, ctl, n, W.sym, w0, w0 + wn);
  note_launch();
  CK(launch_reconstruct(W.sym, reinterpret_cast<const float *>(raw), W.oidx, W.oval, kmax,
                        reinterpret_cast<const u64 *>(&ctl->n_outliers), g, radius, level_eb,
                        nlev, variant, order, y, st));
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// ---- Lorenzo predictor (pipeline.py:123-150, 202-203) ----------------------
uint64_t cszi_compress_lorenzo_workspace_size(const cszi_geom *g, int32_t radius,
                                              const cszi_caps *caps) {
  return layout_compress_lz(g, radius, caps, nullptr, nullptr, nullptr) + 256;
}

static int lz_compress_body(const float *x, const cszi_geom *g, int32_t mode_rel, double eb,
                            int32_t R, const cszi_caps *caps, int32_t pass2, uint8_t *payload,
                            void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, cudaStream_t st) {
  CK(check_geom(g, R));
  CompressWS W;
  float *rec = nullptr;
  const u64 need = layout_compress_lz(g, R, caps, workspace, &W, &rec);
  if (ws_bytes < need) return CSZI_E_CAPACITY;
  const u64 n = grid_n(g);
  const u64 nbins = 2 * (u64)R;
  const u64 raw_cap = raw_capacity(g, R, caps);
  CK(launch_ctl_init(ctl, st));
  CK(launch_range(x, n, ctl, st));  // value_range (pipeline.py:124)
  CK(launch_lorenzo_eb(ctl, eb, mode_rel, R, st));
  CK(launch_lorenzo(0, x, rec, W.sym, g, ctl, 0.0, R, nullptr, nullptr, nullptr, 0, st));
  CK(launch_hist_sym(W.sym, n, R, W.hist, st));
  uint8_t *raw = pass2 ? W.raw : payload;
  uint8_t *lengths = raw;  // no anchor section
  CK(launch_codebook(W.hist, (int)nbins, lengths, W.words, ctl, st, true));
  const u64 head = nbins;
  const bool in_place = ((reinterpret_cast<uintptr_t>(raw) + head) & 3) == 0;
  uint32_t *bits_out = in_place ? reinterpret_cast<uint32_t *>(raw + head) : W.bits;
  CK(launch_encode(0, W.sym, n, R, lengths, W.words, bits_out, caps->bits_cap, x, W.oidx, W.oval,
                   caps->outlier_cap, W.enc_scratch, ctl, st, 0, 0, nullptr, W.hist, true));
  k_assemble<<<grid_for(n / 16), 256, 0, st>>>(raw, head, reinterpret_cast<uint8_t *>(W.bits),
                                                W.oidx, W.oval, x, raw_cap, caps->bits_cap,
                                                caps->outlier_cap, ctl, pass2 ? 0 : 1,
                                                in_place ? 1 : 0);
  note_launch();
  if (pass2)
    CK(launch_pass2_encode(raw, reinterpret_cast<const u64 *>(&ctl->raw_len), raw_cap, payload,
                           W.p2_scratch, ctl, st));
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int cszi_compress_lorenzo(const float *x, const cszi_geom *g, int32_t mode_rel, double eb,
                          int32_t radius, const cszi_caps *caps, int32_t pass2, uint8_t *payload,
                          void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, void *stream) {
  if (!x || !g || !caps || !ctl || !payload) return CSZI_E_INVALID_ARG;
  std::string k("L");
  for (const void *q : {(const void *)x, (const void *)payload, (const void *)workspace,
                        (const void *)ctl})
    key_add(k, q);
  key_add(k, *g);
  key_add(k, mode_rel);
  key_add(k, eb);
  key_add(k, radius);
  key_add(k, *caps);
  key_add(k, pass2);
  key_add(k, ws_bytes);
  return run_graphed(std::move(k), reinterpret_cast<cudaStream_t>(stream), [&](cudaStream_t st) {
    return lz_compress_body(x, g, mode_rel, eb, radius, caps, pass2, payload, workspace,
                            ws_bytes, ctl, st);
  });
}

static int lz_decompress_body(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                              const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                              double eb_abs, int32_t table_mode, float *y, void *workspace,
                              uint64_t ws_bytes, cszi_ctl *ctl, cudaStream_t st) {
  CK(check_geom(g, radius));
  DecompressWS W;
  const u64 need = layout_decompress(g, radius, reinterpret_cast<const u64 *>(sec_len),
                                     payload_len, 1, workspace, &W);
  if (ws_bytes < need) return CSZI_E_CAPACITY;
  const u64 n = grid_n(g);
  const u64 nbins = 2 * (u64)radius;
  const u64 raw_len = sec_len[0] + sec_len[1] + sec_len[2] + sec_len[3];
  if (sec_len[1] != nbins) return CSZI_E_MALFORMED;
  CK(launch_ctl_init(ctl, st));
  const uint8_t *raw = payload;
  if (pass2) {
    CK(launch_pass2_decode(payload, payload_len, W.raw, raw_len, W.p2_scratch, ctl, st, 1));
    raw = W.raw;
  }
  // an anchor section, if a crafted archive carries one, is ignored as the
  // reference ignores it for Lorenzo archives
  const uint8_t *lengths = raw + sec_len[0];
  const uint8_t *bits = lengths + sec_len[1];
  const uint8_t *outl = bits + sec_len[2];
  CK(launch_canonical(lengths, (int)nbins, nullptr, W.dec_tables, ctl, st, pass2 ? raw_len : 0));
  CK(launch_decode(bits, sec_len[2], n, radius, W.dec_tables, W.sym, 0, W.dec_scratch, ctl, st,
                   table_mode, 32, 0, n));
  const u64 kmax = sec_len[3] >= 8 ? (sec_len[3] - 8) / 12 : 0;
  k_outliers_parse<<<grid_for(kmax), 256, 0, st>>>(outl, sec_len[3], n, W.oidx, W.oval, W.sym,
                                                   ctl);
  note_launch();
  k_outliers_mark<<<grid_for(kmax), 256, 0, st>>>(W.oidx, ctl, n, W.sym, 0, n);
  note_launch();
  CK(launch_lorenzo(1, nullptr, y, W.sym, g, ctl, dmul_host(2.0, eb_abs), radius, W.oidx, W.oval,
                    reinterpret_cast<const u64 *>(&ctl->n_outliers), 0, st));
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int cszi_decompress_lorenzo(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                            const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                            double eb_abs, int32_t table_mode, float *y, void *workspace,
                            uint64_t ws_bytes, cszi_ctl *ctl, void *stream) {
  if (!payload || !sec_len || !g || !ctl || !y) return CSZI_E_INVALID_ARG;
  std::string k("M");
  for (const void *q : {(const void *)payload, (const void *)y, (const void *)workspace,
                        (const void *)ctl})
    key_add(k, q);
  key_add(k, payload_len);
  key_add(k, pass2);
  k.append(reinterpret_cast<const char *>(sec_len), 4 * sizeof(uint64_t));
  key_add(k, *g);
  key_add(k, radius);
  key_add(k, eb_abs);
  key_add(k, table_mode);
  key_add(k, ws_bytes);
  return run_graphed(std::move(k), reinterpret_cast<cudaStream_t>(stream), [&](cudaStream_t st) {
    return lz_decompress_body(payload, payload_len, pass2, sec_len, g, radius, eb_abs, table_mode,
                              y, workspace, ws_bytes, ctl, st);
  });
}

// lorenzo_predict_quantize (lorenzo.py:22-33): x -> symbols (q + R, 0 for an
// outlier); rec: float[n] scratch
int cszi_lorenzo_predict(const float *x, const cszi_geom *g, double eb_abs, int32_t radius,
                         uint16_t *sym, float *rec, cszi_ctl *ctl, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(check_geom(g, radius));
  CK(launch_ctl_init(ctl, st));
  CK(launch_lorenzo_eb(ctl, eb_abs, 0, radius, st));
  return launch_lorenzo(0, x, rec, sym, g, ctl, 0.0, radius, nullptr, nullptr, nullptr, 0, st);
}

// lorenzo_reconstruct (lorenzo.py:36-53): symbols (0xFFFF at outliers) -> y
int cszi_lorenzo_reconstruct(const uint16_t *sym, const uint64_t *out_idx, const float *out_val,
                             uint64_t n_out, const cszi_geom *g, double eb_abs, int32_t radius,
                             float *y, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!g || !sym || !y) return CSZI_E_INVALID_ARG;
  if (radius < 1 || radius > 32767) return CSZI_E_INVALID_ARG;
  return launch_lorenzo(1, nullptr, y, const_cast<uint16_t *>(sym), g, nullptr,
                        dmul_host(2.0, eb_abs), radius, reinterpret_cast<const u64 *>(out_idx),
                        out_val, nullptr, n_out, st);
}

int cszi_ctl_fetch(const cszi_ctl *ctl, cszi_ctl *host, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(host, ctl, sizeof(cszi_ctl), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return CSZI_E_CUDA;
  return CSZI_OK;
}

int cszi_ctl_init(cszi_ctl *ctl, void *stream) {
  return launch_ctl_init(ctl, reinterpret_cast<cudaStream_t>(stream));
}

int cszi_range(const float *x, uint64_t n, cszi_ctl *ctl, void *stream) {
  return launch_range(x, n, ctl, reinterpret_cast<cudaStream_t>(stream));
}

int cszi_scan_field(const float *x, uint64_t n, cszi_ctl *ctl, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(launch_ctl_init(ctl, st));
  return launch_range(x, n, ctl, st);
}

int cszi_tune(const float *x, const cszi_geom *g, const cszi_params *p, int32_t *samples,
              cszi_ctl *ctl, void *stream) {
  CK(check_geom(g, p->radius));
  return launch_tune(x, g, p, ctl, samples, reinterpret_cast<cudaStream_t>(stream));
}

int cszi_sample_gather(const float *x, const cszi_geom *g, int32_t *vals, void *stream) {
  return launch_sample_gather(x, g, vals, reinterpret_cast<cudaStream_t>(stream));
}

int cszi_tune_from_samples(const int32_t *vals, const cszi_geom *g, const cszi_params *p,
                           cszi_ctl *ctl, void *stream) {
  CK(check_geom(g, p->radius));
  return launch_tune_from_samples(vals, g, p, ctl, reinterpret_cast<cudaStream_t>(stream));
}

// ---- sharded compress glue (distributed.py) --------------------------------
int cszi_shard_scan(const float *x, uint64_t n_own, uint64_t flat0, const cszi_geom *g,
                    cszi_ctl *ctl, int64_t *keys, int32_t *samples, void *stream) {
  if (!g || !ctl || !keys || !samples || (n_own && !x)) return CSZI_E_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(launch_ctl_init(ctl, st));
  if (n_own) {
    CK(launch_range(x, n_own, ctl, st));
    CK(launch_sample_gather(x, g, samples, st));
  } else {
    cudaMemsetAsync(samples, 0, sizeof(int32_t) * CSZI_SAMPLE_WORDS, st);
  }
  k_shard_keys<<<1, 32, 0, st>>>(ctl, flat0, keys);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int cszi_shard_set_range(cszi_ctl *ctl, const int64_t *keys, void *stream) {
  if (!ctl || !keys) return CSZI_E_INVALID_ARG;
  k_shard_set_range<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(ctl, keys);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int cszi_shard_piece_bits(const uint64_t *hist, const uint8_t *lengths, int32_t nbins,
                          int64_t *out, void *stream) {
  if (!hist || !lengths || !out || nbins < 1) return CSZI_E_INVALID_ARG;
  k_shard_piece_bits<<<1, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const u64 *>(hist), lengths, nbins, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int cszi_shard_counts(const cszi_ctl *ctl, int64_t *out, void *stream) {
  if (!ctl || !out) return CSZI_E_INVALID_ARG;
  k_shard_counts<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(ctl, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int cszi_shard_assemble(int32_t np, const float *const *anchors, const uint64_t *na,
                        const uint8_t *lengths, int32_t nbins, const uint8_t *const *bits,
                        const uint64_t *bit0, const uint64_t *nbits,
                        const uint64_t *const *oidx, const float *const *oval,
                        const uint64_t *nout, int32_t pass2, uint8_t *raw, uint64_t raw_cap,
                        uint8_t *payload, void *workspace, uint64_t ws_bytes, cszi_ctl *ctl,
                        void *stream) {
  if (np < 1 || !anchors || !na || !lengths || !bits || !bit0 || !nbits || !oidx || !oval ||
      !nout || !raw || !ctl || (pass2 && (!payload || !workspace)))
    return CSZI_E_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  u64 off = 0, total_bits = 0, kt = 0;
  for (int i = 0; i < np; ++i) {
    total_bits += nbits[i];
    kt += nout[i];
    off += 4 * na[i];
  }
  const u64 head = off + (u64)nbins;
  const u64 nbytes = (total_bits + 7) / 8;
  const u64 words = (total_bits + 31) / 32 + 1;
  const u64 raw_len = head + nbytes + 8 + 12 * kt;
  if (head + 4 * words > raw_cap || raw_len > raw_cap) return CSZI_E_CAPACITY;
  if (pass2 && ws_bytes < p2enc_scratch_bytes(raw_len)) return CSZI_E_CAPACITY;
  off = 0;
  for (int i = 0; i < np; ++i) {
    if (na[i]) cudaMemcpyAsync(raw + off, anchors[i], 4 * na[i], cudaMemcpyDeviceToDevice, st);
    off += 4 * na[i];
  }
  cudaMemcpyAsync(raw + off, lengths, (size_t)nbins, cudaMemcpyDeviceToDevice, st);
  // bit pieces: each was packed at its global bit phase (distributed.py), so
  // a word-aligned section takes them as whole words, ORed at their word
  // offsets (a piece's first and last words are shared with its neighbours)
  cudaMemsetAsync(raw + head, 0, 4 * words, st);
  const bool aligned = ((reinterpret_cast<uintptr_t>(raw) + head) & 3) == 0;
  for (int i = 0; i < np; ++i) {
    if (!nbits[i]) continue;
    const u64 ph = bit0[i] & 31;
    if (aligned) {
      const u64 nw = (ph + nbits[i] + 31) / 32;
      u64 blocks = (nw + 255) / 256;
      if (blocks > 4096) blocks = 4096;
      k_or_words<<<(unsigned)blocks, 256, 0, st>>>(
          reinterpret_cast<uint32_t *>(raw + head) + bit0[i] / 32,
          reinterpret_cast<const uint32_t *>(bits[i]), nw);
      note_launch();
    } else {  // odd R: the section is not word-aligned; shift the pieces in
      CK(launch_concat_bits(raw + head, bit0[i] - ph, bits[i], ph + nbits[i], st));
    }
  }
  // outlier section: count, then the pieces' (index, value) records
  uint8_t *os = raw + head + nbytes;
  u64 r0 = 0;
  for (int i = 0; i < np; ++i) {
    if (nout[i]) {
      k_shard_records<<<grid_for(nout[i]), 256, 0, st>>>(
          reinterpret_cast<const u64 *>(oidx[i]), oval[i], nout[i], os + 8 + 12 * r0);
      note_launch();
    }
    r0 += nout[i];
  }
  k_shard_tail<<<1, 32, 0, st>>>(os, kt, raw_len, pass2 ? 0 : 1, ctl);
  note_launch();
  if (pass2)
    CK(launch_pass2_encode(raw, reinterpret_cast<const u64 *>(&ctl->raw_len), raw_len, payload,
                           workspace, ctl, st));
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int cszi_find_cuts(const uint8_t *bytes, uint64_t lo, uint64_t hi, int64_t *out, void *stream) {
  if (!bytes || !out) return CSZI_E_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long *fl = reinterpret_cast<unsigned long long *>(out + 2);  // scratch
  const unsigned long long init[2] = {~0ull, 0ull};
  cudaMemcpyAsync(fl, init, sizeof(init), cudaMemcpyHostToDevice, st);
  if (hi > lo + 2) {
    k_find_cuts<<<grid_for(hi - lo), 256, 0, st>>>(bytes, lo, hi, fl, fl + 1);
    note_launch();
  }
  k_cuts_out<<<1, 1, 0, st>>>(fl, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

uint64_t cszi_slab_anchor_count(const cszi_geom *g) { return slab_anchor_count(g); }

uint64_t cszi_encode_sym_workspace_size(uint64_t n) { return enc_scratch_bytes(n) + 256; }

int cszi_encode_sym_at(const uint16_t *sym, uint64_t n, int32_t radius, const uint8_t *lengths,
                       const uint32_t *words, const float *x, uint64_t idx_offset,
                       uint32_t bit_base, uint8_t *out, uint64_t cap_bytes, uint64_t *out_idx,
                       float *out_val, uint64_t out_cap, void *workspace, cszi_ctl *ctl,
                       void *stream) {
  if ((reinterpret_cast<uintptr_t>(out) & 3) || bit_base > 31) return CSZI_E_INVALID_ARG;
  return launch_encode(0, sym, n, radius, lengths, words, reinterpret_cast<uint32_t *>(out),
                       cap_bytes, x, reinterpret_cast<u64 *>(out_idx), out_val, out_cap,
                       workspace, ctl, reinterpret_cast<cudaStream_t>(stream), idx_offset,
                       bit_base);
}

int cszi_encode_sym_nz(const uint16_t *sym, uint64_t n, int32_t radius, const uint8_t *lengths,
                       const uint32_t *words, const float *x, uint64_t idx_offset,
                       uint32_t bit_base, uint8_t *out, uint64_t cap_bytes, uint64_t *out_idx,
                       float *out_val, uint64_t out_cap, const uint32_t *nzmap,
                       const uint64_t *hist, void *workspace, cszi_ctl *ctl, void *stream) {
  if ((reinterpret_cast<uintptr_t>(out) & 3) || bit_base > 31 || !nzmap || !hist)
    return CSZI_E_INVALID_ARG;
  return launch_encode(0, sym, n, radius, lengths, words, reinterpret_cast<uint32_t *>(out),
                       cap_bytes, x, reinterpret_cast<u64 *>(out_idx), out_val, out_cap,
                       workspace, ctl, reinterpret_cast<cudaStream_t>(stream), idx_offset,
                       bit_base, nzmap, reinterpret_cast<const u64 *>(hist), false);
}

int cszi_encode_sym(const uint16_t *sym, uint64_t n, int32_t radius, const uint8_t *lengths,
                    const uint32_t *words, const float *x, uint64_t idx_offset, uint8_t *out,
                    uint64_t cap_bytes, uint64_t *out_idx, float *out_val, uint64_t out_cap,
                    void *workspace, cszi_ctl *ctl, void *stream) {
  return cszi_encode_sym_at(sym, n, radius, lengths, words, x, idx_offset, 0, out, cap_bytes,
                            out_idx, out_val, out_cap, workspace, ctl, stream);
}

int cszi_concat_bits(uint8_t *dst, uint64_t dst_bit, const uint8_t *src, uint64_t nbits,
                     void *stream) {
  return launch_concat_bits(dst, dst_bit, src, nbits, reinterpret_cast<cudaStream_t>(stream));
}

int cszi_pack_outliers(const uint64_t *idx, const float *val, uint64_t k, uint8_t *out,
                       void *stream) {
  return launch_pack_outliers(reinterpret_cast<const u64 *>(idx), val, k, out,
                              reinterpret_cast<cudaStream_t>(stream));
}

int cszi_predict(const float *x, const cszi_geom *g, int32_t radius, int32_t exact,
                 uint16_t *sym, uint64_t *hist, cszi_ctl *ctl, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(check_geom(g, radius));
  cudaMemsetAsync(hist, 0, 8 * 2 * (size_t)radius, st);
  return launch_predict(x, g, radius, ctl, sym, reinterpret_cast<u64 *>(hist), exact != 0, st);
}

int cszi_predict_nz(const float *x, const cszi_geom *g, int32_t radius, int32_t exact,
                    uint16_t *sym, uint64_t *hist, uint32_t *nzmap, int32_t *nz_done,
                    cszi_ctl *ctl, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(check_geom(g, radius));
  cudaMemsetAsync(hist, 0, 8 * 2 * (size_t)radius, st);
  bool nz = false;
  const int rc = launch_predict(x, g, radius, ctl, sym, reinterpret_cast<u64 *>(hist), exact != 0,
                                st, nzmap, &nz);
  if (nz_done) *nz_done = nz ? 1 : 0;
  return rc;
}

int cszi_reconstruct(const uint16_t *sym, const float *anchors, const uint64_t *out_idx,
                     const float *out_val, uint64_t n_out, const cszi_geom *g, int32_t radius,
                     const double *level_eb, int32_t nlev, const int32_t variant[3],
                     const int32_t order[3], float *y, void *stream) {
  CK(check_geom(g, radius));
  return launch_reconstruct(sym, anchors, reinterpret_cast<const u64 *>(out_idx), out_val, n_out,
                            nullptr, g, radius, level_eb, nlev, variant, order, y,
                            reinterpret_cast<cudaStream_t>(stream));
}

int cszi_interp_level(float *recon, const float *source, int32_t *codes, uint8_t *is_outlier,
                      const float *outlier_values, const float *anchor_block, const cszi_geom *g,
                      int64_t stride, double level_eb, const int32_t variant[3],
                      const int32_t order[3], int32_t radius, int32_t mode, void *stream) {
  if (!g || g->rank < 1 || g->rank > 3 || !recon || !codes || !is_outlier || !anchor_block ||
      (mode == 0 && !source) || (mode == 1 && !outlier_values))
    return CSZI_E_INVALID_ARG;
  return launch_interp_level(recon, source, codes, is_outlier, outlier_values, anchor_block, g,
                             stride, level_eb, variant, order, radius, mode,
                             reinterpret_cast<cudaStream_t>(stream));
}

int cszi_gather_anchors(const float *x, const cszi_geom *g, float *out, void *stream) {
  return launch_gather_anchors(x, g, out, reinterpret_cast<cudaStream_t>(stream));
}

int cszi_histogram_i32(const int32_t *codes, uint64_t n, int32_t radius, uint64_t *counts,
                       cszi_ctl *ctl, void *stream) {
  if (radius < 1) return CSZI_E_INVALID_ARG;
  return launch_hist_i32(codes, n, radius, reinterpret_cast<u64 *>(counts), ctl,
                         reinterpret_cast<cudaStream_t>(stream));
}

int cszi_codebook(const uint64_t *counts, uint32_t nbins, uint8_t *lengths, uint32_t *words,
                  cszi_ctl *ctl, void *stream) {
  return launch_codebook(reinterpret_cast<const u64 *>(counts), (int)nbins, lengths, words, ctl,
                         reinterpret_cast<cudaStream_t>(stream));
}

uint64_t cszi_dec_tables_size(uint32_t nbins) { return dec_tables_bytes((int)nbins); }

int cszi_canonical(const uint8_t *lengths, uint32_t nbins, uint32_t *words, void *dec_tables,
                   cszi_ctl *ctl, void *stream) {
  return launch_canonical(lengths, (int)nbins, words, dec_tables, ctl,
                          reinterpret_cast<cudaStream_t>(stream));
}

uint64_t cszi_huff_encode_workspace_size(uint64_t n) { return enc_scratch_bytes(n) + 256; }

int cszi_huff_encode_i32(const int32_t *codes, uint64_t n, int32_t radius,
                         const uint8_t *lengths, const uint32_t *words, uint8_t *out,
                         uint64_t cap, void *workspace, cszi_ctl *ctl, void *stream) {
  if (reinterpret_cast<uintptr_t>(out) & 3) return CSZI_E_INVALID_ARG;
  return launch_encode(1, codes, n, radius, lengths, words, reinterpret_cast<uint32_t *>(out),
                       cap, nullptr, nullptr, nullptr, 0, workspace, ctl,
                       reinterpret_cast<cudaStream_t>(stream), 0);
}

uint64_t cszi_huff_decode_workspace_size(uint64_t nbytes, int32_t table_mode) {
  return dec_scratch_bytes(nbytes, table_mode) + 256;
}

int cszi_huff_decode_i32(const uint8_t *stream_bytes, uint64_t nbytes, uint64_t n,
                         int32_t radius, const void *dec_tables, int32_t *codes,
                         int32_t table_mode, int32_t lmax, void *workspace, cszi_ctl *ctl,
                         void *stream) {
  return launch_decode(stream_bytes, nbytes, n, radius, dec_tables, codes, 1, workspace, ctl,
                       reinterpret_cast<cudaStream_t>(stream), table_mode, lmax, 0, n);
}

uint64_t cszi_pass2_encode_workspace_size(uint64_t n) { return p2enc_scratch_bytes(n) + 256; }

int cszi_pass2_encode(const uint8_t *in, const uint64_t *n_dev, uint64_t n, uint8_t *out,
                      void *workspace, cszi_ctl *ctl, void *stream) {
  return launch_pass2_encode(in, reinterpret_cast<const u64 *>(n_dev), n, out, workspace, ctl,
                             reinterpret_cast<cudaStream_t>(stream));
}

uint64_t cszi_pass2_decode_workspace_size(uint64_t n) { return p2dec_scratch_bytes(n) + 256; }

int cszi_pass2_decode(const uint8_t *in, uint64_t n, uint8_t *out, uint64_t cap,
                      int32_t expand, void *workspace, cszi_ctl *ctl, void *stream) {
  return launch_pass2_decode(in, n, out, cap, workspace, ctl,
                             reinterpret_cast<cudaStream_t>(stream), expand);
}

}  // extern "C"

extern "C" {
// ABI self-check for bindings: sizes of the shared structs.
uint64_t cszi_launch_count(void) { return g_launches.load(); }

void cszi_abi_sizes(uint64_t out[4]) {
  out[0] = sizeof(cszi_geom);
  out[1] = sizeof(cszi_params);
  out[2] = sizeof(cszi_caps);
  out[3] = sizeof(cszi_ctl);
}
}
