/*
 * cszi.h — C ABI of libcszi.so, the B200-native (sm_100a) cuSZ-i hot path.
 *
 * The reference package (ebcomp, pure Python + numba) has no native FFI; its
 * drop-in boundary is the Python API  ebcomp.compress / ebcomp.decompress
 * (pkg/src/ebcomp/pipeline.py:66-78, :166).  Each entry point below replaces
 * one stage of that path and cites the reference function whose semantics it
 * reproduces bit-for-bit.  The Python host layer (paper_2312_05492_b200/) is
 * the only caller; see INTEGRATION.md for the ctypes binding.
 *
 * Conventions
 *  - extern "C", no exceptions cross the ABI; every function returns an int
 *    status (CSZI_OK or a negative CSZI_E_* code; the E_* codes map 1:1 onto
 *    the ebcomp.errors classes, CSZI_E_CUDA is a CUDA runtime failure).
 *  - All device pointers are caller-owned (torch tensors on the host side);
 *    scratch comes from a caller-provided workspace sized by the matching
 *    *_workspace_size() query.  Sizes and indices are 64-bit everywhere.
 *  - Every call is stream-ordered on the caller's cudaStream_t (passed as
 *    void*) and returns without synchronising; results that are data
 *    dependent (bit counts, outlier counts, payload length, tuned config,
 *    error flags) are written into a device-resident cszi_ctl record that
 *    the caller copies back once at the end.
 *  - Grids are 1..3-D float32, C order, slowest axis first (grid.py:19-38).
 *    Internally a rank-r grid is padded to 3-D with leading extent-1 axes.
 */
#ifndef CSZI_H
#define CSZI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:8-95) ------------------------------------- */
#define CSZI_OK 0
#define CSZI_E_NONFINITE (-1)        /* NonFiniteValue      grid.py:60-62     */
#define CSZI_E_INCONSISTENT (-2)     /* Inconsistent        predictor.py:150  */
#define CSZI_E_LENGTH_OVERFLOW (-3)  /* LengthOverflow      huffman.py:97     */
#define CSZI_E_EMPTY_HISTOGRAM (-4)  /* EmptyHistogram      huffman.py:82     */
#define CSZI_E_TRUNCATED (-5)        /* TruncatedStream     huffman.py:200    */
#define CSZI_E_CORRUPT (-6)          /* Corrupt             pass2.py:80       */
#define CSZI_E_MALFORMED (-7)        /* MalformedSection    archive.py:195    */
#define CSZI_E_UNKNOWN_SYMBOL (-8)   /* UnknownSymbol       huffman.py:176    */
#define CSZI_E_OUT_OF_RANGE (-9)     /* OutOfRange          huffman.py:71     */
#define CSZI_E_LENGTH_MISMATCH (-10) /* LengthMismatch      archive.py:155    */
#define CSZI_E_OUTLIER_INDEX (-11)   /* outlier index >= n (numpy IndexError) */
#define CSZI_E_INVALID_ARG (-20)
#define CSZI_E_UNSUPPORTED (-21)
#define CSZI_E_CAPACITY (-22) /* a caller buffer is smaller than the data */
#define CSZI_E_CUDA (-30)

/* Bits of cszi_ctl.flags (device-detected conditions; host raises in the
 * reference's check order). */
#define CSZI_F_NONFINITE (1u << 0)
#define CSZI_F_EB_NONPOSITIVE (1u << 1)
#define CSZI_F_LENGTH_OVERFLOW (1u << 2)
#define CSZI_F_EMPTY_HISTOGRAM (1u << 3)
#define CSZI_F_TRUNCATED (1u << 4)
#define CSZI_F_P2_CORRUPT (1u << 5)
#define CSZI_F_P2_LENGTH (1u << 6)
#define CSZI_F_OUTLIER_COUNT (1u << 7)
#define CSZI_F_OUTLIER_ORDER (1u << 8)
#define CSZI_F_OUTLIER_INDEX (1u << 9)
#define CSZI_F_CAPACITY (1u << 10)
#define CSZI_F_UNKNOWN_SYMBOL (1u << 11)

#define CSZI_MAX_LEVELS 16

/* Padded-3D geometry of one grid plus its predictor layout
 * (predictor.py:79-105 ChunkLayout, pipeline.py:159-163 _layout_for). */
typedef struct cszi_geom {
  int32_t rank;        /* 1..3 (original rank)                            */
  int32_t pad_;
  int64_t ext[3];      /* padded extents, slowest first                   */
  int64_t stride;      /* anchor stride S (power of two)                  */
  int64_t tile[3];     /* super-chunk tile per padded axis (1 if padded)  */
  int64_t slab[2];     /* owned global z range [z0, z1) of a z-slab shard;
                          {0, 0} = the whole grid.  Shard buffers hold planes
                          [z0, min(z1 + 1, ext[0])) (one closing halo plane);
                          3-D default layout only.                          */
} cszi_geom;

/* Host-provided compression parameters (pipeline.py:66-101). */
typedef struct cszi_params {
  int32_t mode_rel;        /* 1 = "rel", 0 = "abs"                         */
  int32_t radius;          /* quant_radius R (>= 2)                        */
  double eb;               /* eb as given                                  */
  int32_t have_alpha;      /* alpha known on the host (override or rel)    */
  int32_t have_variants;   /* variants override                            */
  int32_t have_order;      /* dim_order override                           */
  int32_t pad_;
  double alpha;            /* used when have_alpha                          */
  double alpha_pow[CSZI_MAX_LEVELS]; /* alpha ** (level-1), level = 1..    */
  int32_t variant[3];      /* padded-axis variants (override)               */
  int32_t order[3];        /* padded-axis dim order (override), rank items  */
  int32_t exact;           /* 1: force the true-division quantizer          */
  int32_t pad2_;
} cszi_params;

/* Device-resident control record: written by kernels, copied back once.  */
typedef struct cszi_ctl {
  /* range reduction (grid.py:104-108, grid.py:60-62) */
  uint32_t vmin_key;       /* order-preserving float keys (atomicMin/Max)  */
  uint32_t vmax_key;
  uint64_t first_nonfinite; /* UINT64_MAX when every value is finite        */
  /* tuned configuration (tuning.py:93-129) */
  double vmin, vmax, rng;
  double eb_abs, alpha;
  double level_eb[CSZI_MAX_LEVELS]; /* coarse -> fine                       */
  double inv_e2[CSZI_MAX_LEVELS];   /* 1 / (2 * level_eb)                  */
  double err_sum[3][2];
  int64_t sample_count[3];
  int32_t variant[3];      /* padded-axis variants                          */
  int32_t order[3];        /* padded-axis pass order (rank items used)      */
  int32_t nlev;
  int32_t radius;
  /* entropy stage */
  uint64_t bits;           /* Huffman bitstream length in bits              */
  uint64_t n_outliers;
  uint64_t raw_len;        /* sections concatenated (pre pass-2)            */
  uint64_t payload_len;    /* stored payload (post pass-2)                  */
  uint64_t decoded_symbols;
  uint32_t flags;          /* CSZI_F_* */
  uint32_t max_len;        /* longest code length                           */
  uint64_t scratch[8];
} cszi_ctl;

/* ---- whole-path entry points ------------------------------------------ */

/* Capacities for data-dependent outputs.  If a run overflows one of them,
 * CSZI_F_CAPACITY is set and the caller retries with larger values (the
 * worst case is bits_cap = 4*n bytes, outlier_cap = n). */
typedef struct cszi_caps {
  uint64_t bits_cap;     /* bytes for the Huffman bitstream              */
  uint64_t outlier_cap;  /* outlier records                               */
} cszi_caps;

/* Workspace bytes for cszi_compress on a grid of this geometry. */
uint64_t cszi_compress_workspace_size(const cszi_geom *g, int32_t radius, const cszi_caps *caps);

/* Device payload capacity (bytes) for cszi_compress. */
uint64_t cszi_payload_capacity(const cszi_geom *g, int32_t radius, const cszi_caps *caps);

/*
 * compress — pipeline.py:66-156 for predictor="interp", pass-2 codec 0.
 * x: device float32[n].  range_done != 0: ctl already holds the range and
 * finite scan of x (cszi_range ran at Grid construction) — only the output
 * fields are reset.  Writes the stored payload (pass-2 encoded when
 * pass2 != 0, else the raw section concatenation) to `payload`, and the
 * tuned config, section lengths (ctl->bits, n_outliers, raw_len,
 * payload_len) and CSZI_F_* flags to ctl.
 */
int cszi_compress(const float *x, const cszi_geom *g, const cszi_params *p,
                  const cszi_caps *caps, int32_t pass2, int32_t range_done, uint8_t *payload,
                  void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, void *stream);

/* Workspace bytes for cszi_decompress. */
uint64_t cszi_decompress_workspace_size(const cszi_geom *g, int32_t radius,
                                        const uint64_t sec_len[4], uint64_t payload_len);

/*
 * decompress — pipeline.py:166-204 (predictor="interp").
 * payload: device bytes of the stored payload; sec_len: the four
 * pre-pass-2 section lengths from the header; level_eb: eb_abs /
 * alpha ** (level-1) coarse -> fine (computed by the host as plan_levels
 * does); variant/order: padded-axis ids.  table_mode != 0 forces the exact
 * transfer-table Huffman decode (used when ctl->scratch[1] reports that the
 * speculative decode did not converge).  Writes y (float32[n]).
 */
int cszi_decompress(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                    const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                    const double *level_eb, int32_t nlev, const int32_t variant[3],
                    const int32_t order[3], int32_t table_mode, float *y, void *workspace,
                    uint64_t ws_bytes, cszi_ctl *ctl, void *stream);

/* ---- Lorenzo predictor (pipeline.py:123-150 / :202-203, lorenzo.py) ----
 * compress(predictor="lorenzo"): range scan, eb_abs (rel: eb * range when
 * the range is positive, else eb), the Lorenzo recurrence (wavefront tiles
 * on the GPU, bit-exact with _kernels.py:104-215), histogram, codebook,
 * Huffman, sections (no anchor section) and pass-2.  ctl->eb_abs, bits,
 * n_outliers, payload_len and flags as for cszi_compress.  The payload
 * capacity of cszi_payload_capacity() suffices. */
uint64_t cszi_compress_lorenzo_workspace_size(const cszi_geom *g, int32_t radius,
                                              const cszi_caps *caps);
int cszi_compress_lorenzo(const float *x, const cszi_geom *g, int32_t mode_rel, double eb,
                          int32_t radius, const cszi_caps *caps, int32_t pass2, uint8_t *payload,
                          void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, void *stream);
/* decompress of a Lorenzo archive (an anchor section is ignored); workspace size:
 * cszi_decompress_workspace_size(). */
int cszi_decompress_lorenzo(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                            const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                            double eb_abs, int32_t table_mode, float *y, void *workspace,
                            uint64_t ws_bytes, cszi_ctl *ctl, void *stream);
/* lorenzo_predict_quantize (lorenzo.py:22-33): symbols q + radius (0 for an
 * outlier) of x under the absolute bound eb_abs; rec: float32[n] scratch
 * (the reconstruction). */
int cszi_lorenzo_predict(const float *x, const cszi_geom *g, double eb_abs, int32_t radius,
                         uint16_t *sym, float *rec, cszi_ctl *ctl, void *stream);
/* lorenzo_reconstruct (lorenzo.py:36-53): symbols q + radius (0xFFFF at an
 * outlier, whose value is looked up in out_idx / out_val) -> y. */
int cszi_lorenzo_reconstruct(const uint16_t *sym, const uint64_t *out_idx, const float *out_val,
                             uint64_t n_out, const cszi_geom *g, double eb_abs, int32_t radius,
                             float *y, void *stream);

/* ---- stage entry points (fine-grained API of the reference) ------------ */

/* ctl := initial state (range keys reset, counters and flags zero). */
int cszi_ctl_init(cszi_ctl *ctl, void *stream);
/* Stream-ordered copy of a device ctl into host memory (pinned for an
 * asynchronous copy) followed by a stream synchronisation: the one host
 * read-back of a compress / decompress call. */
int cszi_ctl_fetch(const cszi_ctl *ctl, cszi_ctl *host, void *stream);

/* value_range + finite scan (grid.py:60-62, :104-108) into ctl. */
int cszi_range(const float *x, uint64_t n, cszi_ctl *ctl, void *stream);

/* cszi_ctl_init + cszi_range in one call (the Grid constructor's device
 * path, grid.py:19-63): one host call less before the first launch. */
int cszi_scan_field(const float *x, uint64_t n, cszi_ctl *ctl, void *stream);

/* profile_samples + select_config + plan_levels (tuning.py:42-129,
 * predictor.py:122-136) on a ctl holding the range of x; samples is a
 * device scratch of CSZI_SAMPLE_WORDS int32. */
int cszi_tune(const float *x, const cszi_geom *g, const cszi_params *p, int32_t *samples,
              cszi_ctl *ctl, void *stream);

/* compress_predict (predictor.py:395-420) on a tuned ctl:
 * sym uint16[n] = q + R (0 for outliers, R at anchors), hist uint64[2R]
 * (outliers and anchors counted as symbol R).  exact != 0 forces the
 * true-division quantizer (validation of the reciprocal fast path). */
int cszi_predict(const float *x, const cszi_geom *g, int32_t radius, int32_t exact,
                 uint16_t *sym, uint64_t *hist, cszi_ctl *ctl, void *stream);

/* cszi_predict that also writes the non-R bitmap nzmap (bit j of word w set
 * when symbol 32w + j is not R; (planes of x) * ny * nx / 8 bytes) when the
 * layout allows it (3-D default layout, nx % 32 == 0): *nz_done = 1 then. */
int cszi_predict_nz(const float *x, const cszi_geom *g, int32_t radius, int32_t exact,
                    uint16_t *sym, uint64_t *hist, uint32_t *nzmap, int32_t *nz_done,
                    cszi_ctl *ctl, void *stream);

/* Inverse interpolation (predictor.py:423-465) from uint16 symbols
 * (0xFFFF marks an outlier whose value is found in out_idx/out_val). */
int cszi_reconstruct(const uint16_t *sym, const float *anchors, const uint64_t *out_idx,
                     const float *out_val, uint64_t n_out, const cszi_geom *g, int32_t radius,
                     const double *level_eb, int32_t nlev, const int32_t variant[3],
                     const int32_t order[3], float *y, void *stream);

/* interpolate_level (predictor.py:367-392): the per-dimension passes of
 * ONE level (stride s, bound level_eb) over a device reconstruction buffer
 * recon[ext] (float32, C order), in dim order `order` (padded axes), with the
 * anchor lattice restored from anchor_block (lattice row-major) after each
 * pass.  mode 0 = Compress (reads source, writes recon, codes = q or 0,
 * is_outlier 0/1 for every pass point), mode 1 = Decompress (reads codes,
 * is_outlier, outlier_values[ext]; writes recon).  Replaces the reference's
 * numpy _run_pass / _split_pass (predictor.py:283-364). */
int cszi_interp_level(float *recon, const float *source, int32_t *codes, uint8_t *is_outlier,
                      const float *outlier_values, const float *anchor_block, const cszi_geom *g,
                      int64_t stride, double level_eb, const int32_t variant[3],
                      const int32_t order[3], int32_t radius, int32_t mode, void *stream);

/* gather_anchors (predictor.py:250-256): lattice row-major float32 values
 * (of the anchor planes inside g->slab when a slab is set). */
int cszi_gather_anchors(const float *x, const cszi_geom *g, float *out, void *stream);
uint64_t cszi_slab_anchor_count(const cszi_geom *g);

/* ---- sharded compress glue (multi-GPU z-slabs) ---------------
 * One call per slab and step of distributed.compress_slabs_batch (no
 * reference counterpart: the reference's only split is the thread pool of
 * predictor.py:347-364, whose output is byte-identical by construction).
 * cszi_shard_scan: ctl reset, range + finite scan of the n_own owned values,
 *   tuner sample gather (zeros for an empty slab), and keys[3] =
 *   (vmin key, -vmax key, first non-finite flat index + flat0 or INT64_MAX),
 *   ready for an all-reduce MIN.
 * cszi_shard_set_range: the reduced keys back into ctl.
 * cszi_shard_piece_bits: *out = sum(hist[i] * lengths[i]) (the slab's
 *   Huffman piece length in bits, outliers coded as R).
 * cszi_shard_counts: out[2] = (ctl->bits, ctl->n_outliers) after an encode. */
int cszi_shard_scan(const float *x, uint64_t n_own, uint64_t flat0, const cszi_geom *g,
                    cszi_ctl *ctl, int64_t *keys, int32_t *samples, void *stream);
int cszi_shard_set_range(cszi_ctl *ctl, const int64_t *keys, void *stream);
int cszi_shard_piece_bits(const uint64_t *hist, const uint8_t *lengths, int32_t nbins,
                          int64_t *out, void *stream);
int cszi_shard_counts(const cszi_ctl *ctl, int64_t *out, void *stream);

/* Distributed pass-2 encode (sharded compress): out[0] / out[1] = the first /
 * last index i in [lo + 2, hi) of bytes where a run of >= 2 zero bytes ends
 * (bytes[i-2] == bytes[i-1] == 0 != bytes[i]), -1 if none.  The zero-run
 * codec (pass2.py:30-67) has a segment boundary there whatever precedes the
 * run, so a stream cut at such points encodes piecewise to the same bytes.
 * out must hold 4 int64 (out[2..3] is scratch). */
int cszi_find_cuts(const uint8_t *bytes, uint64_t lo, uint64_t hi, int64_t *out, void *stream);

/* ---- sharded decompress split by Huffman chunk ranges -------
 * The stages of cszi_decompress over one workspace of
 * cszi_decompress_workspace_size bytes (same arguments throughout; g->slab
 * = the rank's z-slab):
 *   cszi_decompress_prologue: ctl reset, pass-2 decode, code tables;
 *   cszi_huff_chunks(sec_len[2]) = M, the stream's 256-bit chunk count;
 *   cszi_decompress_sync_range: speculative decode + synchronisation of
 *     chunks [h0, h1) (entry: the range's first entry bit, or UINT64_MAX for
 *     the speculative exit of chunk h0 - 1, which *entry_used receives);
 *     writes X / K / D[h0, h1) of full-length (M) arrays of chunk exits,
 *     symbol counts and dead flags; ctl->scratch[1] != 0: not converged;
 *   (the caller all-gathers X / K / D and repeats a rank's range with the
 *    true entry X[h0 - 1] when it differs from *entry_used)
 *   cszi_decompress_write_window: counts scan, truncation check, symbols of
 *     the slab's window;
 *   cszi_decompress_epilogue: outlier section, reconstruction of the slab
 *     into y ((slab[1] - slab[0]) ny nx floats).
 * The result equals cszi_decompress with the same geometry. */
int cszi_decompress_prologue(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                             const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                             void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, void *stream);
uint64_t cszi_huff_chunks(uint64_t nbytes);
int cszi_decompress_sync_range(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                               const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                               uint64_t h0, uint64_t h1, uint64_t entry, uint64_t *X,
                               uint32_t *K, uint8_t *D, uint64_t *entry_used, void *workspace,
                               uint64_t ws_bytes, cszi_ctl *ctl, void *stream);
int cszi_decompress_write_window(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                                 const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                                 const uint64_t *X, uint32_t *K, const uint8_t *D,
                                 void *workspace, uint64_t ws_bytes, cszi_ctl *ctl, void *stream);
/* Pass-2 decode split by 1 KiB chunks of the encoded payload (sharded
 * decompress): tables of chunks [c0, c1) into full-length arrays (M =
 * cszi_p2d_chunks(n); tab: M x 129 bytes, ctab: M x 129 uint32); the caller
 * all-gathers them; cszi_p2d_resolve (every rank: chain, counts, scan ->
 * E, cnt, off of M entries, ctl->raw_len); cszi_p2d_expand writes the raw
 * bytes of chunks [c0, c1) at their offsets (only the ranges a rank needs).
 * cszi_decompress_raw_offset: where the workspace's raw buffer starts;
 * cszi_decompress_prologue_raw: the prologue for a raw payload already
 * expanded there (ctl reset + code tables). */
uint64_t cszi_p2d_chunks(uint64_t n);
uint64_t cszi_p2d_resolve_scratch_size(uint64_t n);
int cszi_p2d_tables(const uint8_t *in, uint64_t n, uint64_t c0, uint64_t c1, uint8_t *tab,
                    uint32_t *ctab, void *stream);
int cszi_p2d_resolve(const uint8_t *tab, const uint32_t *ctab, uint64_t n, uint8_t *E,
                     uint32_t *cnt, uint64_t *off, void *scratch, cszi_ctl *ctl, void *stream);
int cszi_p2d_expand(const uint8_t *in, uint64_t n, const uint8_t *E, const uint64_t *off,
                    const uint32_t *cnt, uint64_t c0, uint64_t c1, uint8_t *out, uint64_t cap,
                    cszi_ctl *ctl, void *stream);
uint64_t cszi_decompress_raw_offset(const cszi_geom *g, int32_t radius,
                                    const uint64_t sec_len[4], uint64_t payload_len);
int cszi_decompress_prologue_raw(uint64_t payload_len, const uint64_t sec_len[4],
                                 const cszi_geom *g, int32_t radius, void *workspace,
                                 uint64_t ws_bytes, cszi_ctl *ctl, void *stream);
int cszi_decompress_epilogue(const uint8_t *payload, uint64_t payload_len, int32_t pass2,
                             const uint64_t sec_len[4], const cszi_geom *g, int32_t radius,
                             const double *level_eb, int32_t nlev, const int32_t variant[3],
                             const int32_t order[3], float *y, void *workspace, uint64_t ws_bytes,
                             cszi_ctl *ctl, void *stream);

/* Root of the sharded compress (replaces the whole-field _field_sections /
 * serialize payload, pipeline.py:59-63, archive.py:102-127, for slab
 * pieces): raw = the np anchor pieces (na[i] floats each, slab order) ||
 * code lengths (nbins bytes) || bitstream || outlier section (count, then
 * the pieces' records), then pass-2 into payload when pass2 != 0 (else raw
 * is the payload).  bits[i] is slab i's piece packed at global bit bit0[i]:
 * its word 0 holds global bits from (bit0[i] & ~31); nbits[i] bits.  Host
 * arrays of device pointers.  ctl->raw_len / payload_len are set on the
 * device.  raw_cap >= 4 sum(na) + nbins + 4 (total_bits / 32 + 2) +
 * 8 + 12 sum(nout); workspace >= cszi_pass2_encode_workspace_size(raw). */
int cszi_shard_assemble(int32_t np, const float *const *anchors, const uint64_t *na,
                        const uint8_t *lengths, int32_t nbins, const uint8_t *const *bits,
                        const uint64_t *bit0, const uint64_t *nbits,
                        const uint64_t *const *oidx, const float *const *oval,
                        const uint64_t *nout, int32_t pass2, uint8_t *raw, uint64_t raw_cap,
                        uint8_t *payload, void *workspace, uint64_t ws_bytes, cszi_ctl *ctl,
                        void *stream);

/* profile_samples split for sharding (tuning.py:42-74): gather the packed
 * sample values (float32 bit patterns, 0 where the point lies outside the
 * owned planes of g->slab) ... */
#define CSZI_SAMPLE_WORDS (64 * 3 * 5)
int cszi_sample_gather(const float *x, const cszi_geom *g, int32_t *vals, void *stream);
/* ... and select_config + plan_levels from the (all-reduced) samples; ctl
 * must hold the global range keys. */
int cszi_tune_from_samples(const int32_t *vals, const cszi_geom *g, const cszi_params *p,
                           cszi_ctl *ctl, void *stream);

/* Huffman-encode predictor symbols (uint16, 0 = outlier sentinel) with a
 * global flat-index offset for the outlier records; ctl->bits /
 * ctl->n_outliers receive the counts.  out is 4-byte aligned. */
uint64_t cszi_encode_sym_workspace_size(uint64_t n);
int cszi_encode_sym(const uint16_t *sym, uint64_t n, int32_t radius, const uint8_t *lengths,
                    const uint32_t *words, const float *x, uint64_t idx_offset, uint8_t *out,
                    uint64_t cap_bytes, uint64_t *out_idx, float *out_val, uint64_t out_cap,
                    void *workspace, cszi_ctl *ctl, void *stream);
/* The same with the stream packed from bit bit_base (0..31) of out's first
 * word: a z-slab shard packs its piece at its global bit phase, so the root
 * merges pieces with word copies (multi-GPU compress). */
int cszi_encode_sym_at(const uint16_t *sym, uint64_t n, int32_t radius, const uint8_t *lengths,
                       const uint32_t *words, const float *x, uint64_t idx_offset,
                       uint32_t bit_base, uint8_t *out, uint64_t cap_bytes, uint64_t *out_idx,
                       float *out_val, uint64_t out_cap, void *workspace, cszi_ctl *ctl,
                       void *stream);

/* cszi_encode_sym_at driven by the bitmap of cszi_predict_nz; hist = the
 * histogram of these n symbols (gives the stream length up front).  out_val
 * is not written: an outlier's value is x[out_idx - idx_offset]. */
int cszi_encode_sym_nz(const uint16_t *sym, uint64_t n, int32_t radius, const uint8_t *lengths,
                       const uint32_t *words, const float *x, uint64_t idx_offset,
                       uint32_t bit_base, uint8_t *out, uint64_t cap_bytes, uint64_t *out_idx,
                       float *out_val, uint64_t out_cap, const uint32_t *nzmap,
                       const uint64_t *hist, void *workspace, cszi_ctl *ctl, void *stream);

/* dst (zeroed, bytes) |= nbits of src placed at bit offset dst_bit (MSB-first). */
int cszi_concat_bits(uint8_t *dst, uint64_t dst_bit, const uint8_t *src, uint64_t nbits,
                     void *stream);

/* archive.py:184-189 outlier section: u64 count + packed (u64, f32) pairs. */
int cszi_pack_outliers(const uint64_t *idx, const float *val, uint64_t k, uint8_t *out,
                       void *stream);

/* build_histogram (huffman.py:60-74): int32 codes -> uint64[2R];
 * out-of-range codes set bit 31 of ctl->flags. */
int cszi_histogram_i32(const int32_t *codes, uint64_t n, int32_t radius, uint64_t *counts,
                       cszi_ctl *ctl, void *stream);

/* _code_lengths + canonical words (huffman.py:77-160):
 * counts uint64[nbins] -> lengths uint8[nbins], words uint32[nbins]. */
int cszi_codebook(const uint64_t *counts, uint32_t nbins, uint8_t *lengths, uint32_t *words,
                  cszi_ctl *ctl, void *stream);

/* Codebook.from_lengths (huffman.py:128-160): canonical words and, when
 * dec_tables != NULL, the decoder tables (cszi_dec_tables_size bytes). */
uint64_t cszi_dec_tables_size(uint32_t nbins);
int cszi_canonical(const uint8_t *lengths, uint32_t nbins, uint32_t *words, void *dec_tables,
                   cszi_ctl *ctl, void *stream);

/* huffman_encode (huffman.py:167-182): int32 codes -> MSB-first stream in
 * out (cap bytes, 4-byte aligned); ctl->bits <- exact bit count. */
uint64_t cszi_huff_encode_workspace_size(uint64_t n);
int cszi_huff_encode_i32(const int32_t *codes, uint64_t n, int32_t radius,
                         const uint8_t *lengths, const uint32_t *words, uint8_t *out,
                         uint64_t cap, void *workspace, cszi_ctl *ctl, void *stream);

/* huffman_decode (huffman.py:185-202): exactly n int32 codes from nbytes
 * of stream; CSZI_F_TRUNCATED in ctl->flags on failure. */
uint64_t cszi_huff_decode_workspace_size(uint64_t nbytes, int32_t table_mode);
int cszi_huff_decode_i32(const uint8_t *stream_bytes, uint64_t nbytes, uint64_t n,
                         int32_t radius, const void *dec_tables, int32_t *codes,
                         int32_t table_mode, int32_t lmax, void *workspace, cszi_ctl *ctl,
                         void *stream);

/* pass2_encode codec 0 (pass2.py:50-67): ctl->payload_len <- output size;
 * out capacity >= n + n/128 + 1.  n_dev: device pointer to the byte count
 * (n is its upper bound). */
uint64_t cszi_pass2_encode_workspace_size(uint64_t n);
int cszi_pass2_encode(const uint8_t *in, const uint64_t *n_dev, uint64_t n, uint8_t *out,
                      void *workspace, cszi_ctl *ctl, void *stream);

/* pass2_decode codec 0 (pass2.py:70-86): ctl->raw_len <- decoded size
 * (always); with expand != 0 also writes out (cap bytes).  Literal overrun
 * sets CSZI_F_P2_CORRUPT; cap overflow sets CSZI_F_CAPACITY. */
uint64_t cszi_pass2_decode_workspace_size(uint64_t n);
int cszi_pass2_decode(const uint8_t *in, uint64_t n, uint8_t *out, uint64_t cap,
                      int32_t expand, void *workspace, cszi_ctl *ctl, void *stream);

/* Library build identification. */
const char *cszi_version(void);

/* sizeof(cszi_geom), sizeof(cszi_params), sizeof(cszi_caps), sizeof(cszi_ctl)
 * — lets a binding verify its struct mirrors at load time. */
void cszi_abi_sizes(uint64_t out[4]);

/* Number of kernels this library has launched in this process. */
uint64_t cszi_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CSZI_H */
