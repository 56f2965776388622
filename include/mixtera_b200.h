/* C-ABI of the B200-native Mixtera hot path (libmxb200.so).
 *
 * Plain pointers and sizes only: no torch or Python types cross this
 * boundary. "device" arguments are CUDA device pointers on the current
 * device, "host" arguments are ordinary host memory, `stream` is a
 * cudaStream_t (NULL = legacy default stream). Every function returns an int
 * status (MX_OK = 0, MX_EXHAUSTED = 1, negative = error); the message of the
 * last error on the calling thread is mx_last_error().
 *
 * The reference (mixplane, pure Python) has no FFI: its seams are the Python
 * duck types called from server.py. Each entry point below replaces one of
 * them (reference file:line in brackets); INTEGRATION.md shows the ctypes
 * binding a maintainer adds on the reference side.
 *
 * Error codes map to the reference's exception types (errors.py:4-45):
 *   MX_ERR_QUERY -> QueryError, MX_ERR_INDEX -> IndexBuildError,
 *   MX_ERR_MIXTURE -> MixtureError, MX_ERR_FEEDBACK -> FeedbackError,
 *   MX_ERR_DATA -> DataReadError, MX_ERR_INVALID -> ValueError.
 */
#ifndef MIXTERA_B200_H
#define MIXTERA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MX_OK 0
#define MX_EXHAUSTED 1
#define MX_ERR_CUDA (-1)
#define MX_ERR_INVALID (-2)
#define MX_ERR_QUERY (-3)
#define MX_ERR_INDEX (-4)
#define MX_ERR_MIXTURE (-5)
#define MX_ERR_FEEDBACK (-6)
#define MX_ERR_DATA (-7)
#define MX_ERR_UNSUPPORTED (-8)

#define MX_MAX_PROPS 16

typedef struct mx_index mx_index;
typedef struct mx_gen mx_gen;

/* Last error message of the calling thread ("" when none). */
const char* mx_last_error(void);
/* ABI version; bumps on any signature change. */
int mx_abi_version(void);
/* Kernels this library has launched since it was loaded (all streams). */
int64_t mx_launch_count(void);
/* Per-phase CUDA-event timing on the launching stream: phases are
 * "scan_runs" (the stage-1 streaming kernel alone), "radix_sort",
 * "index_scans", "cursor_layout", "cursor_shuffle", "plan", "emit".
 * on = 1: every phase; on = 2: "scan_runs" only (two event records per job,
 * for timed loops); 0: off. */
int mx_profile_enable(int on);
int mx_profile_reset(void);
int mx_profile_read(const char* phase, double* total_ms, int64_t* count);

/* ------------------------------------------------------------------ stage 1
 * Columnar catalog + filter, encoded by the host (codec.py):
 *   columns[p]   device int32[n_samples], property p in NAME order (-1 = null),
 *                files concatenated in ascending file-id order;
 *   lut          host uint32, property p occupies [lut_offsets[p], lut_offsets[p+1]):
 *                entry (code+1) = packed-key contribution | 0x80000000 if the
 *                code fails the conjunctive filter (catalog.py:459-511);
 *   field_shift/field_width: bit position of property p's value-rank field;
 *   key strings: piece (key_string_base[p] + rank - 1) is
 *                escape(prop) ":" escape(v1) "," ... (mixtures.py:118-121).
 */
typedef struct mx_catalog_desc {
  int32_t n_props;
  const int32_t* const* columns;
  const uint32_t* lut;
  const int32_t* lut_offsets;
  int64_t n_samples;
  int32_t n_files;
  const int64_t* file_offsets; /* device int64[n_files+1] */
  const int32_t* file_ds;      /* host int32[n_files] */
  const int64_t* file_ids;     /* host int64[n_files], ascending */
  uint32_t key_bits;
  uint32_t rank_mask;
  const uint32_t* field_shift; /* host [n_props] */
  const uint32_t* field_width; /* host [n_props] */
  const uint8_t* key_strings;
  const int64_t* key_string_offsets; /* host [n_pieces+1] */
  const int32_t* key_string_base;    /* host [n_props] */
  /* Row-tuple layout (ABI 2). 0 = one code column per property, as above.
   * > 0 = the catalog stores its rows dictionary-encoded: columns[0..n_columns)
   * hold row-tuple codes and lut/lut_offsets have n_columns segments whose
   * entry (code+1) is the tuple's whole packed key | 0x80000000 if any of its
   * property codes fails the filter (the sum / OR of the per-property entries,
   * codec.py). n_key_pieces = number of key-string pieces (the per-property
   * cardinalities are then not derivable from lut_offsets). */
  int32_t n_columns;
  int32_t n_key_pieces;
  /* bytes per code: 4 (int32, also when 0) or 2 (u16 codes; a row-tuple
   * dictionary of <= 65,536 tuples). Columns must be 16-byte (int32) / 8-byte
   * (u16) aligned for the vector-load path; others take the scalar path. */
  int32_t column_bytes;
} mx_catalog_desc;

/* Fused filter + interval detection + index build
 * [MetadataCatalog.filter_intervals catalog.py:549-605 + build_index
 *  index.py:88-115, called from server.py:112-115]. Errors: MX_ERR_QUERY for
 * an un-keyable (all-null) sample or an empty catalog. An empty result is a
 * valid index with 0 keys (the server raises "matches no samples"). */
int mx_index_build(const mx_catalog_desc* desc, void* stream, mx_index** out);
/* Index from explicit interval rows [build_index(rows, workers) index.py:88-115,
 * the reference's entry point when rows come from anywhere but the catalog
 * (tests, composed paths)]. Host arrays [n_rows]: key = 1-based rank of the
 * row's component key in MixtureKey.sort_key order (so the packed key order
 * is the key order), file = index into the file table, which is sorted by
 * (dataset id, file id); start / end half-open. Key strings: piece k-1 is the
 * canonical string of key rank k (mixtures.py:118-121), offsets [n_keys+1].
 * On the device: sort by (key, file, start), reject empty intervals and
 * overlaps inside one (key, file) (MX_ERR_INDEX, index.py:32-47), merge
 * adjacent intervals, then the same key / block / cumulative tables as
 * mx_index_build. The result does not depend on the row order (= workers). */
typedef struct mx_rows_desc {
  int64_t n_rows;
  const uint32_t* key;
  const uint32_t* file;
  const uint32_t* start;
  const uint32_t* end;
  int32_t n_files;
  const int32_t* file_ds;  /* host int32[n_files] */
  const int64_t* file_ids; /* host int64[n_files] */
  int32_t n_keys;
  uint32_t key_bits;       /* bits of the largest rank (<= 31) */
  const uint8_t* key_strings;
  const int64_t* key_string_offsets; /* host [n_keys+1] */
} mx_rows_desc;
int mx_index_build_rows(const mx_rows_desc* desc, void* stream, mx_index** out);
int mx_index_free(mx_index* index);
int mx_index_sizes(const mx_index* index, int64_t* n_keys, int64_t* n_blocks,
                   int64_t* n_intervals, int64_t* n_samples);
/* Realized component keys in MixtureKey.sort_key order [ChunkerIndex
 * component_keys/key_sample_counts index.py:59-73]: host outputs [n_keys]. */
int mx_index_export_keys(const mx_index* index, uint32_t* packed, int64_t* samples);
/* Flat interval table in (key, dataset, file, start) order
 * [ChunkerIndex._index index.py:50-55]: host outputs [n_intervals]. */
int mx_index_export_intervals(const mx_index* index, uint32_t* key_rank, int32_t* ds,
                              int64_t* file_id, uint32_t* start, uint32_t* end);

/* ------------------------------------------------------------------ stage 2
 * Generator = per-key RangeCursor layouts + seeded component order
 * [ChunkGenerator.__init__ chunks.py:136-146, RangeCursor index.py:126-147].
 * cursor_prefix = stable-hash message prefix for (job_seed, "cursor"),
 * chunk_prefix  = prefix for (job_seed, "chunk") (seeding.py:18-33);
 * order_seed    = derive_seed(job_seed, "component-order"). */
int mx_gen_create(mx_index* index, const uint8_t* cursor_prefix, int32_t cursor_prefix_len,
                  const uint8_t* chunk_prefix, int32_t chunk_prefix_len, uint64_t order_seed,
                  void* stream, mx_gen** out);
int mx_gen_free(mx_gen* gen);

/* Mixture in force for the next plan [MixtureSpec mixtures.py:187-252].
 * allow: host uint32 [n_mkeys][allow_words]; bit (allow_base[p] + r) of mixture
 * key m says whether a component holding value-rank r (0 = null) of property p
 * matches m on p (mixtures.py:100-109). weights: host double [n_mkeys] in
 * MixtureKey.sort_key order. */
typedef struct mx_mixture_desc {
  int32_t n_mkeys;
  const uint32_t* allow;
  int32_t allow_words;
  const int32_t* allow_base; /* host [n_props] */
  const double* weights;
  int64_t chunk_size;
  int32_t strict;
} mx_mixture_desc;

/* Plan and emit up to max_chunks chunks under `mix`, exactly the sequence
 * max_chunks calls of ChunkGenerator.generate(spec) would return
 * [chunks.py:194-230, redistribute_best_effort :109-130, apportion
 * mixtures.py:158-184]. n_out = chunks emitted; MX_EXHAUSTED when the plan
 * ended with generate() returning None (report via mx_gen_report). */
int mx_gen_plan(mx_gen* gen, const mx_mixture_desc* mix, int64_t max_chunks, int64_t* n_out);
/* Same for generate_arbitrary(chunk_size) [chunks.py:232-253]. */
int mx_gen_plan_arbitrary(mx_gen* gen, int64_t chunk_size, int64_t max_chunks, int64_t* n_out);
/* Sizes of the last plan's result. */
int mx_gen_result_sizes(const mx_gen* gen, int64_t* n_chunks, int64_t* n_ranges);
/* Copy the last plan's chunks to host: chunk_offsets [n_chunks+1] (into the
 * range arrays), chunk_ids / seeds [n_chunks], ranges [n_ranges] sorted per
 * chunk by (mixture key, file, start), merged (chunks.py:169-192). `mkey` is
 * the mixture-key index (or the component rank for arbitrary chunks). */
int mx_gen_result_copy(const mx_gen* gen, int64_t* chunk_offsets, int64_t* chunk_ids, uint64_t* seeds,
                       uint32_t* mkey, int32_t* ds, int64_t* file_id, uint32_t* start, uint32_t* end);
/* Device views of the same result (valid until the next plan/free). */
int mx_gen_result_device(const mx_gen* gen, const int64_t** chunk_offsets, const uint64_t** seeds,
                         const uint32_t** mkey, const uint32_t** file_index, const uint32_t** start,
                         const uint32_t** end);
/* Copy of the last plan's result into caller DEVICE buffers: chunk_offsets
 * [n_chunks+1], pieces [n_ranges] (file_index = index into the file table). */
int mx_gen_result_export(const mx_gen* gen, int64_t* chunk_offsets, uint32_t* mkey, uint32_t* file_index,
                         uint32_t* start, uint32_t* end, void* stream);
/* Canonical chunk bytes of the last plan on the device [Chunk.serialize
 * chunks.py:54-93, canonical_json seeding.py:36-42]. key_json: the JSON-quoted
 * canonical strings of the result's keys (mixture keys, or component keys for
 * arbitrary chunks), key_rank their ranks in string order; file_rank: rank of
 * every file of the index in (str(ds), str(fid)) order; mixture_json: the
 * spec's canonical JSON ("null" for arbitrary chunks). */
typedef struct mx_json_desc {
  int64_t n_keys;
  const uint8_t* key_json;
  const int64_t* key_json_off; /* [n_keys+1] */
  const uint32_t* key_rank;    /* [n_keys] */
  const uint32_t* file_rank;   /* [n_files] */
  const uint8_t* mixture_json;
  int32_t mixture_len;
} mx_json_desc;
int mx_gen_result_json(mx_gen* gen, const mx_json_desc* desc, int64_t* total_bytes, void* stream);
/* Host copy of the serialized result: bytes [total_bytes], offsets [n_chunks+1]. */
int mx_gen_result_json_copy(const mx_gen* gen, uint8_t* bytes, int64_t* offsets);
/* Shortfall report of the last generate() that returned None: host [n_mkeys]. */
int mx_gen_report(const mx_gen* gen, int64_t* remaining);
/* Remember / restore the cursor state and next chunk id on the device (used
 * to rewind a look-ahead plan to the last chunk handed to the caller). */
int mx_gen_mark(mx_gen* gen);
int mx_gen_reset_to_mark(mx_gen* gen);
int mx_gen_next_chunk_id(const mx_gen* gen, int64_t* next_id);
int mx_gen_set_next_chunk_id(mx_gen* gen, int64_t next_id);
/* Cursor checkpoint form {pos, offset} per component rank
 * [RangeCursor.state_dict/load_state index.py:180-189]: host [n_keys]. */
int mx_gen_get_cursors(const mx_gen* gen, int64_t* pos, int64_t* offset);
int mx_gen_set_cursors(mx_gen* gen, const int64_t* pos, const int64_t* offset);
/* Component order as component ranks: host [n_keys]. */
int mx_gen_component_order(const mx_gen* gen, uint32_t* order);
/* RangeCursor._ranges of one component: host outputs sized by n_ranges. */
int mx_gen_cursor_ranges(const mx_gen* gen, uint32_t comp, int64_t* n_ranges, int32_t* ds,
                         int64_t* file_id, uint32_t* start, uint32_t* end, int64_t capacity);

/* ------------------------------------------------------------------ multi-GPU
 * File-sharded index. Rank r indexes the contiguous global
 * file range [file_lo, file_hi) with mx_index_build (local file indices
 * 0..file_hi-file_lo-1), exports its (key, file) block table, and after an
 * all-gather of the tables builds the hybrid index whose keys, blocks, cursor
 * shuffles and chunk plans are those of the whole catalog
 * [RangeCursor index.py:126-147 over files of every rank]. Chunks planned on
 * a hybrid index hold only this rank's pieces; mx_chunks_merge interleaves the
 * ranks' chunk CSRs into the global (mixture key, file, start) order. */

/* Device rows uint32[n_blocks][4] = (packed key, file_base + file index,
 * samples, intervals), in (packed key, file) order. */
int mx_index_block_table(const mx_index* index, int64_t file_base, uint32_t* rows, void* stream);
/* Host copy of the realized packed keys [n_keys] (ascending). */
int mx_index_packed_keys(const mx_index* index, uint32_t* packed);

typedef struct mx_shard_desc {
  int32_t world, rank;
  int64_t file_lo, file_hi;      /* this rank's global file indices */
  int32_t n_files;               /* global file table: */
  const int32_t* file_ds;        /*   host [n_files] dataset ids (nondecreasing) */
  const int64_t* file_ids;       /*   host [n_files] file ids */
  const uint32_t* tables;        /* device uint32[world][cap][4] gathered block rows */
  const int64_t* counts;         /* host [world] rows per rank */
  int64_t cap;
  const uint32_t* global_keys;   /* host [n_global_keys] sorted union of packed keys */
  int64_t n_global_keys;
} mx_shard_desc;

int mx_index_build_sharded(const mx_index* local, const mx_shard_desc* desc, void* stream, mx_index** out);
/* Sharded cursor state: a key whose frontier lies inside another rank's
 * block reports pos = offset = -1 (mx_gen_get_cursors) / consumed = -1
 * (mx_gen_cursor_to_consumed); the owner reports the value, so a MAX
 * all-reduce over ranks completes it. */
int mx_gen_cursor_to_consumed(const mx_gen* gen, const int64_t* pos, const int64_t* offset, int64_t* consumed);
int mx_gen_set_consumed(mx_gen* gen, const int64_t* consumed);
/* Root-side merge of `world` per-rank chunk CSRs of the same n_chunks chunks:
 * offs device int64[world][n_chunks+1]; piece arrays device uint32[world][cap]
 * (rank q's pieces at q*cap). Outputs: out_off device int64[n_chunks+1],
 * pieces device uint32[sum of ranks' pieces]. */
int mx_chunks_merge(int32_t world, int64_t n_chunks, int64_t cap, const int64_t* offs, const uint32_t* mkey,
                    const uint32_t* file_index, const uint32_t* start, const uint32_t* end, int64_t* out_off,
                    uint32_t* out_mkey, uint32_t* out_file_index, uint32_t* out_start, uint32_t* out_end,
                    void* stream);

/* Key-partitioned multi-GPU (parallel.build_partitioned). Each global key is
 * OWNED by one rank; every rank sends the block rows of mx_index_block_table
 * (global file indices) to the keys' owners. The owner builds an index of
 * one pseudo-interval [0, samples) per (key, file) block of its keys over the
 * GLOBAL file table (key codec copied from `like`), and a generator on it:
 * its per-key cursor shuffles are the reference's over the key's files of
 * the whole catalog [RangeCursor index.py:126-147], so mx_gen_block_offsets
 * gives each block's offset in its key's cursor stream (device uint64[n_rows],
 * in the order of the rows given to mx_index_build_owner). The same call on
 * rows (packed key, 0, total samples) gives the key-level index every rank
 * plans on (global per-key totals; chunks.py:188-259 only needs those).
 * dense_key_bits > 0: the rows are already file-ordered within each key
 * (every source's (key, file)-sorted rows concatenated in rank order) and
 * row[3] holds a dense key rank increasing with the packed key, < 2^bits:
 * one stable sort pass per 8 bits instead of a (file, key) sort. */
int mx_index_build_owner(const mx_index* like, const uint32_t* rows, int64_t n_rows, int32_t n_files,
                         const int32_t* file_ds, const int64_t* file_ids, int32_t dense_key_bits, void* stream,
                         mx_index** out);
int mx_gen_block_offsets(mx_gen* gen, uint64_t* offsets, void* stream);
/* Plans of `gen` (on a key-level index) then emit only `local`'s pieces:
 * block b of local key k is the key's cursor stream at blk_off[b] (device
 * uint64[n_blocks]); key_g (device uint32[n_keys]) = its rank in gen's index;
 * file_lo = global index of local file 0. The buffers must outlive the
 * generator's plans. Mixtures of <= 32 keys sharing no component (others:
 * MX_ERR_UNSUPPORTED); pass local == NULL to detach. */
int mx_gen_set_local(mx_gen* gen, const mx_index* local, const uint64_t* blk_off, const uint32_t* key_g,
                     int64_t file_lo);
/* Chunk-owner output (no rank gathers every piece). With
 * handoff on, a plan of a partitioned generator stops after the cut: its
 * pieces, grouped by global chunk, stay in the generator (mx_gen_handoff:
 * device offsets int64[n_chunks + 1], pieces uint32[n_pieces][4] = (mixture
 * key, global file index, start, end)). The caller sends each chunk owner the
 * pieces of its chunks (one all-to-all; rank r owns a contiguous chunk range)
 * with their per-chunk counts, and the owner finishes ITS chunks:
 * counts device int32[world][n_own], pieces device uint32[n_pieces][4]
 * source-major then chunk-major. The result (mx_gen_result_*) then holds the
 * owned chunks (ids chunk_lo..), normalised as the single-GPU path does. */
int mx_gen_set_handoff(mx_gen* gen, int32_t on);
int mx_gen_handoff(const mx_gen* gen, int64_t* n_chunks, int64_t* n_pieces, const int64_t** chunk_offsets,
                   const uint32_t** pieces);
int mx_gen_finish_owned(mx_gen* gen, int32_t world, int64_t chunk_lo, int64_t n_own, int64_t n_global,
                        const int32_t* counts, const uint32_t* pieces, int64_t n_pieces, void* stream);

/* ------------------------------------------------------------ registration
 * Metadata registration from JSON-lines bytes in HBM [MetadataCatalog.
 * register_dataset catalog.py:323-435, _parse_one_file catalog.py:246-262,
 * iter_records formats.py:47-56, JsonFieldParser catalog.py:168-183,
 * _normalize_values catalog.py:186-232]; SURVEY.md §8f-3.
 *
 * buf: device bytes, 16-byte aligned, n_bytes a multiple of 16, every file
 * newline-terminated (padding after the last newline is not a line).
 * Records = non-empty lines in order. Call once with rec_start == NULL to get
 * n_records (and n_lines), then with device int64 outputs [n_records]: the
 * record's byte range [start, end) and its global line index. */
int mx_jsonl_records(const uint8_t* buf, int64_t n_bytes, int64_t* rec_start, int64_t* rec_end,
                     int64_t* rec_line, int64_t capacity, int64_t* n_records, int64_t* n_lines, void* stream);
/* Per record and requested top-level field (names: device bytes + offsets
 * [n_fields+1], n_fields <= 32), device outputs [n_records][n_fields]:
 * kind 0 missing / 1 value / 2 host / 3 present without a value (null, []);
 * nelem = distinct elements of the normalised value; hash_a/hash_b = 128-bit
 * hash of the normalised value (sorted distinct element hashes);
 * value_start/value_len = byte span of a string value's content, or
 * ~start / length of a list value. host[n_records] = 1: the record needs the
 * host's json.loads + parser + normalisation (invalid JSON, escapes in a
 * key or a requested value, numbers / booleans / nested values in a
 * requested field, NaN / Infinity, BOM, NUL, > 8 list elements). */
int mx_jsonl_extract(const uint8_t* buf, const int64_t* rec_start, const int64_t* rec_end, int64_t n_records,
                     const uint8_t* field_names, const int64_t* field_offsets, int32_t n_fields, uint8_t* kind,
                     uint8_t* nelem, uint64_t* hash_a, uint64_t* hash_b, int64_t* value_start, int32_t* value_len,
                     uint8_t* host, void* stream);

/* ------------------------------------------------------------ client modes
 * Tokenized processing mode [ChunkStreamer.tokenized client.py:451-506,
 * tokenizers.py]; SURVEY.md §8f-4.
 * mx_jsonl_tokenize: per record (spans from mx_jsonl_records) the tokens of
 * the top-level string field `field`: tokenizer 0 = ByteTokenizer (UTF-8
 * bytes of the decoded string), 1 = WhitespaceTokenizer (str.split() pieces,
 * stable_hash("tok", piece) % vocab_size). tokens == NULL: counts[n_records]
 * and host[n_records] (1 = the host tokenizer must handle the record: no
 * string value, non-object record, escaped key, lone surrogate). Otherwise
 * writes the device-path records' tokens at offsets[r] (device int64). */
int mx_jsonl_tokenize(const uint8_t* buf, const int64_t* rec_start, const int64_t* rec_end, int64_t n_records,
                      const uint8_t* field, int32_t field_len, int32_t tokenizer, uint32_t vocab_size,
                      const int64_t* offsets, int64_t* counts, int32_t* tokens, uint8_t* host, void* stream);
/* Packing of one chunk's key streams into n_windows windows of
 * seqs_per_window sequences of sequence_length tokens (device arrays):
 * window slot i holds key slot_key[i]'s sequences [slot_first[i],
 * slot_first[i+1]) of the window; key m owns samples [key_off[m],
 * key_off[m+1]) (global record ids, iterator order) with exclusive token
 * prefix sample_prefix; outputs int32 [n_windows*seqs_per_window*L] tokens
 * and tags (key_tag[m] per token). */
int mx_pack_tokens(int64_t n_windows, int32_t sequence_length, int32_t n_slots, const int32_t* slot_key,
                   const int32_t* slot_first, const int32_t* key_count, const int64_t* key_off,
                   const int64_t* samples, const int64_t* sample_prefix, const int64_t* token_offsets,
                   const int32_t* tokens, const int32_t* key_tag, int32_t seqs_per_window, int32_t* out_tokens,
                   int32_t* out_tags, void* stream);

/* ------------------------------------------------------------------ stage 3
 * Per-domain loss reduction [per_domain_loss client.py:582-598]: device
 * f32 losses[n], int32 tags[n] in [0, n_domains) -> device f64 sums, int64
 * counts [n_domains] (overwritten). MX_ERR_DATA on a tag out of range. */
int mx_domain_loss(const float* losses, const int32_t* tags, int64_t n, int32_t n_domains,
                   double* sums, int64_t* counts, void* stream);
/* Batched power-law fit [fit_power_law ado.py:121-168]: domain d's points
 * are [point_offsets[d], point_offsets[d+1]) of n[] / loss[] (device f64);
 * geom: device f64[49] = numpy.geomspace(1e-6, 1, 49). out_law: device f64
 * [n_domains][4] = (epsilon, beta, alpha, fallback). */
int mx_fit_power_law(int32_t n_domains, const int64_t* point_offsets, const double* n,
                     const double* loss, const double* geom, double* out_law, void* stream);
/* ADO mixture update [AdoState.compute_pi/_floored ado.py:273-319]. Device
 * f64 state vectors of length k: mu, credit, law (k x 4, NaN row = no law),
 * pi_bar (in/out), pi (out). shared_n = _shared_n(t). Writes pi; advances
 * pi_bar with count *pi_bar_count (device int64, incremented). */
int mx_ado_pi(int32_t k, const double* mu, const double* credit, const double* law,
              double shared_n, double p_min, double smoothing, double* pi_bar,
              int64_t* pi_bar_count, double* pi, void* stream);
/* credit <- (1 - rate) * credit + rate * pi [AdoState.record_step ado.py:241-243]. */
int mx_ado_credit(int32_t k, double rate, const double* pi, double* credit, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MIXTERA_B200_H */
