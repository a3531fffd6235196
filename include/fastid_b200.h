/*
 * fastid_b200.h -- C ABI of the B200-native FastID comparison path.
 *
 * Plain pointers and sizes only.  Every entry point returns a fastid_status;
 * on failure fastid_last_error() holds a thread-local message.  Functions
 * taking a `stream` accept a cudaStream_t passed as void* (NULL = default
 * stream) and DEVICE pointers; they enqueue work and return without syncing.
 * fastid_run_kernel takes HOST pointers and is synchronous.
 *
 * Reference interfaces each entry replaces (paths under the reference
 * package pkg/src/fastid/):
 *   fastid_run_kernel        run_naive_kernel        kernel.py:350-353
 *                            run_blocked_kernel      kernel.py:317-347
 *                            Executor.run seam       scheduler.py:221-240
 *   fastid_compare_full      _naive_kernel / _blocked_worker kernel.py:224-269
 *                            (behind compare_naive / compare_blocked kernel.py:283-314)
 *   fastid_pack_bits         codec.pack              codec.py:118-127
 *   fastid_pack_genotypes    codec.encode_genotype + pack codec.py:99-127
 *   fastid_load_words        Panel words -> device rows (Panel kernel.py:68-129)
 *   fastid_compare_topk      no reference equivalent; the
 *   fastid_compare_threshold derivation of compare_naive's matrix, see DESIGN.md
 *   fastid_merge_topk        multi-device combine (paper future work)
 *
 * Device row layout: every profile row occupies fastid_row_stride(L) bytes
 * (a multiple of 16), holding the panel's words in their native little-endian
 * byte order followed by zero fill.  Bit order inside a row does not affect the
 * score as long as both operands share it, so u32 and u64 panels load as-is.
 */
#ifndef FASTID_B200_H
#define FASTID_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FASTID_API __attribute__((visibility("default")))
#else
#define FASTID_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FASTID_ABI_VERSION 1

enum fastid_status {
    FASTID_OK = 0,
    FASTID_E_INVALID = 1,     /* bad argument (maps to ValueError)                */
    FASTID_E_MISMATCH = 2,    /* incompatible panels (maps to PanelMismatchError) */
    FASTID_E_CUDA = 3,        /* CUDA runtime/driver failure                      */
    FASTID_E_CAPACITY = 4,    /* output buffer too small; count still reported    */
    FASTID_E_NOMEM = 5,       /* device allocation failed                         */
    FASTID_E_UNSUPPORTED = 6, /* formulation/shape not supported on this device   */
    FASTID_E_FORMAT = 7,      /* malformed panel text (maps to PanelFormatError)  */
    FASTID_E_CORRUPT = 8      /* nonzero padding (maps to CorruptProfileError)    */
};

enum fastid_formulation {
    FASTID_AUTO = 0,       /* the measured winner (tensor, mxf4)               */
    FASTID_POPC = 1,       /* CUDA cores: LOP3 (and-not) + POPC over u32 words  */
    FASTID_TENSOR_I8 = 2,  /* tcgen05.mma kind::i8 on 0/1-unpacked tiles        */
    FASTID_TENSOR_F4 = 3   /* tcgen05.mma kind::mxf4 (e2m1 0/1, unit scales)    */
};

/* The overloaded semiring's "multiply" (FastID Eq. 1 and the paper's variants,
 * PAPER.md:39-45), OR-ed into any `formulation` argument:
 *   FASTID_OP_ANDNOT  popcount(known AND NOT unknown) -- the reference's score
 *                     (kernel.py:33-35); the default (0)
 *   FASTID_OP_AND     popcount(known AND unknown): shared minor alleles
 *   FASTID_OP_XOR     popcount(known XOR unknown): Hamming distance
 * The reference implements only AND-NOT; AND and XOR have no reference
 * counterpart and are checked against a numpy restatement. */
enum fastid_operator {
    FASTID_OP_ANDNOT = 0,
    FASTID_OP_AND = 0x100,
    FASTID_OP_XOR = 0x200
};
#define FASTID_OP_MASK 0x300

FASTID_API int fastid_abi_version(void);
FASTID_API const char* fastid_last_error(void);
/* bytes per device row for a panel of bit_length loci: ceil(L / 128) * 16 */
FASTID_API int64_t fastid_row_stride(int64_t bit_length);
/* largest k accepted by fastid_compare_topk */
FASTID_API int fastid_max_k(void);
/* Kernels this library has enqueued so far in this process (all devices and
 * streams): a measurement aid -- bench.py reads it around its timed region. */
FASTID_API unsigned long long fastid_launch_count(void);
/* 1 if `formulation` can run panels of bit_length loci on this build, else 0 */
FASTID_API int fastid_supports(int formulation, int64_t bit_length);

/* ---- profile encoder ---------------------------------------------------- */

/* Copy `rows` panel rows of src_row_bytes each (u32/u64 words, little-endian)
 * into the aligned device layout, zero-filling each row to dst_stride. */
FASTID_API int fastid_load_words(const void* src, int64_t rows, int64_t src_row_bytes, void* dst,
                      int64_t dst_stride, void* stream);

/* Pack a (rows x bit_length) 0/1 byte matrix into MSB-first words of
 * word_bits (32|64) exactly as codec.pack, written in the device layout. */
FASTID_API int fastid_pack_bits(const uint8_t* bits, int64_t rows, int64_t bit_length, int word_bits,
                     void* dst, int64_t dst_stride, void* stream);

/* Encode (rows x n_loci) genotype codes (0=MM, 1=Mm, 2=mM, 3=mm) into
 * 2*n_loci minor-allele bits (codec.GENOTYPE_BITS) and pack as above. */
FASTID_API int fastid_pack_genotypes(const uint8_t* codes, int64_t rows, int64_t n_loci, int word_bits,
                          void* dst, int64_t dst_stride, void* stream);

/* ---- comparison --------------------------------------------------------- */

/* out[i * ld_out + j] = popcount(refs_i AND NOT queries_j) for all i < n_refs,
 * j < n_queries.  refs / queries are device rows of `stride` bytes.  `out` may
 * be a view into a wider matrix (ld_out >= n_queries): no element outside
 * [0, n_refs) x [0, n_queries) is written. */
FASTID_API int fastid_compare_full(const void* refs, int64_t n_refs, const void* queries, int64_t n_queries,
                        int64_t stride, int64_t bit_length, uint32_t* out, int64_t ld_out,
                        int formulation, void* stream);

/* Workspace bytes fastid_compare_topk needs for this shape. */
FASTID_API int fastid_topk_workspace(int64_t n_refs, int64_t n_queries, int k, int formulation,
                          size_t* bytes);

/* Per query j: the k (score, known index) pairs with the smallest scores,
 * ordered by (score asc, index asc), restricted to score <= max_score.
 * Outputs are [n_queries][k]; unused slots hold score 0xFFFFFFFF, index -1.
 * Reported indices are ref_base + local row. */
FASTID_API int fastid_compare_topk(const void* refs, int64_t n_refs, const void* queries, int64_t n_queries,
                        int64_t stride, int64_t bit_length, int k, uint32_t max_score,
                        int64_t ref_base, uint32_t* top_scores, int64_t* top_index,
                        void* workspace, size_t workspace_bytes, int formulation, void* stream);

/* The first half of fastid_compare_topk: only the comparison kernel, leaving
 * *n_lists candidate lists of *list_len entries per query in the workspace
 * (indices at *index_offset, scores at *score_offset bytes from workspace,
 * list-major [n_lists][n_queries][list_len]) for fastid_merge_topk. */
FASTID_API int fastid_topk_partials(const void* refs, int64_t n_refs, const void* queries, int64_t n_queries,
                                    int64_t stride, int64_t bit_length, int k, uint32_t max_score,
                                    int64_t ref_base, void* workspace, size_t workspace_bytes,
                                    int formulation, void* stream, int* n_lists, int* list_len,
                                    size_t* index_offset, size_t* score_offset);

/* Every (query j, known i, score) with score <= threshold, in no particular
 * order.  *hit_count (device) receives the total number of hits; only the first
 * `capacity` are stored. */
FASTID_API int fastid_compare_threshold(const void* refs, int64_t n_refs, const void* queries,
                             int64_t n_queries, int64_t stride, int64_t bit_length,
                             uint32_t threshold, int64_t ref_base, uint32_t* hit_query,
                             int64_t* hit_ref, uint32_t* hit_score, int64_t capacity,
                             unsigned long long* hit_count, int formulation, void* stream);

/* Merge n_lists candidate lists, each [n_queries][k_in] sorted by (score, index),
 * into the first k per query (lists laid out list-major). */
FASTID_API int fastid_merge_topk(const uint32_t* cand_scores, const int64_t* cand_index, int n_lists,
                      int64_t n_queries, int k_in, int k, uint32_t* top_scores,
                      int64_t* top_index, void* stream);

/* ---- prepared database (resident known panel + tensor image) ------------- */

/* A known panel prepared for repeated queries: for the tensor formulations
 * the handle owns a device "tensor image" of the panel -- every known tile
 * already in the tcgen05 operand layout (e2m1 / u8), built once here -- so the
 * comparison kernels stream it with bulk copies instead of unpacking bits per
 * query batch.  The packed rows `refs` must stay alive while the handle does.
 * Image size: fastid_db_image_bytes (about 4x (mxf4) / 8x (i8) the packed rows). */
typedef struct fastid_db fastid_db;

FASTID_API size_t fastid_db_image_bytes(int64_t n_refs, int64_t bit_length, int formulation);
FASTID_API int fastid_db_create(const void* refs, int64_t n_refs, int64_t stride, int64_t bit_length,
                                int formulation, void* stream, fastid_db** out);
/* As fastid_db_create, but the image is built into the caller's device buffer
 * `image` (at least fastid_db_image_bytes(n_refs, bit_length, formulation)
 * bytes), which the handle does not own or free.  With it a panel whose whole
 * image does not fit is searched chunk by chunk at the image kernels' speed:
 * one reusable buffer, a handle per chunk of rows (ref_base = chunk offset). */
FASTID_API int fastid_db_create_in(const void* refs, int64_t n_refs, int64_t stride, int64_t bit_length,
                                   int formulation, void* image, size_t image_bytes, void* stream, fastid_db** out);
FASTID_API int fastid_db_destroy(fastid_db* db);
/* The operator (FASTID_OP_*) of the handle's later comparisons (default
 * AND-NOT; fastid_db_create also takes it OR-ed into `formulation`).  The image
 * serves every operator.  XOR on an i8 image needs each known row's popcount:
 * computed once on first use (that call synchronises its stream); the mxf4
 * image needs none (a signed unknown operand, tensor.cu unpack_f4_xor). */
FASTID_API int fastid_db_set_operator(fastid_db* db, int op);
FASTID_API int fastid_db_formulation(const fastid_db* db);

/* Execution variants of a prepared database.  Every option computes the same
 * result (bit-exact); they only select among kernel paths, so tests can reach
 * each one.  Options apply to later calls on this handle only. */
enum fastid_db_option {
    FASTID_OPT_NO_CTA_PAIRS = 1,      /* single-CTA kernel instead of CTA pairs       */
    FASTID_OPT_NO_TMA_STORE = 2,      /* full matrix by per-element stores            */
    FASTID_OPT_NO_SPARE_PAIRS = 4,    /* no spare-pair grid on the SMs left over      */
    FASTID_OPT_NARROW_TMA_STORE = 8   /* per-warp (32-unknown) TMA-store blocks       */
};
/* Set (value != 0) or clear one FASTID_OPT_* bit of the handle. */
FASTID_API int fastid_db_set_option(fastid_db* db, int option, int value);
/* The handle's current FASTID_OPT_* bits (-1 for NULL). */
FASTID_API int fastid_db_options(const fastid_db* db);

/* As fastid_compare_full / fastid_topk_partials / fastid_compare_threshold with
 * the database's refs, stride, bit_length and formulation. */
FASTID_API int fastid_db_compare_full(const fastid_db* db, const void* queries, int64_t n_queries,
                                      uint32_t* out, int64_t ld_out, void* stream);
FASTID_API int fastid_db_topk_partials(const fastid_db* db, const void* queries, int64_t n_queries, int k,
                                       uint32_t max_score, int64_t ref_base, void* workspace,
                                       size_t workspace_bytes, void* stream, int* n_lists, int* list_len,
                                       size_t* index_offset, size_t* score_offset);
FASTID_API int fastid_db_compare_threshold(const fastid_db* db, const void* queries, int64_t n_queries,
                                           uint32_t threshold, int64_t ref_base, uint32_t* hit_query,
                                           int64_t* hit_ref, uint32_t* hit_score, int64_t capacity,
                                           unsigned long long* hit_count, void* stream);

/* ---- host-buffer drop-in (synchronous) ----------------------------------- */

/* Executor.run semantics: ref_words (n_refs x n_words), query_words
 * (n_queries x n_words), or (n_words x n_queries) when queries_transposed,
 * words of word_bits (32|64), out (n_refs x n_queries) u32, all HOST memory.
 * Uses a per-thread device context on the current CUDA device. */
FASTID_API int fastid_run_kernel(const void* ref_words, int64_t n_refs, const void* query_words,
                      int64_t n_queries, int64_t n_words, int word_bits, int queries_transposed,
                      uint32_t* out, int formulation);

/* The same comparison with the u32 rows appended, in row order, to the open
 * file descriptor `fd` instead of a host array -- the payload of the
 * reference's FIDM score file (BinaryScoreSink.put, io.py:244-255; the caller
 * writes the 21-byte header, io.py:29-31).  The rows land at the
 * descriptor's current offset (which must be seekable) via parallel
 * pwrite(2) straight from pinned staging; on return the offset is past the
 * last row.  Synchronous. */
FASTID_API int fastid_run_kernel_fd(const void* ref_words, int64_t n_refs, const void* query_words,
                                    int64_t n_queries, int64_t n_words, int word_bits, int queries_transposed,
                                    int fd, int formulation);

/* Top-k over a known panel in HOST memory that need not fit on the device:
 * the rows stream through the GPU in chunks of `chunk_rows` (0 = automatic,
 * ~512 MB of packed rows), the upload of chunk c+1 overlapping the fused
 * compare + top-k of chunk c, and every chunk's lists are merged into the
 * running lists on the device.  Same result as fastid_compare_topk over the
 * whole panel (global known indices = ref_base + row, ties to the lower index);
 * row-major host words in, host top_scores [n_queries][k] (u32, 0xFFFFFFFF =
 * empty) and top_index [n_queries][k] (i64, -1 = empty) out.  Page-locked
 * `ref_words` upload without a staging copy.  Replaces the reference's batched
 * pipeline over a panel larger than one batch (plan_batches scheduler.py:108-140,
 * run_pipeline scheduler.py:270-419) for a top-k-reducing sink. */
FASTID_API int fastid_run_topk(const void* ref_words, int64_t n_refs, const void* query_words, int64_t n_queries,
                               int64_t n_words, int word_bits, int k, uint32_t max_score, int64_t ref_base,
                               uint32_t* top_scores, int64_t* top_index, int64_t chunk_rows, int formulation);

/* ---- measurement ------------------------------------------------------- */

/* Pipe-peak probe (roofline denominator): launches an MMA-only (tensor
 * formulations) or LOP3+POPC-only (FASTID_POPC) kernel, one CTA per SM, with
 * `iters` inner iterations; *work receives the bit-pairs it performs.  Time it
 * with CUDA events on `stream`.  `scratch` is >= 4 * SM-count bytes of device
 * memory. */
FASTID_API int fastid_probe_peak(int formulation, int iters, void* scratch, double* work, void* stream);
/* Diagnostic variants of the tensor probe (variant bit 0: one accumulator for
 * every MMA; bit 1: concurrent 28 KB bulk copies from `src` into shared memory). */
FASTID_API int fastid_probe_tmem_read(int x, int warps, int iters, void* scratch, double* work, void* stream);
/* Diagnostic: MMA stream concurrent with `readers` warps of TMEM loads; sink = 2*SMs u64. */
FASTID_API int fastid_probe_contention(int iters, int readers, void* sink, void* stream);
FASTID_API int fastid_probe_variant(int formulation, int variant, int iters, void* scratch, const void* src,
                                    int64_t src_bytes, double* work, void* stream);
/* Timing-experiment switches and per-tile traces are not part of this library:
 * they exist only in the separate experiments build (_fastid_b200_diag.so,
 * include/fastid_b200_diag.h). */

/* ---- bulk panel ingest (host) ------------------------------------------- */

/* Parse the reference's text panel format (io.load_panel, io.py:45-127):
 * `#bits=<L>` header, `#` comments, blank lines, `<id><TAB><hex>` profiles,
 * universal newlines.  Same validation order and messages as the reference
 * (FASTID_E_FORMAT -> PanelFormatError, FASTID_E_CORRUPT -> CorruptProfileError,
 * first offending line wins).  Words are word_width (32|64) bits, native
 * endian, row-major n x ceil(L/W).  n_threads <= 0: all hardware threads. */
typedef struct fastid_parsed_panel fastid_parsed_panel;
FASTID_API int fastid_parse_panel(const char* text, int64_t len, int word_width, int n_threads,
                                  fastid_parsed_panel** out);
FASTID_API int fastid_parsed_panel_shape(const fastid_parsed_panel* p, int64_t* n_profiles, int64_t* bit_length,
                                         int64_t* n_words, int64_t* id_bytes);
/* words: n x n_words words; ids: id_bytes bytes (UTF-8, the ids joined by
 * '\n'); id_offsets: n + 1 byte offsets of each id in ids (last = id_bytes).
 * Any pointer may be NULL. */
FASTID_API int fastid_parsed_panel_copy(const fastid_parsed_panel* p, void* words, char* ids, int64_t* id_offsets);
FASTID_API void fastid_parsed_panel_free(fastid_parsed_panel* p);

#ifdef __cplusplus
}
#endif

#endif /* FASTID_B200_H */
