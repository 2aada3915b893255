/*
 * seqcdc.h -- C ABI of the B200-native SeqCDC boundary-detection library
 * (libseqcdc.so, built from paper_2505_21194_b200/csrc/).
 *
 * The operation is SeqCDC chunking (Udayashankar & Al-Kiswany, "Vectorized
 * Sequence-Based Chunking for Data Deduplication", arXiv 2505.21194;
 * PAPER.md lines are cited as P:n):
 *
 *   A stream is split into chunks; a chunk boundary is inserted right after
 *   the first run of SeqLength bytes that is strictly increasing (Increasing
 *   mode) or strictly decreasing (Decreasing mode) (§3.1).  Each
 *   chunk's scan starts (min_size - SeqLength) bytes after the chunk start
 *   (§3.2).  Whenever SkipTrigger pairs of adjacent bytes in the
 *   opposing order have been counted since the scan (re)started, the scan
 *   jumps SkipSize bytes ahead and resets its counters (§3.3;
 *   P:225-231).  If no boundary is found first, the chunk ends at
 *   chunk start + max_size (§4).  The last chunk ends at the end of the
 *   stream.  The readings of the paper's ambiguous points (SeqLength counts
 *   bytes; skip when the count REACHES SkipTrigger; the scan resumes SkipSize
 *   bytes past the second byte of the triggering pair; equal bytes are neither
 *   favourable nor opposing; unsigned byte order) are listed in DESIGN.md.
 *
 * Conventions for every entry point:
 *   - Pointers named d_* are DEVICE pointers (cudaMalloc / PyTorch CUDA
 *     memory) on the current CUDA device; h_* are host pointers.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  All device work is enqueued on it; the host never blocks.
 *     Results are valid once the stream has been synchronised.
 *   - Cut offsets are uint64 EXCLUSIVE chunk ends, strictly increasing; for a
 *     non-empty stream the last cut equals its length.  An empty stream has
 *     no cuts.  The result is a pure function of (bytes, params): it does not
 *     depend on alignment, segmenting, batch layout or GPU count.
 *   - Return codes: SEQCDC_OK, or an error detected on the host BEFORE any
 *     work is enqueued (nothing is launched then).  Asynchronous CUDA faults
 *     surface at the next synchronisation, per CUDA convention.
 *   - No exceptions cross the ABI.  Calls are thread-safe and reentrant;
 *     concurrent calls on different streams are allowed.
 *   - Memory: the caller owns every pointer it passes.  If d_workspace is
 *     NULL the library takes scratch memory from its own per-device,
 *     stream-ordered pool (cudaMallocFromPoolAsync/cudaFreeAsync on `stream`)
 *     and keeps no pointer after the enqueued work completes.
 */
#ifndef SEQCDC_H_
#define SEQCDC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEQCDC_OK 0
#define SEQCDC_EINVAL 1   /* bad parameters or arguments */
#define SEQCDC_ENOMEM 2   /* workspace allocation failed or too small */
#define SEQCDC_ECUDA 3    /* a CUDA call failed while enqueuing */

#define SEQCDC_INCREASING 0
#define SEQCDC_DECREASING 1
#define SEQCDC_MAX_SEQ_LENGTH 16   /* implementation limit on SeqLength */

/* seqcdc_params_t.flags: compare bytes as SIGNED int8 instead of unsigned
 * (the alternative reading of P:215's untyped mm512_cmpgt; DESIGN.md c6). */
#define SEQCDC_FLAG_SIGNED 1u
/* seqcdc_params_t.flags: SeqLength counts favourable COMPARISONS instead of
 * bytes (the alternative reading of P:153, DESIGN.md c1): a chunk ends after a
 * run of L favourable pairs (L+1 bytes); scanning still starts at chunk start
 * + min - L.  Equivalent to the bytes reading with (L+1, min+1).
 * L <= SEQCDC_MAX_SEQ_LENGTH - 1 with this flag. */
#define SEQCDC_FLAG_PAIRS 2u

/* Written to *d_ncuts if the device detects inconsistent batch offsets
 * (non-monotone, or d_offsets[ns]-d_offsets[0] != total_bytes). */
#define SEQCDC_NCUTS_BAD_INPUT UINT64_MAX

/* SeqCDC parameters ("SeqLength, SkipTrigger and SkipSize"; Table I,
 * P:291-306; min/max chunk sizes P:378). */
typedef struct seqcdc_params {
    uint32_t mode;          /* SEQCDC_INCREASING or SEQCDC_DECREASING      */
    uint32_t seq_length;    /* L: bytes in a qualifying strict run, 2..16 */
    uint32_t skip_trigger;  /* T: opposing pairs that trigger a skip, >= 1 */
    uint32_t skip_size;     /* S: bytes jumped past the triggering pair's second
                               byte; 0 disables skipping                    */
    uint64_t min_size;      /* >= L; scanning starts at chunk start + min - L */
    uint64_t max_size;      /* >= min_size; forced cut                        */
    uint32_t flags;         /* 0, or SEQCDC_FLAG_SIGNED | SEQCDC_FLAG_PAIRS          */
    uint32_t reserved;      /* must be 0                                             */
} seqcdc_params_t;

/* SEQCDC_OK if *p is acceptable, SEQCDC_EINVAL otherwise (mode not 0/1,
 * L < 2 or L > SEQCDC_MAX_SEQ_LENGTH (- 1 with SEQCDC_FLAG_PAIRS), T == 0,
 * min < L, max < min, unknown flags, reserved != 0, p == NULL). */
int seqcdc_validate_params(const seqcdc_params_t *p);

/* Table I row for avg_kib in {4, 8, 16} with min = avg/2 and
 * max = 2*avg (BASELINE.json configs; the paper's 1 KB min at 4 KB, is
 * not used).  SEQCDC_EINVAL for other sizes or a bad mode. */
int seqcdc_default_params(uint32_t avg_kib, uint32_t mode, seqcdc_params_t *out);

/* Upper bound on the number of cuts of one n-byte stream: ceil(n / min)
 * (every non-final chunk has >= min bytes); 0 for n == 0. */
uint64_t seqcdc_max_cuts(uint64_t n, const seqcdc_params_t *p);

/* Upper bound on the cuts of a batch: total_bytes / min + nstreams. */
uint64_t seqcdc_max_cuts_batch(uint64_t total_bytes, uint32_t nstreams, const seqcdc_params_t *p);

/* Bytes of device scratch a call with these sizes needs (pass a buffer of at
 * least this size as d_workspace to avoid the internal pool). */
size_t seqcdc_workspace_size(uint64_t total_bytes, uint32_t nstreams, const seqcdc_params_t *p);

/*
 * Chunk one stream d_in[0..n).
 *   d_in     device, any alignment, n bytes, read-only.
 *   d_cuts   device uint64[seqcdc_max_cuts(n, p)] (capacity is a documented
 *            precondition the device cannot check).
 *   d_ncuts  device uint64[1]: number of cuts written.
 *   d_workspace/ws_bytes: optional caller scratch (see above), else NULL/0.
 * Errors: SEQCDC_EINVAL (bad params, NULL pointers with n > 0),
 * SEQCDC_ENOMEM, SEQCDC_ECUDA.
 * Walker: streams of >= 16 GiB whose runs need <= 4 favourable pairs and whose
 * max_size <= 16 KiB (the Table I 4/8 KiB rows) run on the per-lane sparse
 * walker, everything else on the warp walker; the environment
 * variable SEQCDC_WALKER=warp|lane forces one.  The result never depends on it.
 */
int seqcdc_chunk(const uint8_t *d_in, uint64_t n, const seqcdc_params_t *p,
                 uint64_t *d_cuts, uint64_t *d_ncuts,
                 void *d_workspace, size_t ws_bytes, void *stream);

/*
 * Chunk `nstreams` independent streams ("files are chunked independently";
 * boundaries never span streams).  Stream j is d_in[d_offsets[j] ..
 * d_offsets[j+1]); d_offsets is a device uint64[nstreams+1], non-decreasing,
 * and total_bytes must equal d_offsets[nstreams] - d_offsets[0] (the host
 * sizes the work from it).  Cuts are written stream after stream as offsets
 * into d_in (i.e. absolute: d_offsets[j] + local cut); stream j's cuts are
 * d_cuts[d_cut_index[j] .. d_cut_index[j+1]) with d_cut_index a device
 * uint64[nstreams+1]; *d_ncuts = total.  d_cuts capacity:
 * seqcdc_max_cuts_batch(total_bytes, nstreams, p).
 */
int seqcdc_chunk_batch(const uint8_t *d_in, const uint64_t *d_offsets, uint32_t nstreams,
                       uint64_t total_bytes, const seqcdc_params_t *p,
                       uint64_t *d_cuts, uint64_t *d_cut_index, uint64_t *d_ncuts,
                       void *d_workspace, size_t ws_bytes, void *stream);

/*
 * Range calls: the building blocks of the multi-GPU layer (one huge stream
 * sharded over P ranks; paper_2505_21194_b200/dist.py).  A
 * rank holds the range [R, R + range_len) of the stream in d_buf[0 ..
 * range_len) followed by a right halo: d_buf[range_len .. buf_len) holds the
 * next bytes of the stream.  buf_len is treated as the end of the stream, so
 * a non-final range needs a halo of at least max_size - 1 bytes (then no
 * chunk starting in the range sees it); the final range has buf_len ==
 * range_len == the rest of the stream.  "The next cut depends only on the
 * previous cut" (f(base) reads only [base, f(base)) and
 * the stream end) is what makes a range chunkable before its true first
 * chunk start is known.
 *
 * seqcdc_range_chunk: the chain of chunks that starts at local offset `entry`
 * (as if a cut were there; 0 <= entry <= range_len), up to and including its
 * first cut >= range_len (the "overhang": where the next range's first chunk
 * starts) -- or the end of the stream.  Cuts are written as global offsets
 * (global_offset + local).  entry == range_len gives 0 cuts.  d_cuts capacity:
 * seqcdc_range_max_cuts(buf_len, range_len, p).  Workspace as for
 * seqcdc_chunk.  Errors: SEQCDC_EINVAL (bad params, range_len > buf_len,
 * entry > range_len, NULL pointers), SEQCDC_ENOMEM, SEQCDC_ECUDA.
 */
uint64_t seqcdc_range_max_cuts(uint64_t buf_len, uint64_t range_len, const seqcdc_params_t *p);
int seqcdc_range_chunk(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                       uint64_t global_offset, const seqcdc_params_t *p, uint64_t *d_cuts,
                       uint64_t *d_ncuts, void *d_workspace, size_t ws_bytes, void *stream);

/*
 * seqcdc_range_resync: the TRUE chain of the range, given its true first
 * chunk start `entry` (local; the previous range's overhang minus R) and a
 * speculative chain d_spec[0 .. *d_spec_n) of the same range (global offsets,
 * from seqcdc_range_chunk).  One warp re-walks from `entry` until a cut also
 * present in d_spec (a merge: from there on both chains coincide) or until its
 * first cut >= range_len.  Writes the true chain (re-walked prefix + reused
 * speculative suffix) to d_cuts (capacity seqcdc_range_max_cuts; must not
 * alias d_spec), its length to *d_ncuts, and d_status[4] = {merged (1/0),
 * re-walked cuts, merge index in d_spec, overhang (global)}.  A range whose
 * re-walk did not merge has a new overhang, which the next range must be
 * re-synchronised from (dist.py repeats the exchange until nothing changes).
 * Errors as for seqcdc_range_chunk.
 */
int seqcdc_range_resync(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                        uint64_t global_offset, const seqcdc_params_t *p, const uint64_t *d_spec,
                        const uint64_t *d_spec_n, uint64_t *d_cuts, uint64_t *d_ncuts,
                        uint64_t *d_status, void *stream);

/*
 * seqcdc_range_resync_dev: the same, with the true entry read on the device
 * from *d_entry as a GLOBAL offset (e.g. straight out of an NCCL all_gather of
 * the overhangs), so the whole exchange can be enqueued without a host sync.
 * An entry before the range is clamped to its start, one at or past the range
 * end gives 0 cuts (d_status[0] = 2, d_status[3] = the entry).
 */
int seqcdc_range_resync_dev(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len,
                            const uint64_t *d_entry, uint64_t global_offset, const seqcdc_params_t *p,
                            const uint64_t *d_spec, const uint64_t *d_spec_n, uint64_t *d_cuts,
                            uint64_t *d_ncuts, uint64_t *d_status, void *stream);

/*
 * After chunking (§2): "Each data
 * chunk is hashed using a collision-resistant hashing algorithm, such as
 * SHA-256 ... to obtain a fingerprint"; "the fingerprint is compared
 * against a database of previously observed fingerprints"; space
 * savings = (original - deduplicated) / original (Eq. 1).
 * Both calls read the chunk count on the device (d_ncuts, e.g. the one
 * seqcdc_chunk wrote) so they can be enqueued behind it without a host sync;
 * max_cuts (host) bounds it and sizes the grids.
 *
 * seqcdc_fingerprint: d_digests[32*i .. +32) = SHA-256 (FIPS 180-4) of chunk
 * i = d_in[c_{i-1} .. c_i), c_{-1} = 0, with c = d_cuts (exclusive ends,
 * offsets into d_in).  d_digests: device, >= 32*max_cuts bytes, 16-byte
 * aligned.  Errors: SEQCDC_EINVAL (NULL pointers, misaligned d_digests),
 * SEQCDC_ECUDA.
 */
int seqcdc_fingerprint(const uint8_t *d_in, const uint64_t *d_cuts, const uint64_t *d_ncuts,
                       uint64_t max_cuts, uint8_t *d_digests, void *stream);

/* Bytes of scratch seqcdc_dedup needs for up to max_cuts chunks (its hash set). */
size_t seqcdc_dedup_workspace_size(uint64_t max_cuts);

/*
 * seqcdc_dedup: duplicate detection over the chunks' digests.  Chunk i is a
 * first occurrence iff no chunk j < i has the same digest; d_first[i] = 1/0
 * (d_first may be NULL) and *d_unique_bytes = the summed sizes of first
 * occurrences (the bytes a dedup store keeps).  d_ws/ws_bytes: scratch of
 * seqcdc_dedup_workspace_size(max_cuts) bytes, or NULL to allocate
 * stream-ordered.  Deterministic (the smallest index of each digest wins).
 * Errors: SEQCDC_EINVAL, SEQCDC_ENOMEM, SEQCDC_ECUDA.
 */
int seqcdc_dedup(const uint8_t *d_digests, const uint64_t *d_cuts, const uint64_t *d_ncuts, uint64_t max_cuts,
                 uint8_t *d_first, uint64_t *d_unique_bytes, void *d_workspace, size_t ws_bytes, void *stream);

/*
 * One-exchange sharding (dist.py's device protocol).
 *
 * A range's exchange block is uint64 [3 + tail_max] = {overhang, number of
 * cuts, tail_n, tail[0 .. tail_max)}.
 *
 * seqcdc_range_chunk_tail: seqcdc_range_chunk that also fills the block:
 * d_summary[0..2) = {overhang (the range's last cut), number of cuts}
 * (optional) and the chain continued past the overhang for up to tail_max
 * cuts, stopping before any chunk that would reach past buf_len (so only
 * fully determined chunks are written): d_tail[0] = the overhang, d_tail[1..]
 * the next cuts (global offsets), *d_tail_n = their number (0 when the
 * range's valid chain does not come from its last segment -- the next range
 * then re-walks instead).  The halo must hold those chunks (about tail_max *
 * max_size bytes).  The range's last segment is shortened so this extra walk
 * stays off the critical path.
 *
 * seqcdc_range_merge_tail: the next range's side.  d_prev = the previous
 * range's block (e.g. a row of an NCCL all_gather).  The true chain of this
 * range starts at that overhang; the first tail cut that is also in this
 * range's speculative list d_spec is a merge, and the result (d_cuts,
 * *d_ncuts, d_status as for seqcdc_range_resync) is the tail up to it plus the
 * speculative cuts after it -- no walking.  Without a merge inside the tail,
 * one warp re-walks from the overhang.  d_sum3 (optional) = {final overhang,
 * number of cuts, *d_spec_ov} for the second exchange.  All enqueued, no host
 * sync.
 */
int seqcdc_range_chunk_tail(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                            uint64_t global_offset, const seqcdc_params_t *p, uint64_t *d_cuts,
                            uint64_t *d_ncuts, uint32_t tail_max, uint64_t *d_tail, uint64_t *d_tail_n,
                            uint64_t *d_summary, void *d_workspace, size_t ws_bytes, void *stream);
int seqcdc_range_merge_tail(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t global_offset,
                            const seqcdc_params_t *p, const uint64_t *d_prev, uint32_t tail_max,
                            const uint64_t *d_spec, const uint64_t *d_spec_n, uint64_t *d_cuts,
                            uint64_t *d_ncuts, uint64_t *d_status, const uint64_t *d_spec_ov, uint64_t *d_sum3,
                            void *stream);

/* Fused exchange over peer memory ("fused alternative": the
 * overhang block is published from inside the producing kernel instead of by
 * an NCCL all_gather).
 *
 * seqcdc_xchg_alloc: a zeroed device buffer of `bytes` for this rank's
 * mailbox (cudaMalloc, owned by the caller until seqcdc_xchg_free) and its
 * SEQCDC_IPC_HANDLE_BYTES-byte CUDA IPC handle (written to ipc_handle) for the
 * other processes.  seqcdc_xchg_open maps another process's mailbox (same
 * node; peer access over NVLink is enabled lazily) into this process:
 * *d_peer is writable from kernels until seqcdc_xchg_close.  A process cannot
 * open its own handle (SEQCDC_ECUDA).
 *
 * seqcdc_range_chunk_tail_push: seqcdc_range_chunk_tail (d_summary required)
 * whose final kernel also stores the block [overhang, number of cuts, tail_n,
 * tail[0..tail_n)] into d_peer_blk (a mapped peer mailbox, 3 + tail_max
 * uint64) and then releases flag_value to *d_peer_flag at system scope.
 *
 * seqcdc_range_merge_tail_wait: seqcdc_range_merge_tail whose first kernel
 * waits (on the device, no host sync) until *d_flag >= flag_value (acquire,
 * system scope), then reads the previous range's block from d_mailbox.  After
 * timeout_ns without the flag it reports an empty range with overhang
 * UINT64_MAX, so d_sum3[0] != d_sum3[2] and the caller falls back to the
 * collective protocol.  flag_value must increase from call to call (a step
 * counter); the mailbox is reused. */
/* seqcdc_xchg_put_rows / seqcdc_xchg_wait_rows: a small all-gather over peer
 * memory (the step's second exchange).  Each rank's table holds nranks rows of
 * nwords + 1 uint64; put_rows stores d_src[0..nwords) into row `row` of every
 * rank's table (d_tables: a DEVICE array of nranks table addresses, mapped with
 * seqcdc_xchg_open, this rank's own included) and then releases `step` into the
 * row's last word; wait_rows waits on the device until every row of this
 * rank's table carries `step`, copies the rows' data packed into d_out
 * (optional, nranks * nwords uint64) and writes *d_status = 0 (1 after
 * timeout_ns, d_out untouched).
 * `step` must change from call to call; callers alternate two tables so that
 * a rank one step ahead never overwrites a row still being read. */
#define SEQCDC_IPC_HANDLE_BYTES 64
int seqcdc_xchg_put_rows(const uint64_t *d_src, uint32_t nwords, uint64_t *const *d_tables, uint32_t nranks,
                         uint32_t row, uint64_t step, void *stream);
int seqcdc_xchg_wait_rows(const uint64_t *d_table, uint32_t nwords, uint32_t nranks, uint64_t step,
                          uint64_t timeout_ns, uint64_t *d_status, uint64_t *d_out, void *stream);
int seqcdc_xchg_alloc(size_t bytes, void **d_buf, void *ipc_handle);
int seqcdc_xchg_open(const void *ipc_handle, void **d_peer);
int seqcdc_xchg_close(void *d_peer);
int seqcdc_xchg_free(void *d_buf);
int seqcdc_range_chunk_tail_push(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                                 uint64_t global_offset, const seqcdc_params_t *p, uint64_t *d_cuts,
                                 uint64_t *d_ncuts, uint32_t tail_max, uint64_t *d_tail, uint64_t *d_tail_n,
                                 uint64_t *d_summary, void *d_workspace, size_t ws_bytes, uint64_t *d_peer_blk,
                                 uint64_t *d_peer_flag, uint64_t flag_value, void *stream);
int seqcdc_range_merge_tail_wait(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t global_offset,
                                 const seqcdc_params_t *p, const uint64_t *d_mailbox, uint32_t tail_max,
                                 const uint64_t *d_spec, const uint64_t *d_spec_n, uint64_t *d_cuts,
                                 uint64_t *d_ncuts, uint64_t *d_status, const uint64_t *d_spec_ov, uint64_t *d_sum3,
                                 const uint64_t *d_flag, uint64_t flag_value, uint64_t timeout_ns, void *stream);

/* Testing / tuning knob: force the segment length G (rounded up to a
 * multiple of max_size, and to at least max_size) used to split streams into
 * speculative chains; 0 restores the automatic choice.  Process-global.  The
 * cut list never depends on it (tests/test_gpu_parity.py checks this). */
int seqcdc_set_segment_bytes(uint64_t g);

/* Profiling (used by bench.py): when enabled, each call records CUDA events
 * on its stream around its phases.  seqcdc_profile_collect() synchronises on
 * them and writes summed milliseconds ms[0] = segment setup, ms[1] = the walk
 * kernel (the hot loop), ms[2] = stitch + fallback + scan + copy, ms[3] = whole
 * call, and the number of calls; it then clears the records.  Enabling or
 * disabling also clears them.  Process-global. */
int seqcdc_profile_enable(int on);
int seqcdc_profile_collect(double *ms, uint64_t *ncalls);

/* Number of CUDA kernels this library has launched so far in this process
 * (all entry points, all devices; monotone).  Host-only, never blocks.  The
 * bench reports the difference across its timed region as its launch count. */
uint64_t seqcdc_launch_count(void);

/* Human-readable name of a return code (static string). */
const char *seqcdc_strerror(int code);

/* Library build/tuning info (static string: tile/stage sizes, arch). */
const char *seqcdc_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SEQCDC_H_ */
