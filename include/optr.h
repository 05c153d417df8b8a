/*
 * optr.h -- C ABI of the B200-native OptiReduce TAR+RHT hot path.
 *
 * One shared library (paper_2310_06993_b200/liboptr.so) exports these
 * entry points.  They take plain pointers and sizes (device pointers unless
 * noted), enqueue on the caller's CUDA stream, never synchronise the host
 * unless the comment says so, and return an int status.  No torch types.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/ubar/):
 *
 *   optr_derive_seed          hadamard.py:31-34   derive_seed
 *   optr_pcg64_output         hadamard.py:49-50   PCG64(SeedSequence(seed)) stream (k-th draw)
 *   optr_rht_signs            hadamard.py:49-51   RhtContext.signs  (bit-packed, +1 = 1)
 *   optr_fwht                 hadamard.py:76-90   fwht_in_place
 *   optr_rht_encode           hadamard.py:93-102  rht_encode
 *   optr_rht_decode           hadamard.py:105-123 rht_decode (+ EmptyReceptionError)
 *   optr_*_f64                hadamard.py:76-123 in float64, bit-identical
 *   optr_masks_host           datagram.py:70-72,111-124 send-side coin, as packet bitmaps
 *   optr_coin_packets         datagram.py:70-72,122 the coin of any sender's k-th packets
 *   optr_mean_received        collectives.py:77-94 _mean_received
 *   optr_ring_*               collectives.py:248-292 ring_allreduce arithmetic
 *   optr_packetize / _depacketize  wire.py:36-85,176-208 header codec + framing
 *   optr_tar_local            runner.py:211-276 run_generation hot path (encode ->
 *                             collectives.py:97-150 tar_allreduce -> decode) for n
 *                             workers co-resident on one GPU (the SimSession shape)
 *   optr_comm_* / optr_tar    the same path with one worker per GPU (one process per
 *                             GPU), peers' buffers mapped over NVLink (CUDA IPC)
 *
 * Status codes map to the reference's exceptions in the Python facade:
 *   OPTR_EINVAL -> ValueError, OPTR_EEMPTY -> EmptyReceptionError,
 *   OPTR_ECUDA / OPTR_ENOMEM -> RuntimeError.
 */
#ifndef OPTR_H_
#define OPTR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OPTR_OK 0
#define OPTR_EINVAL 1
#define OPTR_EEMPTY 2
#define OPTR_ECUDA 3
#define OPTR_ENOMEM 4

#define OPTR_MAX_WORKERS 16

/* element types of caller buffers (the wire / aggregate is always fp32) */
#define OPTR_F32 0
#define OPTR_BF16 1

/* mask kinds */
#define OPTR_MASK_NONE 0   /* lossless channel, collectives.py:321-401            */
#define OPTR_MASK_COIN 1   /* datagram coin, counter-indexed PCG64 (bit-exact)     */
#define OPTR_MASK_BITMAP 2 /* caller-supplied packet bitmaps (captured sim masks) */

/*
 * Drop masks, per packet.  Packet k of a (stage, dst, src) transfer covers
 * shard entries [k*epp, min((k+1)*epp, len)).  Stage 1 carries shard
 * owned_shard(dst), stage 2 carries owned_shard(src) (collectives.py:117-137).
 * Bitmap layout (u32 words, bit k%32 of word k/32, 1 = delivered):
 *   word index = ((stage * n + dst) * n + src) * words_per_pair + k / 32,
 *   stage in {0 (stage 1), 1 (stage 2)}, words_per_pair from optr_mask_words.
 */
typedef struct {
  int32_t kind;          /* OPTR_MASK_*                                        */
  int32_t epp;           /* entries per packet = max_payload / 4 (350)         */
  uint64_t seed;         /* COIN: sender src draws from SeedSequence([seed,src]) */
  double drop_prob;      /* COIN: packet dropped iff random() < drop_prob      */
  const uint32_t* bitmap;/* BITMAP: device pointer in the layout above         */
  /* COIN: host array of n draws each sender's stream made before this call
   * (a DatagramEndpoint keeps one generator for every run(), datagram.py:70-72,
   * so its k-th collective continues the stream); NULL = fresh streams.     */
  const uint64_t* stream_offsets;
} optr_mask_spec;

/* ------------------------------------------------------------ host helpers */
uint64_t optr_derive_seed(uint64_t job_seed, uint64_t bucket_id, uint64_t generation);
/* k-th u64 output of PCG64(SeedSequence(entropy[0..n_entropy))) */
uint64_t optr_pcg64_output(const uint64_t* entropy, int n_entropy, uint64_t k);
int64_t optr_next_pow2(int64_t n);
/* u32 words per (stage,dst,src) pair for a vector of `dim` entries */
int64_t optr_mask_words(int64_t dim, int n, int epp);
/* host computation of the coin bitmaps (same layout; no GPU needed) */
int optr_masks_host(uint32_t* bitmap_host, int64_t dim, int n, int rotation,
                    uint64_t seed, double drop_prob, int epp);
/* keep[i] = 1 iff packet start+i of sender src's datagram coin stream is
 * delivered (PCG64(SeedSequence([seed, src])).random() >= drop_prob,
 * datagram.py:70-72,122), counter-indexed: any collective's per-packet
 * drops in its own send order (host, no GPU needed). */
int optr_coin_packets(uint64_t seed, int src, uint64_t start, int64_t count, double drop_prob,
                      uint8_t* keep_host);
/* library build/version string */
const char* optr_version(void);

/* ------------------------------------------------------------- codec (GPU) */
/* Rademacher signs as D bits (bit k of word k/32; 1 = +1).  D = power of 2. */
int optr_rht_signs(uint32_t* sign_bits, int64_t dim, uint64_t seed, void* stream);

/* Unnormalised Sylvester FWHT of fp32 v[0..dim) in place; dim = 2^k. */
int optr_fwht(float* v, int64_t dim, void* stream);

/* y[0..dim) = H (signs * pad(x[0..L))) / sqrt(dim).  x is OPTR_F32/BF16. */
int optr_rht_encode(const void* x, int dtype_in, int64_t L, float* y, int64_t dim,
                    uint64_t seed, void* stream);

/* out[0..L) = signs * H(mask ? y : 0) * (dim/count) / sqrt(dim).
 * mask: device bytes (1 = received) or NULL for all received.
 * Synchronises the stream to read count; returns OPTR_EEMPTY if count == 0
 * (hadamard.py:117-118).  out dtype OPTR_F32/BF16. */
int optr_rht_decode(const float* y, const uint8_t* mask, int64_t dim, int64_t L,
                    uint64_t seed, void* out, int dtype_out, void* stream);

/* Float64 codec in the reference's own arithmetic (numpy float64 callers):
 * the same butterfly stages in the same order as hadamard.py:76-90, so the
 * results are bit-identical to the reference's fwht_in_place / rht_encode /
 * rht_decode (hadamard.py:76-123).  optr_rht_decode_f64 synchronises the
 * stream to read the received count (OPTR_EEMPTY when it is 0). */
int optr_fwht_f64(double* v, int64_t dim, void* stream);
int optr_rht_encode_f64(const double* x, int64_t L, double* y, int64_t dim, uint64_t seed, void* stream);
int optr_rht_decode_f64(const double* y, const uint8_t* mask, int64_t dim, int64_t L, uint64_t seed,
                        double* out, void* stream);

/* collectives.py:77-94 _mean_received on the GPU: out = float32(sum in
 * ascending node order of own (i == rank) and peers[i] (as given, zero where
 * missing) / sum of (1 for own, masks[i] for peers)), 0 where the count is 0,
 * accumulated in float64 -- bit-identical to the reference.  peers, masks:
 * HOST arrays of n device pointers; peers[i] NULL = no data from i (skipped),
 * masks[i] NULL = every entry of peers[i] received (1 byte per entry). */
int optr_mean_received(const float* own, const float* const* peers, const uint8_t* const* masks, int n,
                       int rank, int64_t len, float* out, void* stream);

/* Ring baseline steps (collectives.py:248-292), float64 partial sums:
 * optr_ring_cast: out = float32(chunk); optr_ring_step: gather == 0 ->
 * chunk += data, gather == 1 -> chunk[mask] = data[mask] (mask NULL = all);
 * optr_ring_finish: out = float32(buf / nodes). */
int optr_ring_cast(const double* chunk, int64_t n, float* out, void* stream);
int optr_ring_step(double* chunk, const float* data, const uint8_t* mask, int64_t n, int gather, void* stream);
int optr_ring_finish(const double* buf, int nodes, int64_t len, float* out, void* stream);

/* Datagram framing on the GPU (wire.py:36-85,176-208).  Packet k of a shard
 * of n_entries float32 values sits at packets + k*stride (stride >=
 * 9 + max_payload): a 9-byte big-endian header (bucket_id u16, byte_offset
 * u32 = base_byte_offset + k*max_payload, timeout_share u8, flags u8 = last-
 * percentile tag | incast << 1, reserved 0) then the payload bytes.  The
 * final max(1, total/100) packets carry the tag.  OPTR_EINVAL for the
 * reference's HeaderError ranges; max_payload must be a multiple of 4.
 * optr_depacketize zero-fills shard_out / mask_out, then lands every
 * delivered packet (delivered[k] != 0, or all when NULL) at its header's
 * offset; packets with a bad header (reserved byte, bucket id, offset) are
 * skipped and counted in *errors (device u32). */
int optr_packetize(const float* shard, int64_t n_entries, int bucket_id, uint32_t base_byte_offset,
                   int max_payload, int timeout_share, int incast, uint8_t* packets, int64_t stride,
                   void* stream);
int optr_depacketize(const uint8_t* packets, int64_t n_packets, int64_t stride, const uint8_t* delivered,
                     int bucket_id, uint32_t base_byte_offset, int max_payload, float* shard_out,
                     uint8_t* mask_out, int64_t n_entries, unsigned int* errors, void* stream);

/* ------------------------------------------- TAR+RHT, n workers on one GPU */
/* Workspace bytes for optr_tar_local. */
size_t optr_tar_local_workspace(int n, int64_t L, int ht, int epp);

/*
 * One generation of runner.py:211-276 for n co-resident workers:
 *   ht: signs from derive_seed(job_seed, bucket_id, generation) (the runner
 *       passes bucket_id = generation % 65536, runner.py:219-222),
 *       y_w = rht_encode(x_w) (fp32 wire), TAR with rotation, decode per worker
 *       (count 0 -> zeros, runner.py:255-256);
 *   !ht: TAR of x_w directly.
 * x[w], out[w]: device pointers to L elements of dtype_in / dtype_out.
 * received_out: optional device array [2][n] of u64 received entries per
 *   (stage, dst) -- the numbers NodeStats/StageOutcome derive loss from.
 * got_out: optional device bytes [n][dim] = AllReduceResult.received.
 */
int optr_tar_local(const void* const* x, void* const* out, int n, int64_t L,
                   int dtype_in, int dtype_out, uint64_t job_seed, uint64_t bucket_id,
                   uint64_t generation, int rotation, int ht, const optr_mask_spec* masks,
                   void* workspace,
                   size_t workspace_bytes, uint64_t* received_out, uint8_t* got_out,
                   void* stream);

/* Same as optr_tar_local but the caller's stream does not wait: the call
 * runs on the library's work stream of `slot` (0 or 1) after the caller's
 * prior work, so two consecutive buckets overlap.  Calls on the same slot
 * run in order; x, out, workspace and the outputs of a slot must stay
 * untouched until optr_local_join. */
int optr_tar_local_async(const void* const* x, void* const* out, int n, int64_t L,
                         int dtype_in, int dtype_out, uint64_t job_seed, uint64_t bucket_id,
                         uint64_t generation, int rotation, int ht, const optr_mask_spec* masks,
                         void* workspace, size_t workspace_bytes, uint64_t* received_out,
                         uint8_t* got_out, int slot, void* stream);
/* Make `stream` wait for every optr_tar_local_async call issued so far. */
int optr_local_join(void* stream);

/* --------------------------------------- TAR+RHT, one worker per GPU (IPC) */
typedef struct optr_comm_s* optr_comm;

/* Allocate, on CUDA device `device`, this rank's symmetric buffers for
 * buckets up to max_len entries.  Every rank calls it with the same n,
 * max_len and epp. */
int optr_comm_create(optr_comm* out, int device, int rank, int n, int64_t max_len, int epp);
/* Bytes of the opaque IPC handle blob each rank must share with all peers. */
size_t optr_comm_handle_bytes(void);
int optr_comm_get_handle(optr_comm c, void* handle_out);
/* all_handles: n blobs of optr_comm_handle_bytes(), rank order.  Maps every
 * peer's buffers (cudaIpcOpenMemHandle) and checks peer access. */
int optr_comm_open(optr_comm c, const void* all_handles);
int optr_comm_destroy(optr_comm c);

/* This rank's part of one generation (same semantics as optr_tar_local for
 * worker `rank`): x, out are this rank's L-element buffers.
 * received_out: optional device u64[2] (stage1, stage2) for this rank. */
int optr_tar(optr_comm c, const void* x, void* out, int64_t L, int dtype_in,
             int dtype_out, uint64_t job_seed, uint64_t bucket_id, uint64_t generation,
             int rotation, int ht, const optr_mask_spec* masks, uint64_t* received_out,
             void* stream);

/* Same as optr_tar, but the caller's stream does not wait for the result:
 * the call runs on the communicator's work stream of its call parity, so
 * consecutive buckets overlap (one bucket's NVLink stages with the next
 * bucket's encode).  x and out must stay valid and untouched until
 * optr_comm_join.  At most two calls are in flight per parity ordering. */
int optr_tar_async(optr_comm c, const void* x, void* out, int64_t L, int dtype_in,
                   int dtype_out, uint64_t job_seed, uint64_t bucket_id, uint64_t generation,
                   int rotation, int ht, const optr_mask_spec* masks, uint64_t* received_out,
                   void* stream);
/* Make `stream` wait for every optr_tar_async call issued so far. */
int optr_comm_join(optr_comm c, void* stream);

/* Per-call transport report (device memory, written by the call): the
 * numbers StageOutcome / NodeStats carry (simdriver.py:26-45,328-341). */
typedef struct {
  uint64_t received[2];  /* entries this rank received, stage 1 / stage 2   */
  uint64_t cut[2];       /* entries the mask model delivered but a stage
                            deadline cut off (counted as lost)            */
  uint64_t t_open_ns;    /* device global timer: this rank's stage 1 opened */
  uint64_t t_stage1_ns;  /* its last stage-1 (owner) unit was published     */
  uint64_t t_stage2_ns;  /* its last stage-2 tile landed                    */
} optr_tar_stats;

/* optr_tar with OptiReduce's bounded stage 1 (UBT hard bound t_B,
 * transport.py:102-108, simdriver.py:323-326 / datagram.py:165-207): on the
 * fused plan an owner waits for a peer's encoded tile at most
 * stage1_deadline_ns after it opened the stage, then aggregates without it;
 * the cut entries count as lost (stats->cut[0]) and cut_units (optional,
 * device u32 per stage-1 unit of 2^T/UPT entries) gets each unit's bitmask of
 * cut peers.  0 = unbounded; the barrier path (other shapes) never cuts.
 * stats: optional device optr_tar_stats.  async: as optr_tar_async. */
int optr_tar_bounded(optr_comm c, const void* x, void* out, int64_t L, int dtype_in, int dtype_out,
                     uint64_t job_seed, uint64_t bucket_id, uint64_t generation, int rotation, int ht,
                     const optr_mask_spec* masks, uint64_t stage1_deadline_ns, optr_tar_stats* stats,
                     uint32_t* cut_units, int async, void* stream);

/* Cap the persistent fused kernel at `ctas` CTAs (0 = SMs x occupancy): in
 * DDP the kernel waits on peers while backward compute wants the SMs. */
int optr_comm_set_fused_grid(optr_comm c, int ctas);

/* Device-side all-rank barrier on `stream` (flags over NVLink). */
int optr_comm_barrier(optr_comm c, void* stream);

/* Entries per stage-1 unit of the fused plan for (dim, n) -- the granularity
 * of optr_tar_bounded's deadline cut-offs; 0 when the shape takes the
 * barrier path (no cut-offs). */
int64_t optr_fused_unit_entries(int64_t dim, int n);

/* --------------------------------------------------------- instrumentation */
/* Kernel classes timed when timing is enabled. */
#define OPTR_K_PREP 0       /* signs + masks + counts                        */
#define OPTR_K_ENC_FIRST 1  /* first encode FWHT pass (reads x, signs, pad)  */
#define OPTR_K_ENC_MID 2    /* middle encode passes (in place)              */
#define OPTR_K_ENC_LAST 3   /* last encode pass (writes the fp32 wire)      */
#define OPTR_K_AGG 4        /* stage-1 masked mean at the owner             */
#define OPTR_K_DEC_FIRST 5  /* stage-2 gather + first decode pass           */
#define OPTR_K_DEC_MID 6
#define OPTR_K_DEC_LAST 7   /* last decode pass (scale, sign, cast, out)    */
#define OPTR_K_ASSEMBLE 8   /* stage-2 gather without RHT                   */
#define OPTR_K_BARRIER 9
#define OPTR_K_OTHER 10
#define OPTR_K_ENC_MEAN 11  /* one GPU: last encode pass of every worker fused
                               with the stage-1 mean (wire never written)   */
#define OPTR_K_FUSED 12     /* multi-GPU: contiguous encode + stage 1 + stage 2
                               + contiguous decode, one persistent launch  */
#define OPTR_K_SMALL 13     /* multi-GPU buckets <= 2^20 entries: the whole call
                               in one cooperative launch                    */
#define OPTR_K_CLASSES 14
/* Enable (1) / disable (0) CUDA-event timing of every kernel launch. */
int optr_timing_enable(int on);
/* Debug: event trace of the fused multi-GPU kernel into a device buffer of
 * gridDim * per_cta uint4 records (null disables); per_cta < 0 instead points
 * the small-bucket kernels' phase stamps (u64 globaltimer ns: [64][16] per
 * call epoch for tar_small_kernel, [16] for tar_small_local_kernel) at the
 * buffer.  Not thread-safe. */
int optr_debug_trace(void* dev_buf, int64_t per_cta);
/* Synchronise recorded events and return, per class, the summed device
 * milliseconds, the launch count and the worker-passes those launches
 * covered (a launch over k co-resident workers counts k) since the last
 * reset; then reset.  Any pointer may be NULL. */
int optr_timing_collect(double* ms_out, int64_t* launches_out, int64_t* units_out);
/* Kernels this library launched since load (all classes, any device). */
int64_t optr_launch_count(void);

/* --------------------------------------------------------------- probes */
/* Measurement helpers for the NVLink / HBM peaks (tools/nvlink_probe.py). */
int optr_probe_enable_peer(int device, int peer);
/* float4 grid-stride copy of `bytes` (multiple of 16) on `device`; either
 * pointer may be a peer allocation (SM pull / push over NVLink). */
int optr_probe_copy(void* dst, const void* src, int64_t bytes, int blocks, int device, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* OPTR_H_ */
