/*
 * twb200.h — C ABI of libtwb200, the B200 engine for the Revati/timewarp hot path
 * (arXiv 2601.00397): batch-duration prediction, Timekeeper min-advance, and the
 * lockstep discrete-event loop, evaluated in bulk over many serving configs.
 *
 * Conventions (all entry points):
 *   - every data pointer is a DEVICE pointer allocated by the caller (the library
 *     never allocates except the small scratch noted per call); sizes are element
 *     counts unless the name says bytes;
 *   - work is enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *     default stream) and is stream-ordered; calls never synchronize;
 *   - return 0 on success, otherwise a TW_E* code; tw_last_error() gives text.
 *     Per-element domain errors (EmptyBatch, NegativeDuration, TableMiss) are NOT
 *     call failures: they are written as negative codes into the output arrays,
 *     and the Python shim re-raises the reference's exception classes.
 *   - reentrant; one host thread per device is the intended use.
 *
 * The reference is pure Python; the boundary a maintainer binds is its plugin
 * surface (see INTEGRATION.md for the ctypes stubs):
 *   predictor plugin   pkg/src/timewarp/predictor.py:100-266 (predict(batch, hw) -> ns)
 *   Timekeeper core    pkg/src/timewarp/timekeeper.py:68-366 (BarrierCore.handle/_resolve)
 *   event loop         pkg/src/timewarp/oracle.py:49-180     (simulate / _plan)
 */
#ifndef TWB200_H
#define TWB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TWB200_ABI_VERSION 2 /* 2: tw_predict_one_sync lost dev_io; tw_core_abort / set_suppress; TW_PRED_NAN / OVERFLOW */

/* ---- call status codes ---------------------------------------------------- */
#define TW_OK 0
#define TW_EINVAL 1    /* bad argument (null pointer, size, malformed blob) */
#define TW_ECUDA 2     /* CUDA launch/runtime error */
#define TW_ENOSMEM 3   /* predictor blob or per-warp state exceeds shared memory */
#define TW_ECALLBACK 4 /* a host callback of the native BarrierCore failed (tw_core_abort) */

/* ---- per-element prediction codes (negative int64 in out_ns) -------------- */
#define TW_PRED_EMPTY_BATCH (-1)      /* predictor.py:95-97   EmptyBatch       */
#define TW_PRED_NEGATIVE (-2)         /* predictor.py:143-145 NegativeDuration */
#define TW_PRED_TABLE_MISS (-3)       /* predictor.py:240-242 TableMiss        */
#define TW_PRED_BAD_DESC (-4)         /* desc_id out of range (host bug)       */
#define TW_PRED_NAN (-5)              /* predictor.py:142 round(nan): ValueError */
#define TW_PRED_OVERFLOW (-6)         /* round(+-inf): OverflowError; or a duration
                                         beyond int64 ns (the reference returns a
                                         Python int there: engine limit)          */

/* ---- predictor set ("pset") blob ------------------------------------------ */
/* One contiguous, 16-byte aligned byte blob holding every predictor a sweep uses:
 *   tw_pset_header | tw_pred_desc[n_desc] | table pool | bulk-lookup section
 * A table (kind TABLE) occupies, at byte offset `table_off` from the blob start:
 *   int32 paxis[np] (sorted, unique) | int32 daxis[nd] (sorted, unique) |
 *   (pad to 8) | int64 grid_us[np*nd] (row-major [p][d]; TW_TABLE_HOLE = no row) |
 *   fp64 rp[np], rd[nd]: RN(1 / (axis[k+1] - axis[k])) per interval (last unused) |
 *   int16 lutp[34][2], lutd[34][2]: for b = bitlen(v - axis[0]), the floor index of v
 *   (largest i with axis[i] <= v) lies in [lut[b][0], lut[b][1]] |
 *   int32 grid32[np*nd] (only when desc.pad == 1: every value < 2^31 us)
 * Bulk-lookup section (derived data for the bulk predictor kernels; byte offsets
 * below are from the blob start and stored in 16-byte units):
 *   uint32 qhdr[n_desc][2] (padded to 16 B): w0 = quads16 | prec16 << 16,
 *     w1 = drec16 | nd << 16 | TW_QHDR_FAST (bit 31: the table takes the fast path)
 *   axis record sets, one per DISTINCT axis (tables on a common grid share them):
 *     int32 rec[32][4] = {lo, hi, info, 0} for b = bitlen(v), v >= 0: every v of
 *     that bit length inside [axis[0], axis[n-1]] has floor index i = info & 0xffff
 *     (info < 0: the bucket straddles several intervals -> generic path);
 *     lo = axis[i], hi = axis[i+1] (axis[i] at the last index); v outside [lo, hi]
 *     is outside the axis
 *   int32 quads[np][nd][4] per fast table = {c[i][j], c[i+1][j], c[i][j+1],
 *     c[i+1][j+1]} (indices clamped at the last row/column; holes = -1)
 * The event loop needs only the first core_bytes (tw_sim_many accepts that as
 * pset_bytes; passing the whole blob lets its prediction-cache misses use the
 * bulk-lookup section); the bulk predictor kernels take the whole blob. The blob is
 * built on host (paper_2601_00397_b200/predictor.py::PredictorSet) and staged into
 * shared memory by each CTA with cp.async.bulk (TMA), except in tw_sim_many's
 * throughput variant, which reads it from global memory. */
#define TW_QHDR_FAST 0x80000000u
#define TW_PSET_MAGIC 0x54534550u /* "PEST" little-endian */
#define TW_PRED_CONSTANT 0        /* predictor.py:100-111 */
#define TW_PRED_LINEAR 1          /* predictor.py:114-146 */
#define TW_PRED_TABLE 2           /* predictor.py:149-242 */
/* grid cell with no calibration row (table values may be negative: TablePredictor(rows)
 * accepts them, predictor.py:164-170; only from_csv rejects them); the int32 copy of a
 * grid, present only when every value lies in [0, 2^31), marks holes with -1 */
#define TW_TABLE_HOLE (-9223372036854775807LL - 1)
#define TW_TABLE_HOLE32 (-1)

typedef struct tw_pset_header {
  uint32_t magic;
  uint32_t version;     /* 2 */
  int32_t n_desc;
  int32_t total_bytes;  /* whole blob, multiple of 16 */
  int32_t core_bytes;   /* header | descs | table pool: all the event loop reads */
  int32_t fast_off;     /* == core_bytes: start of the bulk-lookup section (below) */
  int32_t n_axis_sets;  /* distinct table axes in the bulk-lookup section */
  int32_t reserved;
} tw_pset_header;       /* 32 B */

typedef struct tw_pred_desc {
  int32_t kind;                /* TW_PRED_* */
  int32_t allow_extrapolation; /* TABLE: nearest-row fallback (predictor.py:238-239) */
  int64_t constant_us;         /* CONSTANT: duration_us (>= 0, checked on host) */
  double base_us;              /* LINEAR coefficients, applied left to right:     */
  double per_prefill_token_us; /* ((base + kp*P) + kd*D) + kc*C, each op rounded  */
  double per_decode_us;        /* in fp64, no FMA (predictor.py:137-142)          */
  double per_context_token_us;
  int32_t table_off; /* TABLE: byte offset of paxis from blob start */
  int32_t np;        /* TABLE: prefill-axis length */
  int32_t nd;        /* TABLE: decode-axis length  */
  int32_t pad;       /* TABLE: 1 = an int32 copy of the grid follows the LUTs */
} tw_pred_desc; /* 64 B */

/* ---- bulk predictor (kernel 2 of the north star) -------------------------- */
/* out_ns[i] = predict(features i) in ns (multiple of 1000) or a TW_PRED_* code.
 * Durations are whole microseconds x 1000, so a value < 0 that is a multiple of 1000 is a
 * (negative) duration from a table with negative rows and any other value < 0 is a code.
 * Features are the reference's BatchComposition totals (predictor.py:69-84):
 * P = total_prefill_tokens, D = num_decodes, C = total_context; a batch is empty
 * iff it has no slots, which the feature-only entry point encodes as
 * P == 0 && D == 0 && C < 0 (C = -1 marks "no slots": predictor.py:83-84). */
int tw_predict_features(const void* pset, int64_t pset_bytes, const int32_t* P,
                        const int32_t* D, const int64_t* C, const int32_t* desc_id,
                        int64_t n, int64_t* out_ns, void* stream);

/* Fused batch-feature extraction + prediction over CSR batches (kernels 1+2).
 * Batch b owns slots [batch_off[b], batch_off[b+1]); a slot is a PrefillChunk
 * (slot_tok >= 0: chunk_tokens, slot_ctx: context_len_before) or a DecodeSlot
 * (slot_tok == -1, slot_ctx: context_len) — predictor.py:47-61.
 * slot_tok / slot_ctx must be 16-byte aligned and readable up to the next multiple
 * of 4 elements past the last slot (tiles of slots move with TMA bulk copies).
 * feat_out (optional, may be NULL) receives int64 {P, D, C} per batch. */
int tw_predict_batches(const void* pset, int64_t pset_bytes, const int64_t* batch_off,
                       const int32_t* slot_tok, const int32_t* slot_ctx,
                       const int32_t* desc_id, int64_t n_batches, int64_t* feat_out,
                       int64_t* out_ns, void* stream);

/* One batch, synchronously, for the live engine's per-step predict() (engine.py:684):
 * host_slots holds int32 tok[n_slots] then int32 ctx[n_slots] (slot encoding as in
 * tw_predict_batches). The call stages them in caller-owned pinned host memory
 * (io_bytes >= 8*n_slots + 8), which a one-warp kernel reads and answers in place
 * (zero-copy under UVA), reading the predictor blob from global
 * memory; the call then polls the answer word in the pinned buffer instead of
 * synchronizing `stream` (which it does only if no answer arrives within 200 ms, to
 * report the kernel's error). *out_ns receives ns or a TW_PRED_* code. */
int tw_predict_one_sync(const void* pset, int64_t pset_bytes, const int32_t* host_slots,
                        int32_t n_slots, int32_t desc_id, void* pinned_io, int64_t io_bytes,
                        int64_t* out_ns, void* stream);

/* Resident predictor service (the live engine's per-step predict(), engine.py:684):
 * tw_service_start launches one persistent warp on its own non-blocking stream that
 * serves requests through a mailbox in mapped pinned host memory; tw_service_predict
 * (host_slots: int32 tok[n_slots] then ctx[n_slots]) writes a request and spins until
 * the answer arrives (ns or a TW_PRED_* code in *out_ns); tw_service_stop ends the
 * kernel and frees the mailbox. One caller thread per service. */
typedef struct tw_service tw_service;
int tw_service_start(const void* pset, int64_t pset_bytes, int32_t max_slots, tw_service** out);
int tw_service_predict(tw_service* service, const int32_t* host_slots, int32_t n_slots,
                       int32_t desc_id, int64_t* out_ns);
/* The same request with the batch's features extracted on the host (P = total prefill
 * tokens, D = number of decodes, C = total context; predictor.py:69-84; each < 2^48):
 * one 32-byte mailbox read on the device, no slot transfer. The caller answers an empty
 * batch itself (EmptyBatch): (P, D, C) of a non-empty batch are predicted as given. */
int tw_service_predict_features(tw_service* service, int64_t total_prefill_tokens, int64_t num_decodes,
                                int64_t total_context, int32_t desc_id, int64_t* out_ns);
int tw_service_stop(tw_service* service);

/* Device self-test of the predictor's reciprocal-based exact division against the
 * hardware's correctly rounded __ddiv_rn on n pseudo-random operand pairs; adds the
 * number of differing quotients to *mismatches (device counter, caller-zeroed). */
int tw_selftest_division(int64_t n, uint64_t seed, unsigned long long* mismatches, void* stream);

/* ---- Timekeeper (kernel 3): BarrierCore op-stream replay ------------------ */
/* One op stream per Timekeeper instance ("config"); every stream is replayed
 * by one warp with the BarrierCore state machine (timekeeper.py:131-366) on a
 * FakeClock (pkg/tests/_support.py:25-38). Actors are identified by their
 * registration index (client ids "actor1", "observer2", ... map to 0, 1, ...). */
#define TW_OP_REGISTER_ACTOR 0    /* arg ignored                              */
#define TW_OP_REGISTER_OBSERVER 1
#define TW_OP_SEAL 2
#define TW_OP_JUMP 3              /* client, arg = absolute target ns          */
#define TW_OP_ENTER 4             /* client, group (small int), arg = expected */
#define TW_OP_DEREGISTER 5        /* client                                    */
#define TW_OP_ADVANCE_CLOCK 6     /* arg = ns the FakeClock moves forward      */
#define TW_OP_BAD_CLIENT 7        /* any op naming an unknown client id        */

/* ack codes written per op (errors.py:12-45, wire.py MalformedBody) */
#define TW_ACK_OK 0
#define TW_ACK_REGISTRATION_SEALED 1
#define TW_ACK_NO_ACTORS 2
#define TW_ACK_UNKNOWN_CLIENT 3
#define TW_ACK_INVALID_STATE 4
#define TW_ACK_ROLE_VIOLATION 5
#define TW_ACK_INVALID_DELTA 6
#define TW_ACK_EXPECTED_MISMATCH 7
#define TW_ACK_TOO_MANY 8 /* > TW_TK_MAX_CLIENTS clients or groups (engine limit) */

#define TW_TK_MAX_CLIENTS 32
#define TW_TK_MAX_GROUPS 32
/* tw_tk_replay_wide: the same replay for streams with up to 1,024 clients and 64 groups */
#define TW_TK_MAX_CLIENTS_WIDE 1024
#define TW_TK_MAX_GROUPS_WIDE 64

typedef struct tw_tk_op {
  int64_t arg;
  int32_t type;   /* TW_OP_* */
  int16_t client; /* registration index */
  int16_t group;  /* collective group index */
} tw_tk_op;       /* 16 B */

typedef struct tw_tk_event {
  int64_t offset_ns; /* CLOCK_UPDATE offset, or COLLECTIVE_RELEASE group  */
  int64_t seq;       /* CLOCK_UPDATE seq, or release generation           */
  int64_t wall_ns;   /* FakeClock stamp                                   */
  int32_t kind;      /* 0 = CLOCK_UPDATE (incl. suppressed), 1 = RELEASE  */
  int32_t op_index;  /* op that triggered it                              */
} tw_tk_event;       /* 32 B */

typedef struct tw_tk_final {
  int64_t offset_ns;
  int64_t seq;
  int64_t wall_ns;
  int64_t rounds;     /* resolves */
  int64_t broadcasts; /* CLOCK_UPDATEs (including suppressed ones) */
  int64_t n_events;   /* total events produced (may exceed capacity) */
  int32_t status;     /* 0 ok, 1 event buffer overflow, 2 engine limit hit */
  int32_t pad;
  int64_t pad2;
} tw_tk_final; /* 64 B */

/* Streams are CSR: stream s owns ops [op_off[s], op_off[s+1]); its events go to
 * ev[ev_off[s] ..  ev_off[s+1]) (capacity; excess counted, not written).
 * wall0_ns[s]: FakeClock start; cooldown_ns[s]: BarrierCore cooldown (>= 0);
 * suppress[s]: suppress_broadcasts flag. ack: one int32 per op. */
int tw_tk_replay(const tw_tk_op* ops, const int64_t* op_off, int32_t n_streams,
                 const int64_t* wall0_ns, const int64_t* cooldown_ns,
                 const uint8_t* suppress, int32_t* ack, tw_tk_event* ev,
                 const int64_t* ev_off, tw_tk_final* fin, void* stream);

/* The same replay for wide streams (up to TW_TK_MAX_CLIENTS_WIDE clients and
 * TW_TK_MAX_GROUPS_WIDE groups; BarrierCore has no limit): one warp per stream with its
 * client and group state in shared memory, lanes striding over clients. */
int tw_tk_replay_wide(const tw_tk_op* ops, const int64_t* op_off, int32_t n_streams,
                      const int64_t* wall0_ns, const int64_t* cooldown_ns,
                      const uint8_t* suppress, int32_t* ack, tw_tk_event* ev,
                      const int64_t* ev_off, tw_tk_final* fin, void* stream);

/* tw_tk_resolve for any A >= 1: eligible_words holds ceil(A/32) uint32 words per
 * Timekeeper (bit a of word a/32 = actor a eligible); one warp per Timekeeper. */
int tw_tk_resolve_wide(int64_t* pending, const uint32_t* eligible_words, int32_t n_cfg, int32_t A,
                       int64_t cooldown_ns, int64_t* offset_ns, int64_t* seq, int64_t* wall_ns,
                       int64_t* last_bcast_ns, int8_t* broadcast, void* stream);

/* Bulk min-advance (the _try_resolve/_resolve arithmetic, timekeeper.py:318-366)
 * for C independent Timekeepers with A actor slots each, one round:
 * pending[c*A + a] = requested target or INT64_MAX (no request / not eligible);
 * eligible_mask[c] bit a = actor a is active and not exempt. A round resolves
 * iff sealed (assumed) and every eligible actor has a pending target. State
 * arrays (offset/seq/wall/last_bcast; last_bcast = INT64_MIN means None) are
 * updated in place; broadcast[c] = 1 when a CLOCK_UPDATE is emitted, 0 when the
 * round resolved silently, -1 when it did not resolve. Pending entries of
 * resolved configs are reset to INT64_MAX (pending.clear()). Requires A <= 32. */
int tw_tk_resolve(int64_t* pending, const uint32_t* eligible_mask, int32_t n_cfg,
                  int32_t A, int64_t cooldown_ns, int64_t* offset_ns, int64_t* seq,
                  int64_t* wall_ns, int64_t* last_bcast_ns, int8_t* broadcast,
                  void* stream);

/* ---- lockstep event loop (kernel 4): oracle.simulate over many configs ---- */
#define TW_POLICY_MIXED 0               /* engine.py:46-48 */
#define TW_POLICY_PREFILL_PRIORITIZED 1

#define TW_SIM_TIMEKEEPER 1u /* flags: drive virtual time through per-config BarrierCore rounds */

typedef struct tw_sim_cfg {
  /* EngineConfig (engine.py:98-133) */
  int32_t chunk_size;
  int32_t max_batch_tokens;
  int32_t max_running;
  int32_t kv_block_tokens;
  int32_t kv_capacity_blocks;
  int32_t workers_per_replica; /* TP */
  int32_t pp_stages;           /* PP */
  int32_t policy;              /* TW_POLICY_* */
  int32_t pred_id;             /* descriptor index in the pset */
  int32_t workload_id;         /* index into the workload CSR */
  int64_t epoch_ns;            /* simulate(epoch_ns=...) (oracle.py:53) */
  int64_t tk_cooldown_ns;      /* Timekeeper cooldown J for the actor grid */
  uint32_t flags;              /* TW_SIM_* */
  int32_t pad;
} tw_sim_cfg; /* 64 B */

/* status codes per config */
#define TW_SIM_OK 0
#define TW_SIM_STALLED_ACTIVE 1  /* oracle.py:184-188 */
#define TW_SIM_STALLED_KV 2      /* oracle.py:189-193 */
#define TW_SIM_PRED_ERROR 3      /* predictor raised; pred_code holds TW_PRED_* */
#define TW_SIM_CAPACITY 4        /* max_running exceeds the launch's slot capacity */
#define TW_SIM_BAD_CONFIG 5      /* EngineConfig validation failed (engine.py:109-120); the
                                    config never ran: final_now_ns = epoch, counters 0 */
#define TW_SIM_EVENT_OVERFLOW 6  /* flag bit (status |= 1<<8) when the dump was truncated */

typedef struct tw_sim_result {
  int64_t final_now_ns; /* virtual time when the loop drained (max FINISHED ts) */
  int64_t steps;        /* non-empty batches = predictions */
  int64_t events;       /* token events emitted */
  uint64_t digest;      /* order-sensitive digest of the event stream (tw_event_hash) */
  int64_t tk_seq;       /* Timekeeper CLOCK_UPDATE count (TW_SIM_TIMEKEEPER)            */
  int64_t tk_offset_ns; /* final Timekeeper offset                                       */
  int64_t tk_wall_ns;   /* final FakeClock wall. The three tk_* fields are the IDEALIZED */
                        /* protocol (workers between steps or parked count as exempt):   */
                        /* the minimum wall a live run needs; DESIGN.md §5 measures the  */
                        /* reference live stack against it                               */
  int32_t status;       /* TW_SIM_* (+ overflow bit) */
  int32_t pred_code;    /* TW_PRED_* when status == TW_SIM_PRED_ERROR */
} tw_sim_result;        /* 64 B */

/* event kinds (engine.py:57-60) and the dump record */
#define TW_EV_FIRST_TOKEN 0
#define TW_EV_OUTPUT_TOKEN 1
#define TW_EV_FINISHED 2
typedef struct tw_event {
  int64_t ts_ns;
  int32_t step;
  int32_t req_kind; /* (request index << 2) | kind */
} tw_event;         /* 16 B */

/* Workloads are CSR over requests already sorted stably by offset (oracle.py:60):
 * workload w owns requests [wl_off[w], wl_off[w+1]).
 * order: permutation of config ids (largest estimated cost first) that the
 * persistent CTAs pull from a device work counter; may be NULL (identity).
 * req_first_ns / req_finish_ns (optional): per (config, request) FIRST_TOKEN and
 * FINISHED timestamps at [req_base[c] + i]; unset entries are left untouched.
 * ev / ev_off (optional): audited configs get their full event stream in
 * ev[ev_off[c] .. ev_off[c+1]). slot_capacity: per-warp active-list capacity,
 * normally max(max_running) over the configs (configs above it finish with
 * TW_SIM_CAPACITY). Up to 4096 the slot state lives in shared memory (capacities
 * whose state does not fit 4 warps per CTA run fewer warps per CTA); above 4096 it
 * lives in scratch (one slice per resident warp). scratch: device memory of
 * scratch_bytes >= tw_sim_scratch_bytes(n_cfg, slot_capacity) (64 bytes up to 4096;
 * less than that above 4096 runs fewer resident warps, down to one slice); its first
 * 4 bytes are zeroed by the call (work counter).
 * Two variants of the same kernel, picked by n_cfg: up to 8 configs per SM (every
 * config resident on its own warp: latency-bound), each CTA stages pset_bytes of the
 * blob in shared memory; above that (throughput-bound), or when the blob does not fit
 * in shared memory, the blob is read from global memory so that shared memory holds
 * only slot state and 4 CTAs of <= 128 registers fit per SM. Results are identical. */
int tw_sim_many(const void* pset, int64_t pset_bytes, const tw_sim_cfg* cfgs,
                int32_t n_cfg, const int32_t* order, const int64_t* wl_off,
                const int64_t* req_offset_ns, const int32_t* req_prompt,
                const int32_t* req_output, tw_sim_result* results,
                const int64_t* req_base, int64_t* req_first_ns, int64_t* req_finish_ns,
                const int64_t* ev_off, tw_event* ev, int32_t slot_capacity, void* scratch,
                int64_t scratch_bytes, void* stream);
/* scratch bytes tw_sim_many wants for these sizes (64 up to slot capacity 4096) */
int64_t tw_sim_scratch_bytes(int32_t n_cfg, int32_t slot_capacity);
/* Scratch bytes for the latency regime's busy-period segments (0: n_cfg is not in that
 * regime). With scratch_bytes >= this (total_requests = req_base[n_cfg]), req_base given,
 * no event dump and slot capacity <= 4096, tw_sim_many splits each config's arrivals at
 * likely regeneration points (an arrival that finds the engine empty restarts the
 * timeline, oracle.py:78-83), simulates the segments speculatively in parallel and joins
 * the valid pieces (serially re-running any piece whose boundary was not one), so one
 * config's serial chain no longer bounds the sweep. Records and stamps are identical to
 * the serial loop's, except that when a config stops early (stall or prediction error)
 * stamps a speculative segment wrote past the stop are reset to -1. */
int64_t tw_sim_seg_scratch_bytes(int32_t n_cfg, int64_t total_requests);
/* Opt-in statistics of the segmented path for the next tw_sim_many calls on this thread
 * (device pointer, 8 int32 per config; NULL disables): {segments, pieces joined from a
 * segment's run, pieces re-run serially by the join pass, Timekeeper carry-overs refused,
 * segments out of log / overrun room, stops that were not regeneration points of the next
 * run, 0, 0}. */
int tw_sim_set_seg_stats(int32_t* per_config_8xi32);

/* Launch geometry the library picked for the last tw_sim_many on this thread
 * (for the bench's roofline bookkeeping). */
int tw_sim_last_launch(int32_t* grid, int32_t* block, int32_t* smem_bytes,
                       int32_t* slot_capacity);
/* Which event loop the last tw_sim_many on this thread ran: 0 latency variant (one warp
 * per config), 1 throughput variant, 2 busy-period segments (plan, segments, Timekeeper
 * replays, join; the geometry above is the segments kernel's), 3 slot state in scratch. */
int tw_sim_last_path(void);

/* Opt-in instrumentation for the next tw_sim_many calls on this thread: when set
 * (device pointer, 16 int64 per config; NULL disables), each config records
 * {SM cycles, normal steps, macro runs, steps covered by runs, Timekeeper cycles,
 * run-event cycles, Timekeeper broadcasts, arrival cycles, plan cycles, admission
 * cycles, predict cycles, apply cycles, 0, 0, 0, 0}. */
int tw_sim_set_profile(int64_t* per_config_16xi64);
/* Debug mode for the next tw_sim_many calls on this thread: when set (device pointer,
 * 8 int32 per config; NULL disables), the event loop runs its invariant-checking build
 * (sim_check.cu) and records per config {iterations checked, virtual time went back,
 * slot overran its prompt/output, incremental KV-block counter != recomputation
 * (engine.py:359-369), Timekeeper offset/seq/wall went back, V != wall + offset or V
 * short of the step end, last broadcast after the wall, event count != sum(max(output,
 * 1) + 1)}: all but the first must stay 0. Results are identical to the normal build. */
int tw_sim_set_checks(int32_t* per_config_8xi32);

/* ---- per-config latency metrics: metrics.py:62-253 ------ */
/* RunReport.summary() of an oracle-mode run (runner.py:339-365), reduced on device
 * from the per-request stamps tw_sim_many wrote: TTFT = first - epoch - offset,
 * e2e = finish - epoch - offset, TPOT = (finish - first) / (output - 1) for outputs
 * > 1 (metrics.py:49-62); nearest-rank p50/p90/p99 with rank = ceil(p/100.0 * n)
 * (metrics.py:65-71) and mean = Python sum()/len, i.e. Neumaier-compensated
 * summation in request order (CPython >= 3.12 sum of floats) then one division. */
#define TW_METRICS_OK 0
#define TW_METRICS_INCOMPLETE 1  /* some request has no FINISHED stamp (IncompleteLog) */
#define TW_METRICS_SIM_FAILED 2  /* the config's tw_sim_result status is not OK      */
#define TW_METRICS_TOO_LARGE 3   /* more requests than max_requests                   */

typedef struct tw_latency_stats {
  double p50, p90, p99, mean;
  int64_t count; /* 0: no values (the summary omits the entry) */
} tw_latency_stats; /* 40 B */

typedef struct tw_run_metrics {
  int64_t num_requests;
  int64_t output_tokens;
  int64_t virtual_elapsed_ns; /* max FINISHED - epoch (metrics.py:245) */
  double tokens_per_virtual_s;
  tw_latency_stats ttft, e2e, tpot;
  int32_t status; /* TW_METRICS_* */
  int32_t n_missing;
} tw_run_metrics; /* 160 B */

/* One CTA per config. Requests of config c are workload cfgs[c].workload_id's
 * (CSR as in tw_sim_many) with stamps at req_base[c] + i (-1 = never stamped).
 * sim (optional): tw_sim_many's records; a non-OK status gives TW_METRICS_SIM_FAILED.
 * sum_order (optional, per workload request, CSR like the workload): the position
 * of each request in the caller's arrival list, which sets the order of the
 * compensated TPOT sum; NULL = the engine's (stable-sorted) order, which is the
 * caller's order for sorted arrival lists such as generate_arrivals produces.
 * max_requests: an upper bound on any workload's size. Up to ~28,000 requests the
 * per-request keys (8 B each) live in shared memory; above that they live in the
 * caller's global scratch (less than tw_metrics_scratch_bytes, down to one slice of
 * 8*max_requests bytes, runs fewer CTAs; none gives TW_ENOSMEM). With the full
 * tw_metrics_scratch_bytes the scratch also holds each config's TPOT values (8 B per
 * request) and a second kernel sums them one lane per config (CPython's compensated
 * sum, same order); with less, one thread of the config's CTA sums them. */
int tw_metrics_many(const tw_sim_cfg* cfgs, int32_t n_cfg, const int64_t* wl_off,
                    const int64_t* req_offset_ns, const int32_t* req_output,
                    const int64_t* req_base, const int64_t* req_first_ns,
                    const int64_t* req_finish_ns, const tw_sim_result* sim,
                    const int32_t* sum_order, int32_t max_requests, void* scratch,
                    int64_t scratch_bytes, tw_run_metrics* out, void* stream);
/* bytes of global scratch tw_metrics_many wants for these sizes (the TPOT rows, plus the
 * keys above ~28,000 requests) */
int64_t tw_metrics_scratch_bytes(int32_t n_cfg, int32_t max_requests);

/* ---- native BarrierCore for the live Timekeeper --------- */
/* Host C++ (no GPU): the reference's single-threaded protocol state machine
 * (timekeeper.py:68-398) behind an opaque handle. Replaces `BarrierCore(...)` in
 * TimekeeperServer (timekeeper.py:435-440) through the Python shim
 * NativeBarrierCore (paper_2601_00397_b200/barrier_core.py). Clients are
 * registration indices (ids "actor<n>"/"observer<n>" in registration order); group
 * ids are caller-assigned small integers. Not thread-safe: one state thread owns a
 * core, as in the reference. */
typedef struct tw_core tw_core;

#define TW_MSG_REGISTER 0 /* wire.MessageType */
#define TW_MSG_SEAL 1
#define TW_MSG_JUMP_REQUEST 2
#define TW_MSG_COLLECTIVE_ENTER 3
#define TW_MSG_DEREGISTER 4
#define TW_MSG_OTHER 5 /* any type clients may not send -> TW_EINVAL (MalformedBody) */
#define TW_ROLE_ACTOR 0
#define TW_ROLE_OBSERVER 1

typedef struct tw_core_msg {
  int32_t type;   /* TW_MSG_* */
  int32_t client; /* registration index; -1 = absent or never issued */
  int32_t role;   /* REGISTER: TW_ROLE_*, -1 = unknown role (MalformedBody) */
  int32_t group;  /* COLLECTIVE_ENTER: group handle, -1 = missing group_id */
  int64_t target; /* JUMP_REQUEST target ns (valid iff has_target) */
  int64_t expected;
  int32_t has_target, has_expected;
} tw_core_msg; /* 40 B */

typedef struct tw_core_ack {
  int32_t error;      /* TW_ACK_* (0 = no error) */
  int32_t client;     /* REGISTER: the new client's index; else the request's */
  int32_t group;      /* COLLECTIVE_ENTER: the request's group */
  int32_t resolve;    /* 1: deliver the ack, then call tw_core_try_resolve */
  int64_t offset_ns;  /* REGISTER_ACK offset */
  int64_t seq;        /* REGISTER_ACK seq */
  int64_t generation; /* COLLECTIVE_ENTER generation (ExpectedMismatch: the open size) */
} tw_core_ack;        /* 40 B */

#define TW_REC_REGISTER 0 /* structured log records (timekeeper.py log_record) */
#define TW_REC_SEAL 1
#define TW_REC_REQUEST 2
#define TW_REC_COLLECTIVE_ENTER 3
#define TW_REC_COLLECTIVE_RELEASE 4
#define TW_REC_DEREGISTER 5
#define TW_REC_RESOLVE 6
#define TW_REC_BROADCAST 7

typedef struct tw_core_record {
  int32_t kind; /* TW_REC_* */
  int32_t client, role, group;
  int64_t wall_ns, offset_ns, seq, target_ns, expected, generation, t_min_ns;
  int32_t num_actors, eligible, broadcast, suppressed;
  int32_t n_items, pad;
  const int32_t* items;        /* release: members; resolve: pending clients (id order) */
  const int64_t* item_targets; /* resolve: their targets */
} tw_core_record;

#define TW_EMIT_CLOCK_UPDATE 0
#define TW_EMIT_COLLECTIVE_RELEASE 1
typedef struct tw_core_emit {
  int32_t kind, group;
  int64_t offset_ns, seq, generation;
} tw_core_emit;

typedef struct tw_core_state_t {
  int64_t offset_ns, seq, last_broadcast_wall_ns, barrier_open_since_ns;
  int32_t sealed, has_last_broadcast, has_barrier_open, n_clients;
  int32_t n_groups, eligible, n_pending, n_active_actors;
} tw_core_state_t;

typedef int64_t (*tw_core_clock_fn)(void* user);             /* wall ns */
typedef void (*tw_core_sleep_fn)(void* user, double seconds); /* sleep(wait_ns / 1e9) */
typedef void (*tw_core_emit_fn)(void* user, const tw_core_emit* ev);
typedef void (*tw_core_log_fn)(void* user, const tw_core_record* rec);

/* emit / log_record may be NULL; clock / sleep may be NULL for the host realtime clock
 * (CLOCK_REALTIME ns, the reference's wall_now) and nanosleep. Returns TW_EINVAL for a
 * negative cooldown. */
int tw_core_new(int64_t cooldown_ns, int32_t suppress_broadcasts, tw_core_clock_fn clock,
                tw_core_sleep_fn sleep, tw_core_emit_fn emit, tw_core_log_fn log_record,
                void* user, tw_core** out);
int tw_core_free(tw_core* core);
/* One inbound message: validates and mutates state, fills the ack (protocol errors
 * are ack.error, not call failures); TW_EINVAL = MalformedBody. */
int tw_core_handle(tw_core* core, const tw_core_msg* msg, tw_core_ack* ack);
int tw_core_try_resolve(tw_core* core);
/* From inside a clock / sleep / emit / log callback: the callback failed. The core
 * unwinds as soon as the callback returns and the call in progress returns TW_ECALLBACK,
 * keeping the state changed so far (as the reference core does when a callback raises). */
int tw_core_abort(tw_core* core);
/* BarrierCore.suppress_broadcasts is a plain attribute the reference re-reads on every
 * resolve (timekeeper.py:351-363): this updates it on a live core. */
int tw_core_set_suppress(tw_core* core, int32_t suppress_broadcasts);
int tw_core_state(const tw_core* core, tw_core_state_t* st);
/* flags: 1 active, 2 exempt, 4 has a pending target (pending_target) */
int tw_core_client(const tw_core* core, int32_t idx, int32_t* role, int32_t* flags,
                   int64_t* pending_target);
/* flags: 1 exists, 2 expected set, 4 open; members sorted by client id (<= cap). */
int tw_core_group(const tw_core* core, int32_t group, int64_t* generation, int64_t* expected,
                  int64_t* open_since_ns, int32_t* flags, int32_t* members, int32_t cap,
                  int32_t* n_members);

/* ---- bulk Poisson workload generation ------------------- */
/* generate_arrivals for source "poisson" (workload.py:118-144), one thread per
 * workload, bit-exact with numpy's Generator (PCG64, ziggurat exponential, Lemire
 * bounded integers). The host seeds each workload: state/inc are
 * np.random.default_rng(seed).bit_generator.state (128-bit values split hi/lo). */
#define TW_TOKENS_FIXED 0   /* TokenDist kind "fixed": value a, no draw */
#define TW_TOKENS_UNIFORM 1 /* TokenDist kind "uniform": integers(a, b + 1) */

typedef struct tw_wl_spec {
  uint64_t state_hi, state_lo, inc_hi, inc_lo; /* PCG64 state after seeding */
  double scale;                                /* 1.0 / qps (exponential scale) */
  int32_t prompt_kind, prompt_a, prompt_b;
  int32_t output_kind, output_a, output_b;
  int32_t has_uint32;  /* PCG64 32-bit buffer (0 after seeding) */
  uint32_t uinteger;
} tw_wl_spec;          /* 72 B */

/* Workload w fills requests [wl_off[w], wl_off[w+1]) of offset_ns (cumulative
 * int(round(gap_s * 1e9))), prompt, output. status[w] = 0, or 1 + the index of the
 * first request with a non-positive token count (WorkloadError, workload.py:137-140). */
int tw_generate_poisson(const tw_wl_spec* specs, int32_t n_wl, const int64_t* wl_off,
                        int64_t* offset_ns, int32_t* prompt, int32_t* output, int32_t* status,
                        void* stream);

/* ---- misc ------------------------------------------------------------------ */
int tw_abi_version(void);
const char* tw_last_error(void);
/* Number of kernel launches this thread has issued through the library. */
int64_t tw_launch_count(void);

#ifdef __cplusplus
}
#endif

/* ---- the event digest, shared by the CUDA path and the oracle ------------- */
/* digest = sum over events k (0-based, emission order) of tw_event_hash(k, ...)
 * mod 2^64, with tw_event_hash = M(req, kind) * L(k, ts, step):
 *   M = tw_mix64(req*C1 + kind*C2 + C3) | 1   (odd: a pseudo-random multiplier per
 *       request and event kind; req = index in the stable-sorted arrivals)
 *   L = k*A + ts*B + step*G + 1               (A, B, G odd)
 * Position-bound (k), and every field change of one event changes the digest
 * (M and the coefficients are odd, so M*coef*delta != 0 mod 2^64 for any
 * delta != 0 mod 2^64); reorderings cancel only with probability ~2^-60.
 * L is linear in (k, ts, step), so the OUTPUT_TOKEN events of a run of identical
 * decode steps sum in closed form per request (tw_event_run_sum). */
#define TW_DIGEST_VERSION 2
#define TW_DIG_A 0x9E3779B97F4A7C15ULL
#define TW_DIG_B 0xD6E8FEB86659FD93ULL
#define TW_DIG_G 0xFF51AFD7ED558CCDULL
#if defined(__CUDACC__)
#define TW_HD __host__ __device__ __forceinline__
#else
#define TW_HD static inline
#endif
TW_HD uint64_t tw_mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}
TW_HD uint64_t tw_event_mult(uint64_t req, uint64_t kind) {
  return tw_mix64(req * 0xC2B2AE3D27D4EB4FULL + kind * 0x165667B19E3779F9ULL + 0x27D4EB2F165667C5ULL) | 1ULL;
}
/* the step-uniform part of L: ts*B + step*G + 1 */
TW_HD uint64_t tw_event_u(int64_t ts, int64_t step) {
  return (uint64_t)ts * TW_DIG_B + (uint64_t)step * TW_DIG_G + 1ULL;
}
TW_HD uint64_t tw_event_hash(uint64_t k, uint64_t req, uint64_t kind, int64_t ts, int64_t step) {
  return tw_event_mult(req, kind) * (k * TW_DIG_A + tw_event_u(ts, step));
}
/* sum of L over the m events k = k0 + (j-1)*stride, ts = ts0 + j*d, step = step0 + j
 * (j = 1..m): one request's OUTPUT_TOKENs over m identical steps of duration d */
TW_HD uint64_t tw_event_run_sum(uint64_t m, uint64_t k0, uint64_t stride, int64_t ts0, int64_t d, int64_t step0) {
  const uint64_t t1 = (m & 1ULL) ? m * ((m + 1ULL) >> 1) : (m >> 1) * (m + 1ULL); /* sum j     */
  const uint64_t t0 = t1 - m;                                                      /* sum j - 1 */
  return m * (k0 * TW_DIG_A + tw_event_u(ts0, step0)) + TW_DIG_A * stride * t0 +
         ((uint64_t)d * TW_DIG_B + TW_DIG_G) * t1;
}

#endif /* TWB200_H */

/* layout checks (the Python mirrors in paper_2601_00397_b200/_lib.py assert the same) */
#ifdef __cplusplus
static_assert(sizeof(tw_pred_desc) == 64, "tw_pred_desc");
static_assert(sizeof(tw_tk_op) == 16, "tw_tk_op");
static_assert(sizeof(tw_tk_event) == 32, "tw_tk_event");
static_assert(sizeof(tw_tk_final) == 64, "tw_tk_final");
static_assert(sizeof(tw_sim_cfg) == 64, "tw_sim_cfg");
static_assert(sizeof(tw_sim_result) == 64, "tw_sim_result");
static_assert(sizeof(tw_event) == 16, "tw_event");
#else
_Static_assert(sizeof(tw_pred_desc) == 64, "tw_pred_desc");
_Static_assert(sizeof(tw_tk_op) == 16, "tw_tk_op");
_Static_assert(sizeof(tw_tk_event) == 32, "tw_tk_event");
_Static_assert(sizeof(tw_tk_final) == 64, "tw_tk_final");
_Static_assert(sizeof(tw_sim_cfg) == 64, "tw_sim_cfg");
_Static_assert(sizeof(tw_sim_result) == 64, "tw_sim_result");
_Static_assert(sizeof(tw_event) == 16, "tw_event");
#endif
