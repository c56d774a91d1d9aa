// hive_kernels.cuh — launcher interface between the host orchestration
// (hive_host.cu) and the sm_100a kernels (hive_kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include "hive_device.cuh"

namespace hive {

constexpr int BLOCK = 256;
constexpr int WARPS_PER_BLOCK = BLOCK / 32;
// Lanes per operation for each probe kernel: defaults
// chosen by ncu measurement; HIVE_G_FIND / HIVE_G_INSERT / HIVE_G_ERASE /
// HIVE_G_SLOW (1, 2, 4 or 8) override them for experiments.
constexpr int G_FIND = 4, G_INSERT = 4, G_ERASE = 2, G_SLOW = 2;
constexpr int MINB_FIND_DEFAULT = 6;           // 40 regs: 3.60 ms vs 3.79 (48 regs) vs 4.60 (32, spills)
constexpr int MINB_DEFAULT = 4;          // 4 blocks/SM => <= 64 registers (ncu: 74-80 regs left 36% warps active)
constexpr int PART_CHUNK = 8192;         // max elements per warp in the stable partition
constexpr int PART_UNROLL = 4;           // rows of 32 elements whose loads are in flight together
constexpr int MAX_PARTS = 64;
#ifndef HIVE_TWO_CHOICE_T
#define HIVE_TWO_CHOICE_T 0
#endif
// Thresholded two-choice placement in the insert fast path (reading A-21):
// below this many free slots in b1 the emptier of b1 / b2 is claimed; 0 =
// first-fit b1 then b2.  Build-time (-DHIVE_TWO_CHOICE_T=t, HIVE_NVCC_DEFINES).
constexpr uint32_t TWO_CHOICE_T = HIVE_TWO_CHOICE_T;
#ifndef HIVE_CLAIM_ROT
#define HIVE_CLAIM_ROT 0
#endif
// claim placement (hive_kernels.cu c_claim_rot; 0 measured fastest; 1 / 2 for
// experiments: -DHIVE_CLAIM_ROT=r through HIVE_NVCC_DEFINES)
constexpr uint32_t CLAIM_ROT_DEFAULT = HIVE_CLAIM_ROT;

#ifndef HIVE_VICTIM_LOOK
#define HIVE_VICTIM_LOOK 8
#endif
// Step 3 victim choice: 0 = rotating slot; v > 0 = the first of v candidate
// slots (v / G per lane) whose resident's other bucket is a split one.  8 from
// the A/B in profiles/r02b_victim_ab.txt (cfg2 Step 3 1.22 -> 0.88 ms, cfg3
// 3.58 -> 3.91 G ops/s); build-time -DHIVE_VICTIM_LOOK=v for experiments.
constexpr int VICTIM_LOOK = HIVE_VICTIM_LOOK;

// Modes of the stable partition (shard routing).  Mixed-batch classification
// and the election's hash partition have their own kernels (k_classify,
// k_elect_hist / k_elect_scatter); values 0 and 2 are retired.
enum PartMode { PART_ROUTE = 1, PART_ROUTE_KEYS = 3, PART_ROUTE_P2P = 4, PART_ROUTE_PAD = 5 };

// Peer-memory exchange: the owners' inbox / count /
// result buffers of up to MAX_PEERS shards, passed by value.  Every buffer is
// laid out by region: source (or owner) r's records sit at [r * region, ...).
constexpr int MAX_PEERS = 8;
struct PeerDest {
    uint64_t* kv[MAX_PEERS];                 // owner p's inbox records (value << 32 | key)
    uint8_t* ops[MAX_PEERS];                 // owner p's inbox opcodes (nullable)
    unsigned long long* cnt[MAX_PEERS];      // owner p's per-source record counts
    uint32_t* res32[MAX_PEERS];              // source p's result words (return path)
    uint8_t* res8[MAX_PEERS];                // source p's result bytes (return path)
    unsigned long long* sig[MAX_PEERS];      // peer p's signal words [2 phases][MAX_PEERS]
    uint64_t region;                         // records per region
    uint32_t rank;                           // this rank
};
// Signal words per rank: [phase * MAX_PEERS + source] = epoch, then one
// timeout marker.
constexpr int SIG_WORDS = 2 * MAX_PEERS + 1;

struct Grids {                           // persistent grid sizes (blocks)
    int find, insert_fast, insert_slow, erase, dedup, stream, gather;
    int g_find, g_insert, g_slow, g_erase;   // lanes per operation
    int minb;                                // min resident blocks/SM for the mutating kernels
    int minb_find;                           // ... and for k_find
    int minb_slow;                           // ... and for k_insert_slow (HIVE_MINB_SLOW)
};

// Occupancy-derived persistent grid sizes for this device.
Grids query_grids(int num_sms);

// Fill the CRC-32 / CRC-64 constant tables (HASH_CRC) on the current device.
cudaError_t init_hash_tables();

// Calibration gather: random 256 B block reads at k_find's
// access pattern; out[i] = xor of block (fmix32(keys[i]) * n_blocks) >> 32.
cudaError_t launch_gather(const Grids& gr, cudaStream_t s, const uint32_t* keys, uint64_t n,
                          const uint64_t* blocks, uint64_t n_blocks, uint32_t* out, uint32_t mode);

// fix (nullable): the previous phase's duplicate fix-up, run first (mixed batches)
cudaError_t launch_find(const Grids& gr, cudaStream_t s, const uint32_t* keys, const uint32_t* idx,
                        uint64_t n, const uint64_t* n_dev, TableView tv, StashView sv,
                        uint32_t* vals_out, uint8_t* found, const DupFix* fix = nullptr);

// idx2 / n_dev2 / dd2 (nullable): a second op list elected in the same launch
// into its own scratch set (a mixed batch's ERASE list beside its INSERT list).
cudaError_t launch_dedup_elect(int grid, cudaStream_t s, const uint32_t* keys, const uint32_t* idx,
                               uint64_t n, const uint64_t* n_dev, DedupView dd, Ctrl* ctrl,
                               const uint32_t* idx2 = nullptr, const uint64_t* n_dev2 = nullptr,
                               const DedupView* dd2 = nullptr);

cudaError_t launch_insert_fast(const Grids& gr, cudaStream_t s, const uint32_t* keys, const uint32_t* vals,
                               const uint64_t* kvs, const uint32_t* idx, uint64_t n,
                               const uint64_t* n_dev, TableView tv, StashView sv, DedupView dd,
                               uint8_t* status, uint32_t* vals_zero, uint32_t* leftover,
                               uint32_t op_base = 0, bool prof = false);

cudaError_t launch_insert_slow(const Grids& gr, cudaStream_t s, const uint32_t* keys, const uint32_t* vals,
                               const uint64_t* kvs, const uint32_t* leftover, TableView tv,
                               StashView sv, uint32_t max_evictions, uint8_t* status, bool prof = false);

cudaError_t launch_erase(const Grids& gr, cudaStream_t s, const uint32_t* keys, const uint32_t* idx,
                         uint64_t n, const uint64_t* n_dev, TableView tv, StashView sv,
                         DedupView dd, uint8_t* erased, uint32_t* vals_zero, const DupFix* fix = nullptr);

// NEXT-4 monolithic concurrent mixed kernel (one cooperative launch).
// tab: the per-batch group table (tab_mask + 1 words, a power of two >= 2n);
// flag uint8[n], owner_of / leftover uint32[n]; ctrl n_left and slow_next
// must be zero.  mono_grid: the co-resident grid for this device.
int mono_grid(int num_sms);
cudaError_t launch_mixed_mono(int grid, cudaStream_t s, const uint8_t* ops, const uint32_t* keys,
                              const uint32_t* vals, uint64_t n, TableView tv, StashView sv, uint64_t* tab,
                              uint64_t tab_mask, uint8_t* flag, uint32_t* owner_of, uint32_t* leftover,
                              uint32_t max_evictions, uint8_t* result, uint32_t* vals_out);
cudaError_t launch_count_ops(cudaStream_t s, const uint8_t* ops, uint64_t n, uint8_t code,
                             unsigned long long* out);

cudaError_t launch_dup_copy(int grid, cudaStream_t s, const uint32_t* idx, uint64_t n,
                            const uint64_t* n_dev, DedupView dd, uint8_t* out);
// PHASED classification in one pass: counts[c] (zeroed here) = ops of class c
// (0 find, 1 insert, 2 erase), their indices in out_idx[c * stride ...] in
// tile reservation order (not op order); other opcodes: result / value 0.
cudaError_t launch_classify(cudaStream_t s, const uint8_t* ops, uint64_t n, const uint64_t* n_dev,
                            uint64_t* counts, uint32_t* out_idx, uint64_t stride, uint8_t* result_zero,
                            uint32_t* vals_zero, int num_sms, bool counts_zeroed = false);
// hive_mixed's per-batch reset in one launch: ctrl->cls_n, (zero_left) the
// Step-3 cursors, flag[0, fbytes) = 0, dd[0, dwords) = ~0 (either nullable).
cudaError_t launch_batch_prep(cudaStream_t s, Ctrl* ctrl, bool zero_left, uint8_t* flag, uint64_t fbytes,
                              uint64_t* dd, uint64_t dwords, int num_sms);

cudaError_t launch_split(cudaStream_t s, TableView tv, uint32_t n_pairs, Ctrl* ctrl);
cudaError_t launch_merge(cudaStream_t s, TableView tv, uint32_t n_pairs, unsigned long long* abort_at,
                         const unsigned long long* prev_abort, uint64_t prev_pairs);
constexpr int MAX_SEGMENTS = 64;        // linear-hashing rounds crossed by one resize phase

cudaError_t launch_stash_reset(cudaStream_t s, StashView sv);
// a[0, na) and b[0, nb) (64-bit words) set to EMPTY in one launch.
cudaError_t launch_fill2(cudaStream_t s, uint64_t* a, uint64_t na, uint64_t* b, uint64_t nb, int num_sms);

// hive_load_image: spill words of the loaded buckets, stash ring + index + spill bits.
cudaError_t launch_image(cudaStream_t s, TableView tv, uint64_t n_buckets, StashView sv, const uint64_t* stash,
                         uint64_t n_stash);
cudaError_t launch_dump(int grid, cudaStream_t s, TableView tv, uint64_t n_buckets, StashView sv,
                        uint32_t* keys, uint32_t* vals, uint64_t cap);
cudaError_t launch_count_b1(int grid, cudaStream_t s, TableView tv, uint64_t n_buckets, Ctrl* ctrl);

// Stable partition: count -> scan -> scatter.  cnt must hold n_parts * n_warps
// words, part_info 2 * MAX_PARTS words (totals, bases).
uint64_t part_warps(uint64_t n);
// NEXT-1: stable route of this rank's batch straight into the owners' inboxes
// (remote stores over NVLink), then each owner's per-source count.
cudaError_t launch_route_p2p(cudaStream_t s, uint32_t n_shards, uint32_t seed, const uint32_t* keys,
                             const uint32_t* vals, const uint8_t* ops, uint64_t n, uint64_t* cnt,
                             uint64_t* part_info, uint32_t* pos, const PeerDest& pd,
                             unsigned long long* xfail = nullptr);
// Owner, device-count form of the result return (after launch_owner_compact
// over the inbox with cap = region): result j -> source back[j] / region.
cudaError_t launch_return_p2p_back(cudaStream_t s, uint64_t n_upper, const uint64_t* n_dev, uint64_t region,
                                   const uint32_t* back, const uint32_t* res32, const uint8_t* res8,
                                   const PeerDest& pd);
// Owner: gather the per-source inbox regions into contiguous key / value / op arrays.
cudaError_t launch_inbox_compact(cudaStream_t s, uint32_t n_src, uint64_t region, const uint64_t* inbox_kv,
                                 const uint8_t* inbox_ops, const uint64_t* cnt, uint64_t n_total,
                                 uint32_t* keys, uint32_t* vals, uint8_t* ops);
// Owner: write each record's results into its source's result region (remote stores).
cudaError_t launch_return_p2p(cudaStream_t s, uint32_t n_src, const uint64_t* cnt, uint64_t n_total,
                              const uint32_t* res32, const uint8_t* res8, const PeerDest& pd);

// Device-side phase barrier of the peer exchange: every rank stores `epoch`
// into each peer's signal word (release, system scope) after its stores; a
// rank waits (acquire spin, bounded by timeout_ns) until all n sources have.
cudaError_t launch_p2p_signal(cudaStream_t s, uint32_t n, uint32_t phase, uint64_t epoch, const PeerDest& pd);
cudaError_t launch_p2p_wait(cudaStream_t s, uint32_t n, uint32_t phase, uint64_t epoch,
                            unsigned long long* sig_own, uint64_t timeout_ns);

cudaError_t launch_partition(cudaStream_t s, int mode, uint32_t n_parts, uint32_t seed,
                             const uint32_t* keys, const uint32_t* vals, const uint8_t* ops,
                             uint64_t n, uint64_t* cnt, uint64_t* part_info, uint64_t* send_kv,
                             uint8_t* send_ops, uint32_t* pos, const uint32_t* idx = nullptr,
                             const uint64_t* n_dev = nullptr);
cudaError_t launch_elect_partition(cudaStream_t s, const uint32_t* keys, const uint32_t* idx, uint64_t n,
                                   const uint64_t* n_dev, uint32_t n_parts, unsigned long long* gcount,
                                   unsigned long long* cursor, uint64_t* part_info, uint64_t* recs,
                                   int num_sms, const uint32_t* vals = nullptr, uint32_t* rvals = nullptr,
                                   uint8_t* status = nullptr, uint32_t* vals_zero = nullptr);
// Fused INSERT phase with owner election (one cooperative launch): ops
// hash-partitioned into FUSED_PARTS parts (records + values from
// launch_elect_partition with rvals); part q is elected into table (q & 1)
// while part q-1 runs the insert fast path, then Steps 3-4 and the duplicate
// fix-up.  tab0 / tab1: tab_mask + 1 words each, pre-set to the byte patterns
// 0x04 / 0x00 (stale epochs).  ctrl n_left / slow_next must be zero.
constexpr uint32_t FUSED_PARTS = 64;
constexpr uint64_t FUSED_MIN_OPS = 1ull << 21;   // smaller phases: one L2-resident election table
int fused_grid(int num_sms);
cudaError_t launch_insert_fused(int grid, cudaStream_t s, const uint64_t* recs, const uint32_t* rvals,
                                const uint64_t* part_info, uint64_t* tab0, uint64_t* tab1, uint64_t tab_mask,
                                DedupView dd, TableView tv, StashView sv, uint8_t* status, uint32_t* vals_zero,
                                uint32_t* leftover, uint32_t max_evictions, const uint32_t* keys,
                                const uint32_t* vals);
// clear_next (nullable, clear_words even): a sub-table the launch sets to
// EMPTY in its tail (the next part's, so its clear overlaps this election).
cudaError_t launch_dedup_elect_part(int grid, cudaStream_t s, const uint64_t* recs, const uint64_t* part_info,
                                    uint32_t part, DedupView dd, Ctrl* ctrl, uint64_t* clear_next = nullptr,
                                    uint64_t clear_words = 0);

// ---- sharded table over NCCL (include/hive.h "Sharded tables") ------
// Stable route into a padded send buffer of G regions of `cap` records
// (region p = ops owned by shard p, in op order); ops past `cap` of their
// region are not sent (pos = NO_POS, ctrl->xfail counts them).  cnt_send[p] =
// records placed in region p.
constexpr uint32_t NO_POS = 0xFFFFFFFFu;
cudaError_t launch_route_pad(cudaStream_t s, uint32_t n_shards, uint32_t seed, const uint32_t* keys,
                             const uint32_t* vals, const uint8_t* ops, uint64_t n, uint64_t cap, uint64_t* cnt,
                             uint64_t* part_info, uint64_t* send_kv, uint8_t* send_ops, uint32_t* pos,
                             uint64_t* cnt_send, Ctrl* ctrl, const uint32_t* idx = nullptr,
                             const uint64_t* n_dev = nullptr);
// Source-side owner election of a sharded call: groups (key, opcode) --
// opc == nullptr: every op has opcode kind_op -- elect the highest op index,
// flag grouped ops, owner_of for grouped ops, and list = the ops to route
// (*n_list of them).  tab: mask + 1 words (power of two >= 2n).
cudaError_t launch_src_elect(cudaStream_t s, const uint8_t* opc, uint8_t kind_op, const uint32_t* keys, uint64_t n,
                             uint64_t* tab, uint64_t mask, uint8_t* flag, uint32_t* owner_of, uint32_t* list,
                             unsigned long long* n_list, Ctrl* ctrl);
// After the exchange: grouped non-owners copy their owner's results.
cudaError_t launch_src_copy(cudaStream_t s, uint64_t n, const uint8_t* flag, const uint32_t* owner_of, uint8_t* out8,
                            uint32_t* out32);
// Owner: the records of the G received regions (cnt_recv[r] valid in region
// r), in source-rank order, as contiguous keys / values / opcodes; back[j] =
// the padded position record j came from; *n_dev = the total.
// self_kv (nullable): region `self` is read from this buffer (the local send
// buffer: the rank's own records skip the exchange), self_ops likewise.
cudaError_t launch_owner_compact(cudaStream_t s, uint32_t n_src, uint64_t cap, const uint64_t* recv_kv,
                                 const uint8_t* recv_ops, const uint64_t* cnt_recv, uint32_t* keys, uint32_t* vals,
                                 uint8_t* ops, uint32_t* back, uint64_t* n_dev, uint32_t self = 0,
                                 const uint64_t* self_kv = nullptr, const uint8_t* self_ops = nullptr);
// Owner: results of the compacted batch back into the padded layout
// (ret8[back[j]] = r8[j], ret32 likewise; either pair may be null).
cudaError_t launch_owner_return(cudaStream_t s, uint64_t n_upper, const uint64_t* n_dev, const uint32_t* back,
                                const uint8_t* r8, const uint32_t* r32, uint8_t* ret8, uint32_t* ret32);
// Source: out8[i] = in8[pos[i]] (pos == NO_POS: out8 = miss8, out32 = 0; a
// non-zero *poison marks every op HIVE_RESULT_PEER_LOST).
constexpr uint8_t HIVE_RESULT_PEER_LOST = 6;
cudaError_t launch_unroute_pad(cudaStream_t s, const uint32_t* pos, uint64_t n, const uint8_t* in8, uint8_t* out8,
                               const uint32_t* in32, uint32_t* out32, uint8_t miss8,
                               const unsigned long long* poison = nullptr, const uint32_t* idx = nullptr,
                               const uint64_t* n_dev = nullptr);

cudaError_t launch_unroute(cudaStream_t s, const uint32_t* pos, uint64_t n, const uint8_t* in8,
                           uint8_t* out8, const uint32_t* in32, uint32_t* out32);
cudaError_t launch_unpack(cudaStream_t s, const uint64_t* kv, uint64_t n, uint32_t* keys,
                          uint32_t* vals);

// Hash study: out[i] = fn(keys[i]) (fn 0 BitHash1, 1 BitHash2, 2 CRC-32,
// 3 CRC-64 low word) and/or set bit (h mod m) of the `bins` bitmap.
cudaError_t launch_hash(cudaStream_t s, uint32_t fn, const uint32_t* keys, uint64_t n, uint32_t* out,
                        uint32_t* bins, uint64_t m);
cudaError_t launch_popc(cudaStream_t s, const uint32_t* bins, uint64_t words, unsigned long long* total);

}  // namespace hive
