/*
 * hive_oracle.cpp — TEST INFRASTRUCTURE ONLY (see hive_oracle.h).
 *
 * A sequential Hive hash table written step by step from the paper
 * (reference/PAPER.md, arXiv 2510.15095).  Nothing here is blocked, fused or
 * parallel: each op runs the paper's algorithm literally on one core, with
 * the 32 "lanes" of a warp evaluated one after another.  Readings of silent or
 * garbled passages (A-n) are listed in DESIGN.md "Readings of the paper".
 *
 * Parity status of each part is stated in DESIGN.md "Oracle pins"; the only
 * "parity unpinned" items are the unobservable ones (slot placement, stash
 * membership, eviction counts), which are checked by invariants instead.
 */
#include "hive_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace {

/* ---- §III-A packed KV word, PAPER:177-188 -------------------------------- */
/* pair = (value << 32) | key  (widened to 64 bits first, A-5)     */
uint64_t Pack(uint32_t key, uint32_t value) {
    return ((uint64_t)value << 32) | (uint64_t)key;
}
/* key = pair & 0xFFFFFFFFu */
uint32_t UnpackKey(uint64_t pair) { return (uint32_t)(pair & 0xFFFFFFFFull); }
/* value = pair >> 32 */
uint32_t UnpackValue(uint64_t pair) { return (uint32_t)(pair >> 32); }
/* EMPTY is undefined in the paper; reading A-9: all ones, so key
 * 0xFFFFFFFF is reserved. */
const uint64_t EMPTY = ~0ull;
const uint32_t INVALID_KEY = 0xFFFFFFFFu;
const int S = 32;                       /* slots per bucket */
const uint32_t FULL_MASK = 0xFFFFFFFFu; /* Alg. 2 line 2: all 32 slots valid */

/* ---- §III-C Listing 1, PAPER:229-249 (reading A-1: the truncated
 * "return key" returns the full 32-bit mix; reduction is done by addr()). -- */
uint32_t BitHash1(uint32_t key) {
    key = ~key + (key << 15);
    key ^= (key >> 12);
    key += (key << 2);
    key ^= (key >> 4);
    key *= 2057u;
    key ^= (key >> 16);
    return key;
}
uint32_t BitHash2(uint32_t key) {
    key = (key + 0x7ed55d16u) + (key << 12);
    key = (key ^ 0xc761c23cu) ^ (key >> 19);
    key = (key + 0x165667b1u) + (key << 5);
    key = (key + 0xd3a2646cu) ^ (key << 9);
    key = (key + 0xfd7046c5u) + (key << 3);
    key = (key ^ 0xb55a4f09u) ^ (key >> 16);
    return key;
}

/* ---- §III-C / §V-B lookup-based hashes (reading A-26):
 * CRC-32/IEEE and CRC-64/XZ over the 4 little-endian key bytes, written
 * here as the bit-serial definition of a reflected CRC (shift register, one
 * polynomial reduction per input bit) rather than the byte-wise table the
 * paper puts in constant memory -- same function, independent arithmetic. -- */
uint32_t Crc32Bytes(const uint8_t* p, uint64_t n) {
    uint32_t c = 0xFFFFFFFFu;                         /* init all ones */
    for (uint64_t i = 0; i < n; ++i) {
        c ^= p[i];
        for (int bit = 0; bit < 8; ++bit)
            c = (c & 1u) ? (c >> 1) ^ 0xEDB88320u : (c >> 1);   /* reflected 0x04C11DB7 */
    }
    return ~c;                                        /* xorout all ones */
}
uint64_t Crc64Bytes(const uint8_t* p, uint64_t n) {
    uint64_t c = ~0ull;
    for (uint64_t i = 0; i < n; ++i) {
        c ^= p[i];
        for (int bit = 0; bit < 8; ++bit)
            c = (c & 1ull) ? (c >> 1) ^ 0xC96C5795D7870F42ull : (c >> 1);   /* reflected ECMA-182 */
    }
    return ~c;
}
uint32_t Crc32Key(uint32_t key) {
    uint8_t b[4] = {(uint8_t)key, (uint8_t)(key >> 8), (uint8_t)(key >> 16), (uint8_t)(key >> 24)};
    return Crc32Bytes(b, 4);
}
uint32_t Crc64Key(uint32_t key) {   /* low 32 bits of CRC-64 (reading A-26) */
    uint8_t b[4] = {(uint8_t)key, (uint8_t)(key >> 8), (uint8_t)(key >> 16), (uint8_t)(key >> 24)};
    return (uint32_t)Crc64Bytes(b, 4);
}
/* The table's hash pair: 0 = (BitHash1, BitHash2) (the paper's default,
 * §V-B), 1 = (CRC-32, CRC-64) (the lookup-based pair of Fig. 8). */
uint32_t HashPair(uint32_t kind, int which, uint32_t key) {
    if (kind == 1) return which == 1 ? Crc32Key(key) : Crc64Key(key);
    return which == 1 ? BitHash1(key) : BitHash2(key);
}

/* ---- §IV-C addressing: index_mask = 2^m - 1, split pointer;
 * the address rule under a split pointer is Litwin's (reading A-2). -------- */
uint32_t Addr(uint32_t h, uint32_t index_mask, uint32_t split) {
    uint32_t b = h & index_mask;
    if (b < split) b = h & ((index_mask << 1) | 1u);
    return b;
}

/* ---- lane primitives of §III-E/F and §IV-C ---- */
uint32_t Ballot(const bool pred[S]) {
    uint32_t m = 0;
    for (int lane = 0; lane < S; ++lane)
        if (pred[lane]) m |= (1u << lane);
    return m;
}
/* FirstSet: index of the least significant set bit, -1 if none (Alg. 1). */
int FirstSet(uint32_t mask) {
    for (int lane = 0; lane < S; ++lane)
        if (mask & (1u << lane)) return lane;
    return -1;
}
/* my_rank = __popc(mask & ((1u << lane) - 1)) */
uint32_t PrefixRank(uint32_t mask, uint32_t lane) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < lane; ++i)
        if (mask & (1u << i)) ++r;
    return r;
}
/* select_nth_one(mask, r): position of the (r+1)-th set bit (PAPER:542,
 * SPEC:241-249); -1 if fewer than r+1 bits are set. */
int SelectNthOne(uint32_t mask, uint32_t r) {
    uint32_t seen = 0;
    for (int i = 0; i < S; ++i) {
        if (mask & (1u << i)) {
            if (seen == r) return i;
            ++seen;
        }
    }
    return -1;
}
int Popc(uint32_t mask) {
    int c = 0;
    for (int i = 0; i < S; ++i)
        if (mask & (1u << i)) ++c;
    return c;
}

/* MurmurHash3 fmix32: the shard mixer of SURVEY §8(e) (independent of
 * BitHash1/2 so each shard still uses all of its buckets). */
uint32_t Fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

enum class Outcome { Replaced, New, Failed };

struct Table {
    /* configuration (§8(b)) */
    uint64_t max_buckets;
    float lf_grow, lf_shrink;
    uint32_t max_evictions;     /* PAPER:212 (value: reading A-8) */
    uint32_t resize_k;          /* K of PAPER:481 (value: reading A-8) */
    float stash_fraction;       /* PAPER:443 (value: reading A-8) */
    uint64_t n_b_min;

    /* §III-B structure */
    uint32_t m = 0;             /* index_mask = 2^m - 1 */
    uint32_t split = 0;         /* split pointer */
    std::vector<uint64_t> buckets;   /* n_b * 32 packed words */
    std::vector<uint32_t> freeMask;  /* bit i = 1 -> slot i free */

    /* Overflow stash: ring with head/tail; read side
     * indexed by key (reading A-10). */
    std::vector<uint64_t> ring;
    uint64_t head = 0, tail = 0, stash_cap = 0;
    std::unordered_map<uint32_t, uint64_t> stash_index;  /* key -> ring pos */
    std::vector<uint64_t> pending;   /* stash-full entries ("pending") */

    uint64_t count = 0;              /* live keys incl. stash (reading A-19) */
    oracle_stats_t st{};

    uint64_t NB() const { return (1ull << m) + split; }
    uint32_t Mask() const { return (uint32_t)((1ull << m) - 1); }
    uint64_t* Slot(uint64_t b, int lane) { return &buckets[b * S + lane]; }

    uint32_t hash_kind = 0;          /* HashPair kind */
    uint32_t H1(uint32_t k) const { return HashPair(hash_kind, 1, k); }
    uint32_t H2(uint32_t k) const { return HashPair(hash_kind, 2, k); }
    uint32_t B1(uint32_t k) const { return Addr(H1(k), Mask(), split); }
    uint32_t B2(uint32_t k) const { return Addr(H2(k), Mask(), split); }

    /* AltBucket (Alg. 3 line 31): the other candidate; equal candidates ->
     * cur; neither -> first candidate. */
    uint32_t Alt(uint32_t k, uint32_t cur) const {
        uint32_t c1 = B1(k), c2 = B2(k);
        if (cur == c1) return c2;
        if (cur == c2) return c1;
        return c1;
    }

    uint64_t StashCapFor(uint64_t nb) const {
        uint64_t c = (uint64_t)llround((double)stash_fraction * (double)nb * S);
        return std::max<uint64_t>(1024, c);
    }

    /* ---- Alg. 1 ReplacePath(T, b, k, v), PAPER:323-346 ------------------ */
    bool ReplacePath(uint32_t b, uint32_t k, uint32_t v) {
        uint64_t cached_kv[S];
        bool match[S];
        for (int l = 0; l < S; ++l) {           /* line 1: coalesced load */
            cached_kv[l] = *Slot(b, l);
            match[l] = (UnpackKey(cached_kv[l]) == k);   /* line 3 */
        }
        uint32_t M = Ballot(match);              /* line 4 */
        if (M == 0) return false;                /* line 5: early exit */
        int w = FirstSet(M);                     /* line 7 */
        uint64_t old = cached_kv[w];             /* winner lane */
        uint64_t nw = Pack(k, v);
        bool success = false;
        if (*Slot(b, w) == old) {                /* line 10: CAS */
            *Slot(b, w) = nw;
            success = true;
        }
        return success;                          /* line 11: broadcast */
    }

    /* ---- Alg. 2 ClaimThenCommit(T, b, kv), PAPER:348-379 --------------- */
    int ClaimThenCommit(uint32_t b, uint64_t kv) {
        uint32_t mask = freeMask[b];             /* line 1: lane 0 load */
        mask = mask & FULL_MASK;                 /* line 2 */
        if (mask == 0) return -1;                /* line 3 */
        bool cand[S];
        for (int l = 0; l < S; ++l) cand[l] = (mask & (1u << l)) != 0;
        uint32_t C = Ballot(cand);               /* line 4 */
        int winner = FirstSet(C);                /* line 5 */
        int claimed = -1;
        uint32_t slotBit = 1u << winner;         /* line 8 */
        uint32_t old = freeMask[b];              /* line 9: FetchAnd */
        freeMask[b] = old & ~slotBit;
        if (old & slotBit) {                     /* line 10 */
            *Slot(b, winner) = kv;               /* line 11: publish */
            claimed = winner;
        }
        /* line 14 "restore bit if failed" is omitted: reading A-12 (the AND
         * changed nothing when the bit was already clear). */
        return claimed;                          /* line 16: broadcast */
    }

    /* ---- Alg. 3 CuckooEvictAndInsert(T, b0, kv0), PAPER:387-436 ---------
     * Reading A-6: each round = ClaimThenCommit then one eviction; after
     * max_evictions rounds the in-hand entry goes to Step 4.  Reading A-13:
     * the place-without-evict branch claims the bit exactly as Alg. 2.      */
    bool CuckooEvictAndInsert(uint32_t b0, uint64_t* kv_inout) {
        uint64_t kv = *kv_inout;
        uint32_t b = b0;
        uint64_t rounds = 0;
        bool placed = false;
        for (uint32_t kick = 1; kick <= max_evictions; ++kick) {   /* line 2 */
            ++rounds;
            if (ClaimThenCommit(b, kv) >= 0) { placed = true; break; }  /* line 3 */
            st.lock_acq++;                                   /* line 7: Lock */
            uint32_t fm = freeMask[b] & FULL_MASK;           /* line 8 (A-22) */
            if (fm != 0) {                                   /* lines 9-15 */
                int s = FirstSet(fm);
                freeMask[b] = fm & ~(1u << s);
                *Slot(b, s) = kv;
                placed = true;                               /* PlacedWithoutEvict */
                break;
            }
            uint32_t occ = ~fm;                              /* line 17 */
            int s = FirstSet(occ);                           /* line 18 */
            uint64_t victim = *Slot(b, s);                   /* line 19 */
            *Slot(b, s) = kv;                                /* line 21 */
            /* Unlock (line 22); Evicted(s) broadcast (line 26) */
            kv = victim;                                     /* line 33 */
            b = Alt(UnpackKey(kv), b);                       /* line 34 */
        }
        st.step3_rounds += rounds;
        st.max_depth = std::max<uint64_t>(st.max_depth, rounds);
        *kv_inout = kv;
        return placed;                                       /* line 38 */
    }

    /* ---- Step 4: overflow stash push, PAPER:438-443 --------------------- */
    bool StashPush(uint64_t kv) {
        uint64_t h = head, t = tail;             /* head relaxed, tail acquire */
        if (t - h < stash_cap) {
            uint64_t pos = t;                    /* fetch_add(tail) */
            tail = t + 1;
            ring[pos % stash_cap] = kv;          /* index = tail mod capacity */
            stash_index[UnpackKey(kv)] = pos % stash_cap;
            return true;
        }
        pending.push_back(kv);                   /* flagged pending */
        return false;
    }
    /* Stash read side (reading A-10): the live ring slot holding key k. */
    int64_t StashFind(uint32_t k) const {
        auto it = stash_index.find(k);
        if (it == stash_index.end()) return -1;
        uint64_t kv = ring[it->second];
        if (kv == EMPTY || UnpackKey(kv) != k) return -1;
        return (int64_t)it->second;
    }

    /* Steps 2-4 for an entry known to be absent from the table. */
    Outcome Place(uint32_t b1, uint32_t b2, uint64_t kv) {
        if (ClaimThenCommit(b1, kv) >= 0) { st.step2++; return Outcome::New; }
        if (b2 != b1 && ClaimThenCommit(b2, kv) >= 0) { st.step2++; return Outcome::New; }
        st.step3_entries++;
        uint64_t in_hand = kv;
        if (CuckooEvictAndInsert(b1, &in_hand)) {  /* Step 3 starts at b1 */
            st.step3_ok++;
            return Outcome::New;
        }
        st.step4++;
        if (StashPush(in_hand)) return Outcome::New;
        return Outcome::Failed;
    }

    /* ---- §IV-A four-step insert, PAPER:310-319 -------------------------- */
    Outcome Insert(uint32_t k, uint32_t v) {
        uint32_t b1 = B1(k), b2 = B2(k);
        /* Step 1: replace in a candidate bucket (Alg. 1) ... */
        if (ReplacePath(b1, k, v)) { st.step1++; return Outcome::Replaced; }
        if (b2 != b1 && ReplacePath(b2, k, v)) { st.step1++; return Outcome::Replaced; }
        /* ... or in the stash (reading A-11). */
        int64_t sp = StashFind(k);
        if (sp >= 0) { ring[sp] = Pack(k, v); st.step1++; return Outcome::Replaced; }
        Outcome o = Place(b1, b2, Pack(k, v));
        if (o == Outcome::New) count++;
        return o;
    }

    /* ---- Alg. 4 ScanBucketAndDelete(T, b, k), PAPER:448-475 ------------- */
    bool ScanBucketAndDelete(uint32_t b, uint32_t k) {
        uint64_t kv[S];
        bool match[S];
        for (int l = 0; l < S; ++l) {            /* lines 4-5 */
            kv[l] = *Slot(b, l);
            match[l] = (UnpackKey(kv[l]) == k);
        }
        uint32_t M = Ballot(match);              /* line 6 */
        if (M == 0) return false;                /* line 7 */
        int w = FirstSet(M);                     /* line 8 */
        bool success = false;
        uint64_t old = kv[w];
        if (*Slot(b, w) == old) {                /* line 12: CAS -> EMPTY */
            *Slot(b, w) = EMPTY;
            success = true;
        }
        if (success) freeMask[b] |= (1u << w);   /* line 14: publish free slot */
        return success;                          /* line 15 */
    }

    /* §IV-B delete over the d = 2 candidates, then the stash (A-10). */
    bool Erase(uint32_t k) {
        uint32_t b1 = B1(k), b2 = B2(k);
        bool ok = ScanBucketAndDelete(b1, k);
        if (!ok && b2 != b1) ok = ScanBucketAndDelete(b2, k);
        if (!ok) {
            int64_t sp = StashFind(k);
            if (sp >= 0) { ring[sp] = EMPTY; stash_index.erase(k); ok = true; }
        }
        if (ok) count--;
        return ok;
    }

    /* §IV-B lookup: WCME over b1, b2 (winner = lowest matching lane), then
     * the stash; bottom (not found) otherwise. PAPER:444-445. */
    bool Find(uint32_t k, uint32_t* v) {
        uint32_t cands[2] = {B1(k), B2(k)};
        for (int d = 0; d < 2; ++d) {
            if (d == 1 && cands[1] == cands[0]) break;
            bool match[S];
            uint64_t kv[S];
            for (int l = 0; l < S; ++l) {
                kv[l] = *Slot(cands[d], l);
                match[l] = (UnpackKey(kv[l]) == k);
            }
            uint32_t M = Ballot(match);
            if (M != 0) { *v = UnpackValue(kv[FirstSet(M)]); return true; }
        }
        int64_t sp = StashFind(k);
        if (sp >= 0) { *v = UnpackValue(ring[sp]); return true; }
        return false;
    }

    /* Stash drain + reinsertion after a resize.
     * The capacity is recomputed for the new size (reading A-8). */
    void DrainAndReinsert() {
        std::vector<uint64_t> live;
        for (uint64_t p = head; p < tail; ++p) {
            uint64_t kv = ring[p % stash_cap];
            if (kv != EMPTY) live.push_back(kv);
        }
        stash_cap = StashCapFor(NB());
        ring.assign(stash_cap, EMPTY);
        head = tail = 0;
        stash_index.clear();
        for (uint64_t kv : live) {
            uint32_t k = UnpackKey(kv);
            (void)Place(B1(k), B2(k), kv);   /* already counted in `count` */
        }
    }

    /* ---- §IV-C.1 expansion (split), PAPER:490-530 ------------------------ */
    void SplitPair(uint32_t b_src, uint32_t b_dst) {
        uint32_t index_mask = Mask();
        uint32_t next_mask = (index_mask << 1) | 1u;
        bool should_move[S];
        uint64_t kv[S];
        for (int l = 0; l < S; ++l) {
            kv[l] = *Slot(b_src, l);
            should_move[l] = false;
            if (kv[l] == EMPTY) continue;
            uint32_t k = UnpackKey(kv[l]);
            /* reading A-3: the hash that addressed the entry to b_src */
            uint32_t h = ((H1(k) & index_mask) == b_src) ? H1(k) : H2(k);
            should_move[l] = ((h & next_mask) == b_dst);
        }
        uint32_t move_mask = Ballot(should_move);
        for (int l = 0; l < S; ++l) {
            if (!should_move[l]) continue;
            uint32_t my_rank = PrefixRank(move_mask, l);
            *Slot(b_dst, my_rank) = kv[l];
            *Slot(b_src, l) = EMPTY;
        }
        int n_movers = Popc(move_mask);
        freeMask[b_src] |= move_mask;
        uint32_t low = (n_movers == 32) ? 0xFFFFFFFFu : ((1u << n_movers) - 1);  /* A-5 */
        freeMask[b_dst] &= ~low;
    }

    /* expand_batch(K): allocate and split K buckets from split_ptr
     * (PAPER:492-495), advance the round at 2^m. */
    void ExpandBatch() {
        uint64_t round_end = (1ull << m);
        uint64_t n = std::min<uint64_t>(resize_k, round_end - split);
        n = std::min<uint64_t>(n, max_buckets - NB());
        if (n == 0) return;
        uint64_t nb_new = NB() + n;
        buckets.resize(nb_new * S, EMPTY);        /* "allocates K new buckets" */
        freeMask.resize(nb_new, 0xFFFFFFFFu);
        for (uint64_t j = 0; j < n; ++j) {
            uint32_t b_src = split;
            uint32_t b_dst = (uint32_t)(b_src + (1ull << m));
            SplitPair(b_src, b_dst);
            split++;
        }
        if (split == round_end) {
            m++;
            split = 0;
        }
        st.grows++;
        DrainAndReinsert();
    }

    /* ---- §IV-C.2 contraction (merge), PAPER:532-553 ----------------------
     * Reading A-7: at split == 0 re-express (m, 0) as (m-1, 2^(m-1)); merge
     * LIFO pairs (split-1, split-1+2^m).  Returns true if a merge aborted. */
    bool MergePair(uint32_t b_dst, uint32_t b_src) {
        bool live[S];
        uint64_t kv[S];
        for (int l = 0; l < S; ++l) {
            kv[l] = *Slot(b_src, l);
            live[l] = (kv[l] != EMPTY);
        }
        uint32_t occ_mask = Ballot(live);
        uint32_t dst_free = freeMask[b_dst];
        int n_move = Popc(occ_mask), n_free = Popc(dst_free);
        if (n_move > n_free) return false;                    /* PAPER:545 abort */
        uint32_t used_mask = 0;
        for (int l = 0; l < S; ++l) {
            if (!live[l]) continue;
            uint32_t my_rank = PrefixRank(occ_mask, l);
            int pos = SelectNthOne(dst_free, my_rank);
            *Slot(b_dst, pos) = kv[l];
            *Slot(b_src, l) = EMPTY;
            used_mask |= (1u << pos);
        }
        freeMask[b_src] = 0xFFFFFFFFu;
        freeMask[b_dst] &= ~used_mask;
        return true;
    }

    bool ContractBatch() {
        if (NB() <= n_b_min) return false;
        if (split == 0) {                       /* PAPER:551-553 regress */
            m--;
            split = (uint32_t)(1ull << m);
        }
        uint64_t n = std::min<uint64_t>(resize_k, split);
        n = std::min<uint64_t>(n, NB() - n_b_min);
        bool aborted = false;
        for (uint64_t j = 0; j < n; ++j) {
            uint32_t b_dst = split - 1;
            uint32_t b_src = (uint32_t)(b_dst + (1ull << m));
            if (!MergePair(b_dst, b_src)) { aborted = true; st.merge_aborts++; break; }
            split--;
            buckets.resize(NB() * S);           /* the partner bucket is released */
            freeMask.resize(NB());
        }
        /* Reading A-30: a regressed round whose first merge aborted is left at
         * split == 2^m, which is the state (m+1, 0) re-expressed (A-7).  It is
         * written back as (m+1, 0): ExpandBatch's round arithmetic
         * (2^m - split buckets left in the round) needs split < 2^m, and with
         * split == 2^m the table could never grow again. */
        if (split == (uint32_t)(1ull << m)) {
            m++;
            split = 0;
        }
        st.shrinks++;
        DrainAndReinsert();
        return aborted;
    }

    /* Triggers, PAPER:480-483 (timing: reading A-19). */
    void GrowBefore(uint64_t n_ins) {
        if (lf_grow >= 1.0f) return;
        while ((double)(count + n_ins) > (double)lf_grow * (double)NB() * S) {
            uint64_t before = NB();
            ExpandBatch();
            if (NB() == before) break;          /* max capacity reached */
        }
    }
    void ShrinkAfter() {
        if (lf_shrink <= 0.0f) return;
        while ((double)count < (double)lf_shrink * (double)NB() * S && NB() > n_b_min) {
            if (ContractBatch()) break;         /* abort stops (reading A-25) */
        }
    }

    /* ---- PHASED batch contract --------------------------- */
    int InsertPhase(const uint32_t* keys, const uint32_t* vals,
                    const std::vector<uint64_t>& idx, uint8_t* status) {
        std::unordered_set<uint32_t> added;   /* keys absent at phase start */
        int rc = 0;
        for (uint64_t i : idx) {
            uint32_t k = keys[i];
            if (k == INVALID_KEY) { status[i] = 2; continue; }
            uint32_t dummy;
            bool present_now = Find(k, &dummy);
            if (!present_now) added.insert(k);
            bool present_at_start = present_now && !added.count(k);
            Outcome o = Insert(k, vals[i]);
            if (o == Outcome::Failed) { status[i] = 3; rc = 1; }
            else status[i] = present_at_start ? 1 : 0;
        }
        return rc;
    }
    void ErasePhase(const uint32_t* keys, const std::vector<uint64_t>& idx, uint8_t* out) {
        std::unordered_set<uint32_t> erased;
        for (uint64_t i : idx) {
            uint32_t k = keys[i];
            if (k == INVALID_KEY) { out[i] = 0; continue; }
            bool ok = Erase(k);
            if (ok) erased.insert(k);
            out[i] = (ok || erased.count(k)) ? 1 : 0;
        }
    }
    void FindPhase(const uint32_t* keys, const std::vector<uint64_t>& idx,
                   uint32_t* vals_out, uint8_t* found) {
        for (uint64_t i : idx) {
            uint32_t k = keys[i];
            uint32_t v = 0;
            bool f = (k != INVALID_KEY) && Find(k, &v);
            found[i] = f ? 1 : 0;
            if (vals_out) vals_out[i] = f ? v : 0;
        }
    }
};

}  // namespace

struct oracle_table { Table t; };

extern "C" {

oracle_t oracle_create(uint64_t capacity_slots, uint64_t max_capacity_slots,
                       float lf_grow, float lf_shrink, uint32_t max_evictions,
                       uint32_t resize_k, float stash_fraction) {
    auto* o = new oracle_table();
    Table& t = o->t;
    /* Reading A-20: any n_b >= 2, held as (m = floor(log2 n_b), split). */
    uint64_t nb = std::max<uint64_t>(2, (capacity_slots + S - 1) / S);
    uint32_t m = 0;
    while ((2ull << m) <= nb) ++m;
    t.m = m;
    t.split = (uint32_t)(nb - (1ull << m));
    t.max_buckets = max_capacity_slots ? std::max<uint64_t>(nb, (max_capacity_slots + S - 1) / S)
                                       : (1ull << 31);
    t.lf_grow = lf_grow;
    t.lf_shrink = lf_shrink;
    t.max_evictions = max_evictions ? max_evictions : 16;
    t.resize_k = resize_k ? resize_k : 1024;
    t.stash_fraction = stash_fraction;
    t.n_b_min = nb;
    t.buckets.assign(nb * S, EMPTY);
    t.freeMask.assign(nb, 0xFFFFFFFFu);
    t.stash_cap = t.StashCapFor(nb);
    t.ring.assign(t.stash_cap, EMPTY);
    return o;
}

void oracle_destroy(oracle_t o) { delete o; }

static std::vector<uint64_t> Iota(uint64_t n) {
    std::vector<uint64_t> v(n);
    for (uint64_t i = 0; i < n; ++i) v[i] = i;
    return v;
}

int oracle_insert(oracle_t o, const uint32_t* keys, const uint32_t* vals, uint64_t n,
                  uint8_t* status) {
    if (n == 0) return 0;
    o->t.GrowBefore(n);
    return o->t.InsertPhase(keys, vals, Iota(n), status);
}

int oracle_find(oracle_t o, const uint32_t* keys, uint64_t n, uint32_t* vals_out,
                uint8_t* found) {
    o->t.FindPhase(keys, Iota(n), vals_out, found);
    return 0;
}

int oracle_erase(oracle_t o, const uint32_t* keys, uint64_t n, uint8_t* erased) {
    if (n == 0) return 0;
    o->t.ErasePhase(keys, Iota(n), erased);
    o->t.ShrinkAfter();
    return 0;
}

int oracle_mixed(oracle_t o, const uint8_t* op, const uint32_t* keys, const uint32_t* vals,
                 uint64_t n, uint32_t* vals_out, uint8_t* result) {
    /* op: 0 find, 1 insert, 2 erase; other codes are invalid
     * ops and report 0. */
    std::vector<uint64_t> ins, era, fnd;
    for (uint64_t i = 0; i < n; ++i) {
        if (op[i] == 1) ins.push_back(i);
        else if (op[i] == 2) era.push_back(i);
        else if (op[i] == 0) fnd.push_back(i);
        else { result[i] = 0; if (vals_out) vals_out[i] = 0; }
    }
    int rc = 0;
    if (!ins.empty()) {
        o->t.GrowBefore(ins.size());
        rc = o->t.InsertPhase(keys, vals, ins, result);
        if (vals_out) for (uint64_t i : ins) vals_out[i] = 0;
    }
    if (!era.empty()) {
        o->t.ErasePhase(keys, era, result);
        if (vals_out) for (uint64_t i : era) vals_out[i] = 0;
        o->t.ShrinkAfter();
    }
    if (!fnd.empty()) o->t.FindPhase(keys, fnd, vals_out, result);
    return rc;
}

void oracle_get_stats(oracle_t o, oracle_stats_t* out) {
    Table& t = o->t;
    oracle_stats_t s = t.st;
    s.n_buckets = t.NB();
    s.m = t.m;
    s.split = t.split;
    s.count = t.count;
    uint64_t live = 0;
    for (uint64_t p = t.head; p < t.tail; ++p)
        if (t.ring[p % t.stash_cap] != EMPTY) ++live;
    s.stash_live = live;
    s.stash_cap = t.stash_cap;
    s.pending = t.pending.size();
    uint64_t in_b1 = 0;
    for (uint64_t b = 0; b < t.NB(); ++b)
        for (int l = 0; l < S; ++l) {
            uint64_t kv = t.buckets[b * S + l];
            if (kv != EMPTY && t.B1(UnpackKey(kv)) == b) ++in_b1;
        }
    s.in_b1 = in_b1;
    *out = s;
}

uint64_t oracle_dump(oracle_t o, uint32_t* keys, uint32_t* vals, uint64_t cap) {
    Table& t = o->t;
    uint64_t n = 0;
    auto emit = [&](uint64_t kv) {
        if (n < cap && keys) { keys[n] = UnpackKey(kv); if (vals) vals[n] = UnpackValue(kv); }
        ++n;
    };
    for (uint64_t i = 0; i < t.NB() * S; ++i)
        if (t.buckets[i] != EMPTY) emit(t.buckets[i]);
    for (uint64_t p = t.head; p < t.tail; ++p)
        if (t.ring[p % t.stash_cap] != EMPTY) emit(t.ring[p % t.stash_cap]);
    return n;
}

int oracle_check(oracle_t o, char* msg, int msglen) {
    Table& t = o->t;
    auto fail = [&](const char* what, uint64_t a, uint64_t b) {
        if (msg && msglen > 0) snprintf(msg, msglen, "%s (%llu, %llu)", what,
                                        (unsigned long long)a, (unsigned long long)b);
        return 1;
    };
    std::unordered_set<uint32_t> seen;
    uint64_t live = 0;
    for (uint64_t b = 0; b < t.NB(); ++b) {
        for (int l = 0; l < S; ++l) {
            uint64_t kv = t.buckets[b * S + l];
            bool free_bit = (t.freeMask[b] >> l) & 1u;
            /* quiescent freeMask/slot consistency */
            if (free_bit != (kv == EMPTY)) return fail("freeMask/slot mismatch", b, l);
            if (kv == EMPTY) continue;
            uint32_t k = UnpackKey(kv);
            if (k == INVALID_KEY) return fail("reserved key stored", b, l);
            if (!seen.insert(k).second) return fail("duplicate key", k, b);
            /* addressing validity */
            if (t.B1(k) != b && t.B2(k) != b) return fail("key outside its candidates", k, b);
            ++live;
        }
    }
    for (uint64_t p = t.head; p < t.tail; ++p) {
        uint64_t kv = t.ring[p % t.stash_cap];
        if (kv == EMPTY) continue;
        uint32_t k = UnpackKey(kv);
        if (!seen.insert(k).second) return fail("duplicate key (stash)", k, p);
        auto it = t.stash_index.find(k);
        if (it == t.stash_index.end() || it->second != p % t.stash_cap)
            return fail("stash index mismatch", k, p);
        ++live;
    }
    if (live != t.count) return fail("count != scan", t.count, live);
    if (!t.pending.empty()) return fail("pending (stash full) entries", t.pending.size(), 0);
    if (t.st.max_depth > t.max_evictions) return fail("eviction depth over bound", t.st.max_depth, t.max_evictions);
    /* stash entries only come from exhausted Step 3 */
    if (t.st.step4 != t.st.step3_entries - t.st.step3_ok)
        return fail("stash pushes != exhausted Step-3 entries", t.st.step4, t.st.step3_entries - t.st.step3_ok);
    if (t.NB() > t.max_buckets) return fail("over max capacity", t.NB(), t.max_buckets);
    if (msg && msglen > 0) msg[0] = 0;
    return 0;
}

void oracle_expand(oracle_t o, uint32_t k) {
    uint32_t saved = o->t.resize_k;
    o->t.resize_k = k;
    o->t.ExpandBatch();
    o->t.resize_k = saved;
}

int oracle_contract(oracle_t o, uint32_t k) {
    uint32_t saved = o->t.resize_k;
    o->t.resize_k = k;
    bool aborted = o->t.ContractBatch();
    o->t.resize_k = saved;
    return aborted ? 1 : 0;
}

uint32_t oracle_bucket(oracle_t o, uint64_t b, uint64_t* slots32) {
    Table& t = o->t;
    if (b >= t.NB()) return 0;
    for (int l = 0; l < S; ++l) slots32[l] = t.buckets[b * S + l];
    return t.freeMask[b];
}

/* The whole bucket array (n_buckets * 32 packed words) and the live stash
 * entries, for loading the oracle's layout into the GPU table (test hook). */
uint64_t oracle_image(oracle_t o, uint64_t* slots, uint64_t* stash, uint64_t stash_cap) {
    Table& t = o->t;
    if (slots) std::copy(t.buckets.begin(), t.buckets.begin() + t.NB() * S, slots);
    uint64_t n = 0;
    for (uint64_t p = t.head; p < t.tail; ++p) {
        uint64_t kv = t.ring[p % t.stash_cap];
        if (kv == EMPTY) continue;
        if (stash && n < stash_cap) stash[n] = kv;
        ++n;
    }
    return n;
}

uint64_t oracle_pack(uint32_t key, uint32_t value) { return Pack(key, value); }
uint32_t oracle_unpack_key(uint64_t pair) { return UnpackKey(pair); }
uint32_t oracle_unpack_value(uint64_t pair) { return UnpackValue(pair); }
uint32_t oracle_bithash1(uint32_t key) { return BitHash1(key); }
uint32_t oracle_bithash2(uint32_t key) { return BitHash2(key); }
uint32_t oracle_crc32_bytes(const uint8_t* p, uint64_t n) { return Crc32Bytes(p, n); }
uint64_t oracle_crc64_bytes(const uint8_t* p, uint64_t n) { return Crc64Bytes(p, n); }
uint32_t oracle_crc32(uint32_t key) { return Crc32Key(key); }
uint32_t oracle_crc64_lo(uint32_t key) { return Crc64Key(key); }
int oracle_set_hash(oracle_t o, uint32_t kind) {
    if (kind > 1 || o->t.count != 0) return 1;   /* only on an empty table */
    o->t.hash_kind = kind;
    return 0;
}
/* Theorem 1: E[Y] = n - m(1 - (1 - 1/m)^n). */
double oracle_uniform_expected_collisions(uint64_t n, uint64_t m) {
    return (double)n - (double)m * (1.0 - std::pow(1.0 - 1.0 / (double)m, (double)n));
}
/* Y = sum_b (L_b - 1)_+ over m single-slot bins, bin = h mod m (
 * SPEC:187 reading), h = hash `fn` (0 BitHash1, 1 BitHash2, 2 CRC-32,
 * 3 CRC-64 low word) of each key. */
uint64_t oracle_observed_collisions(uint32_t fn, const uint32_t* keys, uint64_t n, uint64_t m) {
    std::vector<uint64_t> load(m, 0);
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t h = fn == 0 ? BitHash1(keys[i]) : fn == 1 ? BitHash2(keys[i])
                   : fn == 2 ? Crc32Key(keys[i]) : Crc64Key(keys[i]);
        ++load[h % m];
    }
    uint64_t y = 0;
    for (uint64_t b = 0; b < m; ++b)
        if (load[b] > 1) y += load[b] - 1;
    return y;
}
uint32_t oracle_addr(uint32_t h, uint32_t index_mask, uint32_t split) { return Addr(h, index_mask, split); }
uint32_t oracle_alt(uint32_t key, uint32_t cur, uint32_t index_mask, uint32_t split) {
    uint32_t c1 = Addr(BitHash1(key), index_mask, split), c2 = Addr(BitHash2(key), index_mask, split);
    if (cur == c1) return c2;
    if (cur == c2) return c1;
    return c1;
}
uint32_t oracle_ballot(const uint8_t* preds32) {
    bool p[S];
    for (int l = 0; l < S; ++l) p[l] = preds32[l] != 0;
    return Ballot(p);
}
int oracle_first_set(uint32_t mask) { return FirstSet(mask); }
uint32_t oracle_prefix_rank(uint32_t mask, uint32_t lane) { return PrefixRank(mask, lane); }
int oracle_select_nth_one(uint32_t mask, uint32_t r) { return SelectNthOne(mask, r); }
uint32_t oracle_fmix32(uint32_t h) { return Fmix32(h); }
/* shard(k) = (uint64(fmix32(k ^ seed)) * G) >> 32 */
uint32_t oracle_shard(uint32_t key, uint32_t seed, uint32_t n_shards) {
    return (uint32_t)(((uint64_t)Fmix32(key ^ seed) * (uint64_t)n_shards) >> 32);
}

}  // extern "C"
