// hive_host.cu — C-ABI implementation (include/hive.h): handle lifecycle, the
// PHASED batch contract (INSERT -> ERASE -> FIND), the
// load-factor triggers of PAPER:480-483 at phase boundaries (reading A-19),
// and bucket-array growth by CUDA virtual memory: the whole max_capacity is
// reserved as one virtual range and 2 MiB physical chunks are mapped as the
// split pointer advances, so a split never copies or rehashes the table
// ("allocates K new buckets").
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hive.h"
#include "hive_kernels.cuh"

using namespace hive;

namespace {

thread_local std::string g_err;

// HIVE_TRACE=1: host-side timing of allocation / mapping / sync points (stderr).
inline bool g_trace() { return getenv("HIVE_TRACE") != nullptr; }
struct Trace {
    const char* what;
    uint64_t arg;
    std::chrono::steady_clock::time_point t0;
    Trace(const char* w, uint64_t a) : what(w), arg(a), t0(std::chrono::steady_clock::now()) {}
    ~Trace() {
        if (!g_trace()) return;
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        fprintf(stderr, "[hive] %-14s %12llu %9.1f us\n", what, (unsigned long long)arg, us);
    }
};

void set_err(cudaError_t e, const char* what, int line) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s at hive_host.cu:%d: %s", what, line, cudaGetErrorString(e));
    g_err = buf;
}
void set_err_drv(CUresult r, const char* what, int line) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s at hive_host.cu:%d: CUresult %d", what, line, (int)r);
    g_err = buf;
}

#define CK(x)                                         \
    do {                                              \
        cudaError_t _e = (x);                         \
        if (_e != cudaSuccess) {                      \
            set_err(_e, #x, __LINE__);                \
            return HIVE_ECUDA;                        \
        }                                             \
    } while (0)
#define CKS(x)                                        \
    do {                                              \
        hive_status _s = (x);                         \
        if (_s != HIVE_OK) return _s;                 \
    } while (0)

// ---- CUDA driver VMM entry points (resolved through the runtime, so the
// library does not link libcuda and loads on GPU-less hosts) ----------------
struct Vmm {
    CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    CUresult (*release)(CUmemGenericAllocationHandle);
    CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*free_va)(CUdeviceptr, size_t);
    CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*unmap)(CUdeviceptr, size_t);
    CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
    bool ok = false;
};

bool load_vmm(Vmm& v) {
    if (v.ok) return true;
    struct { const char* name; void** fn; } tab[] = {
        {"cuMemCreate", (void**)&v.create},       {"cuMemRelease", (void**)&v.release},
        {"cuMemAddressReserve", (void**)&v.reserve}, {"cuMemAddressFree", (void**)&v.free_va},
        {"cuMemMap", (void**)&v.map},             {"cuMemUnmap", (void**)&v.unmap},
        {"cuMemSetAccess", (void**)&v.set_access},
        {"cuMemGetAllocationGranularity", (void**)&v.granularity},
    };
    for (auto& e : tab) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(e.name, e.fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !*e.fn) {
            g_err = std::string("driver entry point missing: ") + e.name;
            return false;
        }
    }
    v.ok = true;
    return true;
}
Vmm g_vmm;

// ---- NCCL, loaded at run time (sharded tables) ------------------------------------
// The library does not link NCCL: libnccl.so.2 is dlopen'ed on first use.  If
// the process has already loaded one (torch's), RTLD_NOLOAD picks that copy,
// so comms made by hive_nccl_comm_init and the calls below share one NCCL.
// ncclComm_t is a pointer and ncclDataType_t / ncclResult_t are int enums; the
// 128-byte ncclUniqueId is passed by value as in nccl.h.
struct NcclUniqueId { char internal[128]; };
enum { NCCL_U8 = 1, NCCL_U32 = 3, NCCL_U64 = 5 };   // ncclUint8 / ncclUint32 / ncclUint64
struct Nccl {
    int (*get_version)(int*) = nullptr;
    int (*get_unique_id)(NcclUniqueId*) = nullptr;
    int (*comm_init_rank)(void**, int, NcclUniqueId, int) = nullptr;
    int (*comm_destroy)(void*) = nullptr;
    int (*comm_count)(void*, int*) = nullptr;
    int (*comm_user_rank)(void*, int*) = nullptr;
    int (*alltoall)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;   // NCCL >= 2.28
    int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*group_start)() = nullptr;
    int (*group_end)() = nullptr;
    const char* (*error_string)(int) = nullptr;
    int version = 0;
    bool ok = false;
};
Nccl g_nccl;
std::mutex g_nccl_mu;

bool load_nccl() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.ok) return true;
    void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!so) so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!so) { g_err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror(); return false; }
    struct { const char* name; void** fn; bool need; } tab[] = {
        {"ncclGetVersion", (void**)&g_nccl.get_version, true},
        {"ncclGetUniqueId", (void**)&g_nccl.get_unique_id, true},
        {"ncclCommInitRank", (void**)&g_nccl.comm_init_rank, true},
        {"ncclCommDestroy", (void**)&g_nccl.comm_destroy, true},
        {"ncclCommCount", (void**)&g_nccl.comm_count, true},
        {"ncclCommUserRank", (void**)&g_nccl.comm_user_rank, true},
        {"ncclAlltoAll", (void**)&g_nccl.alltoall, false},
        {"ncclSend", (void**)&g_nccl.send, true},
        {"ncclRecv", (void**)&g_nccl.recv, true},
        {"ncclGroupStart", (void**)&g_nccl.group_start, true},
        {"ncclGroupEnd", (void**)&g_nccl.group_end, true},
        {"ncclGetErrorString", (void**)&g_nccl.error_string, true},
    };
    for (auto& e : tab) {
        *e.fn = dlsym(so, e.name);
        if (!*e.fn && e.need) { g_err = std::string("NCCL symbol missing: ") + e.name; return false; }
    }
    g_nccl.get_version(&g_nccl.version);
    g_nccl.ok = true;
    return true;
}

void set_err_nccl(int r, const char* what, int line) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s at hive_host.cu:%d: NCCL %d (%s)", what, line, r,
             g_nccl.error_string ? g_nccl.error_string(r) : "?");
    g_err = buf;
}
#define CKN(x)                                        \
    do {                                              \
        int _r = (x);                                 \
        if (_r != 0) {                                \
            set_err_nccl(_r, #x, __LINE__);           \
            return HIVE_ENCCL;                        \
        }                                             \
    } while (0)

uint64_t pow2_at_least(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// A reserved virtual range whose prefix is backed by physical memory.
struct VRange {
    struct Chunk { CUmemGenericAllocationHandle h; size_t off, bytes; };
    CUdeviceptr va = 0;
    size_t reserved = 0, mapped = 0;
    std::vector<Chunk> chunks;
};

}  // namespace

struct hive_table_s {
    hive_config cfg{};
    int dev = 0, num_sms = 0;
    Grids grids{};

    // Growable device arrays: each a reserved VA range backed on demand by
    // physical chunks (never moved, never freed while the table lives).
    size_t gran = 0;
    VRange bk;                         // bucket array
    VRange rg;                         // stash ring
    VRange ix;                         // stash index
    VRange dr;                         // drain staging (stash entries to reinsert)
    VRange sp;                         // spill filter: one u64 per bucket
    CUdeviceptr va = 0;                // == bk.va
    uint64_t max_buckets = 0, nb_min = 0;
    uint64_t nb_at_drain = 0;          // bucket count when the stash was last drained (A-29)
    uint32_t m0 = 0, split0 = 0, m = 0, split = 0;

    // stash ring + index (A-10)
    uint64_t* ring = nullptr;
    uint64_t stash_cap = 0;
    uint64_t* sidx = nullptr;
    uint64_t idx_cap = 0;

    Ctrl* ctrl = nullptr;
    Ctrl* ctrl_h = nullptr;            // pinned mirror
    uint64_t* stage_h = nullptr;       // pinned staging words

    // per-batch scratch (grown on demand)
    uint64_t* dd = nullptr;   uint64_t dd_cap = 0;
    uint32_t* owner = nullptr; uint64_t owner_cap = 0;
    uint8_t* flag = nullptr;  uint64_t flag_cap = 0;
    uint64_t drains = 0;                                 // stash drains launched (hive_mixed bookkeeping)
    // (hive_mixed's paired election carves a second set -- its ERASE phase's
    // table, owner ids and flags -- from the upper halves of these three)
    uint64_t* erec = nullptr; uint64_t erec_cap = 0;     // election records (op << 32 | key)
    uint32_t* rvals = nullptr; uint64_t rvals_cap = 0;   // fused insert: values in record order
    uint64_t* ftab = nullptr; uint64_t ftab_cap = 0;     // fused insert: the two epoch-tagged tables
    int fused_grid = 0;                                  // co-resident grid of k_insert_fused
    unsigned long long* ecount = nullptr;                // per-part counts + cursors
    int mono_grid = 0;                                   // co-resident grid of k_mixed_mono
    uint64_t* einfo = nullptr;                           // per-part totals / bases
    uint32_t* left = nullptr; uint64_t left_cap = 0;
    uint32_t* cls = nullptr;  uint64_t cls_cap = 0;
    uint64_t* cnt = nullptr;  uint64_t cnt_cap = 0;
    uint64_t* pinfo = nullptr;

    // host-buffer pipeline (hive_insert_host / hive_find_host): staging buffers,
    // upload / download streams, and "staging free" events
    uint32_t* hk = nullptr; uint64_t hk_cap = 0;
    uint32_t* hv = nullptr; uint64_t hv_cap = 0;
    uint8_t* hst = nullptr; uint64_t hst_cap = 0;
    uint32_t* fq = nullptr; uint64_t fq_cap = 0;
    uint32_t* fv = nullptr; uint64_t fv_cap = 0;
    uint8_t* ff = nullptr; uint64_t ff_cap = 0;
    cudaStream_t up = nullptr, down = nullptr;
    cudaEvent_t ins_free = nullptr, find_free = nullptr;
    cudaEvent_t ctrl_ev = nullptr;     // hive_mixed: control-block read completed
    std::vector<cudaEvent_t> pipe_ev;

    uint64_t grows = 0, shrinks = 0, merge_aborts = 0;
    uint64_t tail_known = 0;           // stash_tail at the last synchronising read
    // The stash has had no push since its last full reset, which left ring
    // words [0, ring_clean) and index words [0, idx_clean) EMPTY: a resize
    // then clears only the newly exposed words.
    bool stash_clean = false;
    uint64_t ring_clean = 0, idx_clean = 0;
    unsigned long long* aborts = nullptr;   // per-segment first aborting merge pair

    // profiling
    struct Rec { const char* name; cudaEvent_t a, b; uint32_t launches; };
    bool prof = false;
    bool step_prof = false;            // hive_profile level 2: clock64 step breakdown
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    struct Agg { const char* name; double ms; uint64_t n; };
    std::vector<Agg> agg;

    std::atomic<int> busy{0};
    cudaStream_t last = nullptr;

    // ---- sharded table (cfg.nccl_comm != NULL): padded exchange buffers ----
    // Carved from one allocation; tot = nranks * cap records.
    struct Shard {
        void* comm = nullptr;
        int nranks = 1, rank = 0;
        uint64_t cap = 0, tot = 0, batch_max = 0;
        void* base = nullptr;
        uint64_t *send_kv = nullptr, *recv_kv = nullptr, *cnt_send = nullptr, *cnt_recv = nullptr;
        uint64_t *n_dev = nullptr, *pcnt = nullptr, *pinfo = nullptr;
        uint8_t *send_op = nullptr, *recv_op = nullptr, *oc = nullptr;
        uint8_t *r8c = nullptr, *ret8 = nullptr, *rr8 = nullptr;
        uint32_t *pos = nullptr, *kc = nullptr, *vc = nullptr, *back = nullptr;
        uint32_t *r32c = nullptr, *ret32 = nullptr, *rr32 = nullptr;
        // host-buffer calls: device staging of the local batch
        uint32_t *hk = nullptr, *hv = nullptr, *ho32 = nullptr;
        uint8_t *ho8 = nullptr, *hop = nullptr;
        // source-side election (HIVE_SHARD_DEDUP): group table, flags, owners, send list
        void* sbase = nullptr;
        uint64_t* stab = nullptr;
        uint64_t smask = 0;
        uint8_t* sflag = nullptr;
        uint32_t *sowner = nullptr, *slist = nullptr;
        unsigned long long* snlist = nullptr;
    } sh;
    bool sharded() const { return sh.comm != nullptr; }

    // ---- peer-memory exchange (NEXT-1) owner scratch, sized n_src * region ----
    struct Inbox {
        uint64_t cap = 0;
        void* base = nullptr;
        uint32_t *kc = nullptr, *vc = nullptr, *back = nullptr, *r32c = nullptr;
        uint8_t *oc = nullptr, *r8c = nullptr;
        uint64_t* n_dev = nullptr;
    } ib;

    uint64_t nb() const { return (1ull << m) + split; }
    TableView tv() const {
        return TableView{(uint64_t*)va, (uint32_t)((1ull << m) - 1), split, (uint64_t*)sp.va, hkind()};
    }
    StashView sv() const { return StashView{ring, sidx, stash_cap, idx_cap - 1, ctrl}; }
    bool dedup_on() const { return !(cfg.flags & HIVE_KEYS_UNIQUE); }
    uint32_t hkind() const { return (cfg.flags & HIVE_HASH_CRC) ? HASH_CRC : HASH_BITHASH; }
    uint64_t stash_cap_for(uint64_t n_b) const {
        uint64_t c = (uint64_t)llround((double)cfg.stash_fraction * (double)n_b * SLOTS);
        return std::max<uint64_t>(1024, c);
    }
};

namespace {

struct BusyGuard {
    hive_table_s* h;
    bool ok;
    explicit BusyGuard(hive_table_s* t) : h(t) { ok = h->busy.exchange(1) == 0; }
    ~BusyGuard() { if (ok) h->busy.store(0); }
};

cudaEvent_t get_event(hive_table_s* h) {
    if (!h->pool.empty()) {
        cudaEvent_t e = h->pool.back();
        h->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Event pair around one launch when profiling is on.
struct Prof {
    hive_table_s* h;
    const char* name;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    uint32_t launches;                   // kernel launches inside the scope
    Prof(hive_table_s* t, const char* nm, cudaStream_t st, uint32_t nl = 1) : h(t), name(nm), s(st), launches(nl) {
        if (h->prof) {
            a = get_event(h);
            cudaEventRecord(a, s);
        }
    }
    ~Prof() {
        if (h->prof) {
            cudaEvent_t b = get_event(h);
            cudaEventRecord(b, s);
            h->recs.push_back({name, a, b, launches});
        }
    }
};

template <typename T>
hive_status ensure(T*& p, uint64_t& cap, uint64_t need) {
    if (need <= cap && p) return HIVE_OK;
    Trace tr("ensure", need * sizeof(T));
    uint64_t n = std::max<uint64_t>(need, cap * 3 / 2);
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc((void**)&p, n * sizeof(T));
    if (e != cudaSuccess) {
        set_err(e, "cudaMalloc(scratch)", __LINE__);
        return HIVE_ENOMEM;
    }
    cap = n;
    return HIVE_OK;
}

hive_status vrange_reserve(hive_table_s* h, VRange& r, size_t bytes) {
    r.reserved = std::max<size_t>(h->gran, (bytes + h->gran - 1) / h->gran * h->gran);
    CUresult e = g_vmm.reserve(&r.va, r.reserved, 0, 0, 0);
    if (e != CUDA_SUCCESS) { set_err_drv(e, "cuMemAddressReserve", __LINE__); return HIVE_ENOMEM; }
    return HIVE_OK;
}

// Back the first `need` bytes of a range with physical memory.  Growth at least
// doubles what is mapped (whole 2 MiB granules, one cuMemCreate per step):
// cuMemSetAccess / cuMemCreate cost 5-95 ms per call on this system (measured,
// HIVE_TRACE), so a long run of K-bucket splits must cost only a few calls.
// Nothing is ever copied or freed on the way.
hive_status vrange_map(hive_table_s* h, VRange& r, size_t need) {
    need = (need + h->gran - 1) / h->gran * h->gran;
    if (need <= r.mapped) return HIVE_OK;
    Trace tr("vrange_map", need);
    size_t target = std::max(need, 2 * r.mapped);
    target = std::min((target + h->gran - 1) / h->gran * h->gran, r.reserved);
    if (target < need) {
        g_err = "request exceeds the reserved max_capacity";
        return HIVE_ENOMEM;
    }
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = h->dev;
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    const size_t off = r.mapped, bytes = target - r.mapped;
    CUmemGenericAllocationHandle mh;
    CUresult e;
    {
        Trace t1("cuMemCreate", bytes);
        e = g_vmm.create(&mh, bytes, &prop, 0);
    }
    if (e != CUDA_SUCCESS) { set_err_drv(e, "cuMemCreate", __LINE__); return HIVE_ENOMEM; }
    {
        Trace t2("cuMemMap", bytes);
        e = g_vmm.map(r.va + off, bytes, 0, mh, 0);
    }
    if (e != CUDA_SUCCESS) { g_vmm.release(mh); set_err_drv(e, "cuMemMap", __LINE__); return HIVE_ENOMEM; }
    r.chunks.push_back({mh, off, bytes});
    Trace t3("cuMemSetAccess", bytes);
    e = g_vmm.set_access(r.va + off, bytes, &acc, 1);
    if (e != CUDA_SUCCESS) { set_err_drv(e, "cuMemSetAccess", __LINE__); return HIVE_ECUDA; }
    r.mapped = target;
    return HIVE_OK;
}

void vrange_free(VRange& r) {
    if (!r.va) return;
    for (auto& c : r.chunks) {
        g_vmm.unmap(r.va + c.off, c.bytes);
        g_vmm.release(c.h);
    }
    g_vmm.free_va(r.va, r.reserved);
    r = VRange{};
}

hive_status map_buckets(hive_table_s* h, uint64_t n_buckets) {
    CKS(vrange_map(h, h->bk, (size_t)n_buckets * SLOTS * 8));
    return vrange_map(h, h->sp, (size_t)n_buckets * sizeof(uint64_t));
}

hive_status read_ctrl(hive_table_s* h, cudaStream_t s) {
    Trace tr("read_ctrl", 0);
    CK(cudaMemcpyAsync(h->ctrl_h, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    h->tail_known = h->ctrl_h->stash_tail;
    return HIVE_OK;
}

hive_status set_ctrl_word(hive_table_s* h, unsigned long long* field, uint64_t value, cudaStream_t s) {
    if (value == 0) {
        CK(cudaMemsetAsync(field, 0, sizeof(uint64_t), s));
        return HIVE_OK;
    }
    // only used right before a synchronising read, so one staging word suffices
    h->stage_h[0] = value;
    CK(cudaMemcpyAsync(field, h->stage_h, sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    return HIVE_OK;
}

// (Re)size the stash for `cap` entries and clear it (ring + index EMPTY, tail 0).
// Ring and index live in reserved VA ranges: growing maps more memory, the
// index capacity is the power of two >= 2 cap (rebuilt at every drain).
hive_status stash_reset(hive_table_s* h, uint64_t cap, cudaStream_t s) {
    const uint64_t ic = pow2_at_least(2 * cap);
    CKS(vrange_map(h, h->rg, cap * sizeof(uint64_t)));
    CKS(vrange_map(h, h->dr, cap * sizeof(uint64_t)));
    CKS(vrange_map(h, h->ix, ic * sizeof(uint64_t)));
    h->ring = (uint64_t*)h->rg.va;
    h->sidx = (uint64_t*)h->ix.va;
    h->stash_cap = cap;
    h->idx_cap = ic;
    CK(launch_stash_reset(s, h->sv()));
    CKS(set_ctrl_word(h, &h->ctrl->stash_tail, 0, s));
    h->tail_known = 0;
    h->stash_clean = true;
    h->ring_clean = cap;
    h->idx_clean = ic;
    return HIVE_OK;
}

// Resize of an EMPTY stash (tail read as 0 at this phase, so no push since its
// last full reset): the ring and the index are all EMPTY up to the cleared
// extents and the index holds nothing to rehash, so only the words the new
// capacity exposes are cleared (one launch), and stash_tail is already 0.
hive_status stash_resize_empty(hive_table_s* h, uint64_t cap, cudaStream_t s) {
    if (!h->stash_clean) return stash_reset(h, cap, s);
    const uint64_t ic = pow2_at_least(2 * cap);
    CKS(vrange_map(h, h->rg, cap * sizeof(uint64_t)));
    CKS(vrange_map(h, h->dr, cap * sizeof(uint64_t)));
    CKS(vrange_map(h, h->ix, ic * sizeof(uint64_t)));
    h->ring = (uint64_t*)h->rg.va;
    h->sidx = (uint64_t*)h->ix.va;
    const uint64_t r0 = std::min(h->ring_clean, cap), i0 = std::min(h->idx_clean, ic);
    CK(launch_fill2(s, h->ring + r0, cap - r0, h->sidx + i0, ic - i0, h->num_sms));
    h->ring_clean = std::max(h->ring_clean, cap);
    h->idx_clean = std::max(h->idx_clean, ic);
    h->stash_cap = cap;
    h->idx_cap = ic;
    return HIVE_OK;
}

// ---- owner election for in-batch duplicates -------------------
hive_status elect_owners(hive_table_s* h, const uint32_t* keys, const uint32_t* idx, uint64_t n_upper,
                         const uint64_t* n_dev, uint64_t n_batch, DedupView* dd, cudaStream_t s) {
    // Large phases: hash-partition the ops so that each part's sub-table
    // (~32 MB) stays in L2 during its election launch (ncu: 18.5 G elections/s
    // with a 1 GiB table vs 49 G/s L2-resident).
    static const uint64_t sub_bytes = getenv("HIVE_ELECT_MB") ? (uint64_t)atoi(getenv("HIVE_ELECT_MB")) << 20
                                                              : (32ull << 20);
    // sub-table entries per expected part record (HIVE_ELECT_F, experiments)
    static const double fill = getenv("HIVE_ELECT_F") ? atof(getenv("HIVE_ELECT_F")) : 2.5;
    // HIVE_ELECT_JIT=0: clear all sub-tables up front (measured slower)
    static const bool jit = getenv("HIVE_ELECT_JIT") ? atoi(getenv("HIVE_ELECT_JIT")) != 0 : true;
    uint32_t parts = 1;
    while (parts < MAX_PARTS && 2 * n_upper * sizeof(uint64_t) / parts > sub_bytes) parts *= 2;
    const uint64_t sub = pow2_at_least(std::max<uint64_t>(
        1024, parts == 1 ? 2 * n_upper : (uint64_t)(fill * (double)n_upper / parts)));
    CKS(ensure(h->dd, h->dd_cap, sub * parts));
    CKS(ensure(h->owner, h->owner_cap, n_batch));
    CKS(ensure(h->flag, h->flag_cap, n_batch + 1));
    *dd = DedupView{h->dd, sub - 1, h->flag, h->owner, parts, h->flag + n_batch};
    CK(cudaMemsetAsync(h->flag, 0, n_batch + 1, s));
    if (parts == 1 || !jit) CK(cudaMemsetAsync(h->dd, 0xFF, sub * parts * sizeof(uint64_t), s));
    if (parts == 1) {
        Prof p(h, "k_dedup_elect", s);
        CK(launch_dedup_elect(h->grids.dedup, s, keys, idx, n_upper, n_dev, *dd, h->ctrl));
        return HIVE_OK;
    }
    CKS(ensure(h->erec, h->erec_cap, n_upper));
    {
        Prof p(h, "k_elect_partition", s, 3);
        CK(launch_elect_partition(s, keys, idx, n_upper, n_dev, parts, h->ecount, h->ecount + MAX_PARTS,
                                  h->einfo, h->erec, h->num_sms));
    }
    // Each part's sub-table is cleared right before its launch: the memset
    // leaves its lines in L2, where the election's CASes then hit (clearing on
    // a side stream that overlaps the partition and the earlier parts measured
    // slower: the parts then miss L2).  The sub-tables stay
    // intact for the probe kernels' owner lookups.
    // Part q's launch clears part q+1's sub-table in its tail (the election is
    // L2-atomic bound, so the writes use idle HBM time and leave the next
    // table's lines in L2): cfg2 elections 1.51 -> 1.31 ms
    // (profiles/r02c_elect_chain_ab.txt).  HIVE_ELECT_CHAIN=0: a memset before
    // each part instead.
    static const bool chain = !getenv("HIVE_ELECT_CHAIN") || atoi(getenv("HIVE_ELECT_CHAIN")) != 0;
    Prof p(h, "k_dedup_elect", s, parts);
    for (uint32_t q = 0; q < parts; ++q) {
        if (jit && (!chain || q == 0)) CK(cudaMemsetAsync(h->dd + (uint64_t)q * sub, 0xFF, sub * sizeof(uint64_t), s));
        uint64_t* next = (jit && chain && q + 1 < parts) ? h->dd + (uint64_t)(q + 1) * sub : nullptr;
        CK(launch_dedup_elect_part(h->grids.dedup, s, h->erec, h->einfo, q, *dd, h->ctrl, next, next ? sub : 0));
    }
    return HIVE_OK;
}

// Both elections of a mixed batch whose phases each fit one sub-table, in ONE
// launch (hive_mixed, before the control wait): the INSERT list into the first
// scratch set, the ERASE list into the second.  pair_prepare sizes the sets and
// returns the views plus the byte ranges to clear (flags to 0, tables to all
// ones, done by the batch's k_batch_prep); false when a phase would need the
// partitioned election.
struct PairScratch {
    DedupView ins{nullptr, 0, nullptr, nullptr}, era{nullptr, 0, nullptr, nullptr};
    uint8_t* flag = nullptr;
    uint64_t fbytes = 0;
    uint64_t* dd = nullptr;
    uint64_t dwords = 0;
};
bool pair_prepare(hive_table_s* h, uint64_t n_upper, uint64_t n_batch, PairScratch* ps, hive_status* st) {
    static const uint64_t sub_bytes = getenv("HIVE_ELECT_MB") ? (uint64_t)atoi(getenv("HIVE_ELECT_MB")) << 20
                                                              : (32ull << 20);
    *st = HIVE_OK;
    if (2 * n_upper * sizeof(uint64_t) > sub_bytes) return false;
    const uint64_t sub = pow2_at_least(std::max<uint64_t>(1024, 2 * n_upper));
    auto fail = [&](hive_status e) { *st = e; return false; };
    // both scratch sets carved from one allocation each (tables, owner ids,
    // flags); the ERASE set's flags start 16-byte aligned (the duplicate
    // fix-up scans them 16 per load)
    const uint64_t fstride = (n_batch + 1 + 15) & ~15ull;
    if (hive_status e = ensure(h->dd, h->dd_cap, 2 * sub); e != HIVE_OK) return fail(e);
    if (hive_status e = ensure(h->owner, h->owner_cap, 2 * n_batch); e != HIVE_OK) return fail(e);
    if (hive_status e = ensure(h->flag, h->flag_cap, 2 * fstride); e != HIVE_OK) return fail(e);
    ps->ins = DedupView{h->dd, sub - 1, h->flag, h->owner, 1, h->flag + n_batch};
    ps->era = DedupView{h->dd + sub, sub - 1, h->flag + fstride, h->owner + n_batch, 1, h->flag + fstride + n_batch};
    ps->flag = h->flag;
    ps->fbytes = 2 * fstride;
    ps->dd = h->dd;
    ps->dwords = 2 * sub;
    return true;
}

// ---- the INSERT phase (Steps 1-4, owner election, duplicate fix-up) ---------------
// Chunked launch of the fast path for the host pipeline: chunk c covers ops
// [c * chunk, ...) and waits for ready[c] (its values have been uploaded).
struct InsertChunks {
    uint64_t chunk;
    const cudaEvent_t* ready;
};

// The INSERT phase as ONE cooperative launch (k_insert_fused): the ops are
// hash-partitioned with their values, then each part's owner election
// overlaps the previous part's fast path, followed by Steps 3-4 and the
// duplicate fix-up.  Used for large phases with owner election on.
hive_status insert_phase_fused(hive_table_s* h, const uint32_t* keys, const uint32_t* vals, const uint32_t* idx,
                               uint64_t n_upper, const uint64_t* n_dev, uint64_t n_batch, uint8_t* status,
                               uint32_t* vals_zero, cudaStream_t s) {
    const uint64_t per = pow2_at_least(std::max<uint64_t>(1024, (uint64_t)(2.5 * (double)n_upper / FUSED_PARTS)));
    CKS(ensure(h->ftab, h->ftab_cap, 2 * per));
    CKS(ensure(h->owner, h->owner_cap, n_batch));
    CKS(ensure(h->flag, h->flag_cap, n_batch));
    CKS(ensure(h->erec, h->erec_cap, n_upper));
    CKS(ensure(h->rvals, h->rvals_cap, n_upper));
    CKS(ensure(h->left, h->left_cap, std::max<uint64_t>(n_upper, 1)));
    if (!h->fused_grid) h->fused_grid = fused_grid(h->num_sms);
    CK(cudaMemsetAsync(h->flag, 0, n_batch, s));
    CK(cudaMemsetAsync(h->ftab, 0x04, per * sizeof(uint64_t), s));          // epoch 1: stale for even parts
    CK(cudaMemsetAsync(h->ftab + per, 0x00, per * sizeof(uint64_t), s));    // epoch 0: stale for odd parts
    {
        Prof p(h, "k_elect_partition", s, 3);
        CK(launch_elect_partition(s, keys, idx, n_upper, n_dev, FUSED_PARTS, h->ecount, h->ecount + MAX_PARTS,
                                  h->einfo, h->erec, h->num_sms, vals, h->rvals, status, vals_zero));
    }
    CK(cudaMemsetAsync(&h->ctrl->n_left, 0, 2 * sizeof(uint64_t), s));     // n_left + slow_next
    Prof p(h, "k_insert_fused", s);
    CK(launch_insert_fused(h->fused_grid, s, h->erec, h->rvals, h->einfo, h->ftab, h->ftab + per, per - 1,
                           DedupView{h->ftab, per - 1, h->flag, h->owner, FUSED_PARTS}, h->tv(), h->sv(), status,
                           vals_zero, h->left, h->cfg.max_evictions, keys, vals));
    return HIVE_OK;
}

hive_status insert_phase(hive_table_s* h, const uint32_t* keys, const uint32_t* vals,
                         const uint64_t* kvs, const uint32_t* idx, uint64_t n_upper,
                         const uint64_t* n_dev, uint64_t n_batch, uint8_t* status,
                         uint32_t* vals_zero, cudaStream_t s, const InsertChunks* chunks = nullptr,
                         const DedupView* pre = nullptr, DupFix* defer = nullptr, bool left_zeroed = false) {
    const bool dedup = !kvs && h->dedup_on();
    // large phases with election: the fused single-launch form, opt-in with
    // HIVE_FUSED=1 (measured slower than the multi-launch form)
    static const bool fused_ok = getenv("HIVE_FUSED") && atoi(getenv("HIVE_FUSED")) != 0;
    if (dedup && fused_ok && !pre && !chunks && !h->step_prof && n_upper >= FUSED_MIN_OPS)
        return insert_phase_fused(h, keys, vals, idx, n_upper, n_dev, n_batch, status, vals_zero, s);
    DedupView dd{nullptr, 0, nullptr, nullptr};
    if (dedup && pre) dd = *pre;                 // election already enqueued by the caller
    else if (dedup) CKS(elect_owners(h, keys, idx, n_upper, n_dev, n_batch, &dd, s));
    CKS(ensure(h->left, h->left_cap, std::max<uint64_t>(n_upper, 1)));
    static_assert(offsetof(Ctrl, slow_next) == offsetof(Ctrl, n_left) + sizeof(uint64_t), "adjacent");
    if (!left_zeroed) CK(cudaMemsetAsync(&h->ctrl->n_left, 0, 2 * sizeof(uint64_t), s));   // n_left + slow_next
    if (chunks) {
        Prof p(h, "k_insert_fast", s);
        for (uint64_t off = 0, c = 0; off < n_upper; off += chunks->chunk, ++c) {
            CK(cudaStreamWaitEvent(s, chunks->ready[c], 0));
            CK(launch_insert_fast(h->grids, s, keys, vals, nullptr, nullptr,
                                  std::min<uint64_t>(chunks->chunk, n_upper - off), nullptr, h->tv(), h->sv(),
                                  dd, status, nullptr, h->left, (uint32_t)off, h->step_prof));
        }
    } else {
        Prof p(h, kvs ? "k_insert_fast(reinsert)" : "k_insert_fast", s);
        CK(launch_insert_fast(h->grids, s, keys, vals, kvs, idx, n_upper, n_dev, h->tv(),
                              h->sv(), dd, status, vals_zero, h->left, 0, h->step_prof));
    }
    {
        Prof p(h, kvs ? "k_insert_slow(reinsert)" : "k_insert_slow", s);
        CK(launch_insert_slow(h->grids, s, keys, vals, kvs, h->left, h->tv(), h->sv(),
                              h->cfg.max_evictions, status, h->step_prof));
    }
    if (dedup && status && defer) {
        // a mixed batch: the next phase's kernel runs the fix-up first
        *defer = DupFix{dd.flag, dd.owner_of, dd.any, status, n_batch};
    } else if (dedup && status) {
        Prof p(h, "k_dup_copy", s);
        // flags are set only for this phase's ops (the array is per phase), so
        // the dense scan of flag[0, n_batch) replaces a walk of the op list
        // (16 flags per load instead of one random byte per listed op)
        CK(launch_dup_copy(h->grids.stream, s, nullptr, n_batch, nullptr, dd, status));
    }
    return HIVE_OK;
}

// Drain the stash and reinsert its entries with Steps 2-4 after a resize
// (PAPER:214, 443); the capacity follows the new size (reading A-8).  Uses the
// stash tail of the synchronising read that preceded the resize.  The oracle
// drains after every K-bucket batch; the GPU drains once per resize phase
// (stash membership is not observable, count is unchanged either way).
// Expansion-time drains are batched (reading A-29): while the table has grown
// by less than 1/8 since the last drain and the stash is under 1/4 of its
// capacity -- with room for 1/16 of the coming inserts -- the drain waits for
// a later expansion phase.  Contraction always drains (the capacity shrinks).
// HIVE_DRAIN_EVERY=1 drains at every resize phase.
hive_status drain_reinsert(hive_table_s* h, cudaStream_t s, bool growing = false, uint64_t n_ins = 0) {
    static const bool every = getenv("HIVE_DRAIN_EVERY") && atoi(getenv("HIVE_DRAIN_EVERY")) != 0;
    const uint64_t new_cap = h->stash_cap_for(h->nb());
    if (h->tail_known == 0) {
        if (new_cap != h->stash_cap) CKS(stash_resize_empty(h, new_cap, s));
        h->nb_at_drain = h->nb();
        return HIVE_OK;
    }
    if (growing && !every && h->tail_known != ~0ull && 8 * h->nb() < 9 * h->nb_at_drain &&
        4 * h->tail_known < h->stash_cap && h->tail_known + n_ins / 16 < h->stash_cap)
        return HIVE_OK;
    h->nb_at_drain = h->nb();
    ++h->drains;                       // hive_mixed: the Step-3 cursors are no longer zero
    const uint64_t used = std::min<uint64_t>(h->tail_known, h->stash_cap);
    Trace tr("drain", used);
    CKS(vrange_map(h, h->dr, used * sizeof(uint64_t)));
    uint64_t* tmpkv = (uint64_t*)h->dr.va;
    CK(cudaMemcpyAsync(tmpkv, h->ring, used * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    CKS(stash_reset(h, new_cap, s));
    CKS(insert_phase(h, nullptr, nullptr, tmpkv, nullptr, used, nullptr, used, nullptr, nullptr, s));
    h->tail_known = ~0ull;             // unknown until the next read
    return HIVE_OK;
}

// Grow before an INSERT phase (reading A-19): the K-bucket
// expand_batch loop of the oracle is simulated on the host from `count` (it
// depends on nothing else), then executed as one k_split launch per
// linear-hashing round it crosses -- pairs of one round are independent, and a
// round's sources were written by the previous round's launch.
hive_status grow_known(hive_table_s* h, uint64_t count, uint64_t n_ins, cudaStream_t s) {
    uint32_t m = h->m, split = h->split;
    uint64_t batches = 0;
    auto nb = [&]() { return (1ull << m) + split; };
    while ((double)(count + n_ins) > (double)h->cfg.lf_grow * (double)nb() * SLOTS) {
        uint64_t n = std::min<uint64_t>(h->cfg.resize_k, (1ull << m) - split);
        n = std::min<uint64_t>(n, h->max_buckets - nb());
        if (n == 0) break;                // max_capacity reached
        split += (uint32_t)n;
        if (split == (1u << m)) { ++m; split = 0; }
        ++batches;
    }
    if (!batches) return HIVE_OK;
    CKS(map_buckets(h, nb()));
    while (h->m != m || h->split != split) {
        const uint32_t round_end = 1u << h->m;
        const uint32_t stop = (h->m == m) ? split : round_end;
        {
            Prof p(h, "k_split", s);
            CK(launch_split(s, h->tv(), stop - h->split, h->ctrl));
        }
        h->split = stop;
        if (h->split == round_end) { h->m += 1; h->split = 0; }
    }
    h->grows += batches;
    return drain_reinsert(h, s, true, n_ins);
}

hive_status grow_before(hive_table_s* h, uint64_t n_ins, cudaStream_t s) {
    if (h->cfg.lf_grow >= 1.0f || n_ins == 0) return HIVE_OK;
    CKS(read_ctrl(h, s));
    return grow_known(h, h->ctrl_h->count, n_ins, s);
}

// Shrink after an ERASE phase: the oracle's
// contract_batch loop is simulated from `count` into per-round segments of
// LIFO pairs; each segment is one check+apply launch pair that stops at its
// first aborting pair (and merges nothing if an earlier segment aborted);
// one synchronising read returns how far the merges got.
// count_lb: a host-known lower bound on the live count (count at the phase
// start minus the erase ops); when even it is above the contraction threshold
// the device read -- a stream sync -- is skipped.
hive_status shrink_after(hive_table_s* h, cudaStream_t s, int64_t count_lb = -1) {
    if (h->cfg.lf_shrink <= 0.0f || h->nb() <= h->nb_min) return HIVE_OK;
    if (count_lb >= 0 && (double)count_lb >= (double)h->cfg.lf_shrink * (double)h->nb() * SLOTS) return HIVE_OK;
    CKS(read_ctrl(h, s));
    const uint64_t count = h->ctrl_h->count;
    struct Seg { uint32_t m, split0; uint64_t pairs; };
    std::vector<Seg> segs;
    uint32_t m = h->m, split = h->split;
    uint64_t batches = 0;
    auto nb = [&]() { return (1ull << m) + split; };
    while ((double)count < (double)h->cfg.lf_shrink * (double)nb() * SLOTS && nb() > h->nb_min) {
        if (split == 0) { --m; split = 1u << m; }              // regress, A-7
        uint64_t n = std::min<uint64_t>(h->cfg.resize_k, split);
        n = std::min<uint64_t>(n, nb() - h->nb_min);
        if (segs.empty() || segs.back().m != m) {
            if ((int)segs.size() == MAX_SEGMENTS) break;
            segs.push_back({m, split, 0});
        }
        segs.back().pairs += n;
        split -= (uint32_t)n;
        ++batches;
    }
    if (segs.empty()) return HIVE_OK;
    for (size_t i = 0; i < segs.size(); ++i) h->stage_h[8 + i] = segs[i].pairs;
    CK(cudaMemcpyAsync(h->aborts, h->stage_h + 8, segs.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    for (size_t i = 0; i < segs.size(); ++i) {
        TableView tv{(uint64_t*)h->va, (uint32_t)((1ull << segs[i].m) - 1), segs[i].split0, (uint64_t*)h->sp.va,
                     h->hkind()};
        Prof p(h, "k_merge", s, 2);
        CK(launch_merge(s, tv, (uint32_t)segs[i].pairs, h->aborts + i, i ? h->aborts + i - 1 : nullptr,
                        i ? segs[i - 1].pairs : 0));
    }
    CK(cudaMemcpyAsync(h->stage_h + 8, h->aborts, segs.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (size_t i = 0; i < segs.size(); ++i) {
        const uint64_t merged = std::min<uint64_t>(h->stage_h[8 + i], segs[i].pairs);
        h->m = segs[i].m;
        h->split = segs[i].split0 - (uint32_t)merged;
        if (merged < segs[i].pairs) { h->merge_aborts++; break; }
    }
    // Reading A-30: a regressed round that merged nothing leaves split == 2^m,
    // the state (m+1, 0) re-expressed (A-7); write it back as (m+1, 0) so that
    // grow_known's round arithmetic (2^m - split buckets left) holds.
    if (h->split == (1u << h->m)) {
        h->m += 1;
        h->split = 0;
    }
    h->shrinks += batches;
    return drain_reinsert(h, s);
}

hive_status erase_phase(hive_table_s* h, const uint32_t* keys, const uint32_t* idx, uint64_t n_upper,
                        const uint64_t* n_dev, uint64_t n_batch, uint8_t* out, uint32_t* vals_zero,
                        cudaStream_t s, const DedupView* pre = nullptr, const DupFix* carry = nullptr,
                        DupFix* defer = nullptr) {
    const bool dedup = h->dedup_on();
    DedupView dd{nullptr, 0, nullptr, nullptr};
    if (dedup && pre) dd = *pre;                 // election already enqueued by the caller
    else if (dedup) CKS(elect_owners(h, keys, idx, n_upper, n_dev, n_batch, &dd, s));
    {
        Prof p(h, "k_erase", s);
        CK(launch_erase(h->grids, s, keys, idx, n_upper, n_dev, h->tv(), h->sv(), dd, out,
                        vals_zero, carry));
    }
    if (dedup && out && defer) {
        *defer = DupFix{dd.flag, dd.owner_of, dd.any, out, n_batch};     // into the FIND kernel
    } else if (dedup && out) {
        Prof p(h, "k_dup_copy", s);
        CK(launch_dup_copy(h->grids.stream, s, nullptr, n_batch, nullptr, dd, out));   // dense scan
    }
    return HIVE_OK;
}

}  // namespace

// ---- host-buffer pipeline -----------------------------------------------------------
namespace {
// CRC constant tables are per device (module __device__ arrays): fill them once.
bool ensure_hash_tables() {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) { set_err(e, "cudaGetDevice", __LINE__); return false; }
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && done[dev]) return true;
    if (cudaError_t e = init_hash_tables(); e != cudaSuccess) { set_err(e, "init_hash_tables", __LINE__); return false; }
    if (dev < 64) done[dev] = true;
    return true;
}
constexpr uint64_t HOST_CHUNK = 1ull << 22;   // ops per transfer / launch chunk

hive_status pipe_init(hive_table_s* h, size_t n_events) {
    if (!h->up) {
        CK(cudaStreamCreateWithFlags(&h->up, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&h->down, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->ins_free, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->find_free, cudaEventDisableTiming));
        CK(cudaEventRecord(h->ins_free, h->up));
        CK(cudaEventRecord(h->find_free, h->up));
    }
    while (h->pipe_ev.size() < n_events) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->pipe_ev.push_back(e);
    }
    return HIVE_OK;
}
}  // namespace

namespace {
// The PHASED mixed batch: classify, INSERT, ERASE, FIND.  n is
// an upper bound of the batch when n_dev (device word) holds its length.
hive_status mixed_impl(hive_t h, const uint8_t* d_op, const uint32_t* d_keys, const uint32_t* d_vals,
                       uint64_t n, const uint64_t* n_dev, uint32_t* d_vals_out, uint8_t* d_result,
                       cudaStream_t s) {
    // classify: op indices by opcode into 3 regions of n (one pass; order
    // inside a region is not the op order -- every phase is order-free)
    CKS(ensure(h->cls, h->cls_cap, 3 * n));
    // one launch resets the batch's counters and the paired election's
    // scratch (the class counts live in the control block, so the control
    // read below brings them along)
    const bool early = h->cfg.lf_grow < 1.0f;       // elections before the control wait
    PairScratch ps;
    bool pair = false;
    if (early && h->dedup_on()) {
        hive_status e2 = HIVE_OK;
        pair = pair_prepare(h, n, n, &ps, &e2);
        CKS(e2);
    }
    CK(launch_batch_prep(s, h->ctrl, true, pair ? ps.flag : nullptr, pair ? ps.fbytes : 0, pair ? ps.dd : nullptr,
                         pair ? ps.dwords : 0, h->num_sms));
    const uint64_t drains0 = h->drains;
    uint64_t* cls_n = reinterpret_cast<uint64_t*>(h->ctrl->cls_n);
    {
        Prof p(h, "k_classify", s);
        CK(launch_classify(s, d_op, n, n_dev, cls_n, h->cls, n, d_result, d_vals_out, h->num_sms, true));
    }
    const uint64_t* n_find = cls_n + 0;
    const uint64_t* n_ins = cls_n + 1;
    const uint64_t* n_era = cls_n + 2;
    int64_t count_lb = -1;
    DedupView dd_ins{nullptr, 0, nullptr, nullptr}, dd_era{nullptr, 0, nullptr, nullptr};
    bool pre = false, pre_era = false;
    if (early) {                           // one wait: phase sizes + counters
        if (!h->ctrl_ev) CK(cudaEventCreateWithFlags(&h->ctrl_ev, cudaEventDisableTiming));
        CK(cudaMemcpyAsync(h->ctrl_h, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(h->ctrl_ev, s));
        // The owner elections do not depend on the table geometry: enqueue
        // them before waiting, so the GPU has work while the host plans the
        // resize from the count it just read.
        if (pair) {
            dd_ins = ps.ins;
            dd_era = ps.era;
            Prof p(h, "k_dedup_elect", s);
            CK(launch_dedup_elect(h->grids.dedup, s, d_keys, h->cls + n, n, n_ins, dd_ins, h->ctrl, h->cls + 2 * n,
                                  n_era, &dd_era));
            pre = pre_era = true;
        } else if (h->dedup_on()) {          // large batch: the INSERT phase's partitioned election
            CKS(elect_owners(h, d_keys, h->cls + n, n, n_ins, n, &dd_ins, s));
            pre = true;
        }
        {
            Trace tr("read_ctrl", 0);
            CK(cudaEventSynchronize(h->ctrl_ev));
        }
        h->tail_known = h->ctrl_h->stash_tail;
        const uint64_t count0 = h->ctrl_h->count, n_erase = h->ctrl_h->cls_n[2], n_insert = h->ctrl_h->cls_n[1];
        count_lb = count0 > n_erase ? (int64_t)(count0 - n_erase) : 0;
        if (n_insert) CKS(grow_known(h, count0, n_insert, s));
    }
    // each phase's duplicate fix-up runs as the prologue of the next phase's
    // kernel (they write results of different op classes): two launches less.
    // The INSERT fix-up rides in k_erase only when the ERASE phase was elected
    // into the second scratch set (pre_era); otherwise that election reuses
    // the first set's flags and the fix-up must run before it.
    DupFix fix_ins, fix_era;
    CKS(insert_phase(h, d_keys, d_vals, nullptr, h->cls + n, n, n_ins, n, d_result, d_vals_out, s, nullptr,
                     pre ? &dd_ins : nullptr, pre_era ? &fix_ins : nullptr, h->drains == drains0));
    CKS(erase_phase(h, d_keys, h->cls + 2 * n, n, n_era, n, d_result, d_vals_out, s, pre_era ? &dd_era : nullptr,
                    pre_era ? &fix_ins : nullptr, &fix_era));
    CKS(shrink_after(h, s, count_lb));
    Prof p(h, "k_find", s);
    CK(launch_find(h->grids, s, d_keys, h->cls, n, n_find, h->tv(), h->sv(), d_vals_out, d_result, &fix_era));
    return HIVE_OK;
}

// ---- sharded table: padded NCCL exchange (include/hive.h "Sharded tables") -------
enum ShardKind { SK_INSERT = 0, SK_FIND = 1, SK_ERASE = 2, SK_MIXED = 3 };

// Buffers of the padded exchange, carved from one cudaMalloc (allocator calls
// cost 5-95 ms each on this system).
hive_status shard_alloc(hive_table_s* h) {
    auto& S = h->sh;
    const uint64_t tot = S.tot, bm = std::max<uint64_t>(S.batch_max, 1), G = (uint64_t)S.nranks;
    const uint64_t pc = G * part_warps(bm) + 1;
    struct Part { void** p; uint64_t bytes; } parts[] = {
        {(void**)&S.send_kv, tot * 8}, {(void**)&S.recv_kv, tot * 8}, {(void**)&S.cnt_send, G * 8},
        {(void**)&S.cnt_recv, G * 8}, {(void**)&S.n_dev, 8}, {(void**)&S.pcnt, pc * 8},
        {(void**)&S.pinfo, 2 * MAX_PARTS * 8}, {(void**)&S.pos, bm * 4}, {(void**)&S.kc, tot * 4},
        {(void**)&S.vc, tot * 4}, {(void**)&S.back, tot * 4}, {(void**)&S.r32c, tot * 4},
        {(void**)&S.ret32, tot * 4}, {(void**)&S.rr32, tot * 4}, {(void**)&S.hk, bm * 4},
        {(void**)&S.hv, bm * 4}, {(void**)&S.ho32, bm * 4}, {(void**)&S.send_op, tot},
        {(void**)&S.recv_op, tot}, {(void**)&S.oc, tot}, {(void**)&S.r8c, tot}, {(void**)&S.ret8, tot},
        {(void**)&S.rr8, tot}, {(void**)&S.ho8, bm}, {(void**)&S.hop, bm},
    };
    uint64_t total = 0;
    for (auto& q : parts) total += (q.bytes + 255) / 256 * 256;
    Trace tr("shard_alloc", total);
    cudaError_t e = cudaMalloc(&S.base, total);
    if (e != cudaSuccess) { set_err(e, "cudaMalloc(shard buffers)", __LINE__); return HIVE_ENOMEM; }
    uint64_t off = 0;
    for (auto& q : parts) {
        *q.p = (char*)S.base + off;
        off += (q.bytes + 255) / 256 * 256;
    }
    // results of padding positions are never read, but keep them defined
    CK(cudaMemset(S.base, 0, total));
    return HIVE_OK;
}

// One all-to-all of `count` elements per peer: ncclAlltoAll (NCCL >= 2.28) or
// a group of send / recv pairs.  skip_self: the rank's own block is not moved
// (the caller reads it from the send buffer) -- NCCL would copy it locally,
// which at 2^26-op batches costs more than the whole exchange to a peer.
hive_status a2a(hive_table_s* h, const void* send, void* recv, size_t count, int dtype, size_t esize,
                cudaStream_t s, bool skip_self = false) {
    auto& S = h->sh;
    if (g_nccl.alltoall && !skip_self) {
        CKN(g_nccl.alltoall(send, recv, count, dtype, S.comm, s));
        return HIVE_OK;
    }
    CKN(g_nccl.group_start());
    for (int p = 0; p < S.nranks; ++p) {
        if (skip_self && p == S.rank) continue;
        CKN(g_nccl.send((const char*)send + p * count * esize, count, dtype, p, S.comm, s));
        CKN(g_nccl.recv((char*)recv + p * count * esize, count, dtype, p, S.comm, s));
    }
    CKN(g_nccl.group_end());
    return HIVE_OK;
}

// The owner's PHASED batch over a compacted received batch whose length is
// the device word n_dev (n_upper bounds it): the host waits only where the
// phase itself needs a count (growth / contraction enabled).
hive_status owner_phase(hive_table_s* h, int kind, const uint8_t* oc, const uint32_t* kc, const uint32_t* vc,
                        uint64_t n_upper, const uint64_t* n_dev, uint8_t* r8c, uint32_t* r32c, cudaStream_t s) {
    switch (kind) {
        case SK_INSERT:
            if (h->cfg.lf_grow < 1.0f) {             // growth needs the union batch size on the host
                CK(cudaMemcpyAsync(h->stage_h, n_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
                CKS(read_ctrl(h, s));
                if (h->stage_h[0]) CKS(grow_known(h, h->ctrl_h->count, h->stage_h[0], s));
            }
            return insert_phase(h, kc, vc, nullptr, nullptr, n_upper, n_dev, n_upper, r8c, nullptr, s);
        case SK_FIND: {
            Prof p(h, "k_find", s);
            CK(launch_find(h->grids, s, kc, nullptr, n_upper, n_dev, h->tv(), h->sv(), r32c, r8c));
            return HIVE_OK;
        }
        case SK_ERASE:
            CKS(erase_phase(h, kc, nullptr, n_upper, n_dev, n_upper, r8c, nullptr, s));
            return shrink_after(h, s);
        default:
            return mixed_impl(h, oc, kc, vc, n_upper, n_dev, r32c, r8c, s);
    }
}

// One collective op of a sharded handle: route -> all-to-all -> owner phase on
// the union batch (rank order) -> all-to-all back -> unpermute.  Stream-
// ordered; the host waits only where the local phase itself needs a count
// (growth / contraction enabled).
hive_status shard_call(hive_table_s* h, int kind, const uint8_t* d_op, const uint32_t* d_keys,
                       const uint32_t* d_vals, uint64_t n, uint32_t* out32, uint8_t* out8, cudaStream_t s) {
    auto& S = h->sh;
    if (n > S.batch_max) {
        g_err = "sharded call: n exceeds shard_batch_max";
        return HIVE_EINVAL;
    }
    const uint32_t G = (uint32_t)S.nranks;
    const uint64_t cap = S.cap, tot = S.tot;
    const bool mixed = kind == SK_MIXED, vals32 = kind == SK_FIND || kind == SK_MIXED;
    // source-side owner election (HIVE_SHARD_DEDUP): route one op per (key, opcode)
    const bool src_dedup = (h->cfg.flags & HIVE_SHARD_DEDUP) && n;
    if (src_dedup) {
        if (!S.sbase) {
            const uint64_t tabn = pow2_at_least(std::max<uint64_t>(1024, 2 * S.batch_max));
            const uint64_t a = tabn * 8, b = (S.batch_max + 255) / 256 * 256, c = (S.batch_max * 4 + 255) / 256 * 256;
            cudaError_t e = cudaMalloc(&S.sbase, a + b + 2 * c + 256);
            if (e != cudaSuccess) { set_err(e, "cudaMalloc(source election)", __LINE__); return HIVE_ENOMEM; }
            char* q = (char*)S.sbase;
            S.stab = (uint64_t*)q;
            S.smask = tabn - 1;
            S.sflag = (uint8_t*)(q + a);
            S.sowner = (uint32_t*)(q + a + b);
            S.slist = (uint32_t*)(q + a + b + c);
            S.snlist = (unsigned long long*)(q + a + b + 2 * c);
        }
        Prof p(h, "k_src_elect", s, 2);
        static const uint8_t kind_op[4] = {1, 0, 2, 0};            // SK_INSERT, SK_FIND, SK_ERASE, (mixed: opcodes)
        CK(launch_src_elect(s, mixed ? d_op : nullptr, kind_op[kind], d_keys, n, S.stab, S.smask, S.sflag, S.sowner,
                            S.slist, S.snlist, h->ctrl));
    }
    {
        Prof p(h, "k_route_pad", s, 3);
        if (n) {
            CK(launch_route_pad(s, G, HIVE_SHARD_SEED, d_keys, kind == SK_INSERT || mixed ? d_vals : nullptr,
                                mixed ? d_op : nullptr, n, cap, S.pcnt, S.pinfo, S.send_kv,
                                mixed ? S.send_op : nullptr, S.pos, S.cnt_send, h->ctrl,
                                src_dedup ? S.slist : nullptr, src_dedup ? (const uint64_t*)S.snlist : nullptr));
        } else {
            CK(cudaMemsetAsync(S.cnt_send, 0, G * sizeof(uint64_t), s));
        }
    }
    {
        Prof p(h, "nccl_alltoall(fwd)", s, 0);
        // the counts collective in its own call, then one group of point-to-point
        // transfers for the records (and opcodes) to the peers
        CKS(a2a(h, S.cnt_send, S.cnt_recv, 1, NCCL_U64, 8, s));
        CKN(g_nccl.group_start());
        hive_status st = a2a(h, S.send_kv, S.recv_kv, cap, NCCL_U64, 8, s, true);
        if (st == HIVE_OK && mixed) st = a2a(h, S.send_op, S.recv_op, cap, NCCL_U8, 1, s, true);
        CKN(g_nccl.group_end());
        CKS(st);
    }
    {
        Prof p(h, "k_owner_compact", s);
        CK(launch_owner_compact(s, G, cap, S.recv_kv, mixed ? S.recv_op : nullptr, S.cnt_recv, S.kc, S.vc,
                                mixed ? S.oc : nullptr, S.back, S.n_dev, (uint32_t)S.rank, S.send_kv,
                                mixed ? S.send_op : nullptr));
    }
    CKS(owner_phase(h, kind, S.oc, S.kc, S.vc, tot, S.n_dev, S.r8c, S.r32c, s));
    {
        Prof p(h, "k_owner_return", s);
        CK(launch_owner_return(s, tot, S.n_dev, S.back, S.r8c, vals32 ? S.r32c : nullptr, S.ret8,
                               vals32 ? S.ret32 : nullptr));
    }
    {
        Prof p(h, "nccl_alltoall(back)", s, 0);
        CKN(g_nccl.group_start());
        hive_status st = a2a(h, S.ret8, S.rr8, cap, NCCL_U8, 1, s, true);
        if (st == HIVE_OK && vals32) st = a2a(h, S.ret32, S.rr32, cap, NCCL_U32, 4, s, true);
        CKN(g_nccl.group_end());
        CKS(st);
    }
    if (n && (out8 || out32)) {
        // the own region's results stayed in ret8 / ret32: place them where the
        // unpermute reads (a device copy of one region, not an NCCL transfer)
        const uint64_t off = (uint64_t)S.rank * cap;
        CK(cudaMemcpyAsync(S.rr8 + off, S.ret8 + off, cap, cudaMemcpyDeviceToDevice, s));
        if (vals32) CK(cudaMemcpyAsync(S.rr32 + off, S.ret32 + off, cap * 4, cudaMemcpyDeviceToDevice, s));
        Prof p(h, "k_unroute_pad", s, src_dedup ? 2 : 1);
        CK(launch_unroute_pad(s, S.pos, n, S.rr8, out8, out32 ? S.rr32 : nullptr, out32,
                              kind == SK_FIND ? 2 : 4, nullptr, src_dedup ? S.slist : nullptr,
                              src_dedup ? (const uint64_t*)S.snlist : nullptr));
        if (src_dedup) CK(launch_src_copy(s, n, S.sflag, S.sowner, out8, out32));
    }
    return HIVE_OK;
}

}  // namespace

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

void hive_config_default(hive_config* c) {
    if (!c) return;
    c->capacity = 1024ull * SLOTS;
    c->max_capacity = 0;
    c->lf_grow = 0.90f;
    c->lf_shrink = 0.25f;
    c->max_evictions = 16;
    c->resize_k = 1024;
    c->stash_fraction = 0.02f;
    c->flags = 0;
    c->nccl_comm = nullptr;
    c->shard_batch_max = 0;
    c->shard_slack = 0.0625f;
}

const char* hive_status_string(hive_status s) {
    switch (s) {
        case HIVE_OK: return "ok";
        case HIVE_EINVAL: return "invalid argument";
        case HIVE_ENOMEM: return "out of memory";
        case HIVE_ECUDA: return "CUDA error";
        case HIVE_ENCCL: return "NCCL error";
        case HIVE_ESTASHFULL: return "stash full (entries lost)";
        case HIVE_EBUSY: return "handle busy";
        case HIVE_EXCHANGE: return "sharded exchange region full (ops not processed)";
    }
    return "unknown";
}

const char* hive_last_error(void) { return g_err.c_str(); }

hive_status hive_create(const hive_config* cfg, void* stream, hive_t* out) {
    if (!cfg || !out || cfg->capacity == 0 || cfg->stash_fraction < 0.0f) return HIVE_EINVAL;
    if (cfg->lf_grow < 1.0f && cfg->lf_shrink > 0.0f && cfg->lf_shrink >= cfg->lf_grow) return HIVE_EINVAL;
    if (cfg->lf_grow <= 0.0f) return HIVE_EINVAL;
    if (cfg->flags & ~(HIVE_KEYS_UNIQUE | HIVE_HASH_CRC | HIVE_SHARD_DEDUP)) return HIVE_EINVAL;
    if ((cfg->flags & HIVE_SHARD_DEDUP) && (!cfg->nccl_comm || cfg->shard_batch_max >= (1ull << 30)))
        return HIVE_EINVAL;
    if (cfg->nccl_comm && (cfg->shard_batch_max == 0 || cfg->shard_slack < 0.0f)) return HIVE_EINVAL;
    *out = nullptr;
    if (!load_vmm(g_vmm)) return HIVE_ECUDA;
    cudaStream_t s = (cudaStream_t)stream;
    auto* h = new hive_table_s();
    h->cfg = *cfg;
    if (!h->cfg.max_evictions) h->cfg.max_evictions = 16;
    if (!h->cfg.resize_k) h->cfg.resize_k = 1024;
    auto fail = [&](hive_status st) { hive_destroy(h); return st; };
    if (cudaGetDevice(&h->dev) != cudaSuccess) return fail(HIVE_ECUDA);
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->dev);
    h->grids = query_grids(h->num_sms);
    if (!ensure_hash_tables()) return fail(HIVE_ECUDA);

    // A-20: any n_b >= 2, held as (m = floor(log2 n_b), split = n_b - 2^m)
    const uint64_t nb = std::max<uint64_t>(2, (cfg->capacity + SLOTS - 1) / SLOTS);
    uint32_t m = 0;
    while ((2ull << m) <= nb) ++m;
    h->m = h->m0 = m;
    h->split = h->split0 = (uint32_t)(nb - (1ull << m));
    h->nb_min = nb;
    h->nb_at_drain = nb;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    uint64_t maxb = cfg->max_capacity ? (cfg->max_capacity + SLOTS - 1) / SLOTS
                                      : (uint64_t)(total_b / 2 / (SLOTS * 8));
    if (cfg->lf_grow >= 1.0f) maxb = nb;     // growth disabled: reserve exactly the table
    h->max_buckets = std::min<uint64_t>(std::max<uint64_t>(maxb, nb), 1ull << 31);

    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = h->dev;
    CUresult r = g_vmm.granularity(&h->gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS || !h->gran) { set_err_drv(r, "cuMemGetAllocationGranularity", __LINE__); return fail(HIVE_ECUDA); }
    const uint64_t max_stash = h->stash_cap_for(h->max_buckets);
    hive_status st = vrange_reserve(h, h->bk, (size_t)h->max_buckets * SLOTS * 8);
    if (st == HIVE_OK) st = vrange_reserve(h, h->rg, max_stash * sizeof(uint64_t));
    if (st == HIVE_OK) st = vrange_reserve(h, h->ix, pow2_at_least(2 * max_stash) * sizeof(uint64_t));
    if (st == HIVE_OK) st = vrange_reserve(h, h->dr, max_stash * sizeof(uint64_t));
    if (st == HIVE_OK) st = vrange_reserve(h, h->sp, (size_t)h->max_buckets * sizeof(uint64_t));
    if (st != HIVE_OK) return fail(st);
    h->va = h->bk.va;
    // growth-enabled tables start with >= 64 MiB of buckets backed (256 Ki
    // buckets) so that early splits need no driver call
    const uint64_t premap = cfg->lf_grow < 1.0f ? std::min<uint64_t>(h->max_buckets, 1ull << 18) : 0;
    st = map_buckets(h, std::max<uint64_t>(nb, premap));
    if (st != HIVE_OK) return fail(st);

    if (cudaMalloc((void**)&h->ctrl, sizeof(Ctrl)) != cudaSuccess) return fail(HIVE_ENOMEM);
    if (cudaMallocHost((void**)&h->ctrl_h, sizeof(Ctrl)) != cudaSuccess) return fail(HIVE_ENOMEM);
    if (cudaMallocHost((void**)&h->stage_h, (8 + MAX_SEGMENTS) * sizeof(uint64_t)) != cudaSuccess)
        return fail(HIVE_ENOMEM);
    if (cudaMalloc((void**)&h->pinfo, 2 * MAX_PARTS * sizeof(uint64_t)) != cudaSuccess) return fail(HIVE_ENOMEM);
    if (cudaMalloc((void**)&h->einfo, 2 * MAX_PARTS * sizeof(uint64_t)) != cudaSuccess) return fail(HIVE_ENOMEM);
    if (cudaMalloc((void**)&h->ecount, 2 * MAX_PARTS * sizeof(unsigned long long)) != cudaSuccess)
        return fail(HIVE_ENOMEM);
    if (cudaMalloc((void**)&h->aborts, MAX_SEGMENTS * sizeof(unsigned long long)) != cudaSuccess)
        return fail(HIVE_ENOMEM);
    memset(h->ctrl_h, 0, sizeof(Ctrl));
    if (cfg->nccl_comm) {                     // one shard of a hash-partitioned table
        if (!load_nccl()) return fail(HIVE_ENCCL);
        auto& S = h->sh;
        S.comm = cfg->nccl_comm;
        int r = g_nccl.comm_count(S.comm, &S.nranks);
        if (r == 0) r = g_nccl.comm_user_rank(S.comm, &S.rank);
        if (r != 0) { set_err_nccl(r, "ncclCommCount/UserRank", __LINE__); return fail(HIVE_ENCCL); }
        if (S.nranks < 1 || S.nranks > 32) return fail(HIVE_EINVAL);
        S.batch_max = cfg->shard_batch_max;
        const double per = std::ceil((double)S.batch_max / S.nranks * (1.0 + (double)cfg->shard_slack));
        S.cap = std::min<uint64_t>((uint64_t)per + 1024, S.batch_max);
        S.tot = S.cap * (uint64_t)S.nranks;
        if (S.tot >= (1ull << 32) || S.batch_max >= (1ull << 32)) return fail(HIVE_EINVAL);
        st = shard_alloc(h);
        if (st != HIVE_OK) return fail(st);
    }
    st = hive_clear(h, stream);
    if (st != HIVE_OK) return fail(st);
    if (cudaStreamSynchronize(s) != cudaSuccess) return fail(HIVE_ECUDA);
    *out = h;
    return HIVE_OK;
}

hive_status hive_clear(hive_t h, void* stream) {
    if (!h) return HIVE_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    h->m = h->m0;
    h->split = h->split0;
    CK(cudaMemsetAsync((void*)h->va, 0xFF, (size_t)h->nb_min * SLOTS * 8, s));
    CK(cudaMemsetAsync((void*)h->sp.va, 0, (size_t)h->nb_min * sizeof(uint64_t), s));
    CK(cudaMemsetAsync(h->ctrl, 0, sizeof(Ctrl), s));
    CKS(stash_reset(h, h->stash_cap_for(h->nb_min), s));
    h->grows = h->shrinks = h->merge_aborts = 0;
    h->nb_at_drain = h->nb_min;
    h->last = s;
    return HIVE_OK;
}

hive_status hive_destroy(hive_t h) {
    if (!h) return HIVE_EINVAL;
    cudaStreamSynchronize(h->last);
    cudaDeviceSynchronize();
    vrange_free(h->bk);
    vrange_free(h->rg);
    vrange_free(h->ix);
    vrange_free(h->dr);
    vrange_free(h->sp);
    void* bufs[] = {h->ctrl, h->rvals, h->ftab, h->dd, h->owner, h->flag, h->left, h->cls, h->cnt, h->pinfo, h->aborts,
                    h->erec, h->ecount, h->einfo, h->hk, h->hv, h->hst, h->fq, h->fv, h->ff};
    for (auto e : h->pipe_ev) cudaEventDestroy(e);
    if (h->ins_free) cudaEventDestroy(h->ins_free);
    if (h->find_free) cudaEventDestroy(h->find_free);
    if (h->ctrl_ev) cudaEventDestroy(h->ctrl_ev);
    if (h->up) cudaStreamDestroy(h->up);
    if (h->down) cudaStreamDestroy(h->down);
    for (void* b : bufs)
        if (b) cudaFree(b);
    if (h->sh.base) cudaFree(h->sh.base);
    if (h->sh.sbase) cudaFree(h->sh.sbase);
    if (h->ib.base) cudaFree(h->ib.base);
    if (h->ctrl_h) cudaFreeHost(h->ctrl_h);
    if (h->stage_h) cudaFreeHost(h->stage_h);
    for (auto& r : h->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : h->pool) cudaEventDestroy(e);
    delete h;
    return HIVE_OK;
}

hive_status hive_insert(hive_t h, const uint32_t* d_keys, const uint32_t* d_vals, uint64_t n,
                        uint8_t* d_status, void* stream) {
    if (!h) return HIVE_EINVAL;
    if (n == 0 && !h->sharded()) return HIVE_OK;      // sharded calls are collective even when empty
    if ((n && (!d_keys || !d_vals)) || n >= (1ull << 32)) return HIVE_EINVAL;
    BusyGuard g(h);
    if (!g.ok) return HIVE_EBUSY;
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    if (h->sharded()) return shard_call(h, SK_INSERT, nullptr, d_keys, d_vals, n, nullptr, d_status, s);
    CKS(grow_before(h, n, s));
    return insert_phase(h, d_keys, d_vals, nullptr, nullptr, n, nullptr, n, d_status, nullptr, s);
}

hive_status hive_find(hive_t h, const uint32_t* d_keys, uint64_t n, uint32_t* d_vals_out,
                      uint8_t* d_found, void* stream) {
    if (!h) return HIVE_EINVAL;
    if (n == 0 && !h->sharded()) return HIVE_OK;
    // op indices are 32-bit inside the kernels (as for insert / erase / mixed)
    if ((n && (!d_keys || !d_vals_out)) || n >= (1ull << 32)) return HIVE_EINVAL;
    BusyGuard g(h);
    if (!g.ok) return HIVE_EBUSY;
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    if (h->sharded()) return shard_call(h, SK_FIND, nullptr, d_keys, nullptr, n, d_vals_out, d_found, s);
    Prof p(h, "k_find", s);
    CK(launch_find(h->grids, s, d_keys, nullptr, n, nullptr, h->tv(), h->sv(), d_vals_out, d_found));
    return HIVE_OK;
}

hive_status hive_erase(hive_t h, const uint32_t* d_keys, uint64_t n, uint8_t* d_erased, void* stream) {
    if (!h) return HIVE_EINVAL;
    if (n == 0 && !h->sharded()) return HIVE_OK;
    if ((n && !d_keys) || n >= (1ull << 32)) return HIVE_EINVAL;
    BusyGuard g(h);
    if (!g.ok) return HIVE_EBUSY;
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    if (h->sharded()) return shard_call(h, SK_ERASE, nullptr, d_keys, nullptr, n, nullptr, d_erased, s);
    CKS(erase_phase(h, d_keys, nullptr, n, nullptr, n, d_erased, nullptr, s));
    return shrink_after(h, s);
}

hive_status hive_mixed(hive_t h, const uint8_t* d_op, const uint32_t* d_keys, const uint32_t* d_vals,
                       uint64_t n, uint32_t* d_vals_out, uint8_t* d_result, void* stream) {
    if (!h) return HIVE_EINVAL;
    if (n == 0 && !h->sharded()) return HIVE_OK;
    if (n && (!d_op || !d_keys || !d_vals || !d_vals_out || !d_result)) return HIVE_EINVAL;
    if (n >= (1ull << 32)) return HIVE_EINVAL;
    BusyGuard g(h);
    if (!g.ok) return HIVE_EBUSY;
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    if (h->sharded()) return shard_call(h, SK_MIXED, d_op, d_keys, d_vals, n, d_vals_out, d_result, s);
    return mixed_impl(h, d_op, d_keys, d_vals, n, nullptr, d_vals_out, d_result, s);
}

hive_status hive_mixed_concurrent(hive_t h, const uint8_t* d_op, const uint32_t* d_keys, const uint32_t* d_vals,
                                  uint64_t n, uint32_t* d_vals_out, uint8_t* d_result, void* stream) {
    if (!h) return HIVE_EINVAL;
    if (h->sharded()) return HIVE_EINVAL;
    if (n == 0) return HIVE_OK;
    if (!d_op || !d_keys || !d_vals || !d_vals_out || !d_result || n >= (1ull << 31)) return HIVE_EINVAL;
    BusyGuard g(h);
    if (!g.ok) return HIVE_EBUSY;
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    if (h->mono_grid == 0) h->mono_grid = mono_grid(h->num_sms);
    if (h->cfg.lf_grow < 1.0f) {             // grow for the batch's inserts (one wait, as hive_mixed)
        CK(launch_count_ops(s, d_op, n, 1, h->ecount));
        CK(cudaMemcpyAsync(h->stage_h, h->ecount, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CKS(read_ctrl(h, s));
        if (h->stage_h[0]) CKS(grow_known(h, h->ctrl_h->count, h->stage_h[0], s));
    }
    const uint64_t tab = pow2_at_least(std::max<uint64_t>(1024, 2 * n));
    CKS(ensure(h->dd, h->dd_cap, tab));
    CKS(ensure(h->flag, h->flag_cap, n));
    CKS(ensure(h->owner, h->owner_cap, n));
    CKS(ensure(h->left, h->left_cap, n));
    CK(cudaMemsetAsync(&h->ctrl->n_left, 0, 2 * sizeof(uint64_t), s));     // n_left + slow_next
    {
        Prof p(h, "k_mixed_mono", s);
        CK(launch_mixed_mono(h->mono_grid, s, d_op, d_keys, d_vals, n, h->tv(), h->sv(), h->dd, tab - 1, h->flag,
                             h->owner, h->left, h->cfg.max_evictions, d_result, d_vals_out));
    }
    return shrink_after(h, s);
}

hive_status hive_insert_host(hive_t h, const uint32_t* h_keys, const uint32_t* h_vals, uint64_t n,
                             uint8_t* h_status, void* stream) {
    if (!h) return HIVE_EINVAL;
    if (n == 0 && !h->sharded()) return HIVE_OK;
    if ((n && (!h_keys || !h_vals)) || n >= (1ull << 32)) return HIVE_EINVAL;
    BusyGuard g(h);
    if (!g.ok) return HIVE_EBUSY;
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    if (h->sharded()) {                      // stage the local batch, then the collective call
        auto& S = h->sh;
        if (n > S.batch_max) return HIVE_EINVAL;
        if (n) {
            CK(cudaMemcpyAsync(S.hk, h_keys, n * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(S.hv, h_vals, n * 4, cudaMemcpyHostToDevice, s));
        }
        CKS(shard_call(h, SK_INSERT, nullptr, S.hk, S.hv, n, nullptr, h_status ? S.ho8 : nullptr, s));
        if (n && h_status) CK(cudaMemcpyAsync(h_status, S.ho8, n, cudaMemcpyDeviceToHost, s));
        return HIVE_OK;
    }
    const uint64_t nch = (n + HOST_CHUNK - 1) / HOST_CHUNK;
    CKS(pipe_init(h, nch + 3));
    CKS(ensure(h->hk, h->hk_cap, n));
    CKS(ensure(h->hv, h->hv_cap, n));
    CKS(ensure(h->hst, h->hst_cap, n));
    cudaEvent_t* ev = h->pipe_ev.data();          // [0, nch): values ready; nch: keys ready; nch+1, nch+2
    // uploads: all keys first (the election needs the whole batch), then values by chunk
    CK(cudaStreamWaitEvent(h->up, h->ins_free, 0));
    CK(cudaMemcpyAsync(h->hk, h_keys, n * 4, cudaMemcpyHostToDevice, h->up));
    CK(cudaEventRecord(ev[nch], h->up));
    for (uint64_t off = 0, c = 0; off < n; off += HOST_CHUNK, ++c) {
        const uint64_t len = std::min(HOST_CHUNK, n - off);
        CK(cudaMemcpyAsync(h->hv + off, h_vals + off, len * 4, cudaMemcpyHostToDevice, h->up));
        CK(cudaEventRecord(ev[c], h->up));
    }
    CK(cudaStreamWaitEvent(s, ev[nch], 0));
    CKS(grow_before(h, n, s));
    InsertChunks ic{HOST_CHUNK, ev};
    CKS(insert_phase(h, h->hk, h->hv, nullptr, nullptr, n, nullptr, n, h->hst, nullptr, s, &ic));
    CK(cudaEventRecord(h->ins_free, s));
    if (h_status) {
        CK(cudaStreamWaitEvent(h->down, h->ins_free, 0));
        CK(cudaMemcpyAsync(h_status, h->hst, n, cudaMemcpyDeviceToHost, h->down));
        CK(cudaEventRecord(ev[nch + 1], h->down));
        CK(cudaStreamWaitEvent(s, ev[nch + 1], 0));
    }
    return HIVE_OK;
}

hive_status hive_find_host(hive_t h, const uint32_t* h_keys, uint64_t n, uint32_t* h_vals_out,
                           uint8_t* h_found, void* stream) {
    if (!h) return HIVE_EINVAL;
    if (n == 0 && !h->sharded()) return HIVE_OK;
    if ((n && (!h_keys || !h_vals_out)) || n >= (1ull << 32)) return HIVE_EINVAL;
    BusyGuard g(h);
    if (!g.ok) return HIVE_EBUSY;
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    if (h->sharded()) {
        auto& S = h->sh;
        if (n > S.batch_max) return HIVE_EINVAL;
        if (n) CK(cudaMemcpyAsync(S.hk, h_keys, n * 4, cudaMemcpyHostToDevice, s));
        CKS(shard_call(h, SK_FIND, nullptr, S.hk, nullptr, n, S.ho32, h_found ? S.ho8 : nullptr, s));
        if (n) CK(cudaMemcpyAsync(h_vals_out, S.ho32, n * 4, cudaMemcpyDeviceToHost, s));
        if (n && h_found) CK(cudaMemcpyAsync(h_found, S.ho8, n, cudaMemcpyDeviceToHost, s));
        return HIVE_OK;
    }
    const uint64_t nch = (n + HOST_CHUNK - 1) / HOST_CHUNK;
    CKS(pipe_init(h, 2 * nch + 1));
    CKS(ensure(h->fq, h->fq_cap, n));
    CKS(ensure(h->fv, h->fv_cap, n));
    CKS(ensure(h->ff, h->ff_cap, n));
    cudaEvent_t* ev = h->pipe_ev.data();          // [0, nch): uploaded; [nch, 2nch): probed; 2nch: done
    CK(cudaStreamWaitEvent(h->up, h->find_free, 0));
    for (uint64_t off = 0, c = 0; off < n; off += HOST_CHUNK, ++c) {
        const uint64_t len = std::min(HOST_CHUNK, n - off);
        CK(cudaMemcpyAsync(h->fq + off, h_keys + off, len * 4, cudaMemcpyHostToDevice, h->up));
        CK(cudaEventRecord(ev[c], h->up));
    }
    {
        Prof p(h, "k_find", s);
        for (uint64_t off = 0, c = 0; off < n; off += HOST_CHUNK, ++c) {
            const uint64_t len = std::min(HOST_CHUNK, n - off);
            CK(cudaStreamWaitEvent(s, ev[c], 0));
            CK(launch_find(h->grids, s, h->fq + off, nullptr, len, nullptr, h->tv(), h->sv(), h->fv + off,
                           h->ff + off));
            CK(cudaEventRecord(ev[nch + c], s));
            CK(cudaStreamWaitEvent(h->down, ev[nch + c], 0));
            CK(cudaMemcpyAsync(h_vals_out + off, h->fv + off, len * 4, cudaMemcpyDeviceToHost, h->down));
            if (h_found) CK(cudaMemcpyAsync(h_found + off, h->ff + off, len, cudaMemcpyDeviceToHost, h->down));
        }
    }
    CK(cudaEventRecord(h->find_free, s));
    CK(cudaEventRecord(ev[2 * nch], h->down));
    CK(cudaStreamWaitEvent(s, ev[2 * nch], 0));
    return HIVE_OK;
}

hive_status hive_size(hive_t h, uint64_t* out) {
    if (!h || !out) return HIVE_EINVAL;
    CKS(read_ctrl(h, h->last));
    *out = h->ctrl_h->count;
    return h->ctrl_h->failed ? HIVE_ESTASHFULL : h->ctrl_h->xfail ? HIVE_EXCHANGE : HIVE_OK;
}

hive_status hive_stats(hive_t h, hive_stats_t* o) {
    if (!h || !o) return HIVE_EINVAL;
    cudaStream_t s = h->last;
    CKS(set_ctrl_word(h, &h->ctrl->in_b1, 0, s));
    CK(launch_count_b1(h->grids.stream, s, h->tv(), h->nb(), h->ctrl));
    CKS(read_ctrl(h, s));
    const Ctrl& c = *h->ctrl_h;
    memset(o, 0, sizeof *o);
    o->n_buckets = h->nb();
    o->m = h->m;
    o->split = h->split;
    o->count = c.count;
    o->stash_used = std::min<uint64_t>(c.stash_tail, h->stash_cap);
    o->stash_cap = h->stash_cap;
    o->evictions = c.evictions;
    o->max_depth = c.max_depth;
    o->stash_pushes = c.stash_pushes;
    o->leftovers = c.leftovers;
    o->grows = h->grows;
    o->shrinks = h->shrinks;
    o->merge_aborts = h->merge_aborts;
    o->failed = c.failed;
    o->in_b1 = c.in_b1;
    o->mapped_bytes = h->bk.mapped;
    for (int i = 0; i < 8; ++i) o->alg_bytes[i] = c.abytes[i];
    o->step3 = c.step3;
    o->xfail = c.xfail;
    o->elect_overflow = c.eover;
    for (int i = 0; i < 4; ++i) o->step_cycles[i] = c.cyc[i];
    return c.failed ? HIVE_ESTASHFULL : c.xfail ? HIVE_EXCHANGE : HIVE_OK;
}

hive_status hive_dump(hive_t h, uint32_t* d_keys, uint32_t* d_vals, uint64_t cap, uint64_t* n_out,
                      void* stream) {
    if (!h || !n_out || (cap && (!d_keys || !d_vals))) return HIVE_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    CKS(set_ctrl_word(h, &h->ctrl->dump_n, 0, s));
    CK(launch_dump(h->grids.stream, s, h->tv(), h->nb(), h->sv(), d_keys, d_vals, cap));
    CKS(read_ctrl(h, s));
    *n_out = h->ctrl_h->dump_n;
    return HIVE_OK;
}

hive_status hive_load_image(hive_t h, const uint64_t* d_slots, uint64_t n_buckets, const uint64_t* d_stash,
                            uint64_t n_stash, void* stream) {
    if (!h || !d_slots || n_buckets < 2 || n_buckets > h->max_buckets || (n_stash && !d_stash)) return HIVE_EINVAL;
    if (h->sharded()) return HIVE_EINVAL;
    BusyGuard g(h);
    if (!g.ok) return HIVE_EBUSY;
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    uint32_t m = 0;
    while ((2ull << m) <= n_buckets) ++m;
    CKS(map_buckets(h, n_buckets));
    h->m = m;
    h->split = (uint32_t)(n_buckets - (1ull << m));
    const uint64_t cap = h->stash_cap_for(n_buckets);
    if (n_stash > cap) return HIVE_EINVAL;
    CK(cudaMemcpyAsync((void*)h->va, d_slots, n_buckets * SLOTS * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync((void*)h->sp.va, 0, n_buckets * sizeof(uint64_t), s));
    CK(cudaMemsetAsync(h->ctrl, 0, sizeof(Ctrl), s));
    CKS(stash_reset(h, cap, s));
    CK(launch_image(s, h->tv(), n_buckets, h->sv(), d_stash, n_stash));
    if (n_stash) h->stash_clean = false;
    // live count = occupied slots + stash entries: counted by the dump kernel
    CKS(set_ctrl_word(h, &h->ctrl->dump_n, 0, s));
    CK(launch_dump(h->grids.stream, s, h->tv(), n_buckets, h->sv(), nullptr, nullptr, 0));
    CKS(read_ctrl(h, s));
    h->stage_h[2] = h->ctrl_h->dump_n;      // two staging words: both copies are in flight together
    h->stage_h[3] = n_stash;
    CK(cudaMemcpyAsync(&h->ctrl->count, h->stage_h + 2, sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(&h->ctrl->stash_tail, h->stage_h + 3, sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    h->tail_known = n_stash;
    h->nb_at_drain = n_buckets;
    h->grows = h->shrinks = h->merge_aborts = 0;
    return HIVE_OK;
}

hive_status hive_profile(hive_t h, int enable) {
    if (!h) return HIVE_EINVAL;
    h->prof = enable != 0;
    h->step_prof = enable >= 2;
    return HIVE_OK;
}

int hive_profile_read(hive_t h, const char** names, double* ms, uint64_t* launches, int max, int reset) {
    if (!h) return -1;
    for (auto& r : h->recs) {
        float t = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&t, r.a, r.b);
        bool hit = false;
        for (auto& a : h->agg)
            if (strcmp(a.name, r.name) == 0) { a.ms += t; a.n += r.launches; hit = true; break; }
        if (!hit) h->agg.push_back({r.name, (double)t, r.launches});
        h->pool.push_back(r.a);
        h->pool.push_back(r.b);
    }
    h->recs.clear();
    int k = 0;
    for (auto& a : h->agg) {
        if (k < max) {
            if (names) names[k] = a.name;
            if (ms) ms[k] = a.ms;
            if (launches) launches[k] = a.n;
        }
        ++k;
    }
    if (reset) h->agg.clear();
    return k;
}

// Scratch of the stateless routing calls, kept per (device, stream) for the
// life of the process: allocator calls cost 5-95 ms on this system, and two
// streams of one device must not share the count / info words (their launches
// may run concurrently).  The map is guarded by a mutex; a stream's scratch is
// only ever used by launches on that stream, which execute in order.
struct RouteScratch { uint64_t* cnt = nullptr; uint64_t cap = 0; uint64_t* info = nullptr; };
static hive_status route_scratch(cudaStream_t s, RouteScratch** out) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, cudaStream_t>, RouteScratch*>> tab;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    for (auto& e : tab)
        if (e.first.first == dev && e.first.second == s) { *out = e.second; return HIVE_OK; }
    auto* rs = new RouteScratch();
    tab.push_back({{dev, s}, rs});
    *out = rs;
    return HIVE_OK;
}

static hive_status route_impl(int mode, uint32_t n_shards, uint32_t seed, const uint32_t* d_keys,
                              const uint32_t* d_vals, const uint8_t* d_ops, uint64_t n, uint64_t* d_send_kv,
                              uint8_t* d_send_ops, uint32_t* d_pos, uint64_t* d_counts, void* stream) {
    if (n_shards == 0 || n_shards > (uint32_t)MAX_PARTS || !d_counts) return HIVE_EINVAL;
    if (n >= (1ull << 32)) return HIVE_EINVAL;
    if (n && (!d_keys || !d_send_kv || !d_pos || (d_send_ops && !d_ops))) return HIVE_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    RouteScratch* rsp = nullptr;
    CKS(route_scratch(s, &rsp));
    RouteScratch& rs = *rsp;
    const uint64_t E = (uint64_t)n_shards * part_warps(n) + 1;
    CKS(ensure(rs.cnt, rs.cap, E));
    if (!rs.info) CK(cudaMalloc((void**)&rs.info, 2 * MAX_PARTS * sizeof(uint64_t)));
    CK(launch_partition(s, mode, n_shards, seed, d_keys, d_vals, d_ops, n, rs.cnt, rs.info, d_send_kv, d_send_ops,
                        d_pos));
    CK(cudaMemcpyAsync(d_counts, rs.info, n_shards * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    return HIVE_OK;
}

hive_status hive_route(uint32_t n_shards, uint32_t seed, const uint32_t* d_keys, const uint32_t* d_vals,
                       const uint8_t* d_ops, uint64_t n, uint64_t* d_send_kv, uint8_t* d_send_ops,
                       uint32_t* d_pos, uint64_t* d_counts, void* stream) {
    return route_impl(PART_ROUTE, n_shards, seed, d_keys, d_vals, d_ops, n, d_send_kv, d_send_ops, d_pos,
                      d_counts, stream);
}

hive_status hive_route_keys(uint32_t n_shards, uint32_t seed, const uint32_t* d_keys, uint64_t n,
                            uint32_t* d_send_keys, uint32_t* d_pos, uint64_t* d_counts, void* stream) {
    return route_impl(PART_ROUTE_KEYS, n_shards, seed, d_keys, nullptr, nullptr, n, (uint64_t*)d_send_keys,
                      nullptr, d_pos, d_counts, stream);
}

hive_status hive_unroute(const uint32_t* d_pos, uint64_t n, const uint8_t* d_in8, uint8_t* d_out8,
                         const uint32_t* d_in32, uint32_t* d_out32, void* stream) {
    if (n == 0) return HIVE_OK;
    if (!d_pos || ((d_out8 != nullptr) != (d_in8 != nullptr)) || ((d_out32 != nullptr) != (d_in32 != nullptr)))
        return HIVE_EINVAL;
    CK(launch_unroute((cudaStream_t)stream, d_pos, n, d_in8, d_out8, d_in32, d_out32));
    return HIVE_OK;
}

// ---- NEXT-1 peer-memory exchange ------------------------------------------------------
static bool fill_peers(PeerDest& pd, uint32_t n, uint64_t region, uint32_t rank) {
    if (n == 0 || n > (uint32_t)MAX_PEERS || rank >= n || region == 0) return false;
    if ((uint64_t)n * region > (1ull << 32)) return false;     // pos_out is 32-bit
    pd = PeerDest{};
    pd.region = region;
    pd.rank = rank;
    return true;
}

hive_status hive_route_p2p(uint32_t n_shards, uint32_t rank, uint32_t seed, const uint32_t* d_keys,
                           const uint32_t* d_vals, const uint8_t* d_ops, uint64_t n, uint64_t region,
                           uint64_t* const* peer_kv, uint8_t* const* peer_ops, uint64_t* const* peer_cnt,
                           uint32_t* d_pos, uint64_t* d_counts, void* stream) {
    PeerDest pd;
    if (!fill_peers(pd, n_shards, region, rank) || !peer_kv || !peer_cnt || !d_counts) return HIVE_EINVAL;
    if (n && (!d_keys || !d_pos)) return HIVE_EINVAL;
    for (uint32_t p = 0; p < n_shards; ++p) {
        if (!peer_kv[p] || !peer_cnt[p] || (d_ops && (!peer_ops || !peer_ops[p]))) return HIVE_EINVAL;
        pd.kv[p] = peer_kv[p];
        pd.ops[p] = d_ops ? peer_ops[p] : nullptr;
        pd.cnt[p] = (unsigned long long*)peer_cnt[p];
    }
    cudaStream_t s = (cudaStream_t)stream;
    RouteScratch* rsp = nullptr;
    CKS(route_scratch(s, &rsp));
    RouteScratch& rs = *rsp;
    CKS(ensure(rs.cnt, rs.cap, (uint64_t)n_shards * part_warps(n) + 1));
    if (!rs.info) CK(cudaMalloc((void**)&rs.info, 2 * MAX_PARTS * sizeof(uint64_t)));
    CK(launch_route_p2p(s, n_shards, seed, d_keys, d_vals, d_ops, n, rs.cnt, rs.info, d_pos, pd));
    CK(cudaMemcpyAsync(d_counts, rs.info, n_shards * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    return HIVE_OK;
}

hive_status hive_serve_inbox(hive_t h, uint32_t kind, uint32_t n_src, uint32_t rank, uint64_t region,
                             const uint64_t* d_inbox_kv, const uint8_t* d_inbox_ops, const uint64_t* d_cnt,
                             uint32_t* const* peer_res32, uint8_t* const* peer_res8, void* stream) {
    PeerDest pd;
    if (!h || h->sharded() || kind > 3 || !fill_peers(pd, n_src, region, rank) || !d_inbox_kv || !d_cnt)
        return HIVE_EINVAL;
    static const int kinds[4] = {SK_FIND, SK_INSERT, SK_ERASE, SK_MIXED};    // API order -> internal
    const int sk = kinds[kind];
    if (sk == SK_MIXED && !d_inbox_ops) return HIVE_EINVAL;
    const bool vals32 = sk == SK_FIND || sk == SK_MIXED;
    for (uint32_t p = 0; p < n_src; ++p) {
        if (!peer_res8 || !peer_res8[p] || (vals32 && (!peer_res32 || !peer_res32[p]))) return HIVE_EINVAL;
        pd.res8[p] = peer_res8[p];
        pd.res32[p] = vals32 ? peer_res32[p] : nullptr;
    }
    BusyGuard g(h);
    if (!g.ok) return HIVE_EBUSY;
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    auto& I = h->ib;
    const uint64_t tot = (uint64_t)n_src * region;
    if (I.cap < tot) {                         // one allocation, carved (allocator calls are slow here)
        if (I.base) CK(cudaFree(I.base));
        I = hive_table_s::Inbox{};
        const uint64_t a = (tot * 4 + 255) / 256 * 256, b = (tot + 255) / 256 * 256;
        cudaError_t e = cudaMalloc(&I.base, 4 * a + 2 * b + 256);
        if (e != cudaSuccess) { set_err(e, "cudaMalloc(inbox scratch)", __LINE__); return HIVE_ENOMEM; }
        char* q = (char*)I.base;
        I.kc = (uint32_t*)q; I.vc = (uint32_t*)(q + a); I.back = (uint32_t*)(q + 2 * a);
        I.r32c = (uint32_t*)(q + 3 * a); I.oc = (uint8_t*)(q + 4 * a); I.r8c = (uint8_t*)(q + 4 * a + b);
        I.n_dev = (uint64_t*)(q + 4 * a + 2 * b);
        I.cap = tot;
    }
    {
        Prof p(h, "k_owner_compact", s);
        CK(launch_owner_compact(s, n_src, region, d_inbox_kv, sk == SK_MIXED ? d_inbox_ops : nullptr, d_cnt, I.kc,
                                I.vc, sk == SK_MIXED ? I.oc : nullptr, I.back, I.n_dev));
    }
    CKS(owner_phase(h, sk, I.oc, I.kc, I.vc, tot, I.n_dev, I.r8c, I.r32c, s));
    Prof p(h, "k_return_p2p", s);
    CK(launch_return_p2p_back(s, tot, I.n_dev, region, I.back, vals32 ? I.r32c : nullptr, I.r8c, pd));
    return HIVE_OK;
}

hive_status hive_unroute_pad(const uint32_t* d_pos, uint64_t n, const uint8_t* d_in8, uint8_t* d_out8,
                             const uint32_t* d_in32, uint32_t* d_out32, uint8_t miss8, const uint64_t* d_poison,
                             void* stream) {
    if (n == 0) return HIVE_OK;
    if (!d_pos || ((d_out8 != nullptr) != (d_in8 != nullptr)) || ((d_out32 != nullptr) != (d_in32 != nullptr)))
        return HIVE_EINVAL;
    CK(launch_unroute_pad((cudaStream_t)stream, d_pos, n, d_in8, d_out8, d_in32, d_out32, miss8,
                          (const unsigned long long*)d_poison));
    return HIVE_OK;
}

hive_status hive_inbox_compact(uint32_t n_src, uint64_t region, const uint64_t* d_inbox_kv,
                               const uint8_t* d_inbox_ops, const uint64_t* d_cnt, uint64_t n_total,
                               uint32_t* d_keys, uint32_t* d_vals, uint8_t* d_ops, void* stream) {
    if (n_src == 0 || n_src > (uint32_t)MAX_PEERS || !d_cnt) return HIVE_EINVAL;
    if (n_total && (!d_inbox_kv || !d_keys || !d_vals || region == 0 || n_total > (uint64_t)n_src * region ||
                    ((d_ops != nullptr) != (d_inbox_ops != nullptr))))
        return HIVE_EINVAL;
    CK(launch_inbox_compact((cudaStream_t)stream, n_src, region, d_inbox_kv, d_inbox_ops, d_cnt, n_total, d_keys,
                            d_vals, d_ops));
    return HIVE_OK;
}

hive_status hive_return_p2p(uint32_t n_src, uint32_t rank, uint64_t region, const uint64_t* d_cnt,
                            uint64_t n_total, const uint32_t* d_res32, const uint8_t* d_res8,
                            uint32_t* const* peer_res32, uint8_t* const* peer_res8, void* stream) {
    PeerDest pd;
    if (!fill_peers(pd, n_src, region, rank) || !d_cnt || n_total > (uint64_t)n_src * region) return HIVE_EINVAL;
    for (uint32_t p = 0; p < n_src; ++p) {
        if ((d_res32 && (!peer_res32 || !peer_res32[p])) || (d_res8 && (!peer_res8 || !peer_res8[p])))
            return HIVE_EINVAL;
        pd.res32[p] = d_res32 ? peer_res32[p] : nullptr;
        pd.res8[p] = d_res8 ? peer_res8[p] : nullptr;
    }
    CK(launch_return_p2p((cudaStream_t)stream, n_src, d_cnt, n_total, d_res32, d_res8, pd));
    return HIVE_OK;
}

hive_status hive_p2p_signal(uint32_t n, uint32_t rank, uint32_t phase, uint64_t epoch,
                            uint64_t* const* peer_sig, void* stream) {
    PeerDest pd;
    if (!fill_peers(pd, n, 1, rank) || phase > 1 || !peer_sig) return HIVE_EINVAL;
    for (uint32_t p = 0; p < n; ++p) {
        if (!peer_sig[p]) return HIVE_EINVAL;
        pd.sig[p] = (unsigned long long*)peer_sig[p];
    }
    CK(launch_p2p_signal((cudaStream_t)stream, n, phase, epoch, pd));
    return HIVE_OK;
}

hive_status hive_p2p_wait(uint32_t n, uint32_t phase, uint64_t epoch, uint64_t* d_sig, uint64_t timeout_ns,
                          void* stream) {
    if (n == 0 || n > (uint32_t)MAX_PEERS || phase > 1 || !d_sig) return HIVE_EINVAL;
    CK(launch_p2p_wait((cudaStream_t)stream, n, phase, epoch, (unsigned long long*)d_sig, timeout_ns));
    return HIVE_OK;
}

hive_status hive_dev_alloc(uint64_t bytes, void** d_out) {
    if (!d_out || bytes == 0) return HIVE_EINVAL;
    *d_out = nullptr;
    cudaError_t e = cudaMalloc(d_out, bytes);
    if (e != cudaSuccess) { set_err(e, "cudaMalloc", __LINE__); return HIVE_ENOMEM; }
    return HIVE_OK;
}

hive_status hive_dev_free(void* d_ptr) {
    if (d_ptr) CK(cudaFree(d_ptr));
    return HIVE_OK;
}

hive_status hive_ipc_handle(const void* d_ptr, uint8_t* handle_out) {
    if (!d_ptr || !handle_out) return HIVE_EINVAL;
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    memcpy(handle_out, &h, sizeof(h));
    return HIVE_OK;
}

hive_status hive_ipc_open(const uint8_t* handle, void** d_out) {
    if (!handle || !d_out) return HIVE_EINVAL;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    CK(cudaIpcOpenMemHandle(d_out, h, cudaIpcMemLazyEnablePeerAccess));
    return HIVE_OK;
}

hive_status hive_ipc_close(void* d_ptr) {
    if (d_ptr) CK(cudaIpcCloseMemHandle(d_ptr));
    return HIVE_OK;
}

hive_status hive_hash(uint32_t fn, const uint32_t* d_keys, uint64_t n, uint32_t* d_out, void* stream) {
    if (fn > HIVE_FN_CRC64) return HIVE_EINVAL;
    if (n == 0) return HIVE_OK;
    if (!d_keys || !d_out) return HIVE_EINVAL;
    if (!ensure_hash_tables()) return HIVE_ECUDA;
    CK(launch_hash((cudaStream_t)stream, fn, d_keys, n, d_out, nullptr, 1));
    return HIVE_OK;
}

hive_status hive_gather_ceiling(const uint64_t* d_blocks, uint64_t n_blocks, const uint32_t* d_keys,
                                uint64_t n, uint32_t* d_out, void* stream) {
    return hive_gather_ceiling_rw((uint64_t*)d_blocks, n_blocks, d_keys, n, d_out, 0, stream);
}

hive_status hive_gather_ceiling_rw(uint64_t* d_blocks, uint64_t n_blocks, const uint32_t* d_keys, uint64_t n,
                                   uint32_t* d_out, uint32_t mode, void* stream) {
    if (mode > 2) return HIVE_EINVAL;
    if (n == 0) return HIVE_OK;
    if (!d_blocks || !d_keys || !d_out || n_blocks == 0 || n_blocks > (1ull << 32)) return HIVE_EINVAL;
    if ((uintptr_t)d_blocks % 256) return HIVE_EINVAL;
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    static thread_local int grid_dev = -1;
    static thread_local Grids gr{};
    if (grid_dev != dev) {
        gr = query_grids(sms);
        grid_dev = dev;
    }
    CK(launch_gather(gr, (cudaStream_t)stream, d_keys, n, d_blocks, n_blocks, d_out, mode));
    return HIVE_OK;
}

hive_status hive_collisions(uint32_t fn, const uint32_t* d_keys, uint64_t n, uint64_t m,
                            uint64_t* y_out, void* stream) {
    if (fn > HIVE_FN_CRC64 || m == 0 || m > (1ull << 32) || !y_out) return HIVE_EINVAL;
    if (n && !d_keys) return HIVE_EINVAL;
    if (!ensure_hash_tables()) return HIVE_ECUDA;
    cudaStream_t s = (cudaStream_t)stream;
    const uint64_t words = (m + 31) / 32;
    void* buf = nullptr;
    CK(cudaMallocAsync(&buf, words * 4 + 8, s));
    uint32_t* bins = (uint32_t*)((char*)buf + 8);
    unsigned long long* total = (unsigned long long*)buf;
    unsigned long long nonempty = 0;
    cudaError_t e = cudaMemsetAsync(buf, 0, words * 4 + 8, s);
    if (e == cudaSuccess && n) e = launch_hash(s, fn, d_keys, n, nullptr, bins, m);
    if (e == cudaSuccess) e = launch_popc(s, bins, words, total);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&nonempty, total, 8, cudaMemcpyDeviceToHost, s);
    cudaError_t e2 = cudaFreeAsync(buf, s);
    if (e == cudaSuccess) e = e2;
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { set_err(e, "hive_collisions", __LINE__); return HIVE_ECUDA; }
    *y_out = n - nonempty;      // sum_b (L_b - 1)_+ = n - #non-empty bins
    return HIVE_OK;
}

hive_status hive_nccl_unique_id(uint8_t* id_out) {
    if (!id_out) return HIVE_EINVAL;
    if (!load_nccl()) return HIVE_ENCCL;
    NcclUniqueId id;
    CKN(g_nccl.get_unique_id(&id));
    memcpy(id_out, id.internal, sizeof id.internal);
    return HIVE_OK;
}

hive_status hive_nccl_comm_init(int nranks, int rank, const uint8_t* id, void** comm_out) {
    if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return HIVE_EINVAL;
    if (!load_nccl()) return HIVE_ENCCL;
    NcclUniqueId uid;
    memcpy(uid.internal, id, sizeof uid.internal);
    *comm_out = nullptr;
    CKN(g_nccl.comm_init_rank(comm_out, nranks, uid, rank));
    return HIVE_OK;
}

hive_status hive_nccl_comm_destroy(void* comm) {
    if (!comm) return HIVE_OK;
    if (!load_nccl()) return HIVE_ENCCL;
    CKN(g_nccl.comm_destroy(comm));
    return HIVE_OK;
}

hive_status hive_shard_info(hive_t h, int* nranks, int* rank, uint64_t* cap_per_peer) {
    if (!h) return HIVE_EINVAL;
    if (nranks) *nranks = h->sh.nranks;
    if (rank) *rank = h->sh.rank;
    if (cap_per_peer) *cap_per_peer = h->sh.cap;
    return HIVE_OK;
}

hive_status hive_unpack_kv(const uint64_t* d_kv, uint64_t n, uint32_t* d_keys, uint32_t* d_vals,
                           void* stream) {
    if (n == 0) return HIVE_OK;
    if (!d_kv) return HIVE_EINVAL;
    CK(launch_unpack((cudaStream_t)stream, d_kv, n, d_keys, d_vals));
    return HIVE_OK;
}

}  // extern "C"
