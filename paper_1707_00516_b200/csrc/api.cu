// C ABI entry points (include/fastid_b200.h): argument checks, formulation
// dispatch, the top-k workspace protocol and the synchronous host-buffer
// drop-in behind fastid_run_kernel.
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace fastid {

namespace {
thread_local std::string g_error;
}

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_error = buf;
}

const char* get_error() { return g_error.c_str(); }

namespace {
std::atomic<unsigned long long> g_launches{0};
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int num_sms() {
    static std::atomic<int> cached{0};
    int n = cached.load(std::memory_order_relaxed);
    if (!n) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cached.store(n, std::memory_order_relaxed);
    }
    return n;
}

cudaError_t ensure_dynamic_smem(const void* fn, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> set;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    int& cur = set[std::make_pair(dev, fn)];
    if (bytes <= cur) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

namespace {

int list_size_for(int k) { return k <= 8 ? 8 : (k <= 16 ? 16 : 32); }

int resolve_formulation(int formulation, int64_t bit_length) {
    formulation &= ~FASTID_OP_MASK;
    if (formulation == FASTID_AUTO) {
        return tensor_supported(bit_length, FASTID_TENSOR_F4) ? FASTID_TENSOR_F4 : FASTID_POPC;
    }
    return formulation;
}

int check_compare(const void* refs, int64_t n_refs, const void* queries, int64_t n_queries, int64_t stride,
                  int64_t bit_length, int formulation) {
    if (n_refs < 0 || n_queries < 0) FASTID_FAIL(FASTID_E_INVALID, "negative panel size");
    if (bit_length <= 0) FASTID_FAIL(FASTID_E_INVALID, "bit_length must be positive");
    if (stride < row_stride_bytes(bit_length) || stride % 16)
        FASTID_FAIL(FASTID_E_INVALID, "stride %lld is not a multiple of 16 covering %lld bits", (long long)stride,
                    (long long)bit_length);
    if ((n_refs && ((uintptr_t)refs & 15)) || (n_queries && ((uintptr_t)queries & 15)))
        FASTID_FAIL(FASTID_E_INVALID, "panel rows must be 16-byte aligned");
    const int op = formulation & FASTID_OP_MASK;
    if (op != FASTID_OP_ANDNOT && op != FASTID_OP_AND && op != FASTID_OP_XOR)
        FASTID_FAIL(FASTID_E_INVALID, "unknown operator 0x%x", op);
    formulation &= ~FASTID_OP_MASK;
    if (formulation < FASTID_AUTO || formulation > FASTID_TENSOR_F4)
        FASTID_FAIL(FASTID_E_INVALID, "unknown formulation %d", formulation);
    if (formulation >= FASTID_TENSOR_I8 && !tensor_supported(bit_length, formulation))
        FASTID_FAIL(FASTID_E_UNSUPPORTED, "formulation %d does not support bit_length %lld", formulation,
                    (long long)bit_length);
    return FASTID_OK;
}

#ifdef FASTID_EXPERIMENTS
// experiments build only (include/fastid_b200_diag.h): process-global switches
long long* g_trace = nullptr;
int g_trace_tiles = 0;
int g_debug_flags = 0;
#endif

CompareArgs make_args(const void* refs, int64_t n_refs, const void* queries, int64_t n_queries, int64_t stride,
                      int64_t bit_length) {
    CompareArgs a{};
#ifdef FASTID_EXPERIMENTS
    a.trace = g_trace;
    a.trace_tiles = g_trace_tiles;
    a.debug_flags = g_debug_flags;
#endif
    a.refs = (const uint8_t*)refs;
    a.queries = (const uint8_t*)queries;
    a.n_refs = n_refs;
    a.n_queries = n_queries;
    a.stride = stride;
    a.bit_length = bit_length;
    return a;
}

int parts_for(int formulation, int64_t n_refs, int64_t n_queries) {
    return formulation == FASTID_POPC ? popc_parts(n_refs, n_queries)
                                      : tensor_parts(n_refs, n_queries, formulation);
}

int launch(Mode mode, const CompareArgs& a, int formulation, int* n_parts, cudaStream_t stream) {
    if (formulation == FASTID_POPC) return launch_popc(mode, a, n_parts, stream);
    return launch_tensor(mode, a, formulation, n_parts, stream);
}

// ---- host-buffer context for fastid_run_kernel ------------------------------

// A small fixed pool of host threads for parallel memcpy between pinned
// staging and the caller's (pageable, possibly untouched) buffers: one
// thread's memcpy into first-touched pages runs far below PCIe rate.
class CopyPool {
  public:
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    int size() const { return (int)workers_.size(); }
    // fn(lo, hi) over [0, bytes) split in page-aligned parts across the pool
    // (the caller takes part 0); returns when every part is done
    void parallel(size_t bytes, const std::function<void(size_t, size_t)>& fn) {
        const int n = size() + 1;
        if (bytes < ((size_t)4 << 20) || n == 1) {
            fn(0, bytes);
            return;
        }
        const size_t part = ((bytes + n - 1) / n + 4095) & ~(size_t)4095;
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            bytes_ = bytes;
            part_ = part;
            pending_ = size();
            ++gen_;
        }
        cv_.notify_all();
        run_part(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }
    void copy(void* dst, const void* src, size_t bytes) {
        parallel(bytes, [&](size_t lo, size_t hi) { memcpy((char*)dst + lo, (const char*)src + lo, hi - lo); });
    }

  private:
    void run_part(int i) {
        const size_t lo = (size_t)i * part_;
        if (lo >= bytes_) return;
        const size_t hi = lo + part_ < bytes_ ? lo + part_ : bytes_;
        (*fn_)(lo, hi);
    }
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            lk.unlock();
            run_part(i + 1);
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    bool stop_ = false;
    uint64_t gen_ = 0;
    int pending_ = 0;
    const std::function<void(size_t, size_t)>* fn_ = nullptr;
    size_t bytes_ = 0, part_ = 0;
};

struct HostContext {
    int device = -1;
    cudaStream_t stream = nullptr;
    void* buf[4] = {nullptr, nullptr, nullptr, nullptr};  // staging, refs, queries, out
    size_t cap[4] = {0, 0, 0, 0};
    // chunked pipeline: pinned staging and device slots, double-buffered
    void* pin_in[2] = {nullptr, nullptr};
    void* pin_out[2] = {nullptr, nullptr};
    size_t pin_in_cap = 0, pin_out_cap = 0;
    void* dev_slot[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};  // raw, rows, out
    size_t dev_slot_cap[3] = {0, 0, 0};
    cudaEvent_t d2h_done[2] = {nullptr, nullptr};
    cudaEvent_t h2d_done[2] = {nullptr, nullptr};
    CopyPool* pool = nullptr;
    // streamed top-k (fastid_run_topk): uploads on their own stream, overlapped
    // with the comparison of the previous chunk on `stream`
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t raw_free[2] = {nullptr, nullptr};  // the comparison stream has consumed raw slot i
    void* tk[4] = {nullptr, nullptr, nullptr, nullptr};  // aligned rows, tensor image, workspace, candidates
    size_t tk_cap[4] = {0, 0, 0, 0};

    ~HostContext() {
        for (void* p : buf)
            if (p) cudaFree(p);
        for (int i = 0; i < 2; ++i) {
            if (pin_in[i]) cudaFreeHost(pin_in[i]);
            if (pin_out[i]) cudaFreeHost(pin_out[i]);
            for (void* p : dev_slot[i])
                if (p) cudaFree(p);
            if (d2h_done[i]) cudaEventDestroy(d2h_done[i]);
            if (h2d_done[i]) cudaEventDestroy(h2d_done[i]);
        }
        delete pool;
        for (int i = 0; i < 2; ++i)
            if (raw_free[i]) cudaEventDestroy(raw_free[i]);
        for (void* p : tk)
            if (p) cudaFree(p);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (stream) cudaStreamDestroy(stream);
    }
    // both streams idle: nothing in flight still reads or writes a buffer about to be freed
    void quiesce() {
        if (copy_stream) cudaStreamSynchronize(copy_stream);
        cudaStreamSynchronize(stream);
    }
    // device buffer tk[slot] of at least `bytes` (contents not preserved)
    int ensure_tk(int slot, size_t bytes) {
        if (bytes <= tk_cap[slot]) return FASTID_OK;
        quiesce();
        if (tk[slot]) cudaFree(tk[slot]);
        tk[slot] = nullptr;
        tk_cap[slot] = 0;
        if (cudaMalloc(&tk[slot], bytes) != cudaSuccess) {
            cudaGetLastError();
            FASTID_FAIL(FASTID_E_NOMEM, "cudaMalloc of %zu bytes failed", bytes);
        }
        tk_cap[slot] = bytes;
        return FASTID_OK;
    }
    int ensure_pipeline(size_t in_bytes, size_t raw_bytes, size_t rows_bytes, size_t out_bytes) {
        if (!pool) {
            unsigned hc = std::thread::hardware_concurrency();
            pool = new CopyPool((int)(hc > 2 ? (hc > 16 ? 15 : hc - 1) : 1));
        }
        for (int i = 0; i < 2; ++i) {
            if (!d2h_done[i] && cudaEventCreateWithFlags(&d2h_done[i], cudaEventDisableTiming) != cudaSuccess)
                FASTID_FAIL(FASTID_E_CUDA, "cudaEventCreate failed");
            if (!h2d_done[i] && cudaEventCreateWithFlags(&h2d_done[i], cudaEventDisableTiming) != cudaSuccess)
                FASTID_FAIL(FASTID_E_CUDA, "cudaEventCreate failed");
        }
        // A failed allocation leaves both slots of that buffer freed and its
        // capacity 0, so a later call reallocates instead of using a null slot.
        auto grow_pinned = [&](void** slots, size_t& cap, size_t bytes) -> int {
            if (bytes <= cap) return FASTID_OK;
            quiesce();
            for (int i = 0; i < 2; ++i) {
                if (slots[i]) cudaFreeHost(slots[i]);
                slots[i] = nullptr;
            }
            cap = 0;
            for (int i = 0; i < 2; ++i) {
                if (cudaMallocHost(&slots[i], bytes) != cudaSuccess) {
                    cudaGetLastError();
                    for (int j = 0; j < 2; ++j) {
                        if (slots[j]) cudaFreeHost(slots[j]);
                        slots[j] = nullptr;
                    }
                    FASTID_FAIL(FASTID_E_NOMEM, "cudaMallocHost of %zu bytes failed", bytes);
                }
            }
            cap = bytes;
            return FASTID_OK;
        };
        if (int rc = grow_pinned(pin_in, pin_in_cap, in_bytes)) return rc;
        if (int rc = grow_pinned(pin_out, pin_out_cap, out_bytes)) return rc;
        const size_t want[3] = {raw_bytes, rows_bytes, out_bytes};
        for (int j = 0; j < 3; ++j) {
            if (want[j] <= dev_slot_cap[j]) continue;
            quiesce();
            for (int i = 0; i < 2; ++i) {
                if (dev_slot[i][j]) cudaFree(dev_slot[i][j]);
                dev_slot[i][j] = nullptr;
            }
            dev_slot_cap[j] = 0;
            for (int i = 0; i < 2; ++i) {
                if (cudaMalloc(&dev_slot[i][j], want[j]) != cudaSuccess) {
                    cudaGetLastError();
                    for (int m = 0; m < 2; ++m) {
                        if (dev_slot[m][j]) cudaFree(dev_slot[m][j]);
                        dev_slot[m][j] = nullptr;
                    }
                    FASTID_FAIL(FASTID_E_NOMEM, "cudaMalloc of %zu bytes failed", want[j]);
                }
            }
            dev_slot_cap[j] = want[j];
        }
        return FASTID_OK;
    }
    int ensure(int slot, size_t bytes) {
        if (bytes <= cap[slot]) return FASTID_OK;
        quiesce();
        if (buf[slot]) cudaFree(buf[slot]);
        buf[slot] = nullptr;
        cap[slot] = 0;
        if (cudaMalloc(&buf[slot], bytes) != cudaSuccess) {
            cudaGetLastError();
            FASTID_FAIL(FASTID_E_NOMEM, "cudaMalloc of %zu bytes failed", bytes);
        }
        cap[slot] = bytes;
        return FASTID_OK;
    }
};

thread_local HostContext* g_host_ctx = nullptr;
constexpr size_t kPipelineMinBytes = (size_t)64 << 20;  // outputs above this stream through the chunk pipeline
constexpr size_t kChunkOutBytes = (size_t)64 << 20;     // u32 output bytes per chunk

int host_context(HostContext** out) {
    int dev = 0;
    FASTID_CUDA(cudaGetDevice(&dev));
    if (g_host_ctx && g_host_ctx->device != dev) {
        delete g_host_ctx;
        g_host_ctx = nullptr;
    }
    if (!g_host_ctx) {
        auto* c = new HostContext();
        c->device = dev;
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete c;
            FASTID_FAIL(FASTID_E_CUDA, "cudaStreamCreate failed");
        }
        g_host_ctx = c;
    }
    *out = g_host_ctx;
    return FASTID_OK;
}

__global__ void transpose_words_kernel(const uint8_t* __restrict__ src, int64_t n_words, int64_t n_cols,
                                       int word_bytes, uint8_t* __restrict__ dst, int64_t dst_stride) {
    // src is (n_words, n_cols) words; dst row c gets word w of column c.
    const int64_t lanes_per_row = dst_stride / 4;
    const int64_t total = n_cols * lanes_per_row;
    const int64_t used = n_words * word_bytes / 4;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / lanes_per_row;
        const int64_t l = t - c * lanes_per_row;
        uint32_t v = 0;
        if (l < used) {
            const int64_t w = l * 4 / word_bytes;
            const int64_t part = (l * 4) % word_bytes;
            v = *reinterpret_cast<const uint32_t*>(src + (w * n_cols + c) * word_bytes + part);
        }
        reinterpret_cast<uint32_t*>(dst + c * dst_stride)[l] = v;
    }
}

}  // namespace
}  // namespace fastid

using namespace fastid;

extern "C" int fastid_abi_version(void) { return FASTID_ABI_VERSION; }

extern "C" unsigned long long fastid_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

#ifdef FASTID_EXPERIMENTS
// Diagnostics (experiments build only): subsequent tensor launches record, in
// CTA 0, kTrSlots clock64() stamps per tile for the first `tiles` tiles into
// `device_buf` (null = off).
extern "C" FASTID_API int fastid_debug_trace(long long* device_buf, int tiles) {
    g_trace = device_buf;
    g_trace_tiles = device_buf ? tiles : 0;
    return FASTID_OK;
}

// Diagnostics (experiments build only): timing-experiment switches for
// subsequent launches (0 = normal).
extern "C" FASTID_API int fastid_debug_flags(int flags) {
    g_debug_flags = flags;
    return FASTID_OK;
}
#endif
extern "C" const char* fastid_last_error(void) { return get_error(); }
extern "C" int64_t fastid_row_stride(int64_t bit_length) { return bit_length > 0 ? row_stride_bytes(bit_length) : 0; }
extern "C" int fastid_max_k(void) { return kMaxTopK; }
extern "C" int fastid_supports(int formulation, int64_t bit_length) {
    if (bit_length <= 0) return 0;
    const int op = formulation & FASTID_OP_MASK;
    if (op != FASTID_OP_ANDNOT && op != FASTID_OP_AND && op != FASTID_OP_XOR) return 0;
    formulation &= ~FASTID_OP_MASK;
    if (formulation == FASTID_AUTO || formulation == FASTID_POPC) return 1;
    return tensor_supported(bit_length, formulation) ? 1 : 0;
}

namespace {
int compare_full_impl(const void* refs, const void* image, int options, int64_t n_refs, const void* queries, int64_t n_queries,
                      int64_t stride, int64_t bit_length, uint32_t* out, int64_t ld_out, int formulation,
                      void* stream, const uint32_t* ref_popc = nullptr) {
    if (int rc = check_compare(refs, n_refs, queries, n_queries, stride, bit_length, formulation)) return rc;
    if (ld_out < n_queries) FASTID_FAIL(FASTID_E_INVALID, "ld_out smaller than n_queries");
    if (n_refs == 0 || n_queries == 0) return FASTID_OK;
    CompareArgs a = make_args(refs, n_refs, queries, n_queries, stride, bit_length);
    a.image = (const uint8_t*)image;
    a.options = options;
    a.op = formulation & FASTID_OP_MASK;
    a.ref_popc = ref_popc;
    a.out = out;
    a.ld_out = ld_out;
    int parts = 0;
    return launch(kFull, a, resolve_formulation(formulation, bit_length), &parts, (cudaStream_t)stream);
}
}  // namespace

extern "C" int fastid_compare_full(const void* refs, int64_t n_refs, const void* queries, int64_t n_queries,
                                   int64_t stride, int64_t bit_length, uint32_t* out, int64_t ld_out,
                                   int formulation, void* stream) {
    return compare_full_impl(refs, nullptr, 0, n_refs, queries, n_queries, stride, bit_length, out, ld_out, formulation,
                             stream);
}

extern "C" int fastid_topk_workspace(int64_t n_refs, int64_t n_queries, int k, int formulation, size_t* bytes) {
    if (k < 1 || k > kMaxTopK) FASTID_FAIL(FASTID_E_INVALID, "k must be in [1, %d]", kMaxTopK);
    if (!bytes) FASTID_FAIL(FASTID_E_INVALID, "bytes is NULL");
    // formulation AUTO resolves against the shape only through bit_length; the
    // workspace is sized for the larger of the two partitions.
    const int kp = list_size_for(k);
    int parts = popc_parts(n_refs, n_queries);
    for (int f = FASTID_TENSOR_I8; f <= FASTID_TENSOR_F4; ++f) {
        const int p = tensor_parts(n_refs, n_queries, f);
        if (p > parts) parts = p;
    }
    (void)formulation;
    // partial lists + one shared admission bound per unknown
    *bytes = (size_t)parts * (size_t)n_queries * (size_t)kp * (sizeof(uint32_t) + sizeof(int64_t)) +
             (size_t)(n_queries + 4) * (1 + kMinSlots) * sizeof(uint32_t) + 256;
    return FASTID_OK;
}

namespace {
int topk_partials_impl(const void* refs, const void* image, int options, int64_t n_refs, const void* queries, int64_t n_queries,
                       int64_t stride, int64_t bit_length, int k, uint32_t max_score, int64_t ref_base,
                       void* workspace, size_t workspace_bytes, int formulation, void* stream, int* n_lists,
                       int* list_len, size_t* index_offset, size_t* score_offset, const uint32_t* ref_popc = nullptr) {
    if (int rc = check_compare(refs, n_refs, queries, n_queries, stride, bit_length, formulation)) return rc;
    if (k < 1 || k > kMaxTopK) FASTID_FAIL(FASTID_E_INVALID, "k must be in [1, %d]", kMaxTopK);
    if (!n_lists || !list_len || !index_offset || !score_offset) FASTID_FAIL(FASTID_E_INVALID, "NULL out-param");
    if (n_refs == 0 || n_queries == 0) FASTID_FAIL(FASTID_E_INVALID, "empty panels have no partial lists");
    size_t need = 0;
    if (int rc = fastid_topk_workspace(n_refs, n_queries, k, formulation, &need)) return rc;
    if (workspace_bytes < need)
        FASTID_FAIL(FASTID_E_CAPACITY, "workspace of %zu bytes is smaller than the %zu required", workspace_bytes,
                    need);
    // auto, packed rows, a handful of unknowns: the CUDA-core scan reads the packed
    // rows once and beats the tensor kernels there (20M x 1024 loci, top-16:
    // 1 unknown 0.49 vs 1.56 ms, 4: 1.12 vs 1.55, 8: 2.00 vs 1.57; popc.cu)
    const int f = ((formulation & ~FASTID_OP_MASK) == FASTID_AUTO && !image && n_queries <= kScanAutoMaxQueries)
                      ? FASTID_POPC
                      : resolve_formulation(formulation, bit_length);
    const int kp = list_size_for(k);
    const int parts = parts_for(f, n_refs, n_queries);
    CompareArgs a = make_args(refs, n_refs, queries, n_queries, stride, bit_length);
    a.image = (const uint8_t*)image;
    a.options = options;
    a.op = formulation & FASTID_OP_MASK;
    a.ref_popc = ref_popc;
    a.k = k;
    a.kpad = kp;
    a.max_score = max_score;
    a.ref_base = ref_base;
    a.part_index = (int64_t*)(((uintptr_t)workspace + 15) & ~(uintptr_t)15);
    a.part_scores = (uint32_t*)(a.part_index + (size_t)parts * n_queries * kp);
    a.bound = a.part_scores + (size_t)parts * n_queries * kp;
    a.list_min = a.bound + ((n_queries + 3) & ~(int64_t)3);  // 16-B aligned rows of kMinSlots
    FASTID_CUDA(cudaMemsetAsync(a.bound, 0xFF, (size_t)(((n_queries + 3) & ~(int64_t)3) + n_queries * kMinSlots) *
                                                   sizeof(uint32_t),
                                (cudaStream_t)stream));
    int launched_parts = 0;
    if (int rc = launch(kTopK, a, f, &launched_parts, (cudaStream_t)stream)) return rc;
    if (launched_parts > parts) FASTID_FAIL(FASTID_E_INVALID, "internal: partition mismatch");
    *n_lists = launched_parts;
    *list_len = kp;
    *index_offset = (size_t)((uintptr_t)a.part_index - (uintptr_t)workspace);
    *score_offset = (size_t)((uintptr_t)a.part_scores - (uintptr_t)workspace);
    return FASTID_OK;
}
}  // namespace

extern "C" int fastid_topk_partials(const void* refs, int64_t n_refs, const void* queries, int64_t n_queries,
                                    int64_t stride, int64_t bit_length, int k, uint32_t max_score, int64_t ref_base,
                                    void* workspace, size_t workspace_bytes, int formulation, void* stream,
                                    int* n_lists, int* list_len, size_t* index_offset, size_t* score_offset) {
    return topk_partials_impl(refs, nullptr, 0, n_refs, queries, n_queries, stride, bit_length, k, max_score, ref_base,
                              workspace, workspace_bytes, formulation, stream, n_lists, list_len, index_offset,
                              score_offset);
}

extern "C" int fastid_compare_topk(const void* refs, int64_t n_refs, const void* queries, int64_t n_queries,
                                   int64_t stride, int64_t bit_length, int k, uint32_t max_score, int64_t ref_base,
                                   uint32_t* top_scores, int64_t* top_index, void* workspace,
                                   size_t workspace_bytes, int formulation, void* stream) {
    if (int rc = check_compare(refs, n_refs, queries, n_queries, stride, bit_length, formulation)) return rc;
    if (k < 1 || k > kMaxTopK) FASTID_FAIL(FASTID_E_INVALID, "k must be in [1, %d]", kMaxTopK);
    if (n_queries == 0) return FASTID_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (n_refs == 0) {
        FASTID_CUDA(cudaMemsetAsync(top_scores, 0xFF, (size_t)n_queries * k * sizeof(uint32_t), st));
        FASTID_CUDA(cudaMemsetAsync(top_index, 0xFF, (size_t)n_queries * k * sizeof(int64_t), st));
        return FASTID_OK;
    }
    int lists = 0, kp = 0;
    size_t xo = 0, so = 0;
    if (int rc = fastid_topk_partials(refs, n_refs, queries, n_queries, stride, bit_length, k, max_score, ref_base,
                                      workspace, workspace_bytes, formulation, stream, &lists, &kp, &xo, &so))
        return rc;
    return launch_merge((const uint32_t*)((uint8_t*)workspace + so), (const int64_t*)((uint8_t*)workspace + xo),
                        lists, n_queries, kp, k, top_scores, top_index, st);
}

namespace {
int threshold_impl(const void* refs, const void* image, int options, int64_t n_refs, const void* queries, int64_t n_queries,
                   int64_t stride, int64_t bit_length, uint32_t threshold, int64_t ref_base, uint32_t* hit_query,
                   int64_t* hit_ref, uint32_t* hit_score, int64_t capacity, unsigned long long* hit_count,
                   int formulation, void* stream, const uint32_t* ref_popc = nullptr) {
    if (int rc = check_compare(refs, n_refs, queries, n_queries, stride, bit_length, formulation)) return rc;
    if (capacity < 0 || !hit_count) FASTID_FAIL(FASTID_E_INVALID, "bad hit buffers");
    cudaStream_t st = (cudaStream_t)stream;
    FASTID_CUDA(cudaMemsetAsync(hit_count, 0, sizeof(unsigned long long), st));
    if (n_refs == 0 || n_queries == 0) return FASTID_OK;
    CompareArgs a = make_args(refs, n_refs, queries, n_queries, stride, bit_length);
    a.image = (const uint8_t*)image;
    a.options = options;
    a.op = formulation & FASTID_OP_MASK;
    a.ref_popc = ref_popc;
    a.threshold = threshold;
    a.ref_base = ref_base;
    a.hit_query = hit_query;
    a.hit_ref = hit_ref;
    a.hit_score = hit_score;
    a.capacity = capacity;
    a.hit_count = hit_count;
    int parts = 0;
    // auto, packed rows, a handful of unknowns: the CUDA-core scan (as for top-k)
    const int f = ((formulation & ~FASTID_OP_MASK) == FASTID_AUTO && !image && n_queries <= kScanAutoMaxQueries)
                      ? FASTID_POPC
                      : resolve_formulation(formulation, bit_length);
    return launch(kThreshold, a, f, &parts, st);
}
}  // namespace

extern "C" int fastid_compare_threshold(const void* refs, int64_t n_refs, const void* queries, int64_t n_queries,
                                        int64_t stride, int64_t bit_length, uint32_t threshold, int64_t ref_base,
                                        uint32_t* hit_query, int64_t* hit_ref, uint32_t* hit_score,
                                        int64_t capacity, unsigned long long* hit_count, int formulation,
                                        void* stream) {
    return threshold_impl(refs, nullptr, 0, n_refs, queries, n_queries, stride, bit_length, threshold, ref_base,
                          hit_query, hit_ref, hit_score, capacity, hit_count, formulation, stream);
}

// ---- prepared database --------------------------------------------------------

struct fastid_db {
    const void* refs;
    int64_t n_refs, stride, bit_length;
    int formulation;  // resolved
    void* image;      // null for the CUDA-core formulation
    size_t image_bytes;
    int device;
    int options;      // FASTID_OPT_* bits
    bool owns_image;  // false: the caller's buffer (fastid_db_create_in)
    int op = FASTID_OP_ANDNOT;        // fastid_db_set_operator
    uint32_t* ref_popc = nullptr;     // per-row popcounts (XOR on the i8 image), owned
    std::mutex popc_mu;               // guards the lazy ref_popc build (calls may come from several threads)
};

extern "C" size_t fastid_db_image_bytes(int64_t n_refs, int64_t bit_length, int formulation) {
    if (n_refs <= 0 || bit_length <= 0) return 0;
    const int f = resolve_formulation(formulation, bit_length);
    return f == FASTID_POPC ? 0 : tensor_image_bytes(n_refs, bit_length, f);
}

extern "C" int fastid_db_create(const void* refs, int64_t n_refs, int64_t stride, int64_t bit_length,
                                int formulation, void* stream, fastid_db** out) {
    if (!out) FASTID_FAIL(FASTID_E_INVALID, "out is NULL");
    *out = nullptr;
    if (int rc = check_compare(refs, n_refs, refs, 0, stride, bit_length, formulation)) return rc;
    auto* db = new fastid_db{refs, n_refs, stride, bit_length, resolve_formulation(formulation, bit_length),
                             nullptr, 0, 0, 0, true};
    db->op = formulation & FASTID_OP_MASK;
    cudaGetDevice(&db->device);
    if (db->formulation != FASTID_POPC && n_refs > 0) {
        db->image_bytes = tensor_image_bytes(n_refs, bit_length, db->formulation);
        if (cudaMalloc(&db->image, db->image_bytes) != cudaSuccess) {
            cudaGetLastError();
            const size_t want = db->image_bytes;
            delete db;
            FASTID_FAIL(FASTID_E_NOMEM, "cannot allocate the %zu-byte tensor image", want);
        }
        CompareArgs a = make_args(refs, n_refs, refs, 0, stride, bit_length);
        if (int rc = build_tensor_image(a, db->formulation, db->image, (cudaStream_t)stream)) {
            cudaFree(db->image);
            delete db;
            return rc;
        }
    }
    *out = db;
    return FASTID_OK;
}

extern "C" int fastid_db_create_in(const void* refs, int64_t n_refs, int64_t stride, int64_t bit_length,
                                   int formulation, void* image, size_t image_bytes, void* stream, fastid_db** out) {
    if (!out) FASTID_FAIL(FASTID_E_INVALID, "out is NULL");
    *out = nullptr;
    if (int rc = check_compare(refs, n_refs, refs, 0, stride, bit_length, formulation)) return rc;
    const int f = resolve_formulation(formulation, bit_length);
    const size_t need = (f == FASTID_POPC || n_refs == 0) ? 0 : tensor_image_bytes(n_refs, bit_length, f);
    if (need && (!image || image_bytes < need))
        FASTID_FAIL(FASTID_E_CAPACITY, "image buffer of %zu bytes is smaller than the %zu required", image_bytes, need);
    auto* db = new fastid_db{refs, n_refs, stride, bit_length, f, need ? image : nullptr, need, 0, 0, false};
    db->op = formulation & FASTID_OP_MASK;
    cudaGetDevice(&db->device);
    if (need) {
        CompareArgs a = make_args(refs, n_refs, refs, 0, stride, bit_length);
        if (int rc = build_tensor_image(a, f, image, (cudaStream_t)stream)) {
            delete db;
            return rc;
        }
    }
    *out = db;
    return FASTID_OK;
}

extern "C" int fastid_db_set_operator(fastid_db* db, int op) {
    if (!db) FASTID_FAIL(FASTID_E_INVALID, "db is NULL");
    if (op != FASTID_OP_ANDNOT && op != FASTID_OP_AND && op != FASTID_OP_XOR)
        FASTID_FAIL(FASTID_E_INVALID, "unknown operator 0x%x", op);
    db->op = op;
    return FASTID_OK;
}

namespace {
// XOR on the i8 image: the rows' popcounts, computed once per handle on the first XOR
// call (the mxf4 kernels fold them into the MMA, tensor.cu unpack_f4_xor)
int db_ref_popc(fastid_db* db, void* stream, const uint32_t** out) {
    *out = nullptr;
    if (db->op != FASTID_OP_XOR || db->formulation != FASTID_TENSOR_I8 || db->n_refs == 0) return FASTID_OK;
    std::lock_guard<std::mutex> lock(db->popc_mu);
    if (!db->ref_popc) {
        if (cudaMalloc(&db->ref_popc, (size_t)popcount_entries(db->n_refs) * sizeof(uint32_t)) != cudaSuccess) {
            cudaGetLastError();
            db->ref_popc = nullptr;
            FASTID_FAIL(FASTID_E_NOMEM, "cannot allocate %lld row popcounts", (long long)db->n_refs);
        }
        if (int rc = launch_row_popcount((const uint8_t*)db->refs, db->n_refs, popcount_entries(db->n_refs), db->stride,
                                         db->formulation == FASTID_TENSOR_F4, db->ref_popc, (cudaStream_t)stream))
            return rc;
        // later calls may come on other streams: the cache is complete before it is shared
        if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
            FASTID_FAIL(FASTID_E_CUDA, "row popcounts: %s", cudaGetErrorString(cudaGetLastError()));
    }
    *out = db->ref_popc;
    return FASTID_OK;
}
}  // namespace

extern "C" int fastid_db_destroy(fastid_db* db) {
    if (!db) return FASTID_OK;
    if (db->ref_popc) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(db->device);
        cudaFree(db->ref_popc);
        cudaSetDevice(cur);
    }
    if (db->image && db->owns_image) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(db->device);
        cudaFree(db->image);
        cudaSetDevice(cur);
    }
    delete db;
    return FASTID_OK;
}

extern "C" int fastid_db_formulation(const fastid_db* db) { return db ? db->formulation : -1; }

constexpr int kAllOptions =
    FASTID_OPT_NO_CTA_PAIRS | FASTID_OPT_NO_TMA_STORE | FASTID_OPT_NO_SPARE_PAIRS | FASTID_OPT_NARROW_TMA_STORE;

extern "C" int fastid_db_set_option(fastid_db* db, int option, int value) {
    if (!db) FASTID_FAIL(FASTID_E_INVALID, "db is NULL");
    if (option == 0 || (option & ~kAllOptions) || (option & (option - 1)))
        FASTID_FAIL(FASTID_E_INVALID, "unknown database option %d", option);
    db->options = value ? (db->options | option) : (db->options & ~option);
    return FASTID_OK;
}

extern "C" int fastid_db_options(const fastid_db* db) { return db ? db->options : -1; }

extern "C" int fastid_db_compare_full(const fastid_db* db, const void* queries, int64_t n_queries, uint32_t* out,
                                      int64_t ld_out, void* stream) {
    if (!db) FASTID_FAIL(FASTID_E_INVALID, "db is NULL");
    const uint32_t* pr = nullptr;
    if (int rc = db_ref_popc(const_cast<fastid_db*>(db), stream, &pr)) return rc;
    return compare_full_impl(db->refs, db->image, db->options, db->n_refs, queries, n_queries, db->stride, db->bit_length, out,
                             ld_out, db->formulation | db->op, stream, pr);
}

extern "C" int fastid_db_topk_partials(const fastid_db* db, const void* queries, int64_t n_queries, int k,
                                       uint32_t max_score, int64_t ref_base, void* workspace, size_t workspace_bytes,
                                       void* stream, int* n_lists, int* list_len, size_t* index_offset,
                                       size_t* score_offset) {
    if (!db) FASTID_FAIL(FASTID_E_INVALID, "db is NULL");
    const uint32_t* pr = nullptr;
    if (int rc = db_ref_popc(const_cast<fastid_db*>(db), stream, &pr)) return rc;
    return topk_partials_impl(db->refs, db->image, db->options, db->n_refs, queries, n_queries, db->stride, db->bit_length, k,
                              max_score, ref_base, workspace, workspace_bytes, db->formulation | db->op, stream, n_lists,
                              list_len, index_offset, score_offset, pr);
}

extern "C" int fastid_db_compare_threshold(const fastid_db* db, const void* queries, int64_t n_queries,
                                           uint32_t threshold, int64_t ref_base, uint32_t* hit_query,
                                           int64_t* hit_ref, uint32_t* hit_score, int64_t capacity,
                                           unsigned long long* hit_count, void* stream) {
    if (!db) FASTID_FAIL(FASTID_E_INVALID, "db is NULL");
    const uint32_t* pr = nullptr;
    if (int rc = db_ref_popc(const_cast<fastid_db*>(db), stream, &pr)) return rc;
    return threshold_impl(db->refs, db->image, db->options, db->n_refs, queries, n_queries, db->stride, db->bit_length, threshold,
                          ref_base, hit_query, hit_ref, hit_score, capacity, hit_count, db->formulation | db->op, stream, pr);
}

namespace {
// Host-buffer comparison: `out` (host, n_refs x n_queries u32) or, when fd >= 0,
// the same rows appended to file descriptor fd (the FIDM payload).
int run_host(const void* ref_words, int64_t n_refs, const void* query_words, int64_t n_queries, int64_t n_words,
             int word_bits, int queries_transposed, uint32_t* out, int fd, int formulation) {
    if (word_bits != 32 && word_bits != 64) FASTID_FAIL(FASTID_E_INVALID, "word_bits must be 32 or 64");
    if (n_words <= 0 || n_refs < 0 || n_queries < 0) FASTID_FAIL(FASTID_E_INVALID, "bad panel shape");
    if (n_refs == 0 || n_queries == 0) return FASTID_OK;
    HostContext* ctx = nullptr;
    if (int rc = host_context(&ctx)) return rc;
    const int wb = word_bits / 8;
    const int64_t row_bytes = n_words * wb;
    const int64_t bit_length = n_words * word_bits;
    const int64_t stride = row_stride_bytes(bit_length);
    const size_t ref_in = (size_t)n_refs * row_bytes, q_in = (size_t)n_queries * row_bytes;
    const size_t out_bytes = (size_t)n_refs * n_queries * 4;
    const bool chunked = out_bytes > kPipelineMinBytes || fd >= 0;
    if (int rc = ctx->ensure(0, chunked ? q_in : (ref_in > q_in ? ref_in : q_in))) return rc;
    if (!chunked)
        if (int rc = ctx->ensure(1, (size_t)n_refs * stride)) return rc;
    if (int rc = ctx->ensure(2, (size_t)n_queries * stride)) return rc;
    if (!chunked)
        if (int rc = ctx->ensure(3, out_bytes)) return rc;
    cudaStream_t st = ctx->stream;
    // queries first (the staging buffer is reused for the refs)
    FASTID_CUDA(cudaMemcpyAsync(ctx->buf[0], query_words, q_in, cudaMemcpyHostToDevice, st));
    if (queries_transposed) {
        const int64_t work = n_queries * (stride / 4);
        transpose_words_kernel<<<(unsigned)std::min<int64_t>(ceil_div(work, 256), num_sms() * 32), 256, 0, st>>>(
            (const uint8_t*)ctx->buf[0], n_words, n_queries, wb, (uint8_t*)ctx->buf[2], stride);
        FASTID_LAUNCHED("transpose_words_kernel");
    } else if (int rc = fastid_load_words(ctx->buf[0], n_queries, row_bytes, ctx->buf[2], stride, st)) {
        return rc;
    }
    if (chunked) {
        // Chunked pipeline over known rows (the paper's pinned-memory, overlapped
        // transfer design, section IV-C; the reference's stage-in / compute /
        // stage-out lanes, scheduler.py:270-419): while the GPU encodes, compares
        // and copies chunk i into pinned slot i%2, the host threads move chunk i-1
        // from its pinned slot into the caller's `out`.
        const int64_t rows = std::max<int64_t>(1, std::min<int64_t>(n_refs, (int64_t)(kChunkOutBytes / ((size_t)n_queries * 4))));
        const size_t cin = (size_t)rows * row_bytes, cout = (size_t)rows * n_queries * 4;
        if (int rc = ctx->ensure_pipeline(cin, cin, (size_t)rows * stride, cout)) return rc;
        const int64_t n_chunks = ceil_div(n_refs, rows);
        // rows land at the descriptor's current offset (after the caller's header)
        const off_t fd_base = fd >= 0 ? ::lseek(fd, 0, SEEK_CUR) : 0;
        if (fd >= 0 && fd_base < 0) FASTID_FAIL(FASTID_E_INVALID, "fd %d is not seekable", fd);
        auto drain = [&](int64_t c) -> int {  // host side of chunk c: pinned slot -> out
            const int slot = (int)(c & 1);
            const int64_t r0 = c * rows, nr = std::min<int64_t>(rows, n_refs - r0);
            FASTID_CUDA(cudaEventSynchronize(ctx->d2h_done[slot]));
            const size_t nb = (size_t)nr * n_queries * 4;
            if (fd < 0) {
                ctx->pool->copy((char*)out + (size_t)r0 * n_queries * 4, ctx->pin_out[slot], nb);
                return FASTID_OK;
            }
            // straight from the pinned slot to the file (parallel pwrite at the
            // chunk's offset): no intermediate host copy
            const off_t base = fd_base + (off_t)r0 * n_queries * 4;
            std::atomic<int> err{0};
            ctx->pool->parallel(nb, [&](size_t lo, size_t hi) {
                for (size_t done = lo; done < hi;) {
                    const ssize_t w = ::pwrite(fd, (const char*)ctx->pin_out[slot] + done, hi - done, base + (off_t)done);
                    if (w < 0) {
                        if (errno == EINTR) continue;
                        err = errno;
                        return;
                    }
                    done += (size_t)w;
                }
            });
            if (err) FASTID_FAIL(FASTID_E_INVALID, "write to fd %d failed: %s", fd, strerror(err.load()));
            return FASTID_OK;
        };
        for (int64_t c = 0; c < n_chunks; ++c) {
            const int slot = (int)(c & 1);
            const int64_t r0 = c * rows, nr = std::min<int64_t>(rows, n_refs - r0);
            // the slot's previous upload has been consumed before its pinned input is rewritten
            FASTID_CUDA(cudaEventSynchronize(ctx->h2d_done[slot]));
            ctx->pool->copy(ctx->pin_in[slot], (const char*)ref_words + (size_t)r0 * row_bytes, (size_t)nr * row_bytes);
            FASTID_CUDA(cudaMemcpyAsync(ctx->dev_slot[slot][0], ctx->pin_in[slot], (size_t)nr * row_bytes,
                                        cudaMemcpyHostToDevice, st));
            FASTID_CUDA(cudaEventRecord(ctx->h2d_done[slot], st));
            if (int rc = fastid_load_words(ctx->dev_slot[slot][0], nr, row_bytes, ctx->dev_slot[slot][1], stride, st))
                return rc;
            if (int rc = fastid_compare_full(ctx->dev_slot[slot][1], nr, ctx->buf[2], n_queries, stride, bit_length,
                                             (uint32_t*)ctx->dev_slot[slot][2], n_queries, formulation, st))
                return rc;
            FASTID_CUDA(cudaMemcpyAsync(ctx->pin_out[slot], ctx->dev_slot[slot][2], (size_t)nr * n_queries * 4,
                                        cudaMemcpyDeviceToHost, st));
            FASTID_CUDA(cudaEventRecord(ctx->d2h_done[slot], st));
            if (c > 0)
                if (int rc = drain(c - 1)) return rc;
        }
        if (int rc = drain(n_chunks - 1)) return rc;
        FASTID_CUDA(cudaStreamSynchronize(st));
        if (fd >= 0 && ::lseek(fd, fd_base + (off_t)out_bytes, SEEK_SET) < 0)
            FASTID_FAIL(FASTID_E_INVALID, "lseek on fd %d failed", fd);
        return FASTID_OK;
    }
    FASTID_CUDA(cudaMemcpyAsync(ctx->buf[0], ref_words, ref_in, cudaMemcpyHostToDevice, st));
    if (int rc = fastid_load_words(ctx->buf[0], n_refs, row_bytes, ctx->buf[1], stride, st)) return rc;
    if (int rc = fastid_compare_full(ctx->buf[1], n_refs, ctx->buf[2], n_queries, stride, bit_length,
                                     (uint32_t*)ctx->buf[3], n_queries, formulation, st))
        return rc;
    FASTID_CUDA(cudaMemcpyAsync(out, ctx->buf[3], out_bytes, cudaMemcpyDeviceToHost, st));
    FASTID_CUDA(cudaStreamSynchronize(st));
    return FASTID_OK;
}
}  // namespace

extern "C" int fastid_run_kernel(const void* ref_words, int64_t n_refs, const void* query_words, int64_t n_queries,
                                 int64_t n_words, int word_bits, int queries_transposed, uint32_t* out,
                                 int formulation) {
    if (!out && n_refs > 0 && n_queries > 0) FASTID_FAIL(FASTID_E_INVALID, "out is NULL");
    return run_host(ref_words, n_refs, query_words, n_queries, n_words, word_bits, queries_transposed, out, -1,
                    formulation);
}

extern "C" int fastid_run_kernel_fd(const void* ref_words, int64_t n_refs, const void* query_words,
                                    int64_t n_queries, int64_t n_words, int word_bits, int queries_transposed,
                                    int fd, int formulation) {
    if (fd < 0) FASTID_FAIL(FASTID_E_INVALID, "bad file descriptor %d", fd);
    return run_host(ref_words, n_refs, query_words, n_queries, n_words, word_bits, queries_transposed, nullptr, fd,
                    formulation);
}

namespace {
constexpr size_t kStreamChunkBytes = (size_t)512 << 20;  // packed known rows per chunk (auto size)
}  // namespace

// Top-k over a known panel held in HOST memory, streamed through the device
// chunk by chunk: the device-side analogue of the reference's batch planner
// and staging lanes (plan_batches scheduler.py:108-140, run_pipeline
// scheduler.py:270-419) for a panel larger than the device, with the sink
// reducing every batch to per-unknown top-k lists.  Per chunk c (rows
// [c*R, c*R + R)): host threads copy it into pinned slot c%2 (skipped when
// the caller's rows are already page-locked), the copy stream uploads it,
// the comparison stream aligns the rows, builds the chunk's tensor image,
// runs the fused top-k kernel with ref_base + c*R, and merges the chunk's
// lists into the running lists (ties keep the lower global index).  Upload
// of chunk c+1 overlaps the comparison of chunk c.
extern "C" int fastid_run_topk(const void* ref_words, int64_t n_refs, const void* query_words, int64_t n_queries,
                               int64_t n_words, int word_bits, int k, uint32_t max_score, int64_t ref_base,
                               uint32_t* top_scores, int64_t* top_index, int64_t chunk_rows, int formulation) {
    if (word_bits != 32 && word_bits != 64) FASTID_FAIL(FASTID_E_INVALID, "word_bits must be 32 or 64");
    if (n_words <= 0 || n_refs < 0 || n_queries < 0) FASTID_FAIL(FASTID_E_INVALID, "bad panel shape");
    if (k < 1 || k > kMaxTopK) FASTID_FAIL(FASTID_E_INVALID, "k must be in [1, %d]", kMaxTopK);
    if (chunk_rows < 0) FASTID_FAIL(FASTID_E_INVALID, "chunk_rows must be >= 0 (0 = automatic)");
    if (n_queries == 0) return FASTID_OK;
    if (!top_scores || !top_index || !query_words) FASTID_FAIL(FASTID_E_INVALID, "NULL buffer");
    if (n_refs == 0) {  // every list empty, as fastid_compare_topk
        for (int64_t i = 0; i < n_queries * k; ++i) {
            top_scores[i] = 0xFFFFFFFFu;
            top_index[i] = -1;
        }
        return FASTID_OK;
    }
    if (!ref_words) FASTID_FAIL(FASTID_E_INVALID, "NULL buffer");
    HostContext* ctx = nullptr;
    if (int rc = host_context(&ctx)) return rc;
    const int wb = word_bits / 8;
    const int64_t row_bytes = n_words * wb;
    const int64_t bit_length = n_words * word_bits;  // zero padding bits add nothing to any score
    const int64_t stride = row_stride_bytes(bit_length);
    if (!fastid_supports(formulation, bit_length))
        FASTID_FAIL(FASTID_E_UNSUPPORTED, "formulation %d cannot run %lld-bit profiles", formulation,
                    (long long)bit_length);
    const int f = resolve_formulation(formulation, bit_length);
    int64_t rows = chunk_rows > 0 ? chunk_rows : std::max<int64_t>(1, (int64_t)(kStreamChunkBytes / (size_t)stride));
    rows = std::min<int64_t>(rows, n_refs);
    const int64_t n_chunks = ceil_div(n_refs, rows);
    cudaStream_t st = ctx->stream;
    if (!ctx->copy_stream && cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
        FASTID_FAIL(FASTID_E_CUDA, "cudaStreamCreate failed");
    for (int i = 0; i < 2; ++i)
        if (!ctx->raw_free[i] && cudaEventCreateWithFlags(&ctx->raw_free[i], cudaEventDisableTiming) != cudaSuccess)
            FASTID_FAIL(FASTID_E_CUDA, "cudaEventCreate failed");
    // rows already page-locked (cudaHostRegister / cudaMallocHost) upload straight from the caller's array
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, ref_words) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const size_t chunk_in = (size_t)rows * row_bytes;
    const size_t lists_bytes = (size_t)n_queries * k * (sizeof(uint32_t) + sizeof(int64_t));
    if (int rc = ctx->ensure_pipeline(pinned ? 0 : chunk_in, chunk_in, 16, 16)) return rc;
    size_t ws_bytes = 0;
    if (int rc = fastid_topk_workspace(rows, n_queries, k, f, &ws_bytes)) return rc;
    const size_t img_bytes = f == FASTID_POPC ? 0 : tensor_image_bytes(rows, bit_length, f);
    const size_t q_in = (size_t)n_queries * row_bytes;
    if (int rc = ctx->ensure(0, q_in)) return rc;
    if (int rc = ctx->ensure(2, (size_t)n_queries * stride)) return rc;
    if (int rc = ctx->ensure_tk(0, (size_t)rows * stride)) return rc;
    if (img_bytes)
        if (int rc = ctx->ensure_tk(1, img_bytes)) return rc;
    if (int rc = ctx->ensure_tk(2, ws_bytes)) return rc;
    if (int rc = ctx->ensure_tk(3, 3 * lists_bytes + 64)) return rc;
    // candidates: [running | chunk] lists (scores then indices), and the merge target
    uint32_t* cand_s = (uint32_t*)ctx->tk[3];                       // [2][n_q][k]
    int64_t* cand_i = (int64_t*)((uint8_t*)ctx->tk[3] + 2 * (size_t)n_queries * k * sizeof(uint32_t));
    uint32_t* tmp_s = (uint32_t*)((uint8_t*)cand_i + 2 * (size_t)n_queries * k * sizeof(int64_t));
    int64_t* tmp_i = (int64_t*)((uint8_t*)tmp_s + ((size_t)n_queries * k * sizeof(uint32_t) + 15) / 16 * 16);
    const size_t nqk = (size_t)n_queries * k;
    // unknowns: upload and align once
    FASTID_CUDA(cudaMemcpyAsync(ctx->buf[0], query_words, q_in, cudaMemcpyHostToDevice, st));
    if (int rc = fastid_load_words(ctx->buf[0], n_queries, row_bytes, ctx->buf[2], stride, st)) return rc;
    for (int i = 0; i < 2; ++i) {  // no upload may wait on a slot event from an earlier call
        FASTID_CUDA(cudaEventRecord(ctx->raw_free[i], st));
        FASTID_CUDA(cudaEventRecord(ctx->h2d_done[i], ctx->copy_stream));
    }
    // a failure part-way leaves work in flight on both streams: drain them before
    // returning, so no later call frees or refills a buffer still being used
    const int rc_loop = [&]() -> int {
    for (int64_t c = 0; c < n_chunks; ++c) {
        const int slot = (int)(c & 1);
        const int64_t r0 = c * rows, nr = std::min<int64_t>(rows, n_refs - r0);
        const size_t nb = (size_t)nr * row_bytes;
        const void* src = (const uint8_t*)ref_words + (size_t)r0 * row_bytes;
        if (!pinned) {
            // the slot's previous upload has left its pinned staging before it is rewritten
            FASTID_CUDA(cudaEventSynchronize(ctx->h2d_done[slot]));
            ctx->pool->copy(ctx->pin_in[slot], src, nb);
            src = ctx->pin_in[slot];
        }
        FASTID_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->raw_free[slot], 0));
        FASTID_CUDA(cudaMemcpyAsync(ctx->dev_slot[slot][0], src, nb, cudaMemcpyHostToDevice, ctx->copy_stream));
        FASTID_CUDA(cudaEventRecord(ctx->h2d_done[slot], ctx->copy_stream));
        FASTID_CUDA(cudaStreamWaitEvent(st, ctx->h2d_done[slot], 0));
        if (int rc = fastid_load_words(ctx->dev_slot[slot][0], nr, row_bytes, ctx->tk[0], stride, st)) return rc;
        FASTID_CUDA(cudaEventRecord(ctx->raw_free[slot], st));
        if (img_bytes) {
            CompareArgs a = make_args(ctx->tk[0], nr, ctx->tk[0], 0, stride, bit_length);
            if (int rc = build_tensor_image(a, f, ctx->tk[1], st)) return rc;
        }
        int lists = 0, kp = 0;
        size_t xo = 0, so = 0;
        if (int rc = topk_partials_impl(ctx->tk[0], img_bytes ? ctx->tk[1] : nullptr, 0, nr, ctx->buf[2], n_queries,
                                        stride, bit_length, k, max_score, ref_base + r0, ctx->tk[2], ws_bytes,
                                        f | (formulation & FASTID_OP_MASK), st,
                                        &lists, &kp, &xo, &so))
            return rc;
        const uint32_t* ps = (const uint32_t*)((uint8_t*)ctx->tk[2] + so);
        const int64_t* px = (const int64_t*)((uint8_t*)ctx->tk[2] + xo);
        if (c == 0) {
            if (int rc = launch_merge(ps, px, lists, n_queries, kp, k, cand_s, cand_i, st)) return rc;
            continue;
        }
        // this chunk's lists -> slot 1, then running (slot 0) + slot 1 -> running
        if (int rc = launch_merge(ps, px, lists, n_queries, kp, k, cand_s + nqk, cand_i + nqk, st)) return rc;
        if (int rc = launch_merge(cand_s, cand_i, 2, n_queries, k, k, tmp_s, tmp_i, st)) return rc;
        FASTID_CUDA(cudaMemcpyAsync(cand_s, tmp_s, nqk * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        FASTID_CUDA(cudaMemcpyAsync(cand_i, tmp_i, nqk * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    }
    return FASTID_OK;
    }();
    if (rc_loop != FASTID_OK) {
        ctx->quiesce();
        return rc_loop;
    }
    FASTID_CUDA(cudaMemcpyAsync(top_scores, cand_s, nqk * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    FASTID_CUDA(cudaMemcpyAsync(top_index, cand_i, nqk * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FASTID_CUDA(cudaStreamSynchronize(st));
    return FASTID_OK;
}
