// Shared device helpers for the def-CG B200 kernels.
//
// Rounding policy: element-wise updates that the reference performs as numpy
// array expressions (x += alpha*p, r = r - alpha*Ap, p = beta*p + r - W mu,
// solvers.py:174-193) use explicit __dmul_rn/__dadd_rn so nvcc cannot contract
// them into FMAs; they then round exactly like the reference.  Reductions
// (dot products, GEMV rows) necessarily use a different summation order than
// BLAS / the reference's left-to-right loops; they are deterministic (fixed
// tree, no atomics), so repeated calls are bit-identical like the reference
// (README.md:49-53, test_kernels.py:83-105).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

#include "../../include/defcg_b200.h"

#define DCG_NT 512                      // threads of the persistent / GEMV CTAs
#define DCG_NW (DCG_NT / 32)            // warps per CTA
#define DCG_RB 128                      // rows per GEMV batch (smem partials)
#define DCG_RG 4                        // rows streamed concurrently per thread
#define DCG_QT 16384                    // x-tile (doubles) staged in smem per pass

struct dcg_context {
    int device;
    int sm_count;
    int solve_blocks;        // CTAs of the persistent solve kernel
    size_t smem_optin;
    void* ws;                // device workspace
    size_t ws_bytes;
    void* ws2;               // second workspace: operands of kernels whose callers hold `ws`
    size_t ws2_bytes;
    void* host;              // pinned host scratch for status read-back
    size_t host_bytes;
    cudaEvent_t ev0, ev1;
    long long* d_res;        // result block of the synchronous Ritz extraction
    // pass-1 range tables of the symmetric GEMV, computed on the host once per
    // (n, G) and kept on the device (dcg_sym_table)
    struct SymTable {
        long long n;
        int G;
        long long* d;        // G + 1 first tiles, device
        long long* h;        // pinned staging copy (kept alive with d)
    } symtbl[4];
    int symtbl_next;
    unsigned int* d_sync;    // persistent synchronisation words (dcg_sync_line), zeroed once
};

// device copy of the stored-Gram pass-1 range table tbl[b] = first tile of
// CTA b of G (sym_tile_begin), cached per context
const long long* dcg_sym_table(dcg_context* ctx, cudaStream_t st, long long n, int G);

// ---- persistent synchronisation words ----------------------------------------
// The grid-barrier counters and work counters of the cooperative kernels live
// in a context-owned array that is zeroed once, not in the shared workspace:
// every launch hands its words back at zero itself (dcg_sync_exit: the last
// CTA out resets them), so no memset node precedes the launch -- a memset costs
// ~3 us of stream time (node + launch gap) on the Newton step's critical path.
// One 128-byte line per slot: word 0 (and 1, for a 64-bit counter) the barrier
// or work counter, word 2 the exit counter.  A slot serves one kernel at a
// time (the context is used by one stream at a time, as its workspace is).
enum DcgSyncSlot { DCG_SW_SOLVE = 0, DCG_SW_ZSTAGE1, DCG_SW_TAIL, DCG_SW_APPLY, DCG_SW_APPLY2, DCG_SW_SBLOCK,
                   DCG_SW_XTY, DCG_SW_DERIVS, DCG_SW_SHARD, DCG_SW_SHARDSTEP, DCG_SW_NSLOTS };
static inline unsigned int* dcg_sync_line(dcg_context* ctx, int slot) { return ctx->d_sync + 32 * slot; }

// ---- status plumbing --------------------------------------------------------
// Device-side status block written by single-CTA / persistent kernels.
struct DevStatus {
    int status;
    int pad;
    long long info;
    long long count;         // k_out / T / iterations depending on kernel
    long long aux;
    double value;            // rel residual / loglik ...
    double value2;           // norm_b / psi ...
};

#define DCG_CUDA(call)                                                   \
    do {                                                                  \
        cudaError_t _e = (call);                                          \
        if (_e != cudaSuccess) {                                          \
            dcg_last_cuda_error = _e;                                     \
            return DCG_E_CUDA;                                            \
        }                                                                 \
    } while (0)

extern thread_local cudaError_t dcg_last_cuda_error;

// Kernel-launch accounting (dcg_launch_count): every launch site checks the
// launch and bumps the process-wide counter the benchmark reports.
void dcg_count_launch();
#define DCG_LAUNCHED()                          \
    do {                                        \
        DCG_CUDA(cudaGetLastError());           \
        dcg_count_launch();                     \
    } while (0)

int dcg_ws_reserve(dcg_context* ctx, size_t bytes);
int dcg_ws2_reserve(dcg_context* ctx, size_t bytes);
int dcg_host_reserve(dcg_context* ctx, size_t bytes);

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Launch set-up cached per call site AND per device: function attributes are
// per device, and contexts on different devices may be driven from different
// host threads, so the caches are indexed by the current device and updated
// under a process-wide mutex (the fast path is one atomic load).
#define DCG_MAX_DEVICES 64
static inline int dcg_current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d & (DCG_MAX_DEVICES - 1);
}
std::mutex& dcg_setup_mutex();

// Raise a kernel's dynamic shared-memory limit only when a launch on this
// device needs more than any earlier one at this call site: the attribute call
// otherwise sat on the host between back-to-back launches.
#define DCG_SMEM_ATTR(kern, bytes)                                                                         \
    do {                                                                                                   \
        static std::atomic<long long> dcg_smem_set_[DCG_MAX_DEVICES];                                      \
        const int dev_ = dcg_current_device();                                                             \
        if ((long long)(bytes) > dcg_smem_set_[dev_].load(std::memory_order_acquire)) {                    \
            std::lock_guard<std::mutex> lock_(dcg_setup_mutex());                                          \
            if ((long long)(bytes) > dcg_smem_set_[dev_].load(std::memory_order_relaxed)) {                \
                DCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes))); \
                dcg_smem_set_[dev_].store((long long)(bytes), std::memory_order_release);                 \
            }                                                                                              \
        }                                                                                                  \
    } while (0)

// Occupancy (CTAs per SM) of `kern` at `smem` bytes, cached per device in
// `cache` (one slot per device: smem << 16 | occupancy + 1).
static inline int dcg_occupancy_cached(std::atomic<long long>* cache, const void* kern, int threads, size_t smem,
                                       int* out) {
    const int dev = dcg_current_device();
    const long long v = cache[dev].load(std::memory_order_acquire);
    if (v && (v >> 16) == (long long)smem) {
        *out = (int)(v & 0xFFFF) - 1;
        return DCG_OK;
    }
    int occ = 0;
    DCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
    cache[dev].store(((long long)smem << 16) | (long long)(occ + 1), std::memory_order_release);
    *out = occ;
    return DCG_OK;
}

// ---- CTA barrier ---------------------------------------------------------------
// __syncthreads() is the *aligned* bar.sync: it assumes every warp arrives
// converged.  Independent thread scheduling does not guarantee reconvergence
// after a lane-predicated loop (e.g. only lanes v < nslots load partials), and a
// warp that reaches an aligned barrier while diverged can be counted as arrived
// before its remaining lanes get there -- the CTA is released early (stale
// shared memory) or a later barrier never completes.  The non-aligned form
// counts threads individually, so it is correct for divergent arrival.
__device__ __forceinline__ void cta_sync() { asm volatile("barrier.sync 0;" ::: "memory"); }

// ---- arithmetic without FMA contraction --------------------------------------
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// ---- loads -----------------------------------------------------------------
// Streamed, read-only for the kernel's lifetime (the Gram slab): no L1 allocation.
__device__ __forceinline__ double2 ld_stream2(const double* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
// Data written by other CTAs of the same launch (after a grid barrier): L2 only.
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// ---- reductions (deterministic: fixed butterfly, identical on every lane) ---
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum; every thread receives the same value.  `red` holds >= 33
// doubles of shared scratch.  Contains two CTA barriers.
__device__ __forceinline__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    cta_sync();
    if (lane == 0) red[warp] = v;
    cta_sync();
    double t = (lane < nw) ? red[lane] : 0.0;
    t = warp_sum(t);
    return t;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double block_max(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    cta_sync();
    if (lane == 0) red[warp] = v;
    cta_sync();
    double t = (lane < nw) ? red[lane] : -INFINITY;
    return warp_max(t);
}

// Row partition of [0, n) over `parts` contiguous, balanced ranges.
__host__ __device__ __forceinline__ long long part_begin(long long n, long long parts, long long i) {
    return (n * i) / parts;
}

// ---- host helpers -------------------------------------------------------------
// bump allocator over ctx->ws (reserve the total first, then carve)
struct Arena {
    char* base;
    size_t off;
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = reinterpret_cast<T*>(base + off);
        off += sizeof(T) * count;
        return p;
    }
};
static inline size_t al(size_t bytes) { return (bytes + 255) & ~size_t(255); }
static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Grid barrier for a launch whose CTAs are all co-resident (cooperative
// launch).  `bar` is a monotonic arrival counter, zero at launch: barrier
// instance m completes when it reaches m * nblocks, so a CTA only needs the
// value its own arrival returned -- one release-atomic per CTA and acquire
// polling, no reset and no generation word (two L2 round trips on the
// critical path).  The CTA barrier before the release orders every thread's
// writes ahead of it (cumulativity); warp 0 polls warp-uniformly (lane 0
// loads, __shfl_sync broadcasts) so no lane is left in a divergent spin.
__device__ __forceinline__ unsigned int atom_add_release_gpu(unsigned int* p, unsigned int v) {
    unsigned int old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void dcg_grid_barrier(unsigned int* bar, unsigned int nblocks) {
    cta_sync();
    if (threadIdx.x < 32) {
        unsigned int target = 0;
        if (threadIdx.x == 0) {
            const unsigned int old = atom_add_release_gpu(bar, 1u);
            target = (old / nblocks + 1u) * nblocks;
        }
        target = __shfl_sync(0xffffffffu, target, 0);
        for (;;) {
            unsigned int cur = 0;
            if (threadIdx.x == 0) cur = ld_acquire_gpu(bar);
            cur = __shfl_sync(0xffffffffu, cur, 0);
            if ((int)(cur - target) >= 0) break;
        }
    }
    cta_sync();
}

// Called by ONE thread of every CTA once the CTA is done with line[0..1] (its
// last grid barrier passed / its last counter draw made): the last CTA out
// returns the line to zero for the next launch.  No CTA reads the counter
// after its exit increment, so the reset cannot race a barrier poll.
__device__ __forceinline__ void dcg_sync_exit(unsigned int* line, unsigned int nblocks) {
    __threadfence();
    if (atomicAdd(line + 2, 1u) == nblocks - 1) {
        line[0] = 0u;
        line[1] = 0u;
        line[2] = 0u;
        __threadfence();
    }
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// copy a device status block to the host (synchronises the stream)
int dcg_read_status(dcg_context* ctx, cudaStream_t st, const DevStatus* dev, DevStatus* out);

// Deterministic "last CTA reduces" handshake: every CTA publishes its partials,
// then calls this; exactly one CTA (the last to arrive) gets true and may read
// all partials.  The counter returns to zero for the next launch.
__device__ __forceinline__ bool cta_last_arrival(unsigned int* counter, unsigned int total) {
    __shared__ int s_last;
    __threadfence();
    cta_sync();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(counter, 1u);
        s_last = (prev == total - 1) ? 1 : 0;
        if (s_last) *counter = 0u;
    }
    cta_sync();
    if (s_last) __threadfence();
    return s_last != 0;
}
