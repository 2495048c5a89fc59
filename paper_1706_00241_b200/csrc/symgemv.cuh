// Symmetric GEMV over the lower triangle of a dense, exactly symmetric K.
//
// K1 streams 8 n^2 bytes per product; K = K' lets every element serve twice,
// so this strategy streams only the ~n^2/2 lower-triangle entries (halving
// HBM traffic per CG iteration), as 64 x 64 tiles (I, J <= I) of the padded
// row-major storage:
//
//   pass 1 (all CTAs): the linear tile sequence is split into contiguous
//     ranges of equal estimated cost (a tile-row segment flush and the partial
//     last tile row are weighted), one per CTA.  Tiles flow through a DCG_SYM_STAGES-deep
//     shared-memory ring filled by per-thread 16-byte cp.async copies whose
//     completion is tracked by mbarriers (cp.async.mbarrier.arrive), and
//     released by one arrival per warp: warps never wait on a CTA barrier per
//     tile.  Warp w owns columns 4w..4w+3 of every tile, lane l rows 2l, 2l+1:
//        row part     t_I[r] += K_IJ[r][c] x_J[c]  (registers along a tile-row
//                     segment; one cross-warp reduction per segment -> rowpart)
//        column part  t_J[c] += K_IJ[r][c] x_I[r]  (64-row sum per column as a
//                     6-shuffle warp reduce-scatter -> colpart[tile], off-
//                     diagonal tiles only)
//     The tile is stored XOR-swizzled (16-byte chunk q of row r at q ^ (r/2))
//     so the column-strip reads are bank-conflict free.
//   pass 2 (after a grid barrier): t_i = sum of the segment partials of tile
//     row I plus colpart of the tiles (I', I), I' > I, in a fixed order.  Row
//     i of tile row I costs ~NT - I loads, so rows are split by that weight and
//     each row is reduced by up to 32 lanes of one warp (no CTA barriers).
//
// Both passes are deterministic (no atomics).  Pass 2 touches 2 x 64 doubles
// per tile, ~3% of the tile bytes.
#pragma once
#include "common.cuh"

#define DCG_TB 64
#ifndef DCG_SYM_STAGES
#define DCG_SYM_STAGES 4
#endif
#define DCG_SYM_TILE_DOUBLES (DCG_TB * DCG_TB)
// a ring stage: the tile plus the 64-entry slices v_J and s_J the tile's row
// product needs, so everything a tile consumes arrives with it
#define DCG_SYM_STAGE_DOUBLES (DCG_SYM_TILE_DOUBLES + 2 * DCG_TB)

__host__ __device__ __forceinline__ long long sym_ntiles_side(long long n) { return (n + DCG_TB - 1) / DCG_TB; }
__host__ __device__ __forceinline__ long long sym_ntiles(long long n) {
    const long long nt = sym_ntiles_side(n);
    return nt * (nt + 1) / 2;
}
__host__ __device__ __forceinline__ long long sym_tile_row_base(long long I) { return I * (I + 1) / 2; }
// tile row of linear tile t (tiles (I, 0..I) are consecutive)
__host__ __device__ __forceinline__ long long sym_tile_row(long long t) {
    long long I = (long long)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (sym_tile_row_base(I + 1) <= t) ++I;
    while (sym_tile_row_base(I) > t) --I;
    return I;
}

// ---- packed layout (DCG_OP_DENSE_SYM with d_kp) ------------------------------
// The lower-triangle tiles in pass-1 order, each 64 x 64 tile one contiguous
// 32 KB block, zero beyond n, and stored in the ring's XOR swizzle (element
// (r, c) at r * 64 + 2 ((c / 2) ^ (r / 2 mod 32)) + c mod 2): a tile lands in
// its stage with ONE bulk copy (cp.async.bulk, the TMA engine) and its DRAM
// pages are read sequentially -- measured 6.7 TB/s streamed through a
// 4-stage ring against 6.0 TB/s for the row-major tile of 64 rows x 512 B
// (tools/stream_probe.cu, profiles/r02/stream_probe.jsonl).
__host__ __device__ __forceinline__ long long sym_packed_doubles(long long n) {
    return sym_ntiles(n) * (long long)(DCG_TB * DCG_TB);
}
__host__ __device__ __forceinline__ int sym_swz(int r, int c) { return r * DCG_TB + 2 * ((c >> 1) ^ ((r >> 1) & 31)) + (c & 1); }

// ---- pass-1 partition: equal estimated cost per CTA ---------------------------
// Cost in quarter tiles of the tiles [0, t) (measured per-CTA pass times):
// 4 per tile, +4 per tile-row segment flush (one per completed row: a CTA
// barrier and a 16-way smem sum), +1 per tile of a partial last tile row --
// those move fewer bytes but hold a ring slot for a full loaded-HBM round trip
// and measured ~1.2x a full tile.
__host__ __device__ __forceinline__ long long sym_cost4(long long t, long long n) {
    const long long NT = sym_ntiles_side(n);
    const long long last = (n % DCG_TB) ? sym_tile_row_base(NT - 1) : sym_tile_row_base(NT);
    const long long inlast = t > last ? t - last : 0;
    return 4 * t + inlast + 4 * sym_tile_row(t);
}
// first tile of CTA b of G: smallest t with cost(t) >= ceil(b * total / G)
__host__ __device__ __forceinline__ long long sym_tile_begin(long long n, long long G, long long b) {
    const long long NT = sym_ntiles_side(n), ntt = NT * (NT + 1) / 2;
    if (b <= 0) return 0;
    if (b >= G) return ntt;
    const long long total = sym_cost4(ntt, n);
    const long long goal = (b * total + G - 1) / G;
    long long lo = 0, hi = ntt;
    while (lo < hi) {
        const long long mid = (lo + hi) / 2;
        if (sym_cost4(mid, n) >= goal) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// ---- pass-2 partition: rows weighted by their partial count -------------------
// Row i of tile row I reads NT - 1 - I column partials, ~1 row-segment partial
// and runs the epilogue: weight NT + F - I.  W(i) = weight of rows [0, i).
// F = DCG_SYM_ROW_FIXED prices a row's fixed cost (its row-segment partials,
// the epilogue's loads and store) in partial loads: with F = 3 the last CTA,
// all cheap rows, took 5.5 us against a 3.6 us mean (n = 10k).
#ifndef DCG_SYM_ROW_FIXED
#define DCG_SYM_ROW_FIXED 12
#endif
__host__ __device__ __forceinline__ long long sym_row_work(long long i, long long n) {
    const long long NT = sym_ntiles_side(n) + DCG_SYM_ROW_FIXED;
    const long long I = i / DCG_TB;
    return DCG_TB * (I * NT - I * (I - 1) / 2) + (i - I * DCG_TB) * (NT - I);
}
__host__ __device__ __forceinline__ long long sym_row_begin(long long n, long long G, long long b) {
    if (b <= 0) return 0;
    if (b >= G) return n;
    const long long goal = (b * sym_row_work(n, n) + G - 1) / G;
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) / 2;
        if (sym_row_work(mid, n) >= goal) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// first tile of part b of R over the tile sub-range [t_lo, t_hi) (equal cost;
// t_lo = 0, t_hi = all tiles reproduces sym_tile_begin)
__host__ __device__ __forceinline__ long long sym_tile_begin_range(long long n, long long t_lo, long long t_hi,
                                                                   long long R, long long b) {
    if (b <= 0) return t_lo;
    if (b >= R) return t_hi;
    const long long c0 = sym_cost4(t_lo, n), c1 = sym_cost4(t_hi, n);
    const long long goal = c0 + (b * (c1 - c0) + R - 1) / R;
    long long lo = t_lo, hi = t_hi;
    while (lo < hi) {
        const long long mid = (lo + hi) / 2;
        if (sym_cost4(mid, n) >= goal) hi = mid; else lo = mid + 1;
    }
    return lo;
}

#define DCG_SYM_MAX_CTAS 255
// Shared memory the two passes need (doubles): ring, 2 x 16 x 64 row-flush
// buffers, 2 x STAGES mbarriers, the table of G + 1 pass-1 range starts.
__host__ __device__ __forceinline__ long long sym_smem_doubles() {
    return (long long)DCG_SYM_STAGES * DCG_SYM_STAGE_DOUBLES + 2 * DCG_NW * DCG_TB + 2 * DCG_SYM_STAGES + 2 +
           (DCG_SYM_MAX_CTAS + 1);
}
__device__ __forceinline__ long long* sym_range_table(double* smem) {
    return reinterpret_cast<long long*>(smem + DCG_SYM_STAGES * DCG_SYM_STAGE_DOUBLES + 2 * DCG_NW * DCG_TB +
                                        2 * DCG_SYM_STAGES + 2);
}
// tbl[b] = first tile of CTA b, b = 0..G (all threads call; ends with a barrier)
__device__ __forceinline__ void sym_fill_range_table(long long* tbl, long long n, int R = -1) {
    if (R < 0) R = gridDim.x;
    for (int b = threadIdx.x; b <= R; b += blockDim.x) tbl[b] = sym_tile_begin(n, R, b);
    cta_sync();
}

// ---- async copy and mbarrier primitives ------------------------------------
__device__ __forceinline__ unsigned sym_saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
// K is streamed once per product and is far larger than L2: its lines are
// marked evict-first so they do not push out the vectors and the tile
// partials pass 2 reads back.  (Keeping a fixed slice of the triangle
// L2-resident with evict-last loads instead -- a persisting carve-out of up
// to 96 MB -- cut the solve's DRAM reads by 13% at n = 10^4 and left its time
// unchanged: pass 1 runs at ~94% of the copy peak per CTA and is bound by the
// per-tile issue work, not by HBM; profiles/r02/l2_pin_*.)
__device__ __forceinline__ unsigned long long sym_policy_evict_first() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void sym_cp_async16_full(double* sdst, const double* gsrc, unsigned long long pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sym_saddr(sdst)), "l"(gsrc),
                 "l"(pol));
}
__device__ __forceinline__ void sym_cp_async16_v(double* sdst, const double* gsrc, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sym_saddr(sdst)), "l"(gsrc), "r"(bytes));
}
__device__ __forceinline__ void sym_cp_async16_vfull(double* sdst, const double* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sym_saddr(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void sym_mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sym_saddr(bar)), "r"(count));
}
// arrive once all cp.async previously issued by this thread have completed
__device__ __forceinline__ void sym_mbar_cp_arrive(unsigned long long* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(sym_saddr(bar)) : "memory");
}
__device__ __forceinline__ void sym_mbar_arrive(unsigned long long* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(sym_saddr(bar))
                 : "memory");
}
__device__ __forceinline__ void sym_mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "SYM_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SYM_WAIT_%=;\n\t}\n" ::"r"(sym_saddr(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void sym_mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(sym_saddr(bar)),
                 "r"(bytes)
                 : "memory");
}
// one packed tile (32 KB) into a stage by the bulk-copy (TMA) engine; completion
// is counted in bytes on the stage's full barrier
__device__ __forceinline__ void sym_bulk_tile(double* sdst, const double* gsrc, unsigned long long* bar,
                                              unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
            sym_saddr(sdst)),
        "l"(gsrc), "r"((unsigned)(DCG_SYM_TILE_DOUBLES * sizeof(double))), "r"(sym_saddr(bar)), "l"(pol)
        : "memory");
}

// 16-byte chunk starting at element j of [0, n): bytes to copy (zero-fill beyond n)
__device__ __forceinline__ int sym_chunk_bytes(long long j, long long n) {
    return j < n ? ((j + 1 < n) ? 16 : 8) : 0;
}

// Per-thread copy geometry of a tile: chunk u covers row (tid/32 + 16u), the
// 16-byte chunk q = tid%32 of that row, stored at swizzled chunk q ^ (row/2).
struct SymCopyPlan {
    long long koff[DCG_SYM_TILE_DOUBLES / 2 / DCG_NT];   // element offsets into K
    int soff[DCG_SYM_TILE_DOUBLES / 2 / DCG_NT];         // offsets into the stage
    int crow, c2;
};

__device__ __forceinline__ SymCopyPlan sym_copy_plan(long long ldk) {
    SymCopyPlan pl;
    const int tid = threadIdx.x;
    pl.crow = tid >> 5;
    pl.c2 = (tid & 31) * 2;
#pragma unroll
    for (int u = 0; u < DCG_SYM_TILE_DOUBLES / 2 / DCG_NT; ++u) {
        const int row = pl.crow + 16 * u;
        pl.koff[u] = (long long)row * ldk + pl.c2;
        pl.soff[u] = row * DCG_TB + 2 * ((tid & 31) ^ ((row >> 1) & 31));
    }
    return pl;
}

// Issue this thread's copies of tile (I, J) (top-left element `kt`) and of the
// slices v_J, s_J into stage `dst`.  cp.async.cg reads through L2, so v may
// have been written by other CTAs before the preceding grid barrier.
template <bool kHint>
__device__ __forceinline__ void sym_issue_tile(const double* __restrict__ kt, const SymCopyPlan& pl, long long n,
                                               long long I, long long J, const double* v, const double* s,
                                               double* dst, unsigned long long pol) {
    const int tid = threadIdx.x;
    const long long r_base = I * DCG_TB, c_base = J * DCG_TB;
    if (r_base + DCG_TB <= n) {   // J <= I: the column block is interior as well
#pragma unroll
        for (int u = 0; u < DCG_SYM_TILE_DOUBLES / 2 / DCG_NT; ++u) {
            if constexpr (kHint) sym_cp_async16_full(dst + pl.soff[u], kt + pl.koff[u], pol);
            else sym_cp_async16_vfull(dst + pl.soff[u], kt + pl.koff[u]);
        }
        if (tid < 32) sym_cp_async16_vfull(dst + DCG_SYM_TILE_DOUBLES + 2 * tid, v + c_base + 2 * tid);
        else if (tid < 64 && s)
            sym_cp_async16_vfull(dst + DCG_SYM_TILE_DOUBLES + DCG_TB + 2 * (tid - 32), s + c_base + 2 * (tid - 32));
        return;
    }
#pragma unroll
    for (int u = 0; u < DCG_SYM_TILE_DOUBLES / 2 / DCG_NT; ++u) {
        const long long gr = r_base + pl.crow + 16 * u, gc = c_base + pl.c2;
        const int bytes = gr < n ? sym_chunk_bytes(gc, n) : 0;
        // chunks wholly beyond n are not copied: their stage slots keep earlier
        // (finite) tile data, which only ever meets zero x entries
        // (edge chunks use the plain form: a zero-filling cp.async with an L2
        // cache hint faulted as an illegal instruction on sm_100a)
        if (bytes == 16 && kHint) sym_cp_async16_full(dst + pl.soff[u], kt + pl.koff[u], pol);
        else if (bytes) sym_cp_async16_v(dst + pl.soff[u], kt + pl.koff[u], bytes);
    }
    if (tid < 32) {
        const long long j = c_base + 2 * tid;
        const int bytes = sym_chunk_bytes(j, n);
        sym_cp_async16_v(dst + DCG_SYM_TILE_DOUBLES + 2 * tid, bytes ? v + j : v, bytes);
    } else if (tid < 64 && s) {
        const long long j = c_base + 2 * (tid - 32);
        const int bytes = sym_chunk_bytes(j, n);
        sym_cp_async16_v(dst + DCG_SYM_TILE_DOUBLES + DCG_TB + 2 * (tid - 32), bytes ? s + j : s, bytes);
    }
}

// x'_j = s_j v_j (or v_j), zero beyond n (v read through L2).
__device__ __forceinline__ double sym_xval(const double* v, const double* s, long long j, long long n) {
    if (j >= n) return 0.0;
    const double vv = ld_cg(v + j);
    return s ? mul_rn(__ldg(s + j), vv) : vv;
}

// The ring's mbarriers are initialised once per launch (re-initialising a
// live mbarrier is undefined); every pass then continues the CTA's tile
// sequence number `seq`, from which stage and phase parities follow.
// Row-major storage: every thread copies a share of each tile and arrives
// (DCG_NT arrivals per use).  Packed storage: thread 0 arms the byte count of
// the tile's bulk copy (one arrival), threads 0..63 copy the v / s slices
// and arrive (64 arrivals).
#define DCG_SYM_PK_ARRIVALS 65
// gtbl (optional): the range table precomputed on the host (dcg_sym_table)
__device__ __forceinline__ void sym_ring_init(double* smem, long long n, bool packed = false,
                                              const long long* gtbl = nullptr) {
    unsigned long long* full = reinterpret_cast<unsigned long long*>(
        smem + DCG_SYM_STAGES * DCG_SYM_STAGE_DOUBLES + 2 * DCG_NW * DCG_TB);
    unsigned long long* empty = full + DCG_SYM_STAGES;
    // finite stage contents from the start (row-major edge tiles leave slots
    // uncopied; packed tiles and their slices are always copied whole)
    if (!packed)
        for (int e = threadIdx.x; e < DCG_SYM_STAGES * DCG_SYM_STAGE_DOUBLES; e += blockDim.x) smem[e] = 0.0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int st = 0; st < DCG_SYM_STAGES; ++st) {
            sym_mbar_init(full + st, packed ? DCG_SYM_PK_ARRIVALS : DCG_NT);
            sym_mbar_init(empty + st, DCG_NW);    // one arrival per warp per use
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (gtbl) {
        long long* tbl = sym_range_table(smem);
        for (int b = threadIdx.x; b <= (int)gridDim.x; b += blockDim.x) tbl[b] = __ldg(gtbl + b);
        cta_sync();
    } else {
        sym_fill_range_table(sym_range_table(smem), n);
    }
}

// Packed storage, threads 0..63: the slices v_J, s_J of a tile into its stage
// (16-byte cp.async, zero beyond n) and the stage arrival; thread 0 first arms
// and issues the tile's bulk copy unless it is already in flight.
__device__ __forceinline__ void sym_issue_packed(const double* kt, long long n, long long J, const double* v,
                                                 const double* s, double* dst, unsigned long long* full,
                                                 unsigned long long pol, bool tile) {
    const int tid = threadIdx.x;
    if (tile && tid == 0) {
        sym_mbar_expect_tx(full, (unsigned)(DCG_SYM_TILE_DOUBLES * sizeof(double)));
        sym_bulk_tile(dst, kt, full, pol);
    }
    const long long j = J * DCG_TB + 2 * (tid & 31);
    const int bytes = sym_chunk_bytes(j, n);
    if (tid < 32) sym_cp_async16_v(dst + DCG_SYM_TILE_DOUBLES + 2 * tid, bytes ? v + j : v, bytes);
    else if (s) sym_cp_async16_v(dst + DCG_SYM_TILE_DOUBLES + DCG_TB + 2 * (tid - 32), bytes ? s + j : s, bytes);
    sym_mbar_cp_arrive(full);
}

// Packed storage: tiles of the NEXT pass over the same range whose bulk copies
// were issued at the end of this one (sym_pass1 with prefetch); they overlap
// the grid barriers and vector phases between two products.  A launch that
// ends with copies in flight drains them first.
__device__ __forceinline__ void sym_ring_drain(double* smem, unsigned int seq, int& pending) {
    if (pending <= 0) return;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(
        smem + DCG_SYM_STAGES * DCG_SYM_STAGE_DOUBLES + 2 * DCG_NW * DCG_TB);
    for (int st = 0; st < pending; ++st) {
        const unsigned int q = seq + st;
        if (threadIdx.x < 64) sym_mbar_cp_arrive(full + q % DCG_SYM_STAGES);
        sym_mbar_wait(full + q % DCG_SYM_STAGES, (q / DCG_SYM_STAGES) & 1);
    }
    pending = 0;
}

// Pass 1 over this CTA's tile range.  colpart/rowpart: ntt x 64 doubles.
// `seq` (uniform per CTA) counts the tiles this CTA has pushed through the
// ring in earlier passes of the same launch; it advances by the range length.
// NV = 2: a second vector v2 rides in the stage's s slot (both vectors
// unscaled, s == nullptr) and its partials go to colpart / rowpart + part2 --
// every tile read from HBM serves two products, each with exactly the
// operation sequence of its NV = 1 pass.
// PK: K is the packed tile array (sym_packed_doubles; ldk unused); `pending`
// (uniform per CTA) counts tiles of this range whose bulk copies a previous
// pass already issued, and `prefetch` issues the first DCG_SYM_STAGES - 1
// tiles of the next pass over the same range once this one is consumed.
template <bool kHint = true, int NV = 1, bool PK = false>
__device__ __forceinline__ void sym_pass1(const double* __restrict__ K, long long ldk, long long n, const double* v,
                                          const double* s, double* colpart, double* rowpart, double* smem,
                                          unsigned int& seq, const double* v2 = nullptr, long long part2 = 0,
                                          int* pending = nullptr, bool prefetch = false) {
    static_assert(NV == 1 || NV == 2, "one or two vectors");
    if constexpr (NV == 2) s = v2;   // the s slot of every stage carries v2
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* ring = smem;
    double* rowred = ring + DCG_SYM_STAGES * DCG_SYM_STAGE_DOUBLES;                       // 2 x NW x 64
    unsigned long long* full = reinterpret_cast<unsigned long long*>(rowred + 2 * DCG_NW * DCG_TB);
    unsigned long long* empty = full + DCG_SYM_STAGES;
    const long long* tbl = sym_range_table(smem);
    const long long t0 = tbl[blockIdx.x];
    const long long t1 = tbl[blockIdx.x + 1];
    if (t0 >= t1) return;   // uniform per CTA
    const int ntiles = (int)(t1 - t0);
    const unsigned int q0 = seq;   // global sequence number of tile lt is q0 + lt
    seq += (unsigned int)ntiles;
    long long I = sym_tile_row(t0);
    long long J = t0 - sym_tile_row_base(I);
    const SymCopyPlan pl = sym_copy_plan(ldk);
    const unsigned long long pol = sym_policy_evict_first();
    const long long row_stride = (long long)DCG_TB * ldk;
    // prologue: tiles 0 .. STAGES-2; issue cursor (iI, iJ, ip) follows
    long long iI = I, iJ = J;
    const double* ip = PK ? K + t0 * DCG_SYM_TILE_DOUBLES : K + iI * row_stride + iJ * DCG_TB;
    const int pre = (PK && pending) ? *pending : 0;
#pragma unroll
    for (int st = 0; st < DCG_SYM_STAGES - 1; ++st) {
        if (st < ntiles) {
            const unsigned int q = q0 + st;
            const int stg = q % DCG_SYM_STAGES;
            if constexpr (PK) {
                if (tid < 64) {
                    if (st >= pre && q >= DCG_SYM_STAGES) sym_mbar_wait(empty + stg, ((q / DCG_SYM_STAGES) - 1) & 1);
                    sym_issue_packed(ip, n, iJ, v, s, ring + stg * DCG_SYM_STAGE_DOUBLES, full + stg, pol, st >= pre);
                }
            } else {
                if (q >= DCG_SYM_STAGES) sym_mbar_wait(empty + stg, ((q / DCG_SYM_STAGES) - 1) & 1);
                sym_issue_tile<kHint>(ip, pl, n, iI, iJ, v, s, ring + stg * DCG_SYM_STAGE_DOUBLES, pol);
                sym_mbar_cp_arrive(full + stg);
            }
        }
        if constexpr (PK) {
            if (++iJ > iI) { ++iI; iJ = 0; }
            ip += DCG_SYM_TILE_DOUBLES;
        } else {
            if (++iJ > iI) { ++iI; iJ = 0; ip = K + iI * row_stride; } else { ip += DCG_TB; }
        }
    }
    if (pending) *pending = 0;
    // swizzled offsets of this thread's reads: rows 2l, 2l+1, chunks 2w, 2w+1
    const int key = lane & 31;                                     // (row >> 1) for both rows
    const int o00 = (2 * lane) * DCG_TB + 2 * ((2 * warp) ^ key);
    const int o01 = (2 * lane) * DCG_TB + 2 * ((2 * warp + 1) ^ key);
    const int o10 = o00 + DCG_TB, o11 = o01 + DCG_TB;
    double xI0 = sym_xval(v, NV == 2 ? nullptr : s, I * DCG_TB + 2 * lane, n);
    double xI1 = sym_xval(v, NV == 2 ? nullptr : s, I * DCG_TB + 2 * lane + 1, n);
    double yI0 = 0.0, yI1 = 0.0;
    if constexpr (NV == 2) {
        yI0 = sym_xval(v2, nullptr, I * DCG_TB + 2 * lane, n);
        yI1 = sym_xval(v2, nullptr, I * DCG_TB + 2 * lane + 1, n);
    }
    double row0 = 0.0, row1 = 0.0, rowb0 = 0.0, rowb1 = 0.0;
    long long seg_start = t0;
    int flush = 0;
    for (int lt = 0; lt < ntiles; ++lt) {
        // produce tile lt + STAGES - 1 into the stage tile lt - 1 used
        {
            const int tn = lt + DCG_SYM_STAGES - 1;
            if constexpr (PK) {
                if (tn < ntiles && tid < 64) {
                    const unsigned int q = q0 + tn;
                    const int stg = q % DCG_SYM_STAGES;
                    if (q >= DCG_SYM_STAGES) sym_mbar_wait(empty + stg, ((q / DCG_SYM_STAGES) - 1) & 1);
                    sym_issue_packed(ip, n, iJ, v, s, ring + stg * DCG_SYM_STAGE_DOUBLES, full + stg, pol, true);
                }
                if (++iJ > iI) { ++iI; iJ = 0; }
                ip += DCG_SYM_TILE_DOUBLES;
            } else {
                if (tn < ntiles) {
                    const unsigned int q = q0 + tn;
                    const int stg = q % DCG_SYM_STAGES;
                    if (q >= DCG_SYM_STAGES) sym_mbar_wait(empty + stg, ((q / DCG_SYM_STAGES) - 1) & 1);
                    sym_issue_tile<kHint>(ip, pl, n, iI, iJ, v, s, ring + stg * DCG_SYM_STAGE_DOUBLES, pol);
                    sym_mbar_cp_arrive(full + stg);
                }
                if (++iJ > iI) { ++iI; iJ = 0; ip = K + iI * row_stride; } else { ip += DCG_TB; }
            }
        }
        // consume tile lt
        const unsigned int q = q0 + lt;
        const int stg = q % DCG_SYM_STAGES;
        sym_mbar_wait(full + stg, (q / DCG_SYM_STAGES) & 1);
        const double* tile = ring + stg * DCG_SYM_STAGE_DOUBLES;
        const double2 a0 = *reinterpret_cast<const double2*>(tile + o00);   // row 2l,   cols 4w, 4w+1
        const double2 a1 = *reinterpret_cast<const double2*>(tile + o01);   // row 2l,   cols 4w+2, 4w+3
        const double2 b0 = *reinterpret_cast<const double2*>(tile + o10);   // row 2l+1
        const double2 b1 = *reinterpret_cast<const double2*>(tile + o11);
        const double2 v0 = *reinterpret_cast<const double2*>(tile + DCG_SYM_TILE_DOUBLES + 4 * warp);
        const double2 v1 = *reinterpret_cast<const double2*>(tile + DCG_SYM_TILE_DOUBLES + 4 * warp + 2);
        double x0 = v0.x, x1 = v0.y, x2 = v1.x, x3 = v1.y;
        double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
        if constexpr (NV == 2) {
            const double2 s0 = *reinterpret_cast<const double2*>(tile + DCG_SYM_TILE_DOUBLES + DCG_TB + 4 * warp);
            const double2 s1 = *reinterpret_cast<const double2*>(tile + DCG_SYM_TILE_DOUBLES + DCG_TB + 4 * warp + 2);
            y0 = s0.x;
            y1 = s0.y;
            y2 = s1.x;
            y3 = s1.y;
        } else if (s) {
            const double2 s0 = *reinterpret_cast<const double2*>(tile + DCG_SYM_TILE_DOUBLES + DCG_TB + 4 * warp);
            const double2 s1 = *reinterpret_cast<const double2*>(tile + DCG_SYM_TILE_DOUBLES + DCG_TB + 4 * warp + 2);
            x0 = mul_rn(s0.x, x0);
            x1 = mul_rn(s0.y, x1);
            x2 = mul_rn(s1.x, x2);
            x3 = mul_rn(s1.y, x3);
        }
        __syncwarp();
        if (lane == 0) sym_mbar_arrive(empty + stg);   // this warp is done with the stage
        row0 = fma(a0.x, x0, row0);
        row0 = fma(a0.y, x1, row0);
        row0 = fma(a1.x, x2, row0);
        row0 = fma(a1.y, x3, row0);
        row1 = fma(b0.x, x0, row1);
        row1 = fma(b0.y, x1, row1);
        row1 = fma(b1.x, x2, row1);
        row1 = fma(b1.y, x3, row1);
        if constexpr (NV == 2) {
            rowb0 = fma(a0.x, y0, rowb0);
            rowb0 = fma(a0.y, y1, rowb0);
            rowb0 = fma(a1.x, y2, rowb0);
            rowb0 = fma(a1.y, y3, rowb0);
            rowb1 = fma(b0.x, y0, rowb1);
            rowb1 = fma(b0.y, y1, rowb1);
            rowb1 = fma(b1.x, y2, rowb1);
            rowb1 = fma(b1.y, y3, rowb1);
        }
        if (J < I) {
            // column sums over the tile's 64 rows: warp reduce-scatter of 4 values
            auto colsum = [&](double zI0, double zI1, double* cp) {
                double c0 = fma(b0.x, zI1, a0.x * zI0);
                double c1 = fma(b0.y, zI1, a0.y * zI0);
                double c2 = fma(b1.x, zI1, a1.x * zI0);
                double c3 = fma(b1.y, zI1, a1.y * zI0);
                const bool hi16 = lane & 16;
                const double r0 = __shfl_xor_sync(0xffffffffu, hi16 ? c0 : c2, 16);
                const double r1 = __shfl_xor_sync(0xffffffffu, hi16 ? c1 : c3, 16);
                double k0 = (hi16 ? c2 : c0) + r0;   // columns {0,1} (lanes < 16) or {2,3}
                double k1 = (hi16 ? c3 : c1) + r1;
                const bool hi8 = lane & 8;
                const double r2 = __shfl_xor_sync(0xffffffffu, hi8 ? k0 : k1, 8);
                double cv = (hi8 ? k1 : k0) + r2;    // column 2*hi16 + hi8
                cv += __shfl_xor_sync(0xffffffffu, cv, 4);
                cv += __shfl_xor_sync(0xffffffffu, cv, 2);
                cv += __shfl_xor_sync(0xffffffffu, cv, 1);
                if ((lane & 7) == 0) cp[(t0 + lt) * DCG_TB + 4 * warp + 2 * (lane >> 4) + ((lane >> 3) & 1)] = cv;
            };
            colsum(xI0, xI1, colpart);
            if constexpr (NV == 2) colsum(yI0, yI1, colpart + part2);
        }
        // end of a tile-row segment: diagonal tile reached or last tile of the range
        if (J == I || lt + 1 == ntiles) {
            if constexpr (NV == 1) {
                double* rr = rowred + (flush & 1) * DCG_NW * DCG_TB;
                rr[warp * DCG_TB + 2 * lane] = row0;
                rr[warp * DCG_TB + 2 * lane + 1] = row1;
                cta_sync();
                if (tid < DCG_TB) {
                    double a = 0.0;
#pragma unroll
                    for (int w = 0; w < DCG_NW; ++w) a += rr[w * DCG_TB + tid];
                    rowpart[seg_start * DCG_TB + tid] = a;
                }
            } else {
                // both halves of the flush buffer in use: a second barrier
                // instead of the alternation
                double* rr = rowred + (tid >= DCG_TB ? DCG_NW * DCG_TB : 0);
                rowred[warp * DCG_TB + 2 * lane] = row0;
                rowred[warp * DCG_TB + 2 * lane + 1] = row1;
                rowred[DCG_NW * DCG_TB + warp * DCG_TB + 2 * lane] = rowb0;
                rowred[DCG_NW * DCG_TB + warp * DCG_TB + 2 * lane + 1] = rowb1;
                cta_sync();
                if (tid < 2 * DCG_TB) {
                    const int c = tid & (DCG_TB - 1);
                    double a = 0.0;
#pragma unroll
                    for (int w = 0; w < DCG_NW; ++w) a += rr[w * DCG_TB + c];
                    (tid >= DCG_TB ? rowpart + part2 : rowpart)[seg_start * DCG_TB + c] = a;
                }
                cta_sync();
                rowb0 = rowb1 = 0.0;
            }
            row0 = row1 = 0.0;
            seg_start = t0 + lt + 1;
            ++flush;
        }
        if (++J > I) {
            ++I;
            J = 0;
            if (lt + 1 < ntiles) {
                xI0 = sym_xval(v, NV == 2 ? nullptr : s, I * DCG_TB + 2 * lane, n);
                xI1 = sym_xval(v, NV == 2 ? nullptr : s, I * DCG_TB + 2 * lane + 1, n);
                if constexpr (NV == 2) {
                    yI0 = sym_xval(v2, nullptr, I * DCG_TB + 2 * lane, n);
                    yI1 = sym_xval(v2, nullptr, I * DCG_TB + 2 * lane + 1, n);
                }
            }
        }
    }
    cta_sync();
    if constexpr (PK) {
        // every stage is consumed (the barrier above): the next pass's first
        // tiles go out now, before the grid barriers, without empty waits
        if (prefetch && pending) {
            const int np = ntiles < DCG_SYM_STAGES - 1 ? ntiles : DCG_SYM_STAGES - 1;
            if (tid == 0) {
                for (int st = 0; st < np; ++st) {
                    const unsigned int q = seq + st;
                    const int stg = q % DCG_SYM_STAGES;
                    sym_mbar_expect_tx(full + stg, (unsigned)(DCG_SYM_TILE_DOUBLES * sizeof(double)));
                    sym_bulk_tile(ring + stg * DCG_SYM_STAGE_DOUBLES, K + (t0 + st) * DCG_SYM_TILE_DOUBLES, full + stg,
                                  pol);
                }
            }
            *pending = np;
        }
    }
}

// Pass 2: t_i for rows [q0, q1) (sym_row_begin partition) from the partials;
// epi(i, t_i) runs on one thread per row.  `tbl` is the pass-1 range table of
// `nranges` ranges (one per CTA, or per team of the matrix-free pass 1),
// `red` 512 doubles of shared scratch.  A round covers 32 * nwr consecutive
// rows (lane = row, so a warp's loads of one tile partial are coalesced); the
// 16 / nwr warps sharing a row slice each sum a strided subset of the column
// partials with up to 16 independent loads in flight, then the subsets are
// combined in a fixed order.
// DEEP: two rounds of 16 partial loads in flight before their adds (the
// standalone products; inside the persistent solve kernel, whose pass 1
// shares the register budget, one round measured faster).  a[q] takes its
// partials in the same sequence either way: bitwise the same sums.
template <bool DEEP = false, class Epi>
__device__ __forceinline__ void sym_pass2(long long n, const double* colpart, const double* rowpart, long long q0,
                                          long long q1, const long long* tbl, int nranges, double* red, Epi&& epi) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long NT = sym_ntiles_side(n);
    const long long R = q1 - q0;
    if (R <= 0) return;
    const int nwr = (int)min((R + 31) / 32, (long long)DCG_NW);   // row warps per round
    const int S = DCG_NW / nwr;                                    // warps per row slice
    const int slice = warp / S, sub = warp % S;
    const bool active = slice < nwr;                               // (16 % nwr leftovers idle)
    const int G = nranges;
    for (long long rb = q0; rb < q1; rb += 32LL * nwr) {
        const long long i = rb + 32LL * slice + lane;
        double acc = 0.0;
        if (active && i < q1) {
            const long long I = i / DCG_TB;
            const int r = (int)(i - I * DCG_TB);
            double a[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) a[q] = 0.0;
            // tiles (Ip, I), Ip = I + 1 + sub + S u: base(Ip + S) - base(Ip) =
            // S Ip + S (S + 1) / 2, so the next partial is one pointer add away
            // (the 64-bit row-base products dominated this loop otherwise)
            const int NTi = (int)NT;
            int Ip = (int)I + 1 + sub;
            const double* ptr = colpart + (sym_tile_row_base(Ip) + I) * DCG_TB + r;
            const long long sstep = (long long)S * (S + 1) / 2;
            if constexpr (!DEEP) {
                while (Ip < NTi) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        if (Ip < NTi) {
                            a[q] += ld_cg(ptr);
                            ptr += ((long long)S * Ip + sstep) * DCG_TB;
                            Ip += S;
                        }
                    }
                }
            }
            while (DEEP && Ip < NTi) {
                double v[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    v[q] = 0.0;
                    if (Ip < NTi) {
                        v[q] = ld_cg(ptr);
                        ptr += ((long long)S * Ip + sstep) * DCG_TB;
                        Ip += S;
                    }
                }
#pragma unroll
                for (int q = 0; q < 16; ++q) a[q] += v[q];
#pragma unroll
                for (int q = 0; q < 16; ++q) a[q] += v[16 + q];
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) a[q] += a[q + 8];
            acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
            if (sub == 0) {
                // row segments of tile row I: one starts at J = 0, one at every
                // pass-1 range start inside the row (empty ranges counted once)
                const long long base = sym_tile_row_base(I);
                acc += ld_cg(rowpart + base * DCG_TB + r);
                int lo = 0, hi = G + 1;   // first b with tbl[b] > base
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (tbl[mid] > base) hi = mid; else lo = mid + 1;
                }
                for (int b = lo; b <= G && tbl[b] <= base + I; ++b)
                    if (tbl[b] > tbl[b - 1]) acc += ld_cg(rowpart + tbl[b] * DCG_TB + r);
            }
        }
        if (S > 1) {
            red[tid] = acc;
            cta_sync();
            if (sub == 0 && active && i < q1) {
                double t = acc;
                for (int u = 1; u < S; ++u) t += red[(warp + u) * 32 + lane];
                epi(i, t);
            }
            cta_sync();
        } else if (active && i < q1) {
            epi(i, acc);
        }
    }
}
