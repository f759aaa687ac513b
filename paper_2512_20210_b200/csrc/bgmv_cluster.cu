// bf16 paged BGMV (decode) on thread-block clusters: the hot path behind
// plora_bgmv for bf16 stores.
//
//   y[t, :] += scale · (x[t, :] · A_{a(t)}ᵀ) · B_{a(t)}ᵀ
//
// with A / Bᵀ rows read straight out of the page arena through the device
// page table (the translation PagePool::translate does on the host,
// src/memory.cpp:55-62).
//
// Decomposition.  A job is one adapter's tokens (<= kJobTok) at one
// (layer, proj); its rank rows are cut into chunks of kChunkRows.  A cluster
// of CS CTAs (4 for Llama-7B widths) owns a list of jobs, LPT-balanced on
// the host by weight bytes.  Every CTA of the cluster walks the same chunk
// list: CTA c streams the c-th input slice of the chunk's A rows and the
// c-th output slice of its Bᵀ rows (both independent of the activations, so
// both are in flight at once), computes the partial v_c = x[:, slice_c] ·
// A[rows, slice_c]ᵀ and pushes it into every peer's shared memory with
// st.async (completing bytes on the peer's exchange mbarrier).  After the
// exchange each CTA holds the full v for the chunk and accumulates
// v · Bᵀ[rows, slice_c] in registers; y is read once (TMA, prefetched with
// x at the job's first chunk) and written once at the job's last chunk.  No
// global-memory flags, no atomics; the only cross-CTA traffic is R·T floats
// per chunk over DSMEM.
//
// Pipelining.  Page-producer warps issue 1-D TMA bulk copies (one per page
// piece, L2 evict-first) into two rings: the chunk's A rows (read by the
// shrink) and its Bᵀ rows (read by the expand, after the exchange) live in
// separate slots, so an A slot is recycled as soon as the shrink is done and
// a Bᵀ slot is only filled shortly before the expand needs it — each byte of
// the ring is held for its own consumer's latency, not for the whole
// shrink → exchange → expand chain.  Weights of the next call are issued
// before griddepcontrol.wait (PDL), activations after it.  The shrink runs at
// most kCredit chunks ahead of this CTA's expand (exchange-slot reuse).
#include <cuda_bf16.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "plan.hpp"
#include "ptx.cuh"

namespace plora {
namespace {

constexpr uint32_t kSWarps = 4;  // shrink group
constexpr uint32_t kEWarps = 8;  // expand group
constexpr uint32_t kCWarps = kSWarps + kEWarps;
constexpr uint32_t kCThreads = kCWarps * 32;
constexpr uint32_t kPWarps = 4;                // page producer warps (TMA issue is per-lane serial)
constexpr uint32_t kThreads = kCThreads + (kPWarps + 1) * 32;  // + one control warp
constexpr uint32_t kX = 16;                    // exchange slots (> 2 · kCredit + 1, see shrink_group)
constexpr uint32_t kCredit = 6;                // shrink may lead this CTA's expand by this many chunks
constexpr uint32_t kJobBufs = 4;               // x / y row buffers: jobs in flight (a job is often 1-2 chunks)
constexpr uint32_t kMaxCs = 8;
constexpr uint32_t kMaxSlots = 8;  // per ring (A rows / Bᵀ rows)
constexpr uint32_t kXSlotFloats = kJobTok * kChunkRows * kMaxCs;  // [t][row][src cta]
constexpr uint32_t kSmemBudget = 227 * 1024;  // the sm_100 opt-in maximum per CTA
constexpr uint32_t kMaxSlice = 1024;  // elements per CTA slice (preferred)
constexpr uint32_t kMaxClusters = 64;  // 148 SMs / clusters of >= 4

struct CArgs {
  const char* arena;
  const uint32_t* table;
  const ClusterChunk* chunks;
  const char* x;
  uint64_t x_stride_b;
  // per projection of the launch (chunk record field `proj`): output, its row
  // stride, and where the (layer, proj) block of a rank-r adapter starts
  // (element r · blk_mult)
  char* y[PLORA_MAX_PROJ];
  uint64_t y_stride_b[PLORA_MAX_PROJ];
  uint64_t blk_mult[PLORA_MAX_PROJ];
  // multi-layer launch (plora_bgmv_layers): every cluster's chunk list runs
  // n_layers times; pass li of it serves layer layer0 + li, whose x / y rows
  // are li·x_lstride_b / li·y_lstride_b[proj] bytes further and whose blocks
  // start li·plu elements further (per unit of rank)
  uint32_t n_layers, np;
  uint64_t x_lstride_b;
  uint64_t y_lstride_b[PLORA_MAX_PROJ];
  uint64_t plu;
  uint32_t log2_page;
  uint32_t d_in, d_out;
  uint32_t cs, ks, ns;  // cluster size, slice widths (elements)
  uint32_t na, nbs, a_bytes, b_bytes, jb_bytes;  // ring depths and slot sizes (A rows, Bᵀ rows)
  uint32_t off_b, off_jb, off_xb, off_bar, off_hdr, off_part, off_ring;
  uint32_t fast;  // every row slice lies inside one page (see my_piece)
  float scale;
  uint64_t* trace;  // diagnostics (plora_debug_set_trace) or nullptr
  // cluster c runs chunks [cl_off[c], cl_off[c + 1]): a kernel parameter, so
  // the prologue's first dependent load is the chunk record itself
  uint32_t cl_off[kMaxClusters + 1];
  uint32_t cl_jobs[kMaxClusters];  // jobs in cluster c's list (virtual job ordinals across passes)
};

// Position of virtual chunk v of a cluster's n_layers-fold list: the pass
// (layer offset) and the chunk record's global index.
struct VPos {
  uint32_t li, gi;
};
__device__ __forceinline__ VPos vpos(uint32_t v, uint32_t i0, uint32_t nch) {
  const uint32_t li = v / nch;
  return VPos{li, i0 + (v - li * nch)};
}

constexpr uint32_t kTraceChunks = 64;
__device__ __forceinline__ uint64_t now_ns() {  // SM cycles (cheap; %globaltimer is not)
  return clock64();
}
__device__ __forceinline__ void trace_put(const CArgs& p, uint32_t k, int field) {
  if (p.trace && k < kTraceChunks) p.trace[(blockIdx.x * kTraceChunks + k) * 16 + field] = now_ns();
}

struct Bars {
  uint64_t* afull;   // [kMaxSlots] chunk A rows landed (+ header)
  uint64_t* aempty;  // [kMaxSlots] A slot free (shrink done)
  uint64_t* bfull;   // [kMaxSlots] chunk Bᵀ rows landed (+ header)
  uint64_t* bempty;  // [kMaxSlots] Bᵀ slot free (expand done)
  uint64_t* jfull;   // [kJobBufs] job x / y rows landed
  uint64_t* jempty;  // [kJobBufs] job buffer free
  uint64_t* xfull;   // [kX] all CS partials of a chunk landed
  __device__ explicit Bars(char* smem, uint32_t off) {
    afull = reinterpret_cast<uint64_t*>(smem + off);
    aempty = afull + kMaxSlots;
    bfull = aempty + kMaxSlots;
    bempty = bfull + kMaxSlots;
    jfull = bempty + kMaxSlots;
    jempty = jfull + kJobBufs;
    xfull = jempty + kJobBufs;
  }
};
constexpr uint32_t kBarBytes = (4 * kMaxSlots + 2 * kJobBufs + kX) * 8;
// chunk records of the A slots, of the Bᵀ slots, then the expand's progress
// counter (chunks done, read by the shrink's credit check)
constexpr uint32_t kHdrBytes = 2 * kMaxSlots * sizeof(ClusterChunk) + 16;
// The shrink group runs as two independent subgroups of kSubWarps warps on
// alternating chunks: its per-chunk time is mostly fixed latency, so two
// chunks in flight nearly double its throughput.
constexpr uint32_t kSubWarps = 2;
constexpr uint32_t kSubgroups = kSWarps / kSubWarps;
constexpr uint32_t kPartBytes = kSubgroups * 2 * kSubWarps * kJobTok * kChunkRows * 4;  // shrink partials

struct Slice {  // this CTA's input / output slice
  uint32_t k0, kb, n0, nb;  // first element, width (elements; may be 0 for tiny widths)
  __device__ Slice(const CArgs& p, uint32_t crank) {
    k0 = min(crank * p.ks, p.d_in);
    kb = min(p.ks, p.d_in - k0);
    n0 = min(crank * p.ns, p.d_out);
    nb = min(p.ns, p.d_out - n0);
  }
};

// Shared-memory row stride of a slice row: 16 bytes of padding so the eight
// rows an ldmatrix touches fall in different banks (unpadded 2 KiB rows put
// all eight in the same bank: an 8-way conflict on every fragment load).
__host__ __device__ constexpr uint32_t row_stride(uint32_t elems) { return elems * 2 + 16; }

__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

__device__ __forceinline__ float dot8(const uint4 a, const uint4 b, float acc) {
  acc = fmaf(bf_lo(a.x), bf_lo(b.x), acc);
  acc = fmaf(bf_hi(a.x), bf_hi(b.x), acc);
  acc = fmaf(bf_lo(a.y), bf_lo(b.y), acc);
  acc = fmaf(bf_hi(a.y), bf_hi(b.y), acc);
  acc = fmaf(bf_lo(a.z), bf_lo(b.z), acc);
  acc = fmaf(bf_hi(a.z), bf_hi(b.z), acc);
  acc = fmaf(bf_lo(a.w), bf_lo(b.w), acc);
  acc = fmaf(bf_hi(a.w), bf_hi(b.w), acc);
  return acc;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ---------------------------------------------------------------- producer
// One page piece of a chunk's copies, resolved through the page table.
struct Piece {
  uint32_t phys;    // physical page (loaded from the device page table)
  uint32_t inpage;  // byte offset inside the page
  uint32_t dst;     // byte offset inside the ring slot
  uint32_t len;     // bytes (0 = no piece)
};

struct Rec {  // chunk record fields (ClusterChunk), read from a smem ring
  uint32_t table_off, rank, ntok, flags, row0, nrows, proj, li;
  uint64_t blk;  // block offset multiplier of this chunk's (layer, proj): A starts at rank · blk
  __device__ Rec(const uint32_t* w, const CArgs& p, uint32_t pass) {
    table_off = w[0];
    rank = w[1] & 0xffffu;
    ntok = (w[1] >> 16) & 0xffu;
    flags = w[1] >> 24;
    row0 = w[2] & 0xffffu;
    nrows = (w[2] >> 16) & 0xffu;
    proj = w[2] >> 24;
    li = pass;
    blk = p.blk_mult[proj] + static_cast<uint64_t>(pass) * p.plu;
  }
};

struct PieceGeom {
  uint32_t KB, NB, KSB, NSB, pprA, pprB;
};

// Piece q of chunk `c`'s A rows (isb = false) or Bᵀ rows (isb = true):
// logical page, offset in the page, destination in the slot, length (0 = no
// piece).
__device__ __forceinline__ uint32_t piece_geom(const CArgs& p, const Slice& sl,
                                               const PieceGeom& pg, const Rec& c, bool isb,
                                               uint32_t q, Piece& out) {
  out.len = 0;
  const uint32_t ppr = isb ? pg.pprB : pg.pprA;
  if (q >= c.nrows * ppr) return 0;
  const uint32_t L = p.log2_page;
  const uint64_t a_base = static_cast<uint64_t>(c.rank) * c.blk;  // elements
  const uint32_t r = q / ppr, k = q - r * ppr;
  uint64_t lo;
  uint32_t len, dst;
  if (!isb) {
    lo = (a_base + static_cast<uint64_t>(c.row0 + r) * p.d_in + sl.k0) * 2;
    len = pg.KB;
    dst = r * pg.KSB;
  } else {
    lo = (a_base + static_cast<uint64_t>(c.rank) * p.d_in +
          static_cast<uint64_t>(c.row0 + r) * p.d_out + sl.n0) * 2;
    len = pg.NB;
    dst = r * pg.NSB;
  }
  const uint64_t hi = lo + len, page = (lo >> L) + k;
  const uint64_t a = max(lo, page << L), b = min(hi, (page + 1) << L);
  if (a >= b) return 0;
  out.inpage = static_cast<uint32_t>(a & ((1ull << L) - 1));
  out.dst = dst + static_cast<uint32_t>(a - lo);
  out.len = static_cast<uint32_t>(b - a);
  return static_cast<uint32_t>(page);
}

__device__ __forceinline__ void cp_async_4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Producer lookahead, all through cp.async into two small smem rings so no
// register ever waits on an in-flight load: at chunk i it fetches the record
// of chunk i + 2·kAhead and the page-table entries of chunk i + kAhead, and
// issues chunk i's bulk copies from entries fetched kAhead chunks earlier.
// (Under a busy HBM a dependent global load takes ~1-1.5 µs.)
constexpr int kAhead = 4;
constexpr uint32_t kRecRing = 2 * kAhead;  // records, 32 bytes each
constexpr uint32_t kRingBytes = kRecRing * 32 + kAhead * 32 * 4 * 3;  // records | entries | geometry

// This lane's page piece of chunk c.  Producer warps 0-1 stream the A rows,
// warps 2-3 the Bᵀ rows; the two warps of a ring take alternate chunks.
// Aligned fast path (p.fast: every row slice lies inside one page): lane r
// < 8 copies row r — a shift, no division.  Generic path: pieces 0..31 of
// the role's piece_geom enumeration on the 32 lanes (the rest go through
// the small-page loop).
__device__ __forceinline__ uint32_t my_piece(const CArgs& p, const Slice& sl, const PieceGeom& pg,
                                             const Rec& c, uint32_t pw, uint32_t lane, Piece& x) {
  x.len = 0;
  if (p.fast) {
    const uint32_t r = lane;
    if (r >= c.nrows) return 0;
    const bool isb = pw >= 2;
    const uint64_t lo =
        (isb ? static_cast<uint64_t>(c.rank) * (c.blk + p.d_in) +
                   static_cast<uint64_t>(c.row0 + r) * p.d_out + sl.n0
             : static_cast<uint64_t>(c.rank) * c.blk +
                   static_cast<uint64_t>(c.row0 + r) * p.d_in + sl.k0) * 2;
    x.len = isb ? pg.NB : pg.KB;
    x.dst = isb ? r * pg.NSB : r * pg.KSB;
    x.inpage = static_cast<uint32_t>(lo & ((1ull << p.log2_page) - 1));
    return static_cast<uint32_t>(lo >> p.log2_page);
  }
  return piece_geom(p, sl, pg, c, pw >= 2, lane, x);
}

// Page warp pw of kPWarps (0-1: A ring, 2-3: Bᵀ ring) owns the chunks
// idx ≡ pw (mod 2) of its ring: waits for the chunk's slot, issues all of the
// chunk's page pieces of its ring (my_piece), publishes the chunk record in
// the slot header and arms the slot barrier with the chunk's bytes
// (arrive.expect_tx after the copies: the phase cannot complete before this
// arrival, so the order is safe).  Alternating chunks halve each warp's
// per-chunk issue and lookahead cost (the bulk copies of a warp issue
// serially).  Both ring depths are even, so a slot's previous chunk was this
// warp's own and its parity waits never run a lap ahead.
__device__ void page_producer(const CArgs& p, char* smem, uint32_t crank, uint32_t cl, uint32_t pw) {
  const uint32_t lane = threadIdx.x & 31;
  Bars bar(smem, p.off_bar);
  uint32_t* recring = reinterpret_cast<uint32_t*>(smem + p.off_ring + pw * kRingBytes);  // [kRecRing][8]
  uint32_t* tblring = recring + kRecRing * 8;                                           // [kAhead][32]
  uint2* georing = reinterpret_cast<uint2*>(tblring + kAhead * 32);  // [kAhead][32] {inpage, dst | len << 16}
  const uint32_t* recg = reinterpret_cast<const uint32_t*>(p.chunks);
  const Slice sl(p, crank);
  const uint64_t ef = ptx::policy_evict_first(), el = ptx::policy_evict_last();
  const uint32_t L = p.log2_page;
  PieceGeom pg;
  pg.KB = sl.kb * 2;
  pg.NB = sl.nb * 2;
  pg.KSB = row_stride(p.ks);
  pg.NSB = row_stride(p.ns);
  pg.pprA = pg.KB ? ((pg.KB - 1) >> L) + 2 : 0;  // page pieces per row (upper bound)
  pg.pprB = pg.NB ? ((pg.NB - 1) >> L) + 2 : 0;
  const uint32_t i0 = p.cl_off[cl], nch = p.cl_off[cl + 1] - i0;
  const uint32_t w2 = pw & 1u;
  const uint32_t n = (nch * p.n_layers + 1 - w2) / 2;  // this warp's chunks: idx = 2j + w2
  const uint32_t njobs = p.cl_jobs[cl];
  auto fetch_rec = [&](uint32_t j) {  // 32-byte record of local chunk j: lanes 0, 1 copy 16 bytes each
    if (lane < 2 && j < n)
      ptx::cp_async_16(recring + (j % kRecRing) * 8 + lane * 4,
                       recg + vpos(2 * j + w2, i0, nch).gi * 8 + lane * 4, 16);
  };
  auto fetch_tbl = [&](uint32_t j) {  // page-table entry of this lane's piece of local chunk j
    if (j >= n) return;
    const Rec c(recring + (j % kRecRing) * 8, p, vpos(2 * j + w2, i0, nch).li);
    Piece x{};
    const uint32_t page = my_piece(p, sl, pg, c, pw, lane, x);
    if (x.len)
      cp_async_4(ptx::smem_u32(tblring + (j % kAhead) * 32 + lane), p.table + c.table_off + page);
    // the piece's geometry rides along, so the issue step does not recompute it
    georing[(j % kAhead) * 32 + lane] = make_uint2(x.inpage, x.len ? (x.dst | (x.len << 16)) : 0u);
  };
  // prologue: records 0 .. 2·kAhead-1 (waited), table entries 0 .. kAhead-1 (one group each)
  for (uint32_t j = 0; j < kRecRing; ++j) fetch_rec(j);
  ptx::cp_async_commit();
  cp_async_wait_group<0>();
  __syncwarp();
  for (uint32_t j = 0; j < static_cast<uint32_t>(kAhead); ++j) {
    fetch_tbl(j);
    ptx::cp_async_commit();
  }
#pragma unroll 1
  const bool isb = pw >= 2;
  const uint32_t nslots = isb ? p.nbs : p.na;
  uint64_t* fullb = isb ? bar.bfull : bar.afull;
  uint64_t* emptyb = isb ? bar.bempty : bar.aempty;
  uint32_t* hdr = reinterpret_cast<uint32_t*>(smem + p.off_hdr) + (isb ? kMaxSlots * 8 : 0);
  uint32_t s = w2, ph = 0;  // slot, its phase parity (no division per chunk)
  for (uint32_t j = 0; j < n; ++j) {
    const uint32_t idx = 2 * j + w2;
    cp_async_wait_group<kAhead - 1>();  // table entries of j, record of j + kAhead
    __syncwarp();
    if (pw == 0 && lane == 0) trace_put(p, idx, 6);
    const uint32_t* rw = recring + (j % kRecRing) * 8;
    const Rec c(rw, p, vpos(idx, i0, nch).li);
    char* sb = smem + (isb ? p.off_b + s * p.b_bytes : s * p.a_bytes);
    const uint2 geo = georing[(j % kAhead) * 32 + lane];
    Piece pc;
    pc.inpage = geo.x;
    pc.dst = geo.y & 0xffffu;
    pc.len = geo.y >> 16;
    const uint32_t phys = pc.len ? tblring[(j % kAhead) * 32 + lane] : 0u;
    if (pw == 0 && lane == 0) trace_put(p, idx, 4);
    ptx::mbar_wait(&emptyb[s], ph ^ 1u);
    if (pw == 0 && lane == 0) trace_put(p, idx, 5);
    uint32_t bytes = pc.len;
    const uint64_t pol = (c.flags & kChunkReuse) ? el : ef;  // pages read again by later jobs stay in L2
    if (pc.len)
      ptx::bulk_g2s_hint(sb + pc.dst, p.arena + (static_cast<uint64_t>(phys) << L) + pc.inpage,
                         pc.len, &fullb[s], pol);
    if (!p.fast) {  // small pages: the role's pieces past the first 32, synchronous lookups
      for (uint32_t q = 32 + lane; q < c.nrows * (isb ? pg.pprB : pg.pprA); q += 32) {
        Piece x;
        const uint32_t page = piece_geom(p, sl, pg, c, isb, q, x);
        if (x.len) {
          ptx::bulk_g2s_hint(sb + x.dst,
                             p.arena + (static_cast<uint64_t>(__ldg(p.table + c.table_off + page)) << L) +
                                 x.inpage,
                             x.len, &fullb[s], pol);
          bytes += x.len;
        }
      }
    }
    if (pw == 0 && lane == 0) trace_put(p, idx, 12);
    if (p.fast) {  // the chunk's rows × their slice bytes, no reduction needed
      bytes = c.nrows * (isb ? pg.NB : pg.KB);
    } else {
      bytes = __reduce_add_sync(0xffffffffu, bytes);
    }
    if (lane == 0) {  // publish the record in the slot header, released by the arrival
      // (virtual fields for the consumers: proj byte = pass · np + proj, jord
      // = pass · jobs + jord, so job buffers cycle across passes)
      const uint4* src = reinterpret_cast<const uint4*>(rw);
      uint4* dst = reinterpret_cast<uint4*>(hdr + s * 8);
      uint4 w0 = src[0];
      w0.z = (w0.z & 0x00ffffffu) | ((c.li * p.np + c.proj) << 24);
      w0.w += c.li * njobs;
      dst[0] = w0;
      dst[1] = src[1];
      ptx::mbar_arrive_expect_tx(&fullb[s], bytes);
    }
    __syncwarp();  // the record ring slot is refilled below
    s += 2;
    if (s >= nslots) {
      s -= nslots;
      ph ^= 1u;
    }
    // ---- lookahead: table entries of j + kAhead (its record landed), record of
    // j + 2·kAhead into the ring slot j just vacated
    fetch_tbl(j + kAhead);
    fetch_rec(j + kRecRing);
    ptx::cp_async_commit();
  }
  cp_async_wait_group<0>();
}

// Control warp: at a job's first chunk, loads the job's x / y slices into a
// job buffer — after griddepcontrol.wait, since the activations are written
// by earlier kernels in the stream.
__device__ void control_producer(const CArgs& p, char* smem, uint32_t crank, uint32_t cl) {
  const uint32_t lane = threadIdx.x & 31;
  Bars bar(smem, p.off_bar);
  uint32_t* recring = reinterpret_cast<uint32_t*>(smem + p.off_ring + kPWarps * kRingBytes);
  const uint32_t* recg = reinterpret_cast<const uint32_t*>(p.chunks);
  const Slice sl(p, crank);
  const uint32_t KB = sl.kb * 2, NB = sl.nb * 2, KSB = row_stride(p.ks), NSB = row_stride(p.ns);
  const uint32_t i0 = p.cl_off[cl], nch = p.cl_off[cl + 1] - i0;
  const uint32_t n = nch * p.n_layers;
  auto fetch_rec = [&](uint32_t j) {
    if (lane < 2 && j < n)
      ptx::cp_async_16(recring + (j % kRecRing) * 8 + lane * 4, recg + vpos(j, i0, nch).gi * 8 + lane * 4, 16);
  };
  for (uint32_t j = 0; j < kAhead; ++j) {
    fetch_rec(j);
    ptx::cp_async_commit();
  }
  uint32_t jord = 0;
  bool waited = false;
#pragma unroll 1
  for (uint32_t idx = 0; idx < n; ++idx) {
    cp_async_wait_group<kAhead - 1>();
    __syncwarp();
    const uint32_t* rw = recring + (idx % kRecRing) * 8;
    const Rec c(rw, p, vpos(idx, i0, nch).li);
    if (c.flags & kChunkFirst) {  // the job's x / y slices
      const uint32_t jbuf = jord % kJobBufs, jph = (jord / kJobBufs) & 1u;
      ++jord;
      char* jb = smem + p.off_jb + jbuf * p.jb_bytes;
      const uint32_t tokx = rw[4 + (lane & 3)];
      ptx::mbar_wait(&bar.jempty[jbuf], jph ^ 1u);
      if (!waited) {
        ptx::pdl_wait();
        waited = true;
      }
      if (lane == 0) ptx::mbar_arrive_expect_tx(&bar.jfull[jbuf], c.ntok * (KB + NB));
      __syncwarp();
      if (lane < c.ntok && KB)
        ptx::bulk_g2s(jb + lane * KSB, p.x + c.li * p.x_lstride_b + tokx * p.x_stride_b + sl.k0 * 2, KB,
                      &bar.jfull[jbuf]);
      else if (lane >= 16 && lane - 16 < c.ntok && NB)
        ptx::bulk_g2s(jb + kJobTok * KSB + (lane - 16) * NSB,
                      p.y[c.proj] + c.li * p.y_lstride_b[c.proj] + tokx * p.y_stride_b[c.proj] + sl.n0 * 2,
                      NB, &bar.jfull[jbuf]);
    }
    __syncwarp();
    fetch_rec(idx + kAhead);
    ptx::cp_async_commit();
  }
  cp_async_wait_group<0>();
  if (!waited) ptx::pdl_wait();
}

// ---------------------------------------------------------------- consumers
// Two warp groups work on consecutive chunks at once (their latency chains
// overlap instead of adding up); both contractions run on warp-level tensor
// cores (M = tokens <= 4 is far below a tcgen05 tile and the kernel is
// HBM-bound — the MMAs keep the instruction count per streamed byte low):
//  shrink group (warps 0-3)  D[tok][row] = x[tok, slice] · W[row, slice]ᵀ,
//      m16n8k16, x rows as A and the chunk's 8 A rows as B (ldmatrix), 16
//      k-steps per warp; the 4 warp partials are summed in a fixed order and
//      pushed into every cluster peer's exchange slot (st.async).
//  expand group (warps 4-11)  Dᵀ[col][tok] += Bᵀ[row][col]ᵀ · v[tok][row]ᵀ,
//      m16n8k8 with 16 output columns per MMA (Bᵀ fragments by
//      ldmatrix.trans); v is split into bf16 hi + lo (~16 mantissa bits of
//      the fp32 v) packed side by side in N, so one MMA applies both halves;
//      accumulators stay in registers across a job.
constexpr uint32_t kSThreads = kSWarps * 32;
constexpr uint32_t kEThreads = kEWarps * 32;
constexpr uint32_t kMaxTiles = (1024 / 16 + kEWarps - 1) / kEWarps;  // 16-column expand tiles per warp (ns <= 1024)

__device__ void shrink_group(const CArgs& p, char* smem, uint32_t crank, uint32_t cl) {
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t gq = lane >> 2, cc = lane & 3;
  const Bars bar(smem, p.off_bar);
  const Slice sl(p, crank);
  const uint32_t KSB = row_stride(p.ks);
  const uint32_t ksteps = (sl.kb + 15) / 16;  // the last one may be half (kb % 16 == 8)
  const bool half_tail = (sl.kb & 15u) != 0;
  const uint32_t xb0 = ptx::smem_u32(smem + p.off_xb);
  float* part = reinterpret_cast<float*>(smem + p.off_part);  // [2][warp][tok][row]
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(smem + p.off_hdr);  // A-slot records
  const volatile uint32_t* edone =
      reinterpret_cast<const volatile uint32_t*>(smem + p.off_hdr + 2 * kMaxSlots * sizeof(ClusterChunk));
  const uint32_t n = (p.cl_off[cl + 1] - p.cl_off[cl]) * p.n_layers;
  // ldmatrix lane addressing: A (x rows) = row (lane&7) + 8·((lane>>3)&1), k-half lane>>4
  // (rows >= kJobTok alias row 0: their D rows are discarded); B (W rows, x4 =
  // two k-steps) = row lane&7, k-quarter lane>>3
  const uint32_t xrow = (lane & 7) + ((lane >> 3) & 1) * 8;
  const uint32_t xoff = (xrow < kJobTok ? xrow : 0) * KSB + (lane >> 4) * 16;
  const uint32_t woff = (lane & 7) * KSB + (lane >> 3) * 16;
  const uint32_t sg = w / kSubWarps, sw = w % kSubWarps;  // subgroup, warp within it
  const bool lead = sw == 0 && lane == 0;
#pragma unroll 1
  for (uint32_t idx = sg; idx < n; idx += kSubgroups) {  // this subgroup's chunks
    // (p.na is even: a subgroup's previous chunk in slot s is idx - na, which
    // it consumed itself, so its parity wait is never a ring lap ahead)
    const uint32_t s = idx % p.na, e = idx % kX;
    if (lead) trace_put(p, idx, 14);
    ptx::mbar_wait(&bar.afull[s], (idx / p.na) & 1u);
    if (lead) trace_put(p, idx, 0);
    const ClusterChunk* ch = reinterpret_cast<const ClusterChunk*>(hdr + s * 8);
    const uint32_t ntok = ch->ntok, jord = ch->jord;
    // Every chunk waits for its job's x rows: with two subgroups a job's later
    // chunk can run before (or beside) its first one.  The job buffer cannot be
    // recycled meanwhile (that needs the job's last expand), so the parity is
    // unambiguous.
    ptx::mbar_wait(&bar.jfull[jord % kJobBufs], (jord / kJobBufs) & 1u);
    // Credit: start chunk idx only once this CTA's expand has finished chunk
    // idx - kCredit.  Then arm this chunk's exchange barrier: CS CTAs ×
    // kChunkRows rows × ntok floats.  Peers' st.async may land before this
    // (negative tx count is fine: the phase also needs this arrival).
    // Aliasing bound: a peer's shrink of chunk m + kX needs its expand past
    // m + kX - kCredit, i.e. our partial of that chunk, i.e. our expand past
    // m + kX - 2·kCredit - 1 > m: kX > 2·kCredit + 1 keeps every live phase of
    // an exchange slot distinct.
    if (lead) {
      while (idx >= *edone + kCredit) __nanosleep(32);
      ptx::mbar_arrive_expect_tx(&bar.xfull[e], p.cs * kChunkRows * ntok * 4);
    }
    if (lead) trace_put(p, idx, 15);
    const uint32_t xa = ptx::smem_u32(smem + p.off_jb + (jord % kJobBufs) * p.jb_bytes) + xoff;
    const uint32_t wa = ptx::smem_u32(smem + s * p.a_bytes) + woff;
    // Warp sw takes k-step pairs sw, sw + kSubWarps, ... (<= kPairs of them).  The
    // schedule is software-pipelined by hand — pair j+1's fragment loads are
    // issued before pair j's MMAs, into the other of two register sets (the
    // asm statements keep program order; no register is copied while its
    // load is in flight).
    constexpr uint32_t kPairs = kMaxSlice / 32 / kSubWarps;
    float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
    float d2[4] = {0.f, 0.f, 0.f, 0.f}, d3[4] = {0.f, 0.f, 0.f, 0.f};  // shorter MMA chains
    uint32_t fr[2][3][4];  // [set][W, x k-step 0, x k-step 1]
#pragma unroll
    for (uint32_t j = 0; j <= kPairs; ++j) {
      const uint32_t kn = 2 * (sw + j * kSubWarps);
      if (j < kPairs && kn + 1 < ksteps) {
        ptx::ldsm_x4(wa + kn * 32, fr[j & 1][0]);
        ptx::ldsm_x4(xa + kn * 32, fr[j & 1][1]);
        ptx::ldsm_x4(xa + kn * 32 + 32, fr[j & 1][2]);
      }
      if (j > 0) {
        const uint32_t kp = 2 * (sw + (j - 1) * kSubWarps);
        uint32_t(&f)[3][4] = fr[(j - 1) & 1];
        if (kp + 1 < ksteps) {
          if (half_tail && kp + 1 == ksteps - 1) {  // k 8..15 of the last step lie past the slice
            f[2][2] = f[2][3] = 0u;
            f[0][3] = 0u;
          }
          const uint32_t b0[2] = {f[0][0], f[0][1]}, b1[2] = {f[0][2], f[0][3]};
          ptx::mma_bf16_16816((j & 1) ? d0 : d2, f[1], b0);
          ptx::mma_bf16_16816((j & 1) ? d1 : d3, f[2], b1);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      d0[q] += d2[q];
      d1[q] += d3[q];
    }
    if ((ksteps & 1u) && sw == (ksteps / 2) % kSubWarps) {  // odd number of k-steps: the last one
      const uint32_t k = ksteps - 1;
      uint32_t a0[4], b[4];
      ptx::ldsm_x4(wa + k * 32, b);
      ptx::ldsm_x4(xa + k * 32, a0);
      if (half_tail) {
        a0[2] = a0[3] = 0u;
        b[1] = 0u;
      }
      const uint32_t b0[2] = {b[0], b[1]};
      ptx::mma_bf16_16816(d0, a0, b0);
    }
    // d[0]/d[1] = (tok gq, rows 2cc, 2cc+1).  Each subgroup's partial buffers
    // alternate by its chunk parity: the lead warp reads one before the
    // subgroup's next barrier, which every warp of the subgroup passes before
    // writing that buffer again.
    float* pb = part + (sg * 2 + ((idx / kSubgroups) & 1u)) * kSubWarps * kJobTok * kChunkRows;
    if (gq < kJobTok) {
      float* pw = pb + (sw * kJobTok + gq) * kChunkRows + 2 * cc;
      pw[0] = d0[0] + d1[0];
      pw[1] = d0[1] + d1[1];
    }
    if (lead) trace_put(p, idx, 8);
    if (sg == 0)  // partials written; slot A rows read (constant barrier ids)
      ptx::named_bar_sync(2, kSubWarps * 32);
    else
      ptx::named_bar_sync(3, kSubWarps * 32);
    if (lead) trace_put(p, idx, 9);
    if (sw == 0) {
      if (lane < ntok * kChunkRows) {  // lane = tok · 8 + row: sum the warps, push
        float v = 0.f;
#pragma unroll
        for (uint32_t ww = 0; ww < kSubWarps; ++ww) v += pb[ww * kJobTok * kChunkRows + lane];
        const uint32_t t = lane / kChunkRows, r = lane % kChunkRows;
        const uint32_t local = xb0 + (e * kXSlotFloats + (t * kChunkRows + r) * kMaxCs + crank) * 4;
        const uint32_t lbar = ptx::smem_u32(&bar.xfull[e]);
        for (uint32_t dst = 0; dst < p.cs; ++dst)
          ptx::st_async_b32(ptx::mapa(local, dst), __float_as_uint(v), ptx::mapa(lbar, dst));
      }
      if (lane == 0) {
        trace_put(p, idx, 1);
        ptx::mbar_arrive(&bar.aempty[s]);  // A slot free
      }
    }
  }
}

__device__ void expand_group(const CArgs& p, char* smem, uint32_t crank, uint32_t cl) {
  const uint32_t tid = threadIdx.x - kSThreads, w = tid >> 5, lane = tid & 31;
  const uint32_t gq = lane >> 2, cc = lane & 3;
  const Bars bar(smem, p.off_bar);
  const Slice sl(p, crank);
  const uint32_t NSB = row_stride(p.ns), KSB = row_stride(p.ks);
  const uint32_t* hdr =
      reinterpret_cast<const uint32_t*>(smem + p.off_hdr) + kMaxSlots * 8;  // Bᵀ-slot records
  volatile uint32_t* edone =
      reinterpret_cast<volatile uint32_t*>(smem + p.off_hdr + 2 * kMaxSlots * sizeof(ClusterChunk));
  const uint32_t n = (p.cl_off[cl + 1] - p.cl_off[cl]) * p.n_layers;
  // this warp's 16-column tiles [t0, t1) of the output slice
  const uint32_t ntiles = sl.nb / 16, tpw = (ntiles + kEWarps - 1) / kEWarps;
  const uint32_t t0 = w * tpw, t1 = min(t0 + tpw, ntiles);
  const bool tail8 = (sl.nb & 15u) != 0 && w == kEWarps - 1;  // a last 8-column tile
  ptx::pdl_wait();  // y is written below: the previous call must be complete
  float acc[kMaxTiles + 1][4];
#pragma unroll 1
  for (uint32_t idx = 0; idx < n; ++idx) {
    const uint32_t s = idx % p.nbs, e = idx % kX;
    ptx::mbar_wait(&bar.bfull[s], (idx / p.nbs) & 1u);
    const ClusterChunk* ch = reinterpret_cast<const ClusterChunk*>(hdr + s * 8);
    const uint32_t ntok = ch->ntok, nrows = ch->nrows, flags = ch->flags, jord = ch->jord;
    if (flags & kChunkFirst) {
      ptx::mbar_wait(&bar.jfull[jord % kJobBufs], (jord / kJobBufs) & 1u);  // y rows of the job
#pragma unroll
      for (uint32_t t = 0; t <= kMaxTiles; ++t)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[t][q] = 0.f;
    }
    ptx::mbar_wait(&bar.xfull[e], (idx / kX) & 1u);
    if (tid == 0) trace_put(p, idx, 2);
    // B operand: N packs (token, part): column n = 2·tok + part holds the bf16
    // hi (part 0) or lo (part 1) half of v[tok][row], so one MMA applies both
    // halves and y[tok] = D[·][2·tok] + D[·][2·tok+1].  This lane supplies
    // rows 2cc, 2cc+1 of column gq (tokens >= ntok, rows >= nrows are 0).
    const uint32_t vt = gq >> 1;
    float v0 = 0.f, v1 = 0.f;
    if (vt < ntok) {
      const float* xs = reinterpret_cast<const float*>(smem + p.off_xb) + e * kXSlotFloats;
      const float4* s0 = reinterpret_cast<const float4*>(xs + (vt * kChunkRows + 2 * cc) * kMaxCs);
      const float4* s1 = s0 + kMaxCs / 4;
      float4 q0 = s0[0], q1 = s1[0];
      v0 = (q0.x + q0.y) + (q0.z + q0.w);  // fixed summation order: deterministic
      v1 = (q1.x + q1.y) + (q1.z + q1.w);
      if (p.cs > 4) {
        q0 = s0[1];
        q1 = s1[1];
        v0 += (q0.x + q0.y) + (q0.z + q0.w);
        v1 += (q1.x + q1.y) + (q1.z + q1.w);
      }
      if (2 * cc >= nrows) v0 = 0.f;
      if (2 * cc + 1 >= nrows) v1 = 0.f;
    }
    const uint32_t bhi = pack_bf16x2(v0, v1);
    const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bhi));
    const uint32_t bv = (gq & 1u) ? pack_bf16x2(v0 - hf.x, v1 - hf.y) : bhi;
    if (tid == 0) trace_put(p, idx, 10);
    // Bᵀ rows >= nrows of the slot are stale: mask their halves of the A fragment
    const uint32_t amask =
        (2 * cc < nrows ? 0x0000ffffu : 0u) | (2 * cc + 1 < nrows ? 0xffff0000u : 0u);
    const char* brow = smem + p.off_b + s * p.b_bytes;
    // ldmatrix.trans lane addressing: row (lane&7) of matrix lane>>3 = 8 columns
    const uint32_t brow0 = ptx::smem_u32(brow + (lane & 7) * NSB);
    const uint32_t baddr = brow0 + (lane >> 3) * 16;
#pragma unroll
    for (uint32_t g = 0; g < kMaxTiles; g += 2) {  // two 16-column tiles per ldmatrix.x4
      if (t0 + g < t1) {
        uint32_t a[4];  // a lone last tile also reads the next 16 columns: in-bounds, unused
        ptx::ldsm_x4_trans(baddr + (t0 + g) * 32, a);
#pragma unroll
        for (uint32_t m = 0; m < 2; ++m) {
          if (t0 + g + m < t1) {
            const uint32_t af[2] = {a[2 * m] & amask, a[2 * m + 1] & amask};
            ptx::mma_bf16_1688(acc[g + m], af, bv);
          }
        }
      }
    }
    if (tail8) {  // a final 8-column tile (nb % 16 == 8): MMA rows 8..15 unused
      uint32_t a[2];
      ptx::ldsm_x2_trans(brow0 + ntiles * 32, a);
      const uint32_t af[2] = {a[0] & amask, 0u};
      ptx::mma_bf16_1688(acc[kMaxTiles], af, bv);
    }
    if (tid == 0) trace_put(p, idx, 11);
    if ((flags & kChunkLast) && cc < ntok) {  // y[tok cc] += scale · (hi + lo), once per job
      const char* yrow = smem + p.off_jb + (jord % kJobBufs) * p.jb_bytes + kJobTok * KSB + cc * NSB;
      const uint32_t li = ch->proj / p.np, pj = ch->proj - li * p.np;  // virtual proj byte
      char* yg = p.y[pj] + li * p.y_lstride_b[pj] + ch->tok[cc] * p.y_stride_b[pj] +
                 static_cast<uint64_t>(sl.n0) * 2;
      auto put = [&](uint32_t col, float v) {
        const float o = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(yrow + col * 2));
        *reinterpret_cast<__nv_bfloat16*>(yg + col * 2) = __float2bfloat16_rn(fmaf(p.scale, v, o));
      };
#pragma unroll
      for (uint32_t t = 0; t < kMaxTiles; ++t) {
        if (t0 + t < t1) {  // d0 + d1 = (col gq, tok cc), d2 + d3 = (col gq + 8, tok cc)
          put((t0 + t) * 16 + gq, acc[t][0] + acc[t][1]);
          put((t0 + t) * 16 + gq + 8, acc[t][2] + acc[t][3]);
        }
      }
      if (tail8) put(ntiles * 16 + gq, acc[kMaxTiles][0] + acc[kMaxTiles][1]);
    }
    ptx::named_bar_sync(1, kEThreads);  // slot (and job buffer) reads done
    if (tid == 0) {
      trace_put(p, idx, 3);
      ptx::mbar_arrive(&bar.bempty[s]);
      if (flags & kChunkLast) ptx::mbar_arrive(&bar.jempty[jord % kJobBufs]);
      __threadfence_block();
      *edone = idx + 1;  // credit for the shrink (its exchange slot is read)
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) bgmv_cluster_kernel(const CArgs p) {
  extern __shared__ __align__(128) char smem[];
  ptx::pdl_launch_dependents();  // the next call may start streaming its weights
  const uint32_t crank = ptx::cluster_ctarank();
  const uint32_t cl = blockIdx.x / p.cs;
  if (threadIdx.x == 0) trace_put(p, kTraceChunks - 1, 6);
  if (threadIdx.x == 0) {
    Bars bar(smem, p.off_bar);
    for (uint32_t s = 0; s < kMaxSlots; ++s) {
      ptx::mbar_init(&bar.afull[s], 1);   // the A page warp of the chunk
      ptx::mbar_init(&bar.aempty[s], 1);  // the shrink subgroup of the chunk
      ptx::mbar_init(&bar.bfull[s], 1);   // the Bᵀ page warp of the chunk
      ptx::mbar_init(&bar.bempty[s], 1);           // the expand group
    }
    *reinterpret_cast<uint32_t*>(smem + p.off_hdr + 2 * kMaxSlots * sizeof(ClusterChunk)) = 0u;
    for (uint32_t j = 0; j < kJobBufs; ++j) {
      ptx::mbar_init(&bar.jfull[j], 1);
      ptx::mbar_init(&bar.jempty[j], 1);
    }
    for (uint32_t e = 0; e < kX; ++e) ptx::mbar_init(&bar.xfull[e], 1);
    ptx::fence_mbar_init();
  }
  ptx::cluster_sync();  // peers' exchange barriers are initialised before any st.async
  if (threadIdx.x >= kCThreads + kPWarps * 32)
    control_producer(p, smem, crank, cl);
  else if (threadIdx.x >= kCThreads)
    page_producer(p, smem, crank, cl, (threadIdx.x - kCThreads) >> 5);
  else if (threadIdx.x < kSThreads)
    shrink_group(p, smem, crank, cl);
  else
    expand_group(p, smem, crank, cl);
  ptx::cluster_sync();  // no CTA leaves while a peer may still address its smem
  if (threadIdx.x == 0) trace_put(p, kTraceChunks - 1, 7);
}

std::mutex g_occ_mu;
std::map<std::tuple<int, uint32_t, uint32_t>, int> g_occ;  // (device, cs, smem) -> clusters

int max_clusters(int device, uint32_t cs, uint32_t smem) {
  std::lock_guard<std::mutex> lk(g_occ_mu);
  auto key = std::make_tuple(device, cs, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  PLORA_CUDA(cudaFuncSetAttribute(bgmv_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBudget)));
  int sms = 0;
  PLORA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<uint32_t>(sms) / cs * cs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  PLORA_CUDA(cudaOccupancyMaxActiveClusters(&n, bgmv_cluster_kernel, &cfg));
  if (n <= 0) throw CudaError("bgmv: no cluster of " + std::to_string(cs) + " CTAs fits");
  g_occ[key] = n;
  return n;
}

}  // namespace

ClusterGeom cluster_geom(uint32_t d_in, uint32_t d_out, int device) {
  ClusterGeom g;
  auto slice = [](uint32_t d, uint32_t cs) { return ((d + cs - 1) / cs + 7) / 8 * 8; };
  g.cs = 4;
  while (std::max(slice(d_in, g.cs), slice(d_out, g.cs)) > kMaxSlice && g.cs < kMaxCs) g.cs *= 2;
  g.ks = slice(d_in, g.cs);
  g.ns = slice(d_out, g.cs);
  if (g.ks > kMaxSlice || g.ns > kMaxSlice)  // expand: 4 columns per consumer thread
    throw ValidationError("bf16 BGMV: d_in " + std::to_string(d_in) + " / d_out " +
                          std::to_string(d_out) + " too wide (max " +
                          std::to_string(kMaxSlice * kMaxCs) + ")");
  auto up128 = [](uint32_t b) { return (b + 127) / 128 * 128; };
  g.a_bytes = up128(kChunkRows * row_stride(g.ks));
  g.b_bytes = up128(kChunkRows * row_stride(g.ns));
  g.jb_bytes = up128(kJobTok * (row_stride(g.ks) + row_stride(g.ns)));
  const uint32_t fixed = kJobBufs * g.jb_bytes + kX * kXSlotFloats * 4 + kBarBytes + kHdrBytes + kPartBytes + (kPWarps + 1) * kRingBytes;
  // equal ring depths, the A ring even (two shrink subgroups alternate chunks)
  const uint32_t pairs = fixed < kSmemBudget ? (kSmemBudget - fixed) / (g.a_bytes + g.b_bytes) : 0;
  g.na = std::min<uint32_t>(kMaxSlots, pairs) & ~1u;
  g.nbs = std::min<uint32_t>(kMaxSlots, pairs) & ~1u;  // even: the page warps alternate chunks
  if (g.na < 2 || g.nbs < 2)
    throw ValidationError("bf16 BGMV: d_in " + std::to_string(d_in) + " / d_out " +
                          std::to_string(d_out) + " leave fewer than 2 ring slots");
  g.smem = g.na * g.a_bytes + g.nbs * g.b_bytes + fixed;
  g.n_clusters = std::min<uint32_t>(kMaxClusters, static_cast<uint32_t>(max_clusters(device, g.cs, g.smem)));
  return g;
}

namespace {

void launch(const plora_plan& plan, const ClusterWork& cw, uint32_t layer, const uint32_t* projs,
            uint32_t np, const void* x, uint64_t x_stride, void* const* ys,
            const uint64_t* y_strides, float scale, cudaStream_t stream, uint32_t n_layers = 1,
            uint64_t x_lstride = 0, const uint64_t* y_lstrides = nullptr) {
  const plora_store& st = *plan.store;
  const ModelGeom& gm = st.geom;
  const ClusterGeom& g = cw.geom;
  if (g.n_clusters == 0) return;  // no LoRA token in the batch
  CArgs a{};
  a.arena = st.arena;
  a.table = st.d_table;
  a.chunks = plan.d_cchunks + cw.chunks_off;
  for (uint32_t c = 0; c <= g.n_clusters; ++c) a.cl_off[c] = plan.ccl_off[cw.cl_off + c];
  for (uint32_t c = 0; c < g.n_clusters; ++c) a.cl_jobs[c] = plan.ccl_jobs[cw.cl_off + c];
  if (n_layers == 0 || n_layers * np > 256)
    throw ValidationError("bf16 BGMV: n_layers x projections must be in [1, 256] per launch");
  a.n_layers = n_layers;
  a.np = np;
  a.x_lstride_b = x_lstride * 2;
  a.plu = gm.per_layer_unit;
  a.x = static_cast<const char*>(x);
  a.x_stride_b = x_stride * 2;
  a.log2_page = st.log2_page;
  a.d_in = gm.m.d_in[projs[0]];
  a.d_out = gm.m.d_out[projs[0]];
  if (a.d_in % 8 || a.d_out % 8) throw ValidationError("bf16 BGMV needs d_in and d_out multiples of 8");
  a.cs = g.cs;
  a.ks = g.ks;
  a.ns = g.ns;
  a.na = g.na;
  a.nbs = g.nbs;
  a.a_bytes = g.a_bytes;
  a.b_bytes = g.b_bytes;
  a.jb_bytes = g.jb_bytes;
  a.off_b = g.na * g.a_bytes;
  a.off_jb = a.off_b + g.nbs * g.b_bytes;
  a.off_xb = a.off_jb + kJobBufs * g.jb_bytes;
  a.off_bar = a.off_xb + kX * kXSlotFloats * 4;
  a.off_hdr = a.off_bar + kBarBytes;
  a.off_part = a.off_hdr + kHdrBytes;
  a.off_ring = a.off_part + kPartBytes;
  a.scale = scale;
  const uint64_t P = 1ull << st.log2_page;
  a.fast = a.d_in % a.ks == 0 && a.d_out % a.ns == 0 && P % (2ull * a.ks) == 0 &&
           P % (2ull * a.ns) == 0;
  for (uint32_t i = 0; i < np; ++i) {
    a.y[i] = static_cast<char*>(ys[i]);
    a.y_stride_b[i] = y_strides[i] * 2;
    a.y_lstride_b[i] = y_lstrides ? y_lstrides[i] * 2 : 0;
    a.blk_mult[i] = gm.blk_mult(layer, projs[i]);
    a.fast = a.fast && a.blk_mult[i] % a.ks == 0 && (a.blk_mult[i] + a.d_in) % a.ns == 0 &&
             (n_layers == 1 || a.plu % a.ks == 0);
  }
  a.trace = trace_buffer(g.n_clusters * g.cs * kTraceChunks * 128);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g.n_clusters * g.cs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = g.cs;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  // programmatic dependent launch: this call's weight streaming may overlap
  // the previous call's tail (activations are read after griddepcontrol.wait)
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  PLORA_CUDA(cudaLaunchKernelEx(&cfg, bgmv_cluster_kernel, a));
  count_launch();
}

}  // namespace

void launch_bgmv_cluster(const plora_plan& plan, uint32_t layer, uint32_t proj, const void* x,
                         uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                         cudaStream_t stream) {
  void* ys[1] = {y};
  const uint64_t strides[1] = {y_stride};
  launch(plan, plan.cwork[proj], layer, &proj, 1, x, x_stride, ys, strides, scale, stream);
}

void launch_bgmv_cluster_layer(const plora_plan& plan, uint32_t layer, const void* x,
                               uint64_t x_stride, void* const* ys, const uint64_t* y_strides,
                               float scale, cudaStream_t stream) {
  uint32_t projs[PLORA_MAX_PROJ];
  for (uint32_t i = 0; i < plan.n_layer_proj; ++i) projs[i] = i;
  launch(plan, plan.cwork_layer, layer, projs, plan.n_layer_proj, x, x_stride, ys, y_strides,
         scale, stream);
}

void launch_bgmv_cluster_layers(const plora_plan& plan, uint32_t layer0, uint32_t n_layers,
                                const void* x, uint64_t x_stride, uint64_t x_lstride,
                                void* const* ys, const uint64_t* y_strides,
                                const uint64_t* y_lstrides, float scale, cudaStream_t stream,
                                const ClusterWork* work) {
  uint32_t projs[PLORA_MAX_PROJ];
  for (uint32_t i = 0; i < plan.n_layer_proj; ++i) projs[i] = i;
  launch(plan, work ? *work : plan.cwork_layer, layer0, projs, plan.n_layer_proj, x, x_stride, ys,
         y_strides, scale, stream, n_layers, x_lstride, y_lstrides);
}

namespace {
uint64_t* g_trace = nullptr;
uint64_t g_trace_bytes = 0;
}  // namespace

uint64_t* trace_buffer(uint64_t need_bytes) { return g_trace_bytes >= need_bytes ? g_trace : nullptr; }

}  // namespace plora

extern "C" int plora_debug_set_trace(void* dev_buf, uint64_t bytes) {
  plora::g_trace = static_cast<uint64_t*>(dev_buf);
  plora::g_trace_bytes = dev_buf ? bytes : 0;
  return 0;
}

extern "C" int plora_debug_plan_geom(const plora_plan* plan, uint32_t proj, uint32_t out[8]) {
  using namespace plora;
  return guard([&] {
    if (!plan || !out) throw ValidationError("null plan or out");
    if (proj >= PLORA_MAX_PROJ) throw ValidationError("proj out of range");
    const ClusterWork& cw = plan->cwork[proj];
    const ClusterGeom& g = cw.geom;
    const uint32_t n = g.n_clusters ? plan->ccl_off[cw.cl_off + g.n_clusters] : 0;
    const uint32_t v[8] = {g.cs, g.ks, g.ns, g.na, g.nbs, g.smem, g.n_clusters, n};
    for (int i = 0; i < 8; ++i) out[i] = v[i];
    return 0;
  });
}
