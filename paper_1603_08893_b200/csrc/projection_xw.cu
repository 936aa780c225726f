// x pass for long lines (projection.cpp:137-155: x FFT, ghat, inverse x FFT):
// 512 points with one warp per x-line, 1024 points with the line split over a
// 2-CTA cluster; all HBM traffic by TMA in both directions.
//
// Why (profiles/r2_x512_dbg.md): the streamed pass k_x_stream (one CTA per SM,
// 8 warps walking its tiles in lock-step) took 4.5 ms at 512^3 whatever was
// removed from the memory side -- its transforms alone took 3.2 ms (block
// barriers around every exchange, so the fp64 pipe, shared memory and the
// barriers take turns), and its register stores blocked the warps for as long
// as the 192 KB of a tile took to drain.  Here
//
//  * a tile is (row i of the tensor, y, 8 kz columns) = 3 components x 512 rows
//    x 128 bytes; warp w owns column w and holds its whole 512-point line in
//    registers (lane = 2 t + h: h = 0 the even rows, h = 1 the odd rows, two
//    256-point half-line transforms of 16 lanes x 16 elements joined by the
//    lane-pair radix-2 step of fft_pair.cuh).  The half-line exchange goes
//    through a warp-private 4 KB scratch (real parts, then imaginary parts) with
//    warp-level syncs only, so the eight warps run out of phase and overlap
//    each other's fp64, shared-memory and shuffle phases;
//  * the three 64 KB component buffers are written by tensor-map TMA loads with
//    the 128-byte swizzle (a warp reads its 16-byte column of 8 consecutive
//    rows from 8 different bank groups) and results go back IN PLACE into the
//    warp's own column of a buffer it has already consumed -- no cross-warp
//    dependency -- from where a TMA store writes the tile back;
//  * one copy warp per buffer (their warp group gives its registers to the
//    transform warps, setmaxnreg) issues the buffer's loads and stores: it waits
//    for "all 8 warps have staged this buffer" (mbarrier), stores it, waits until
//    the store has read shared memory and refills the buffer with the next
//    tile's component.
//
// Buffer schedule per tile k (P, Q, R the three buffers):
//   P, Q: A_1(k), A_2(k) arrive -> every warp forms B = xi_y A_1 + xi_z A_2 from
//         its column and writes the PREVIOUS tile's outputs 1 and 2 (still in
//         registers) into the same columns -> staged -> store -> load
//         A_1(k+1), A_2(k+1), almost a whole tile ahead of their use;
//   R:    A_0(k) arrives -> consumed after the first forward transform; output 0
//         goes back into R after the first inverse transform -> staged -> store
//         -> load A_0(k+1), two transforms ahead of its use.
// Same arithmetic, in the same order, as the lane-pair k_x_stream: results are
// bit-identical (tests/test_gpu_projection.py compares the two kernels' outputs).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "bulk.cuh"
#include "fft_pair.cuh"
#include "proj_common.cuh"

namespace fm {
namespace {

constexpr int XN = 512, XH = 256, XTW = 8, XE = 16, XTH = 16;
constexpr int XTILE = XN * XTW * 16;          // bytes of one component tile
constexpr int XSCR = 4096;                    // exchange scratch per warp
// 8 transform warps (two warp groups) + the copy warp's group: 3 warps per SM
// sub-partition would cap every thread at 168 registers, so the copy group
// hands its registers back (setmaxnreg) and the transform groups take 232
constexpr int XTHREADS = 384;
constexpr size_t XSMEM = 1024 + 3 * size_t(XTILE) + XTW * size_t(XSCR) + 256;

// Transposing exchange of the two half-lines of a warp: lane (t, h) hands its
// a[k] to lane (k, h), slot t.  One double per element and round; element p of
// half-line h sits at double index 2 (p ^ ((p >> 4) & 7)) + h, which makes both
// the strided writes (p = 16 t + k) and the unit-stride reads (p = t + 16 m)
// conflict-free for the 16 lanes a 64-bit access serves per wavefront.
// (32-bit shared-space addresses and explicit ld/st.shared: with generic pointers the
// XOR hides the address space and the accesses compile to generic LD / ST.)
__device__ __forceinline__ void exchange(double2 (&v)[XE], unsigned wr0, unsigned rd0) {
#pragma unroll
  for (int part = 0; part < 2; ++part) {
#pragma unroll
    for (int k = 0; k < XE; ++k) {
      const unsigned a = (wr0 ^ unsigned((k & 7) << 4)) + unsigned((k >> 3) << 7);
      asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(part == 0 ? v[k].x : v[k].y) : "memory");
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < XE; ++m) {
      const unsigned a = (rd0 ^ unsigned((m & 7) << 4)) + unsigned(m << 8);
      double x;
      asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(x) : "r"(a) : "memory");
      if (part == 0) v[m].x = x; else v[m].y = x;
    }
    __syncwarp();
  }
}

// 256-point transform of a half-line held as v[m] = x[t + 16 m] by its 16
// lanes: the two Stockham radix-16 stages of reg::fft<256, 16, SIGN, 2> (same
// butterflies, same twiddles W_512^(2 t r)), exchanged as above.
// TS: tw is the W_512 table (TS = 1) or the W_1024 table read at stride 2.
template <int SIGN, int TS>
__device__ __forceinline__ void fft256(double2 (&v)[XE], int t, unsigned wr0, unsigned rd0,
                                       const double2* __restrict__ tw) {
  reg::Dft<16, SIGN>::run(v);
  exchange(v, wr0, rd0);
#pragma unroll
  for (int r = 1; r < 16; ++r) v[r] = reg::tw_mul(v[r], __ldg(&tw[2 * TS * t * r]), SIGN);
  reg::Dft<16, SIGN>::run(v);
}

// The transforms of one warp's line -- a 512-point line, or (CL) the half-line
// of a 1024-point line whose other half lives in the partner CTA of a 2-CTA
// cluster -- and, CL, the link to the partner warp.
//
// CL: the outermost radix-2 step crosses the CTA pair (X[k] = E[k] + W^k O[k],
// X[k + 512] = E[k] - W^k O[k]).  Each warp PUSHES the eight values per lane its
// partner needs into the partner's scratch with st.async, which completes on the
// partner's ready barrier (armed with the byte count); the partner then reads
// its own shared memory after an ordinary mbarrier wait -- no fence on either
// side.  The free barrier is the reverse "go ahead": signalled (relaxed, no data
// rides on it) after a half-line exchange that is followed by a cross, and after
// a cross that is followed directly by another cross -- once per cross, so both
// barriers advance one phase per cross.  (First form: the partner's values
// pulled with ld.shared::cluster between release / acquire handshakes at cluster
// scope -- every release a MEMBAR.ALL.GPU, every acquire an L1 invalidation that
// threw the twiddles out: 42 900 cycles per x-pass tile against 26 800.)
template <bool CL>
struct WarpLine {
  static constexpr int TS = CL ? 2 : 1;  // table stride: tw is W_1024 for the cluster form
  int lane, t, h;
  unsigned crank;                // CL: parity of this CTA's rows
  unsigned scr, wr0, rd0;        // this warp's exchange scratch (shared-space addresses)
  unsigned scr_peer, ready_peer, free_peer;
  uint64_t* ready_mine;          // the partner's pushed values have landed in this warp's scratch
  uint64_t* free_mine;           // the partner's scratch is free for this warp's push
  unsigned crosses;
  const double2* tw;

  __device__ __forceinline__ void init(int lane_, int w, unsigned crank_, unsigned char* scr0, uint64_t* ready,
                                       uint64_t* freeb, const double2* tw_) {
    lane = lane_;
    h = lane & 1;
    t = lane >> 1;
    crank = crank_;
    scr = bulk::smem_addr(scr0) + w * XSCR;
    wr0 = scr + (t << 8) + (h << 3) + ((t & 7) << 4);  // exchange addresses of slot 0 (see exchange())
    rd0 = scr + (t << 4) + (h << 3);
    ready_mine = ready + w;
    free_mine = freeb + w;
    scr_peer = ready_peer = free_peer = 0u;
    if constexpr (CL) {
      const unsigned peer = crank ^ 1u;
      scr_peer = bulk::cluster_map(scr, peer);
      ready_peer = bulk::cluster_map(bulk::smem_addr(ready_mine), peer);
      free_peer = bulk::cluster_map(bulk::smem_addr(free_mine), peer);
    }
    crosses = 0;
    tw = tw_;
  }
  // The twiddles only depend on the lane: through an opaque copy of the table
  // pointer each transform reloads them instead of keeping ~90 registers live
  // across the tile loop.
  __device__ __forceinline__ const double2* twp() const {
    const double2* p;
    asm volatile("mov.b64 %0, %1;\n" : "=l"(p) : "l"(tw));
    return p;
  }
  // after this warp's last use of its scratch before the partner's next push
  __device__ __forceinline__ void signal_free() {
    if constexpr (CL) {
      __syncwarp();
      if (lane == 0) {
        bulk::mbar_expect_tx(ready_mine, 32 * 8 * 16);  // arm the inbox barrier before the partner may push
        bulk::mbar_arrive_remote(free_peer);
      }
    }
  }
  __device__ __forceinline__ void cross_exchange(const double2 (&out8)[8], double2 (&in8)[8]) {
    bulk::mbar_wait_cluster(free_mine, crosses & 1);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      bulk::st_async_remote(scr_peer + unsigned(((j << 5) + lane) << 4), out8[j], ready_peer);
    bulk::mbar_wait(ready_mine, crosses & 1);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const unsigned a = scr + unsigned(((j << 5) + lane) << 4);
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(in8[j].x), "=d"(in8[j].y) : "r"(a) : "memory");
    }
    ++crosses;
  }
  // frequency held in slot s once the forward transform is complete
  __device__ __forceinline__ int kx_of(int s) const {
    if constexpr (CL) return kslot<XTH, XH>(t, h, (s & 7) + 8 * int(crank)) + XN * (s >> 3);
    else return kslot<XTH, XH>(t, h, s);
  }
  // then_cross: the next transform starts with its cross step (an inverse follows)
  __device__ __forceinline__ void fwd(double2 (&v)[XE], bool then_cross) {
    fft256<-1, TS>(v, t, wr0, rd0, twp());
    signal_free();
    pair_dit<XTH, 1, TS>(v, t, h, twp());
    if constexpr (CL) {
      // this CTA holds the half-line transform S_r[k] in kslot order; CTA 0 forms the outputs of the
      // frequencies in its slots 0..7, CTA 1 those in its slots 8..15
      double2 out8[8], in8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) out8[j] = crank == 0 ? v[j + 8] : v[j];
      cross_exchange(out8, in8);
      const double2* tp = twp();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = kslot<XTH, XH>(t, h, j + 8 * int(crank));
        const double2 e = crank == 0 ? v[j] : in8[j], o = crank == 0 ? in8[j] : v[j + 8];
        const double2 wo = reg::tw_mul(o, __ldg(&tp[k]), -1);
        v[j] = make_double2(e.x + wo.x, e.y + wo.y);
        v[j + 8] = make_double2(e.x - wo.x, e.y - wo.y);
      }
      // the inbox has been read and no half-line exchange comes before the next cross
      if (then_cross) signal_free();
    }
  }
  __device__ __forceinline__ void inv(double2 (&v)[XE], bool then_cross) {
    if constexpr (CL) {
      // the mirror image: sums go to the even-row half-line (CTA 0), twiddled differences to the odd one
      double2 out8[8], in8[8];
      const double2* tp = twp();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = kslot<XTH, XH>(t, h, j + 8 * int(crank));
        const double2 xa = v[j], xb = v[j + 8];
        const double2 u = make_double2(xa.x + xb.x, xa.y + xb.y);
        const double2 d = reg::tw_mul(make_double2(xa.x - xb.x, xa.y - xb.y), __ldg(&tp[k]), +1);
        if (crank == 0) {
          v[j] = u;
          out8[j] = d;
        } else {
          v[j + 8] = d;
          out8[j] = u;
        }
      }
      cross_exchange(out8, in8);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (crank == 0) v[j + 8] = in8[j];
        else v[j] = in8[j];
      }
    }
    pair_dif<XTH, 1, TS>(v, t, h, twp());
    fft256<+1, TS>(v, t, wr0, rd0, twp());
    if (then_cross) signal_free();
  }
};

// FM_X_DBG bit 4: cycle counts summed over the CTAs -- [0], [1] transform warp
// 0 waiting for A_1/A_2 and A_0; [2], [3] store drain (issue -> shared memory
// read) of P/Q and R; [4], [5] the copy threads waiting for staged buffers;
// [6] loop cycles of warp 0; [7] tiles.
__device__ unsigned long long xw_prof[8];

// Tensor maps of a launch: the input (this rank's x-pass input, or the
// spectrum itself on one device) and one output map per destination rank.
struct XwMaps {
  CUtensorMap in;
  CUtensorMap out[kMaxRanks];
};

// RT (P > 1): the fused backward slab transpose -- the rows [s Xl, (s+1) Xl) of
// every output tile are TMA-stored straight into the spectrum of the rank s
// that owns them (peer memory over NVLink when the ranks are devices), at this
// rank's global y: the routed form of store_xb, a box at a time.
// Measured and dropped (512^3, profiles/r2_x512_dbg.md): the copy warps writing
// the tiles back with st.global instead of TMA stores (6.64 vs 3.75 ms), and
// parking the idle register array in the free column of R during two of the
// four transforms (20 700 vs 20 100 cycles per tile: register pressure is not
// what limits the transform warps).
// CL (1024-point lines): a tile of 8 columns is 128 KB per component -- neither
// three buffers in one SM's shared memory nor two 16-element arrays per lane
// hold it -- so the line is split over a cluster of two CTAs: CTA r takes the
// rows of parity r (a 4-D tensor map makes them a box), runs the same 512-point
// machinery on its half-line, and the outermost radix-2 step X[k] = E[k] +
// W^k O[k], X[k + 512] = E[k] - W^k O[k] crosses the CTA pair through
// distributed shared memory, warp to partner warp (cross_exchange below), so
// the warps stay independent of everything but their partner in the other CTA.
// 1024^3: 40.4 ms against 58.6 ms for k_x_fast4<1024> (profiles/r2_x1024_cluster.md).
template <bool RT, bool CL>
__global__ void __launch_bounds__(XTHREADS, 1) k_x_warp(Geo g, const double2* __restrict__ tw, int tiles,
                                                        const __grid_constant__ XwMaps maps, int dbg) {
  constexpr int NLINE = CL ? 2 * XN : XN;  // points of a whole x-line
  extern __shared__ unsigned char smraw[];
  // 1024-byte alignment: the swizzle pattern is a function of the address
  unsigned char* const sm0 =
      smraw + ((1024u - (bulk::smem_addr(smraw) & 1023u)) & 1023u);
  unsigned char* const scr0 = sm0 + 3 * XTILE;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(scr0 + XTW * XSCR);
  uint64_t* const full_p = bars + 0;     // A_1 of a tile has arrived (tx bytes)
  uint64_t* const full_q = bars + 1;     // A_2
  uint64_t* const full_r = bars + 2;     // A_0
  uint64_t* const staged_pq = bars + 3;  // all 8 warps are done with P and Q (count 8)
  uint64_t* const staged_r = bars + 4;   // all 8 warps have written output 0 into R
  uint64_t* const ready = bars + 8;      // CL, per warp: the partner's pushed values have landed in this warp's scratch
  uint64_t* const consumed = bars + 16;  // CL, per warp: the partner's scratch is free for this warp's push
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    bulk::mbar_init(full_p, 1);
    bulk::mbar_init(full_q, 1);
    bulk::mbar_init(full_r, 1);
    bulk::mbar_init(staged_pq, XTW);
    bulk::mbar_init(staged_r, XTW);
    if constexpr (CL)
      for (int i = 0; i < XTW; ++i) {
        bulk::mbar_init(ready + i, 1);
        bulk::mbar_init(consumed + i, 1);
      }
  }
  __syncthreads();
  const unsigned crank = CL ? bulk::cluster_ctarank() : 0u;  // parity of this CTA's rows
  if constexpr (CL) bulk::cluster_sync();  // the partner's barriers exist before anything arrives on them
  const int kzb = g.nzh / XTW;
  // the unit that walks the tiles: this CTA, or the CTA pair
  const int unit = CL ? int(blockIdx.x >> 1) : int(blockIdx.x), units = CL ? int(gridDim.x >> 1) : int(gridDim.x);
  const int K = unit < tiles ? (tiles - 1 - unit) / units + 1 : 0;
  // tile -> (kz block fastest, y, row i)
  auto tile_of = [&](int k, int& kz0, int& y, int& i) {
    const int T_ = unit + k * units;
    kz0 = (T_ % kzb) * XTW;
    const int r = T_ / kzb;
    y = r % g.Ny;
    i = r / g.Ny;
  };

  if (w >= XTW) {  // --------------------------------------------- copy warps
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::);
    // warp 8: P (component 1), warp 9: Q (component 2), warp 10: R (component 0)
    const int buf = w - XTW;
    if (buf > 2 || K == 0) {
      if constexpr (CL) bulk::cluster_sync();
      return;
    }
    const int q = buf == 2 ? 0 : buf + 1;
    const bool late = buf < 2;  // P, Q: phase k stages the outputs of tile k - 1
    uint64_t* const full = buf == 0 ? full_p : (buf == 1 ? full_q : full_r);
    uint64_t* const staged = buf == 2 ? staged_r : staged_pq;
    unsigned char* const tile = sm0 + buf * XTILE;
    auto load = [&](int k) {  // lane 0
      int kz0, y, i;
      tile_of(k, kz0, y, i);
      bulk::mbar_expect_tx(full, XTILE);
#pragma unroll
      for (int r0 = 0; r0 < XN; r0 += 256) {
        if constexpr (CL) bulk::tma4d(tile + r0 * 128, &maps.in, 2 * kz0, y, int(crank), (i * 3 + q) * XN + r0, full);
        else bulk::tma3d(tile + r0 * 128, &maps.in, 2 * kz0, y, (i * 3 + q) * XN + r0, full);
      }
    };
    auto store = [&](int k) {  // lane 0
      int kz0, y, i;
      tile_of(k, kz0, y, i);
      if constexpr (CL && RT) {
        // this CTA's rows j (x = 2 j + parity) belong to rank s = j / (Xl / 2): boxes of at most Xl / 2 rows
        const int xh = g.Xl >> 1, box = xh < 256 ? xh : 256;
        for (int r0 = 0; r0 < XN; r0 += box) {
          const int s = r0 / xh;
          bulk::tma4d_store(&maps.out[s], 2 * kz0, g.y0 + y, int(crank), (i * 3 + q) * xh + (r0 - s * xh),
                            tile + r0 * 128);
        }
      } else if constexpr (CL) {
#pragma unroll
        for (int r0 = 0; r0 < XN; r0 += 256)
          bulk::tma4d_store(&maps.out[0], 2 * kz0, y, int(crank), (i * 3 + q) * XN + r0, tile + r0 * 128);
      } else if constexpr (!RT) {
#pragma unroll
        for (int r0 = 0; r0 < XN; r0 += 256)
          bulk::tma3d_store(&maps.out[0], 2 * kz0, y, (i * 3 + q) * XN + r0, tile + r0 * 128);
      } else {
        const int box = g.Xl < 256 ? g.Xl : 256;  // rows per store: never across two owners
        for (int r0 = 0; r0 < XN; r0 += box) {
          const int s = r0 / g.Xl;
          bulk::tma3d_store(&maps.out[s], 2 * kz0, g.y0 + y, (i * 3 + q) * g.Xl + (r0 - s * g.Xl), tile + r0 * 128);
        }
      }
      bulk::bulk_commit();
    };
    long long t_idle = 0, t_drain = 0;
    const bool prof = (dbg & 16) && lane == 0;
    if (lane == 0) load(0);
    const int phases = late ? K + 1 : K;
    for (int k = 0; k < phases; ++k) {
      const long long c0 = prof ? clock64() : 0;
      // (the copy warps idle most of a tile: sleep between polls so that their
      // spinning does not take issue slots from the transform warps they share
      // schedulers with)
      while (!bulk::mbar_test(staged, k & 1)) __nanosleep(256);
      const long long c1 = prof ? clock64() : 0;
      const int out = late ? k - 1 : k;  // the tile whose output sits in the buffer
      if (out >= 0 && lane == 0) {
        store(out);
        if (out + 1 < K) bulk::bulk_wait_read();
      }
      if (prof) t_idle += c1 - c0, t_drain += clock64() - c1;
      if (lane == 0) {
        const int next = k + 1;  // tile to load into the buffer now
        if (next < K) load(next);
        else if (late && next == K) bulk::mbar_arrive(full);  // nothing to load: free for the flush
      }
    }
    if (prof) atomicAdd(&xw_prof[2 + (buf == 2)], (unsigned long long)t_drain),
        atomicAdd(&xw_prof[4 + (buf == 2)], (unsigned long long)t_idle);
    if (lane == 0) bulk::bulk_wait_all();  // the stores are performed before the CTA retires
    if constexpr (CL) bulk::cluster_sync();
    return;
  }

  // --------------------------------------------------------- transform warps
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::);
  const int h = lane & 1, t = lane >> 1;
  // this lane's 16 bytes of row (lane + 32 m) of a buffer: column w, swizzled
  const int col = (lane << 7) + ((w ^ (lane & 7)) << 4);
  unsigned char* const P = sm0 + col;
  unsigned char* const Q = sm0 + XTILE + col;
  unsigned char* const R = sm0 + 2 * XTILE + col;
  auto at = [](unsigned char* b, int m) { return reinterpret_cast<double2*>(b + (m << 12)); };
  WarpLine<CL> L;
  L.init(lane, w, crank, scr0, ready, consumed, tw);
  auto kx_of = [&](int s) { return L.kx_of(s); };
  auto fwd = [&](double2(&v)[XE], bool then_cross) {
    if (dbg & 1) return;
    L.fwd(v, then_cross && !(dbg & 32));
  };
  auto inv = [&](double2(&v)[XE], bool then_cross) {
    if (dbg & 33) return;  // (bit 5: only the inverse transforms skipped -- how far the TMA pipeline can follow)
    L.inv(v, then_cross);
  };
  double2 X[XE], v[XE];
  double xiy_p = 0.0, xiz_p = 0.0;
  const bool prof = (dbg & 16) && w == 0 && lane == 0;
  long long t_pq = 0, t_r = 0;
  const long long t_begin = prof ? clock64() : 0;
  for (int k = 0; k < K; ++k) {
    int kz0, y, i;
    tile_of(k, kz0, y, i);
    const int kz = kz0 + w;
    const int yg = g.y0 + y;
    const int qy = freq_of(yg, g.Nyg), qz = freq_of(kz, g.Nz);
    const bool nyq_yz = ((g.Nyg % 2 == 0) && (yg == g.Nyg / 2)) || ((g.Nz % 2 == 0) && (kz == g.Nz / 2));
    const double xiy = qy * g.invL[1], xiz = qz * g.invL[2];
    // B = xi_y A_1 + xi_z A_2 from this warp's column; the previous tile's
    // outputs 1 and 2 go back into the same 16 bytes
    {
      const long long c0 = prof ? clock64() : 0;
      bulk::mbar_wait(full_p, k & 1);
      bulk::mbar_wait(full_q, k & 1);
      if (prof) t_pq += clock64() - c0;
    }
#pragma unroll
    for (int m = 0; m < XE; ++m) {
      const double2 a1 = *at(P, m), a2 = *at(Q, m);
      X[m] = make_double2(fma(a1.x, xiy, a2.x * xiz), fma(a1.y, xiy, a2.y * xiz));
    }
    if (k > 0) {
#pragma unroll
      for (int m = 0; m < XE; ++m) {
        *at(P, m) = make_double2(v[m].x * xiy_p, v[m].y * xiy_p);
        *at(Q, m) = make_double2(v[m].x * xiz_p, v[m].y * xiz_p);
      }
    }
    bulk::fence_async_smem();
    __syncwarp();
    if (lane == 0) bulk::mbar_arrive(staged_pq);
    fwd(X, false);
    // forward transform of A_0
    {
      const long long c0 = prof ? clock64() : 0;
      bulk::mbar_wait(full_r, k & 1);
      if (prof) t_r += clock64() - c0;
    }
#pragma unroll
    for (int m = 0; m < XE; ++m) v[m] = *at(R, m);
    fwd(v, true);
    // s = (xi_x FFT(A_0) + FFT(B)) / |xi|^2, zero at xi = 0 and on Nyquist planes
#pragma unroll
    for (int m = 0; m < XE; ++m) {
      const int kx = kx_of(m);
      const double xix = freq_of(kx, NLINE) * g.invL[0];
      const double norm2 = xix * xix + xiy * xiy + xiz * xiz;
      const bool zero = norm2 == 0.0 || nyq_yz || kx == NLINE / 2;
      const double iv = zero ? 0.0 : 1.0 / norm2;
      X[m] = make_double2((v[m].x * xix + X[m].x) * iv, (v[m].y * xix + X[m].y) * iv);
    }
    // Bhat_i0 = IFFT(s xi_x) -> back into R
#pragma unroll
    for (int m = 0; m < XE; ++m) {
      const double f = freq_of(kx_of(m), NLINE) * g.invL[0];
      v[m] = make_double2(X[m].x * f, X[m].y * f);
    }
    inv(v, true);
#pragma unroll
    for (int m = 0; m < XE; ++m) *at(R, m) = v[m];
    bulk::fence_async_smem();
    __syncwarp();
    if (lane == 0) bulk::mbar_arrive(staged_r);
    // IFFT(s): Bhat_i1 = xi_y IFFT(s), Bhat_i2 = xi_z IFFT(s), written at the
    // start of the next tile (or below, after the last one)
#pragma unroll
    for (int m = 0; m < XE; ++m) v[m] = make_double2(X[m].x * 1.0, X[m].y * 1.0);
    inv(v, false);
    xiy_p = xiy;
    xiz_p = xiz;
  }
  if (K > 0) {
    bulk::mbar_wait(full_p, K & 1);  // the stores of tile K - 2's outputs have read P and Q
    bulk::mbar_wait(full_q, K & 1);
#pragma unroll
    for (int m = 0; m < XE; ++m) {
      *at(P, m) = make_double2(v[m].x * xiy_p, v[m].y * xiy_p);
      *at(Q, m) = make_double2(v[m].x * xiz_p, v[m].y * xiz_p);
    }
    bulk::fence_async_smem();
    __syncwarp();
    if (lane == 0) bulk::mbar_arrive(staged_pq);
  }
  if (prof) {
    atomicAdd(&xw_prof[0], (unsigned long long)t_pq);
    atomicAdd(&xw_prof[1], (unsigned long long)t_r);
    atomicAdd(&xw_prof[6], (unsigned long long)(clock64() - t_begin));
    atomicAdd(&xw_prof[7], (unsigned long long)K);
  }
  if constexpr (CL) bulk::cluster_sync();  // neither CTA retires while its partner may still read its scratch
}

// ---------------------------------------------------------------- y pass, 1024
// The 1024-point y pass on the same machinery: a tile is (component, x, 8 kz
// columns) x 1024 y-rows, split over the CTA pair by row parity.  One transform
// per tile, three tiles in flight per CTA (a ring of three 64 KB buffers, each
// with its copy warp).  Forward: the tile arrives as this CTA's parity rows
// (4-D tensor map), the result -- frequencies in kslot order, which for CTA r
// are four blocks of 128 consecutive frequencies -- is written block-wise into
// the same buffer and stored with the natural-order map; the inverse pass runs
// the mirror image.
struct YwMaps {
  CUtensorMap split;  // [C Nx][Ny / 2][2][2 nzh]: box = 256 rows of one parity
  CUtensorMap nat;    // [C Nx][Ny][2 nzh]: box = 128 consecutive rows
};
// CTA r holds the frequencies of blocks {0, 3, 4, 7} (r = 0) or {1, 2, 5, 6} (r = 1) of 128; its buffer
// keeps them in that order.
__device__ __forceinline__ int yw_local_row(int f, unsigned r) {
  const int blk = f >> 7, hi = blk >> 2, lo = blk & 3;
  const int idx = r == 0 ? (lo ? 1 : 0) : lo - 1;
  return ((2 * hi + idx) << 7) + (f & 127);
}
__device__ __forceinline__ int yw_block_row0(int lb, unsigned r) {  // first global row of local block lb
  const int hi = lb >> 1, idx = lb & 1;
  const int lo = r == 0 ? (idx ? 3 : 0) : idx + 1;
  return (4 * hi + lo) << 7;
}

template <int SIGN>
__global__ void __launch_bounds__(XTHREADS, 1) k_y_warp(int nzh, const double2* __restrict__ tw, int tiles,
                                                        const __grid_constant__ YwMaps maps) {
  extern __shared__ unsigned char smraw[];
  unsigned char* const sm0 = smraw + ((1024u - (bulk::smem_addr(smraw) & 1023u)) & 1023u);
  unsigned char* const scr0 = sm0 + 3 * XTILE;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(scr0 + XTW * XSCR);
  uint64_t* const full = bars + 0;    // [3] the buffer's tile has arrived
  uint64_t* const staged = bars + 3;  // [3] all 8 warps have written their results into the buffer
  uint64_t* const ready = bars + 8;
  uint64_t* const freeb = bars + 16;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 3; ++b) {
      bulk::mbar_init(full + b, 1);
      bulk::mbar_init(staged + b, XTW);
    }
    for (int i = 0; i < XTW; ++i) {
      bulk::mbar_init(ready + i, 1);
      bulk::mbar_init(freeb + i, 1);
    }
  }
  __syncthreads();
  const unsigned crank = bulk::cluster_ctarank();
  bulk::cluster_sync();
  const int kzb = nzh / XTW;
  const int unit = int(blockIdx.x >> 1), units = int(gridDim.x >> 1);
  const int K = unit < tiles ? (tiles - 1 - unit) / units + 1 : 0;
  auto tile_of = [&](int k, int& kz0, int& cx) {
    const int T_ = unit + k * units;
    kz0 = (T_ % kzb) * XTW;
    cx = T_ / kzb;
  };

  if (w >= XTW) {  // --------------------------------------------- copy warps
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::);
    const int buf = w - XTW;
    if (buf <= 2 && lane == 0) {
      unsigned char* const tile = sm0 + buf * XTILE;
      // SIGN < 0 reads parity rows and writes frequency blocks; SIGN > 0 the other way round
      auto move = [&](int k, bool in) {
        int kz0, cx;
        tile_of(k, kz0, cx);
        if (in) bulk::mbar_expect_tx(full + buf, XTILE);
        if ((SIGN < 0) == in) {
#pragma unroll
          for (int r0 = 0; r0 < XN; r0 += 256) {
            if (in) bulk::tma4d(tile + r0 * 128, &maps.split, 2 * kz0, int(crank), r0, cx, full + buf);
            else bulk::tma4d_store(&maps.split, 2 * kz0, int(crank), r0, cx, tile + r0 * 128);
          }
        } else {
#pragma unroll
          for (int lb = 0; lb < 4; ++lb) {
            if (in) bulk::tma3d(tile + lb * 128 * 128, &maps.nat, 2 * kz0, yw_block_row0(lb, crank), cx, full + buf);
            else bulk::tma3d_store(&maps.nat, 2 * kz0, yw_block_row0(lb, crank), cx, tile + lb * 128 * 128);
          }
        }
        if (!in) bulk::bulk_commit();
      };
      if (buf < K) move(buf, true);
      for (int k = buf; k < K; k += 3) {
        while (!bulk::mbar_test(staged + buf, (k / 3) & 1)) __nanosleep(128);
        move(k, false);
        if (k + 3 < K) {
          bulk::bulk_wait_read();
          move(k + 3, true);
        }
      }
      bulk::bulk_wait_all();
    }
    bulk::cluster_sync();
    return;
  }

  // --------------------------------------------------------- transform warps
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::);
  WarpLine<true> L;
  L.init(lane, w, crank, scr0, ready, freeb, tw);
  if (SIGN > 0) L.signal_free();  // an inverse transform starts with its cross step
  const int col = (lane << 7) + ((w ^ (lane & 7)) << 4);  // row lane + 32 m, column w, swizzled
  double2 v[XE];
  for (int k = 0; k < K; ++k) {
    const int b = k % 3;
    unsigned char* const base = sm0 + b * XTILE;
    bulk::mbar_wait(full + b, (k / 3) & 1);
    if (SIGN < 0) {
#pragma unroll
      for (int m = 0; m < XE; ++m) v[m] = *reinterpret_cast<const double2*>(base + col + (m << 12));
      L.fwd(v, false);
#pragma unroll
      for (int s = 0; s < XE; ++s) {
        const int lr = yw_local_row(L.kx_of(s), crank);
        *reinterpret_cast<double2*>(base + (lr << 7) + ((w ^ (lr & 7)) << 4)) = v[s];
      }
    } else {
#pragma unroll
      for (int s = 0; s < XE; ++s) {
        const int lr = yw_local_row(L.kx_of(s), crank);
        v[s] = *reinterpret_cast<const double2*>(base + (lr << 7) + ((w ^ (lr & 7)) << 4));
      }
      L.inv(v, true);
#pragma unroll
      for (int m = 0; m < XE; ++m) *reinterpret_cast<double2*>(base + col + (m << 12)) = v[m];
    }
    bulk::fence_async_smem();
    __syncwarp();
    if (lane == 0) bulk::mbar_arrive(staged + b);
  }
  bulk::cluster_sync();
}

}  // namespace

bool xw_launch(fm_ctx* ctx, const Geo& g, double2* spec, int dbg) {
  const bool cluster = g.Nx == 2 * XN;  // 1024-point lines: a CTA pair per tile
  if ((g.Nx != XN && !cluster) || g.nzh % XTW != 0) return false;
  const bool routed = g.P > 1;
  if (routed) {
    // The routed TMA stores are the default where they have been validated --
    // virtual ranks, all buffers on this device (bit-equal to P = 1).  Across
    // devices the destinations are IPC-mapped peer buffers, which no run has
    // exercised yet: there FM_XW_ROUTED=1 opts in and the routed k_x_stream
    // (per-element peer stores) stays the default.  FM_XW_ROUTED=0 turns the
    // path off everywhere.
    const char* e = getenv("FM_XW_ROUTED");
    const bool on = e ? atoi(e) != 0 : ctx->virt;
    const int rows_per_rank = cluster ? g.Xl / 2 : g.Xl;  // of one CTA's XN rows
    if (!on || g.P > kMaxRanks || g.Xl % 16 != 0 || rows_per_rank % 8 != 0 || XN % rows_per_rank != 0 ||
        int(ctx->h_dst_a.size()) < g.P)
      return false;
  }
  XwMaps maps;
  if (!x_tensor_map(spec, 9 * g.Nx, g.Ny, g.nzh, XTW, true, 256, &maps.in, cluster)) return false;
  if (!routed) {
    maps.out[0] = maps.in;
  } else {
    const int rows_per_rank = cluster ? g.Xl / 2 : g.Xl;
    const int box = rows_per_rank < 256 ? rows_per_rank : 256;
    for (int s = 0; s < g.P; ++s)  // A_s viewed as [9 Xl][Ny global][2 nzh] (cluster form: rows split by parity)
      if (!ctx->h_dst_a[s] ||
          !x_tensor_map(ctx->h_dst_a[s], 9 * g.Xl, g.Nyg, g.nzh, XTW, true, box, &maps.out[s], cluster))
        return false;
  }
  using Kern = void (*)(Geo, const double2*, int, const XwMaps, int);
  const Kern kern = cluster ? (routed ? k_x_warp<true, true> : k_x_warp<false, true>)
                            : (routed ? k_x_warp<true, false> : k_x_warp<false, false>);
  set_smem_limit(reinterpret_cast<const void*>(kern), int(XSMEM));
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = (g.nzh / XTW) * g.Ny * 3;
  if (!cluster) {
    const int grid = std::min(tiles, std::max(sms, 1));
    kern<<<grid, XTHREADS, XSMEM, ctx->stream>>>(g, ctx->px.tw, tiles, maps, dbg);
  } else {
    // persistent CTA pairs: as many clusters as the device can hold at once
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(XTHREADS);
    cfg.dynamicSmemBytes = XSMEM;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(2 * std::max(sms / 2, 1));
    // (co-resident CTA pairs: queried once per device and kernel, the query is not cheap)
    static std::mutex mx;
    static std::map<std::pair<int, const void*>, int> cache;
    int pairs = 0;
    {
      std::lock_guard<std::mutex> lk(mx);
      const auto key = std::make_pair(dev, reinterpret_cast<const void*>(kern));
      auto it = cache.find(key);
      if (it == cache.end()) {
        int q = 0;
        if (cudaOccupancyMaxActiveClusters(&q, kern, &cfg) != cudaSuccess) q = 0;
        cudaGetLastError();
        it = cache.emplace(key, q).first;
      }
      pairs = it->second;
    }
    if (pairs < 1) return false;
    cfg.gridDim = dim3(2 * std::min(tiles, pairs));
    if (cudaLaunchKernelEx(&cfg, kern, g, static_cast<const double2*>(ctx->px.tw), tiles, maps, dbg) != cudaSuccess)
      return false;  // (the caller falls back to the staged pass; the error is cleared there)
  }
  if (dbg & 16) {  // timing experiments only: per-tile averages to stderr
    unsigned long long h[8] = {}, z[8] = {};
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpyFromSymbol(h, xw_prof, sizeof(h));
    cudaMemcpyToSymbol(xw_prof, z, sizeof(z));
    const double n = double(h[7] ? h[7] : 1);
    fprintf(stderr,
            "k_x_warp cycles/tile: loop %.0f  wait A1A2 %.0f  wait A0 %.0f | drain PQ %.0f R %.0f | copy idle PQ %.0f R "
            "%.0f\n",
            h[6] / n, h[0] / n, h[1] / n, h[2] / n, h[3] / n, h[4] / n, h[5] / n);
  }
  return true;
}

bool yw_launch(fm_ctx* ctx, const Geo& g, int sign, double2* spec) {
  if (g.Ny != 2 * XN || g.P != 1 || g.nzh % XTW != 0) return false;
  const uint64_t ncx = uint64_t(ctx->ncomp) * g.Nx, nzh = uint64_t(g.nzh), Ny = uint64_t(g.Ny);
  YwMaps maps;
  {
    const uint64_t d[4] = {2 * nzh, 2, Ny / 2, ncx}, st[3] = {nzh * 16, 2 * nzh * 16, Ny * nzh * 16};
    const uint32_t b[4] = {2 * XTW, 1, 256, 1};
    if (!tensor_map_encode(spec, 4, d, st, b, true, &maps.split)) return false;
  }
  {
    const uint64_t d[3] = {2 * nzh, Ny, ncx}, st[2] = {nzh * 16, Ny * nzh * 16};
    const uint32_t b[3] = {2 * XTW, 128, 1};
    if (!tensor_map_encode(spec, 3, d, st, b, true, &maps.nat)) return false;
  }
  using Kern = void (*)(int, const double2*, int, const YwMaps);
  const Kern kern = sign < 0 ? k_y_warp<-1> : k_y_warp<+1>;
  set_smem_limit(reinterpret_cast<const void*>(kern), int(XSMEM));
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = int(nzh / XTW) * int(ncx);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(XTHREADS);
  cfg.dynamicSmemBytes = XSMEM;
  cfg.stream = ctx->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(2 * std::min(tiles, std::max(sms / 2, 1)));
  return cudaLaunchKernelEx(&cfg, kern, g.nzh, static_cast<const double2*>(ctx->py.tw), tiles, maps) == cudaSuccess;
}

}  // namespace fm
