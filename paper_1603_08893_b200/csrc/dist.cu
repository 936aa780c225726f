// Slab decomposition of the projection over P ranks.
//
// Rank r owns x-planes [r Xl, (r+1) Xl) of every real field (Xl = Nx/P).
// Passes 1-2 run on that x-slab; pass 2 writes its spectrum pre-packed per
// destination, B_r = [dst][c][xl][yl][kz] (Yl = Ny/P), so the block bound for
// rank d and component c is one contiguous run of Xl*Yl*nzh complex values.
// The all-to-all delivers it to A_d = [c][x][yl][kz] (global x), where the
// block from source s is again contiguous (x in [s Xl, (s+1) Xl)) -- no pack
// or unpack kernels on either side.  Pass 3 runs on the y-slab, the reverse
// all-to-all returns the blocks, pass 4 reads the packed layout.
//
//   virtual mode : all P ranks live on one device; the all-to-all is one
//                  device copy kernel (validates the decomposition exactly
//                  against P = 1 on a single B200).
//   NCCL mode    : one rank per device; grouped ncclSend/ncclRecv per
//                  (peer, component) chunk over NVLink / NVSwitch.
#include <nccl.h>

#include <cstring>

#include <vector>

#include "proj_common.cuh"

namespace fm {

// Offsets (complex elements) of the chunk (src -> dst, component c):
// b_off inside B of rank src, a_off inside A of rank dst.
struct Chunk {
  int64_t b_off, a_off, count;
};

inline Chunk chunk_of(int P, int Nx, int Ny, int nzh, int NC, int src, int dst, int c) {
  const int64_t Xl = Nx / P, Yl = Ny / P;
  const int64_t cnt = Xl * Yl * nzh;
  return Chunk{(int64_t(dst) * NC + c) * cnt, (int64_t(c) * Nx + int64_t(src) * Xl) * Yl * nzh, cnt};
}

// grid: (blocks over a chunk, NC, P*P); dir +1: B -> A, -1: A -> B
__global__ void k_transpose_virtual(double2* __restrict__ A, double2* __restrict__ B, int P, int NC,
                                    int Nx, int Ny, int nzh, int64_t rank_elems, int dir) {
  const int s = blockIdx.z / P, r = blockIdx.z - s * P, c = blockIdx.y;
  const int64_t Xl = Nx / P, Yl = Ny / P;
  const int64_t cnt = Xl * Yl * nzh;
  double2* b = B + int64_t(s) * rank_elems + (int64_t(r) * NC + c) * cnt;
  double2* a = A + int64_t(r) * rank_elems + (int64_t(c) * Nx + int64_t(s) * Xl) * Yl * nzh;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cnt; i += int64_t(gridDim.x) * blockDim.x) {
    if (dir > 0)
      a[i] = b[i];
    else
      b[i] = a[i];
  }
}

static int nccl_check(fm_ctx* ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return FM_OK;
  return set_error(ctx, FM_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

int transpose(fm_ctx* ctx, int dir) {
  const int P = ctx->P, NC = ctx->ncomp;
  if (ctx->virt) {
    const int64_t cnt = int64_t(ctx->Nx / P) * (ctx->Ny / P) * ctx->nzh;
    const int bx = int(std::min<int64_t>(1024, (cnt + 255) / 256));
    k_transpose_virtual<<<dim3(bx, NC, P * P), 256, 0, ctx->stream>>>(ctx->spec, ctx->spec2, P, NC, ctx->Nx,
                                                                       ctx->Ny, ctx->nzh, ctx->spec_rank_elems, dir);
    FM_LAUNCHED(ctx);
    return FM_OK;
  }
  // one rank per device: grouped point-to-point over NVLink
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  const int me = ctx->rank;
  if (int st = nccl_check(ctx, ncclGroupStart(), "ncclGroupStart")) return st;
  for (int peer = 0; peer < P; ++peer) {
    for (int c = 0; c < NC; ++c) {
      // forward: my packed block for `peer` -> peer's A; reverse: A block of `peer` -> its B
      const Chunk out = dir > 0 ? chunk_of(P, ctx->Nx, ctx->Ny, ctx->nzh, NC, me, peer, c)
                                : chunk_of(P, ctx->Nx, ctx->Ny, ctx->nzh, NC, peer, me, c);
      const Chunk in = dir > 0 ? chunk_of(P, ctx->Nx, ctx->Ny, ctx->nzh, NC, peer, me, c)
                               : chunk_of(P, ctx->Nx, ctx->Ny, ctx->nzh, NC, me, peer, c);
      const double2* src = dir > 0 ? ctx->spec2 + out.b_off : ctx->spec + out.a_off;
      double2* dst = dir > 0 ? ctx->spec + in.a_off : ctx->spec2 + in.b_off;
      if (peer == me) {
        FM_CUDA(ctx, cudaMemcpyAsync(dst, src, out.count * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream));
        continue;
      }
      if (int st = nccl_check(ctx, ncclSend(src, size_t(out.count) * 2, ncclDouble, peer, comm, ctx->stream), "ncclSend"))
        return st;
      if (int st = nccl_check(ctx, ncclRecv(dst, size_t(in.count) * 2, ncclDouble, peer, comm, ctx->stream), "ncclRecv"))
        return st;
    }
  }
  return nccl_check(ctx, ncclGroupEnd(), "ncclGroupEnd");
}

// Ordered sum of `count` per-rank values across the distributed ranks:
// all-gather, then every rank adds them in rank order (deterministic and
// identical on all ranks, unlike an all-reduce whose order is NCCL's).
__global__ void k_sum_ranks(const double* __restrict__ g, int P, int count, double* __restrict__ out) {
  const int i = threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int r = 0; r < P; ++r) s += g[r * count + i];
  out[i] = s;
}

int combine_ranks(fm_ctx* ctx, double* d_vals, int count) {
  if (ctx->virt || ctx->P == 1 || !ctx->nccl) return FM_OK;
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  if (int st = nccl_check(ctx, ncclAllGather(d_vals, ctx->d_gather, size_t(count), ncclDouble, comm, ctx->stream),
                          "ncclAllGather"))
    return st;
  k_sum_ranks<<<1, 32, 0, ctx->stream>>>(ctx->d_gather, ctx->P, count, d_vals);
  FM_LAUNCHED(ctx);
  return FM_OK;
}

int combine_min_u64(fm_ctx* ctx, unsigned long long* d_key) {
  if (ctx->virt || ctx->P == 1 || !ctx->nccl) return FM_OK;
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  return nccl_check(ctx, ncclAllReduce(d_key, d_key, 1, ncclUint64, ncclMin, comm, ctx->stream), "ncclAllReduce");
}

int dist_init_nccl(fm_ctx* ctx, const void* unique_id, int nranks, int rank) {
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm;
  if (int st = nccl_check(ctx, ncclCommInitRank(&comm, nranks, id, rank), "ncclCommInitRank")) return st;
  ctx->nccl = comm;
  return FM_OK;
}

void dist_destroy(fm_ctx* ctx) {
  if (ctx->nccl) ncclCommDestroy(static_cast<ncclComm_t>(ctx->nccl));
  ctx->nccl = nullptr;
}

}  // namespace fm

using namespace fm;

extern "C" {

int fm_nccl_unique_id(void* out, int bytes) {
  if (!out || bytes < int(sizeof(ncclUniqueId))) return FM_E_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return FM_E_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return FM_OK;
}

int fm_dist_chunk(int P, int Nx, int Ny, int nzh, int ncomp, int src, int dst, int comp, int64_t* b_off,
                  int64_t* a_off, int64_t* count) {
  if (P < 1 || Nx % P || Ny % P || src < 0 || src >= P || dst < 0 || dst >= P || comp < 0 || comp >= ncomp ||
      !b_off || !a_off || !count)
    return FM_E_INVALID;
  const Chunk ch = chunk_of(P, Nx, Ny, nzh, ncomp, src, dst, comp);
  *b_off = ch.b_off;
  *a_off = ch.a_off;
  *count = ch.count;
  return FM_OK;
}

}  // extern "C"
