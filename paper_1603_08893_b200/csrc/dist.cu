// Slab decomposition of the projection over P ranks.
//
// Rank r owns x-planes [r Xl, (r+1) Xl) of every real field (Xl = Nx/P).
// Passes 1-2 run on that x-slab, pass 3 on the y-slab [r Yl, (r+1) Yl)
// (Yl = Ny/P), passes 4-5 on the x-slab again.  The two slab transposes are
// not separate all-to-all steps: they are fused into the epilogues of the
// passes that produce the data (route_yf / route_xb, proj_common.cuh):
//
//   pass 2 (forward y FFT) stores every element straight into the x-pass
//          input B_d of the rank d that owns its y, at its global x;
//   pass 3 (x FFT, ghat, inverse x FFT) stores every element straight into
//          the spectrum A_s of the rank s that owns its x, at its global y;
//          pass 4 then runs in place on A_s.
//
// On devices the stores go over NVLink / NVSwitch into peer memory mapped
// with CUDA IPC, so the exchange overlaps the FFT arithmetic line by line
// instead of following it; one cross-rank barrier after pass 2 and one after
// pass 3 order the passes (rank_barrier).  In the virtual mode all P ranks'
// buffers live side by side on one device and the same kernels store into
// them -- the decomposition is validated exactly against P = 1 on one B200.
//
// Buffer hazards (why two barriers suffice): B_d is written by every rank's
// pass 2 and read only by d's pass 3, which runs after barrier 1; the next
// application's pass 2 writes B_d again only after barrier 2, i.e. after d's
// pass 3.  A_s is read by s's pass 2 (before barrier 1) and written by the
// pass 3 of every rank (after barrier 1); s's passes 4-5 and the next pass 1
// run after barrier 2.
#include <nccl.h>

#include <cstring>
#include <string>

#include <vector>

#include "proj_common.cuh"

namespace fm {

static int nccl_check(fm_ctx* ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return FM_OK;
  return set_error(ctx, FM_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

int rank_barrier(fm_ctx* ctx) {
  if (!distributed(ctx)) return FM_OK;
  // a one-element all-reduce on the library stream: it starts after this
  // rank's transpose-fused kernel completed (its peer stores performed) and
  // finishes only when every rank's has
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  double* flag = ctx->d_scal + 63;
  return nccl_check(ctx, ncclAllReduce(flag, flag, 1, ncclDouble, ncclSum, comm, ctx->stream), "ncclAllReduce");
}

// Staged transposes, the textbook form: the y
// and x passes run locally and in place; between them every rank packs, per
// destination d, the block of its spectrum that d owns next into a dense
// staging area (strided 2-D copies), exchanges the blocks with grouped
// ncclSend / ncclRecv over NVLink, and unpacks.  With XY = Xl Yl nzh:
//   forward  A_r [c][xl][y][kz]  --pack-->  S_r [d][c][xl][yl][kz]
//            --all-to-all-->  B_d [c][r Xl + xl][yl][kz]      (received in place)
//   backward B_d [c][x][yl][kz] = [c][s][xl][yl][kz]          (sent in place)
//            --all-to-all-->  S_s [d][c][xl][yl][kz]  --unpack-->  A_s [c][xl][d Yl + yl][kz]
// The send / receive pairs order the ranks; no barrier is needed.  In the
// virtual mode the all-to-all is the same set of block copies on this device.
// This is the arm the peer-store transposes are measured against.
int dist_transpose_staged(fm_ctx* ctx, int dir) {
  const int P = ctx->P, nc = ctx->ncomp;
  const int64_t Xl = ctx->Nx / P, Yl = ctx->Ny / P, nzh = ctx->nzh, Ny = ctx->Ny;
  const int64_t XY = Xl * Yl * nzh;                  // complex elements of one (component, source, destination) block
  const size_t row = size_t(Yl) * nzh * sizeof(double2);     // one (c, xl) row of a block
  const size_t pitch_a = size_t(Ny) * nzh * sizeof(double2);  // the same row inside A
  const int r0 = ctx->virt ? 0 : ctx->rank, r1 = ctx->virt ? P : ctx->rank + 1;
  auto A = [&](int r) { return ctx->spec + (ctx->virt ? int64_t(r) * ctx->spec_rank_elems : 0); };
  auto B = [&](int r) { return ctx->spec2 + (ctx->virt ? int64_t(r) * ctx->spec_rank_elems : 0); };
  auto S = [&](int r) { return ctx->spec3 + (ctx->virt ? int64_t(r) * ctx->spec_rank_elems : 0); };
  if (!ctx->spec3) return set_error(ctx, FM_E_INVALID, "staged transpose without its staging buffer");
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  if (dir > 0) {
    for (int r = r0; r < r1; ++r)
      for (int d = 0; d < P; ++d)
        FM_CUDA(ctx, cudaMemcpy2DAsync(S(r) + int64_t(d) * nc * XY, row, A(r) + int64_t(d) * Yl * nzh, pitch_a, row,
                                       size_t(nc) * Xl, cudaMemcpyDeviceToDevice, ctx->stream));
    if (ctx->virt) {
      for (int r = 0; r < P; ++r)
        for (int d = 0; d < P; ++d)
          for (int c = 0; c < nc; ++c)
            FM_CUDA(ctx, cudaMemcpyAsync(B(d) + (int64_t(c) * P + r) * XY, S(r) + (int64_t(d) * nc + c) * XY,
                                         size_t(XY) * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
      const int r = ctx->rank;
      if (int st = nccl_check(ctx, ncclGroupStart(), "ncclGroupStart")) return st;
      for (int d = 0; d < P; ++d)
        for (int c = 0; c < nc; ++c) {
          ncclSend(S(r) + (int64_t(d) * nc + c) * XY, size_t(2 * XY), ncclDouble, d, comm, ctx->stream);
          ncclRecv(B(r) + (int64_t(c) * P + d) * XY, size_t(2 * XY), ncclDouble, d, comm, ctx->stream);
        }
      if (int st = nccl_check(ctx, ncclGroupEnd(), "ncclGroupEnd(forward transpose)")) return st;
    }
  } else {
    if (ctx->virt) {
      for (int d = 0; d < P; ++d)
        for (int s = 0; s < P; ++s)
          for (int c = 0; c < nc; ++c)
            FM_CUDA(ctx, cudaMemcpyAsync(S(s) + (int64_t(d) * nc + c) * XY, B(d) + (int64_t(c) * P + s) * XY,
                                         size_t(XY) * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
      const int d = ctx->rank;
      if (int st = nccl_check(ctx, ncclGroupStart(), "ncclGroupStart")) return st;
      for (int s = 0; s < P; ++s)
        for (int c = 0; c < nc; ++c) {
          ncclSend(B(d) + (int64_t(c) * P + s) * XY, size_t(2 * XY), ncclDouble, s, comm, ctx->stream);
          ncclRecv(S(d) + (int64_t(s) * nc + c) * XY, size_t(2 * XY), ncclDouble, s, comm, ctx->stream);
        }
      if (int st = nccl_check(ctx, ncclGroupEnd(), "ncclGroupEnd(backward transpose)")) return st;
    }
    for (int r = r0; r < r1; ++r)
      for (int d = 0; d < P; ++d)
        FM_CUDA(ctx, cudaMemcpy2DAsync(A(r) + int64_t(d) * Yl * nzh, pitch_a, S(r) + int64_t(d) * nc * XY, row, row,
                                       size_t(nc) * Xl, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return FM_OK;
}

int dist_setup_routes(fm_ctx* ctx) {
  const int P = ctx->P;
  if (P > kMaxRanks) return set_error(ctx, FM_E_UNSUPPORTED, "more slab ranks than kMaxRanks");
  if (ctx->transpose == 1) return FM_OK;  // staged all-to-all: nothing is mapped
  if (!ctx->d_dst_a) FM_CUDA(ctx, cudaMalloc(&ctx->d_dst_a, sizeof(double2*) * kMaxRanks));
  if (!ctx->d_dst_b) FM_CUDA(ctx, cudaMalloc(&ctx->d_dst_b, sizeof(double2*) * kMaxRanks));
  std::vector<double2*> a(kMaxRanks, nullptr), b(kMaxRanks, nullptr);
  if (!distributed(ctx)) {  // virtual ranks: side by side on this device
    for (int r = 0; r < P; ++r) {
      a[r] = ctx->spec + int64_t(r) * ctx->spec_rank_elems;
      b[r] = ctx->spec2 ? ctx->spec2 + int64_t(r) * ctx->spec_rank_elems : nullptr;
    }
  } else {
    // one rank per device: exchange IPC handles of A and B (all-gather over
    // the communicator), map every peer's buffers into this process
    struct Handles {
      cudaIpcMemHandle_t a, b;
      char bus[32];  // PCI bus id of the rank's device
    };
    Handles mine;
    std::memset(&mine, 0, sizeof(mine));
    FM_CUDA(ctx, cudaDeviceGetPCIBusId(mine.bus, int(sizeof(mine.bus)), ctx->device));
    FM_CUDA(ctx, cudaIpcGetMemHandle(&mine.a, ctx->spec));
    FM_CUDA(ctx, cudaIpcGetMemHandle(&mine.b, ctx->spec2));
    char* d_h = nullptr;
    FM_CUDA(ctx, cudaMalloc(&d_h, sizeof(Handles) * P));
    std::vector<Handles> all(P);
    int st = FM_OK;
    if (cudaMemcpy(d_h + sizeof(Handles) * ctx->rank, &mine, sizeof(Handles), cudaMemcpyHostToDevice) != cudaSuccess)
      st = set_error(ctx, FM_E_CUDA, "IPC handle upload");
    if (!st)
      st = nccl_check(ctx,
                      ncclAllGather(d_h + sizeof(Handles) * ctx->rank, d_h, sizeof(Handles), ncclChar,
                                    static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
                      "ncclAllGather(IPC handles)");
    if (!st && cudaStreamSynchronize(ctx->stream) != cudaSuccess) st = set_error(ctx, FM_E_CUDA, "IPC exchange");
    if (!st && cudaMemcpy(all.data(), d_h, sizeof(Handles) * P, cudaMemcpyDeviceToHost) != cudaSuccess)
      st = set_error(ctx, FM_E_CUDA, "IPC handle download");
    cudaFree(d_h);
    if (st) return st;
    // every peer must be a device this process can map: same node, visible,
    // peer access possible -- checked before any handle is opened
    for (int r = 0; r < P; ++r) {
      if (r == ctx->rank) continue;
      all[r].bus[sizeof(all[r].bus) - 1] = 0;
      int dev = -1, ok = 0;
      if (cudaDeviceGetByPCIBusId(&dev, all[r].bus) != cudaSuccess) {
        cudaGetLastError();
        return set_error(ctx, FM_E_UNSUPPORTED,
                         "slab rank " + std::to_string(r) + " runs on device " + all[r].bus +
                             ", which this process cannot see: the peer-store transposes need every rank's "
                             "device visible (or use FM_TRANSPOSE=nccl)");
      }
      if (dev == ctx->device)
        return set_error(ctx, FM_E_UNSUPPORTED, "slab ranks " + std::to_string(ctx->rank) + " and " +
                                                    std::to_string(r) + " share device " + all[r].bus);
      if (cudaDeviceCanAccessPeer(&ok, ctx->device, dev) != cudaSuccess || !ok) {
        cudaGetLastError();
        return set_error(ctx, FM_E_UNSUPPORTED,
                         "no peer access from device " + std::string(mine.bus) + " to " + all[r].bus +
                             " (slab rank " + std::to_string(r) + "): use FM_TRANSPOSE=nccl");
      }
    }
    for (int r = 0; r < P; ++r) {
      if (r == ctx->rank) {
        a[r] = ctx->spec;
        b[r] = ctx->spec2;
        continue;
      }
      void* pa = nullptr;
      void* pb = nullptr;
      FM_CUDA(ctx, cudaIpcOpenMemHandle(&pa, all[r].a, cudaIpcMemLazyEnablePeerAccess));
      ctx->ipc_open.push_back(pa);
      FM_CUDA(ctx, cudaIpcOpenMemHandle(&pb, all[r].b, cudaIpcMemLazyEnablePeerAccess));
      ctx->ipc_open.push_back(pb);
      a[r] = static_cast<double2*>(pa);
      b[r] = static_cast<double2*>(pb);
    }
  }
  ctx->h_dst_a = a;
  FM_CUDA(ctx, cudaMemcpy(ctx->d_dst_a, a.data(), sizeof(double2*) * kMaxRanks, cudaMemcpyHostToDevice));
  FM_CUDA(ctx, cudaMemcpy(ctx->d_dst_b, b.data(), sizeof(double2*) * kMaxRanks, cudaMemcpyHostToDevice));
  return FM_OK;
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
  FM_LAUNCHED_K(ctx, "k_sum_ranks");
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
  for (void* p : ctx->ipc_open) cudaIpcCloseMemHandle(p);
  ctx->ipc_open.clear();
  if (ctx->d_dst_a) cudaFree(ctx->d_dst_a);
  if (ctx->d_dst_b) cudaFree(ctx->d_dst_b);
  ctx->d_dst_a = ctx->d_dst_b = nullptr;
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

int fm_dist_route(int P, int Nx, int Ny, int nzh, int ncomp, int dir, int src, int comp, int i0, int i1, int kz,
                  int32_t* dst_rank, int64_t* dst_index) {
  if (P < 1 || P > kMaxRanks || Nx % P || Ny % P || src < 0 || src >= P || comp < 0 || comp >= ncomp || kz < 0 ||
      kz >= nzh || !dst_rank || !dst_index || (dir != 1 && dir != -1))
    return FM_E_INVALID;
  const int Xl = Nx / P, Yl = Ny / P;
  int d = 0;
  if (dir > 0) {  // y pass of x-slab src: (comp, xl = i0, y = i1, kz)
    if (i0 < 0 || i0 >= Xl || i1 < 0 || i1 >= Ny) return FM_E_INVALID;
    *dst_index = route_yf(Nx, Xl, Yl, nzh, src, comp, i0, i1, kz, d);
  } else {        // x pass of y-slab src: (comp, x = i0, yl = i1, kz)
    if (i0 < 0 || i0 >= Nx || i1 < 0 || i1 >= Yl) return FM_E_INVALID;
    *dst_index = route_xb(Ny, Xl, Yl, nzh, src, comp, i0, i1, kz, d);
  }
  *dst_rank = d;
  return FM_OK;
}

}  // extern "C"
