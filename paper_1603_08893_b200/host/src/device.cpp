#include "device.hpp"

#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <tuple>

#include "fftmech/errors.hpp"
#include "fftmech/placement.hpp"
#include "fftmech/solver.hpp"

namespace fftmech {

namespace {
std::mutex g_placement_mu;
Placement g_placement;
}  // namespace

void set_placement(const Placement& p) {
  if (p.ranks < 1) throw std::invalid_argument("placement: ranks must be >= 1");
  std::lock_guard<std::mutex> lock(g_placement_mu);
  g_placement = p;
}
Placement placement() {
  std::lock_guard<std::mutex> lock(g_placement_mu);
  return g_placement;
}

}  // namespace fftmech

namespace fftmech::detail {

Device::~Device() {
  if (h) fm_ctx_destroy(h);
}

std::shared_ptr<Device> device_for(const GridShape& shape, int tdim, int mode) {
  using Key = std::tuple<int, int, int, int, double, double, double, int, int, int, int, bool>;
  static std::mutex mu;
  static std::map<Key, std::weak_ptr<Device>> registry;
  const Placement where = placement();
  const char* env = std::getenv("FFTMECH_DEVICE");
  const int device = where.device >= 0 ? where.device : (env ? std::atoi(env) : 0);
  const Key key{shape.dim, shape.points[0], shape.points[1], shape.points[2], shape.lengths[0],
                shape.lengths[1], shape.lengths[2], tdim, mode, device, where.ranks, where.staged_transposes};
  std::lock_guard<std::mutex> lock(mu);
  if (auto live = registry[key].lock()) return live;
  auto dev = std::make_shared<Device>();
  dev->shape = shape;
  dev->tdim = tdim;
  dev->mode = mode;
  const int32_t pts[3] = {shape.points[0], shape.points[1], shape.points[2]};
  const double len[3] = {shape.lengths[0], shape.lengths[1], shape.lengths[2]};
  const int st = fm_ctx_create(shape.dim, pts, len, tdim, mode, device, &dev->h);
  if (st == FM_E_INVALID) throw std::invalid_argument("tensor dim must be in [grid dim, 3]");
  if (st != FM_OK) throw Error("fftmech: no usable CUDA device for the sm_100a kernels (status " + std::to_string(st) + ")");
  if (where.ranks > 1) {
    if (where.staged_transposes) check(dev->h, fm_ctx_set_transpose(dev->h, 1), "placement.staged_transposes");
    check(dev->h, fm_ctx_set_virtual_ranks(dev->h, where.ranks), "placement.ranks");
  }
  registry[key] = dev;
  return dev;
}

void throw_status(fm_ctx* h, int status, const std::string& where) {
  fm_error_info info{};
  if (h) fm_last_error_info(h, &info);
  const std::string msg = where + ": " + (h ? fm_last_error(h) : "error");
  switch (status) {
    case FM_E_INVALID: throw std::invalid_argument(msg);
    case FM_E_INVERTED: throw InvertedElement(static_cast<std::size_t>(info.node));
    case FM_E_NOT_SPD: throw NotPositiveDefinite(static_cast<std::size_t>(info.node), info.value);
    case FM_E_SINGULAR: throw SingularTensor(static_cast<std::size_t>(info.node));
    case FM_E_CG_STALLED: throw CgStalled(info.cg_iterations, info.value);
    case FM_E_COMPLEX_RESIDUE: throw ComplexResidue(info.value, 0.0);  // debug mode only (fm_ctx_set_debug)
    default: throw Error(msg);
  }
}

DevField::DevField(const std::shared_ptr<Device>& dev, int ncomp) : dev_(dev) {
  check(dev_->h, fm_field_alloc(dev_->h, ncomp, &f_), "fm_field_alloc");
}
DevField::~DevField() {
  if (f_) fm_field_free(dev_->h, f_);
}
void DevField::upload(std::span<const double> host) {
  check(dev_->h, fm_field_upload(dev_->h, f_, host.data(), static_cast<int64_t>(host.size())), "upload");
}
void DevField::download(std::span<double> host) const {
  check(dev_->h, fm_field_download(dev_->h, f_, host.data(), static_cast<int64_t>(host.size())), "download");
}

}  // namespace fftmech::detail
