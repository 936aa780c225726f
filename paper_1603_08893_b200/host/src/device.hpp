// Internal glue between the drop-in C++ API and the C ABI of libfftmech_b200.so.
#pragma once

#include <memory>
#include <span>
#include <string>

#include "../../../include/fftmech_b200.h"
#include "fftmech/grid.hpp"

namespace fftmech::detail {

// One device context per (grid, tdim, Nyquist mode), shared by the
// projection operator and the models bound to it.
struct Device {
  fm_ctx* h = nullptr;
  GridShape shape;
  int tdim = 3;
  int mode = 0;
  ~Device();
};

std::shared_ptr<Device> device_for(const GridShape& shape, int tdim, int mode);

// Maps an fm_status onto the reference exception hierarchy.
[[noreturn]] void throw_status(fm_ctx* h, int status, const std::string& where);
inline void check(fm_ctx* h, int status, const char* where) {
  if (status != FM_OK) throw_status(h, status, where);
}

// RAII device field on a context.
class DevField {
 public:
  DevField(const std::shared_ptr<Device>& dev, int ncomp);
  ~DevField();
  DevField(const DevField&) = delete;
  DevField& operator=(const DevField&) = delete;
  fm_field* get() const { return f_; }
  void upload(std::span<const double> host);
  void download(std::span<double> host) const;

 private:
  std::shared_ptr<Device> dev_;
  fm_field* f_ = nullptr;
};

}  // namespace fftmech::detail
