// Drop-in run output (reference API: proj/core/include/fftmech/snapshot.hpp,
// SnapshotSink of proj/core/src/run_config.cpp:434-493).
//
// Snapshots are raw little-endian float64 slabs (component-major, one file per
// field) plus a `meta_<k>.json` record; report.csv carries one row per
// increment.  Byte layout pinned to the reference's own records
// (tests/golden/reference_records/).
#pragma once

#include <filesystem>
#include <map>
#include <string>
#include <vector>

#include "fftmech/fields.hpp"
#include "fftmech/solver.hpp"
#include "fftmech/tensor2.hpp"

namespace fftmech {

struct ReportRow {
  std::string increment;
  int newton_iters = 0;
  long cg_iters_total = 0;
  double residual = 0.0;
  double wall_ms = 0.0;
  double eps_bar = 0.0;
};

// `increment,newton_iters,cg_iters_total,residual,wall_ms,eps_bar`, %.17g.
void write_report_csv(const std::filesystem::path& file, const std::vector<ReportRow>& rows);

struct SnapshotFieldData {
  int components = 1;          // 1 for scalars, tdim^2 for tensors
  std::vector<double> values;  // component-major slabs of n values
};

struct Snapshot {
  int increment = 0;
  std::string label;
  GridShape grid;
  int tensor_dim = 3;
  Tensor2 fbar;
  std::map<std::string, SnapshotFieldData> fields;
};

void write_snapshot(const std::filesystem::path& dir, const Snapshot& snap);
Snapshot read_snapshot(const std::filesystem::path& dir, int increment);
std::vector<int> list_snapshots(const std::filesystem::path& dir);
Tensor2Field snapshot_to_field(const Snapshot& snap, const std::string& name);
// Legacy-VTK structured points (x fastest), %.12g.
void write_vtk_snapshot(const std::filesystem::path& file, const Snapshot& snap);

// What a run writes (RunConfig "output" block).
struct OutputOptions {
  std::filesystem::path directory = "fftmech_out";
  std::vector<std::string> fields = {"F", "P", "eq"};  // subset of F, P, eq, epsp
  int stride = 1;                                      // snapshot every stride-th increment
  bool vtk = false;
};

// ProgramSink that accumulates report rows and writes a snapshot every
// `stride` increments.  eq is computed by the model's equivalent_stress_field
// (device kernel fm_equivalent_stress).
class SnapshotSink final : public ProgramSink {
 public:
  explicit SnapshotSink(OutputOptions opts);
  void on_increment(std::size_t index, const Increment& inc, const SolveReport& report, const Tensor2Field& F,
                    const Tensor2Field& P, MaterialModel& model) override;
  void finish() const;
  // Partial report plus failure.json {increment, error}.
  void record_failure(const std::string& label, const std::string& what) const;
  const std::vector<ReportRow>& rows() const { return rows_; }

 private:
  OutputOptions opts_;
  std::vector<ReportRow> rows_;
};

}  // namespace fftmech
