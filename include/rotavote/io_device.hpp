// Device CSV ingest next to the reference's read_correspondences (io.hpp:11-13, io.cpp:66-101):
// the same file format, strictness, exceptions and messages, parsed on the GPU
// (rv_read_correspondences_csv). The reference's io.hpp stays the drop-in for the other I/O
// functions; a maintainer switches its read path by forwarding io.cpp:66-101 to
// read_correspondences_device, or keeps the rows in HBM with
// read_correspondences_to_device and hands them to rv_estimate_single_device.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "angles.hpp"
#include "device.hpp"

namespace rotavote {

namespace detail {
inline void check_csv(rv_status st, int64_t line) {
  if (st == RV_OK) return;
  const std::string m = rv_context_last_error(context());
  if (st == RV_ERR_PARSE) throw ParseError(m, static_cast<int>(line));
  if (st == RV_ERR_EMPTY_FILE) throw EmptyFile(m);
  if (st == RV_ERR_IO) throw IoError(m);
  check(st);
}
}  // namespace detail

// Rows parsed on the device and left there: n x 6 f64 (Correspondence layout), valid until the
// next CSV call on this thread's context.
inline const double* read_correspondences_to_device(const std::string& path, int64_t* n_rows) {
  const double* d = nullptr;
  int64_t line = 0;
  const rv_status st = rv_read_correspondences_csv(detail::context(), path.c_str(), &d, n_rows, &line);
  detail::check_csv(st, line);  // (line read after the call: argument order is unspecified)
  return d;
}

inline std::vector<Correspondence> read_correspondences_device(const std::string& path) {
  int64_t n = 0;
  const double* d = read_correspondences_to_device(path, &n);
  std::vector<double> flat(static_cast<size_t>(n) * 6);
  detail::check(rv_device_to_host(detail::context(), flat.data(), d, static_cast<int64_t>(flat.size() * sizeof(double))));
  std::vector<Correspondence> out(static_cast<size_t>(n));
  for (size_t i = 0; i < out.size(); ++i) {
    const double* r = flat.data() + 6 * i;
    out[i].x = Vec3(r[0], r[1], r[2]);
    out[i].y = Vec3(r[3], r[4], r[5]);
  }
  return out;
}

}  // namespace rotavote
