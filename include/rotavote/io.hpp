// Drop-in for proj/include/rotavote/io.hpp (io.hpp:1-30): the same
// declarations, formats, exceptions and messages (io.cpp:66-205).
//   read_correspondences     parsed ON THE DEVICE (rv_read_correspondences_csv, io_device.hpp):
//                            rows, header rule, strictness and error lines identical to io.cpp:66-101
//   write_correspondences    header + "%.17g" rows (io.cpp:103-110)
//   write_result / read_result
//                            the JSON result document (io.cpp:112-160): an array of objects with
//                            the keys in sorted order, numbers that round-trip bit-exact (shortest
//                            round-trip digits out, std::from_chars in). A small self-contained JSON
//                            writer/reader -- no third-party JSON dependency
//   write_truth / read_truth the truth sidecar (io.cpp:162-193)
//   dump_accumulator         text / binary PGM plots (io.cpp:195-205, voting.cpp:218-239)
// Header-only; a build uses this file INSTEAD of io.cpp.
#pragma once

#include <algorithm>
#include <charconv>
#include <cctype>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <map>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "estimator.hpp"
#include "io_device.hpp"
#include "rotavote/synth.hpp"  // SceneTruth (the reference's synth.hpp, unchanged)
#include "voting.hpp"

namespace rotavote {

enum class DumpFormat { Text, Pgm };

namespace detail {

inline std::ofstream io_out(const std::string& path, std::ios_base::openmode mode = std::ios_base::out) {
  std::ofstream f(path, mode);
  if (!f) throw IoError("cannot open for writing: " + path);
  return f;
}
inline std::ifstream io_in(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open for reading: " + path);
  return f;
}
inline std::string g17(double v) {  // the reference's %.17g
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

// JSON number text for a double: shortest round-trip digits; integral values keep a ".0" and NaN
// / infinities become null (the conventions of the reference's JSON library).
inline std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  char b[64];
  const auto r = std::to_chars(b, b + sizeof b, v);
  std::string s(b, r.ptr);
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}

// Minimal JSON value for the result document: null, number (kept as text), string, array, object.
struct JVal {
  enum Kind { Null, Num, Str, Arr, Obj } kind = Null;
  std::string text;
  std::vector<JVal> items;
  std::map<std::string, JVal> fields;
  const JVal& at(const std::string& k) const {
    const auto it = fields.find(k);
    if (it == fields.end()) throw ParseError("bad result document: missing key '" + k + "'", 0);
    return it->second;
  }
  double num() const {
    if (kind == Null) return std::nan("");
    double v = 0.0;
    const auto r = std::from_chars(text.data(), text.data() + text.size(), v);
    if (kind != Num || r.ec != std::errc{}) throw ParseError("bad result document: expected a number", 0);
    return v;
  }
};

class JParser {
 public:
  explicit JParser(std::string s) : s_(std::move(s)) {}
  JVal parse() {
    JVal v = value();
    ws();
    if (p_ != s_.size()) bad("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void bad(const char* what) const {
    throw ParseError(std::string("bad result document: ") + what + " at offset " + std::to_string(p_), 0);
  }
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\r' || s_[p_] == '\t')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < s_.size() && s_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  std::string str() {
    if (!eat('"')) bad("expected a string");
    std::string out;
    while (p_ < s_.size() && s_[p_] != '"') {
      if (s_[p_] == '\\') {
        if (++p_ >= s_.size()) bad("bad escape");
      }
      out += s_[p_++];
    }
    if (p_ >= s_.size()) bad("unterminated string");
    ++p_;
    return out;
  }
  JVal value() {
    ws();
    if (p_ >= s_.size()) bad("unexpected end");
    JVal v;
    const char c = s_[p_];
    if (c == '[') {
      ++p_;
      v.kind = JVal::Arr;
      if (eat(']')) return v;
      do v.items.push_back(value());
      while (eat(','));
      if (!eat(']')) bad("expected ']'");
    } else if (c == '{') {
      ++p_;
      v.kind = JVal::Obj;
      if (eat('}')) return v;
      do {
        std::string k = str();
        if (!eat(':')) bad("expected ':'");
        v.fields[k] = value();
      } while (eat(','));
      if (!eat('}')) bad("expected '}'");
    } else if (c == '"') {
      v.kind = JVal::Str;
      v.text = str();
    } else if (s_.compare(p_, 4, "null") == 0) {
      p_ += 4;
    } else {
      const size_t b = p_;
      while (p_ < s_.size() && (std::isdigit((unsigned char)s_[p_]) || std::strchr("+-.eE", s_[p_]))) ++p_;
      if (p_ == b) bad("unexpected character");
      v.kind = JVal::Num;
      v.text = s_.substr(b, p_ - b);
    }
    return v;
  }
  std::string s_;
  size_t p_ = 0;
};

}  // namespace detail

inline std::vector<Correspondence> read_correspondences(const std::string& path) {
  return read_correspondences_device(path);
}

inline void write_correspondences(const std::vector<Correspondence>& corrs, const std::string& path) {
  auto f = detail::io_out(path);
  f << "x0,x1,x2,y0,y1,y2\n";
  for (const Correspondence& c : corrs) {
    const double v[6] = {c.x.x(), c.x.y(), c.x.z(), c.y.x(), c.y.y(), c.y.z()};
    for (int k = 0; k < 6; ++k) f << detail::g17(v[k]) << (k == 5 ? '\n' : ',');
  }
}

inline void write_result(const std::vector<RotationEstimate>& estimates, const std::string& path) {
  // one object per estimate, keys sorted, two-space indentation
  std::string out;
  auto line = [&](int depth, const std::string& s) { out.append((size_t)depth * 2, ' ').append(s); };
  auto number_list = [&](int depth, const std::string& key, const std::vector<std::string>& vals, bool last) {
    if (vals.empty()) {
      line(depth, "\"" + key + "\": []" + (last ? "\n" : ",\n"));
      return;
    }
    line(depth, "\"" + key + "\": [\n");
    for (size_t i = 0; i < vals.size(); ++i) line(depth + 1, vals[i] + (i + 1 < vals.size() ? ",\n" : "\n"));
    line(depth, last ? "]\n" : "],\n");
  };
  if (estimates.empty()) {
    out = "[]\n";
  } else {
    out = "[\n";
    for (size_t k = 0; k < estimates.size(); ++k) {
      const RotationEstimate& e = estimates[k];
      line(1, "{\n");
      line(2, "\"angle_rad\": " + detail::json_double(e.angle) + ",\n");
      number_list(2, "axis", {detail::json_double(e.axis.x()), detail::json_double(e.axis.y()),
                              detail::json_double(e.axis.z())}, false);
      line(2, "\"axis_votes\": " + std::to_string(e.axis_votes) + ",\n");
      line(2, "\"elapsed_s\": " + detail::json_double(e.elapsed_s) + ",\n");
      line(2, "\"inlier_count\": " + std::to_string(e.inliers.size()) + ",\n");
      std::vector<std::string> idx;
      idx.reserve(e.inliers.size());
      for (int i : e.inliers) idx.push_back(std::to_string(i));
      number_list(2, "inlier_indices", idx, false);
      std::vector<std::string> m;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) m.push_back(detail::json_double(e.rotation(r, c)));
      number_list(2, "matrix", m, true);
      line(1, k + 1 < estimates.size() ? "},\n" : "}\n");
    }
    out += "]\n";
  }
  auto f = detail::io_out(path);
  f << out;
}

inline std::vector<RotationEstimate> read_result(const std::string& path) {
  auto f = detail::io_in(path);
  const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  const detail::JVal doc = detail::JParser(text).parse();
  std::vector<RotationEstimate> out;
  for (const detail::JVal& item : doc.items) {
    RotationEstimate e;
    const auto& ax = item.at("axis").items;
    if (ax.size() != 3) throw ParseError("bad result document: axis needs 3 numbers", 0);
    e.axis = Vec3(ax[0].num(), ax[1].num(), ax[2].num());
    e.angle = item.at("angle_rad").num();
    const auto& m = item.at("matrix").items;
    if (m.size() != 9) throw ParseError("bad result document: matrix needs 9 numbers", 0);
    for (int i = 0; i < 9; ++i) e.rotation(i / 3, i % 3) = m[(size_t)i].num();
    for (const auto& v : item.at("inlier_indices").items) e.inliers.push_back(static_cast<int>(v.num()));
    e.axis_votes = static_cast<std::uint32_t>(item.at("axis_votes").num());
    e.elapsed_s = item.at("elapsed_s").num();
    out.push_back(std::move(e));
  }
  return out;
}

inline void write_truth(const SceneTruth& truth, const std::string& path) {
  std::ostringstream s;
  s << "rotations " << truth.rotations.size() << '\n';
  for (const Mat3& r : truth.rotations)
    for (int i = 0; i < 9; ++i) s << detail::g17(r(i / 3, i % 3)) << (i == 8 ? '\n' : ' ');
  s << "labels " << truth.labels.size() << '\n';
  for (size_t i = 0; i < truth.labels.size(); ++i) s << (i ? " " : "") << truth.labels[i];
  s << '\n';
  auto f = detail::io_out(path);
  f << s.str();
}

inline SceneTruth read_truth(const std::string& path) {
  auto f = detail::io_in(path);
  SceneTruth t;
  std::string tag;
  std::size_t n = 0;
  if (!(f >> tag >> n) || tag != "rotations") throw ParseError("expected 'rotations N'", 1);
  t.rotations.assign(n, Mat3::Zero());
  for (Mat3& r : t.rotations)
    for (int i = 0; i < 9; ++i)
      if (!(f >> r(i / 3, i % 3))) throw ParseError("truncated rotation matrix", 0);
  if (!(f >> tag >> n) || tag != "labels") throw ParseError("expected 'labels N'", 0);
  t.labels.assign(n, 0);
  for (int& l : t.labels)
    if (!(f >> l)) throw ParseError("truncated label list", 0);
  return t;
}

inline void dump_accumulator(const Accumulator2D& acc, const std::string& path, DumpFormat format) {
  auto f = format == DumpFormat::Pgm ? detail::io_out(path, std::ios_base::out | std::ios_base::binary)
                                     : detail::io_out(path);
  if (format == DumpFormat::Pgm) dump_accumulator_pgm(acc, f);
  else dump_accumulator_text(acc, f);
  if (!f) throw IoError("write failed: " + path);
}

}  // namespace rotavote
