// Ours (not a reference file): the device CSV ingest (include/rotavote/io_device.hpp) against the
// reference's read_correspondences (io.cpp, compiled into this binary as a caller) on the
// reference's own io fixtures plus a writer round trip -- same rows, same exception types and
// messages.
#include <doctest.h>

#include <cstdio>
#include <fstream>
#include <string>

#include "rotavote/io.hpp"
#include "rotavote/io_device.hpp"

using namespace rotavote;

namespace {
std::string tmp_file(const std::string& name, const std::string& text) {
  const std::string p = std::string("/tmp/rv_dropin_io_") + name;
  std::ofstream(p, std::ios::binary) << text;
  return p;
}

template <typename F>
std::string what_of(F&& f) {
  try {
    f();
  } catch (const ParseError& e) {
    return std::string("ParseError:") + e.what() + ":" + std::to_string(e.line);
  } catch (const EmptyFile& e) {
    return std::string("EmptyFile:") + e.what();
  } catch (const IoError& e) {
    return std::string("IoError:") + e.what();
  }
  return "ok";
}
}  // namespace

TEST_CASE("device CSV ingest matches the reference read_correspondences") {
  const char* fixtures[] = {"1,0,0,0,1,0\n0,1,0,-1,0,0\n", "x0,x1,x2,y0,y1,y2\n1,0,0,0,1,0\n",
                            "1,0,0,0,1,0\n1,0,0,0,1\n",  "1,0,0,0,1,0\n1,zero,0,0,1,0\n",
                            "",                          "x0,x1,x2,y0,y1,y2\n",
                            "1,2,3,4,5,6\r\n\r\n7,8,9,10,11,12", "0.1,-2.5e-3,1e300,4.9406564584124654e-324,-0,7\n"};
  int k = 0;
  for (const char* text : fixtures) {
    const std::string p = tmp_file(std::to_string(k++) + ".csv", text);
    std::vector<Correspondence> a, b;
    const std::string ea = what_of([&] { a = read_correspondences(p); });
    const std::string eb = what_of([&] { b = read_correspondences_device(p); });
    if (ea != eb) std::printf("fixture %d: reference '%s' vs device '%s'\n", k - 1, ea.c_str(), eb.c_str());
    CHECK(ea == eb);
    REQUIRE(a.size() == b.size());
    for (size_t i = 0; i < a.size(); ++i) {
      CHECK((a[i].x - b[i].x).norm() == 0.0);
      CHECK((a[i].y - b[i].y).norm() == 0.0);
    }
    std::remove(p.c_str());
  }
  CHECK(what_of([] { read_correspondences_device("/tmp/rv_dropin_io_missing.csv"); }) ==
        what_of([] { read_correspondences("/tmp/rv_dropin_io_missing.csv"); }));
}
