// gen_io_golden.cpp -- golden on-disk weight files written by the UNMODIFIED
// reference (abq::io, /root/reference/proj/include/abq/io.hpp:64-124).
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/ and run
// by tests/golden/make_io_golden.py, which commits the files under
// tests/golden/io/.  Writes, into the directory given as argv[1]:
//   wt_pc4.abqt   QuantizedTensor, per-channel asymmetric 4-bit, 5 x 70
//                 (abq::io::write_quantized; scales are stored as f32)
//   wt_pt3.abqt   per-tensor 3-bit, 3 x 129
//   wt_pc4.abqp   bitpack(codes, planes) of wt_pc4 (abq::io::write_planes)
//   bundle.abqz   "ABQZ" bundle of two layers (name record + ABQT + ABQP per
//                 layer), the layout abqtool's write_bundle emits
//                 (tools/abqtool.cpp:211-237), written with the reference's
//                 own record writers
#include <cstdint>
#include <fstream>
#include <string>

#include "abq/bitplane.hpp"
#include "abq/core.hpp"
#include "abq/io.hpp"
#include "abq/quantizer.hpp"

namespace {

abq::QuantizedTensor make_q(std::uint64_t seed, std::size_t rows, std::size_t cols, unsigned bits,
                            abq::Granularity g) {
  abq::Rng rng(seed);
  abq::Mat w = rng.gauss_matrix(rows, cols, 0.02);
  abq::QuantSpec spec;
  spec.bits = bits;
  spec.scheme = abq::Scheme::Asymmetric;
  spec.granularity = g;
  return abq::quantize(w, spec);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string dir = argv[1];
  const abq::QuantizedTensor a = make_q(31, 5, 70, 4, abq::Granularity::PerChannel);
  const abq::QuantizedTensor b = make_q(32, 3, 129, 3, abq::Granularity::PerTensor);
  {
    auto os = abq::io::detail::open_out(dir + "/wt_pc4.abqt");
    abq::io::write_quantized(os, a);
  }
  {
    auto os = abq::io::detail::open_out(dir + "/wt_pt3.abqt");
    abq::io::write_quantized(os, b);
  }
  {
    auto os = abq::io::detail::open_out(dir + "/wt_pc4.abqp");
    abq::io::write_planes(os, abq::bitpack(a.codes, a.spec.planes()));
  }
  {
    auto os = abq::io::detail::open_out(dir + "/bundle.abqz");
    os.write("ABQZ", 4);
    abq::io::detail::put<std::uint16_t>(os, abq::io::kFormatVersion);
    abq::io::detail::put<std::uint32_t>(os, 2);
    const abq::QuantizedTensor* qs[2] = {&a, &b};
    const char* names[2] = {"up", "down"};
    for (int i = 0; i < 2; ++i) {
      const std::string name = names[i];
      abq::io::detail::put<std::uint16_t>(os, std::uint16_t(name.size()));
      os.write(name.data(), std::streamsize(name.size()));
      abq::io::write_quantized(os, *qs[i]);
      abq::io::write_planes(os, abq::bitpack(qs[i]->codes, qs[i]->spec.planes()));
    }
  }
  return 0;
}
