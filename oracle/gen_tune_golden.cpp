// gen_tune_golden.cpp -- tile candidate lists written by the UNMODIFIED
// reference (abq::enumerate_tile_candidates, /root/reference/proj/include/
// abq/tune.hpp:51-92) for the parity test of the GPU build's tune API.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/ and
// run by tests/golden/make_tune_golden.py, which commits the JSON under
// tests/golden/tune/.  One line per (p, q, m): the candidates in order,
// each as [BM, BN, BK, WM, WN, WK], plus the reference's padding_redundancy
// (tune.hpp:17-23) and tops_of (tune.hpp:129-131) on fixed inputs.
#include <cstdio>

#include "abq/tune.hpp"

int main() {
  const unsigned ps[] = {1, 2, 3, 4, 5, 8};
  const unsigned qs[] = {1, 2, 4, 7, 8};
  const std::size_t ms[] = {1, 7, 64, 128, 1000};
  std::printf("[\n");
  bool first = true;
  for (unsigned p : ps)
    for (unsigned q : qs)
      for (std::size_t m : ms) {
        const auto c = abq::enumerate_tile_candidates(p, q, m, 4096, 4096);
        std::printf("%s{\"p\": %u, \"q\": %u, \"m\": %zu, \"padding\": %.17g, \"candidates\": [", first ? "" : ",\n", p,
                    q, m, abq::padding_redundancy(m, p, abq::TileConfig::mma_m));
        first = false;
        for (std::size_t i = 0; i < c.size(); ++i)
          std::printf("%s[%zu, %zu, %zu, %zu, %zu, %zu]", i ? ", " : "", c[i].BM, c[i].BN, c[i].BK, c[i].WM, c[i].WN,
                      c[i].WK);
        std::printf("]}");
      }
  std::printf(",\n{\"tops_of\": [128, 11008, 4096, 18.5, %.17g]}\n]\n", abq::detail::tops_of(128, 11008, 4096, 18.5));
  return 0;
}
