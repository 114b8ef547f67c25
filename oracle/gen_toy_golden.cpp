// gen_toy_golden.cpp -- model-level golden vectors from the UNMODIFIED reference
// toy block (/root/reference/proj/include/abq/toyblock.hpp:66-282): the seeded
// weights and input, forward_fp, and forward_quant under three configurations
// (W4A4 and W8A8 with init_params; W3A6 with non-trivial balance vectors,
// alpha/beta and the down_proj compensation pair), plus
// first_token_attention_share of each trace.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/ and run
// by tests/golden/make_toy_golden.py (commits tests/golden/toy/toy.json).
#include <cstdio>
#include <string>

#include "abq/toyblock.hpp"

namespace {

void put(const char* name, const abq::Mat& m, bool comma = true) {
  std::printf("\"%s\": {\"rows\": %zu, \"cols\": %zu, \"data\": [", name, m.rows, m.cols);
  for (std::size_t i = 0; i < m.data.size(); ++i) std::printf("%s%.17g", i ? "," : "", m.data[i]);
  std::printf("]}%s\n", comma ? "," : "");
}

void put_vec(const char* name, const std::vector<double>& v) {
  std::printf("\"%s\": [", name);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? "," : "", v[i]);
  std::printf("],\n");
}

}  // namespace

int main() {
  const abq::ToyBlock b = abq::ToyBlock::seeded(7, 16, 2);
  abq::Rng rng(8);
  const abq::Mat x = rng.gauss_matrix(8, 16);
  std::printf("{\"dim\": %zu, \"heads\": %zu, \"hidden\": %zu,\n", b.dim, b.heads, b.hidden);
  put("x", x);
  put("wq", b.wq);
  put("wk", b.wk);
  put("wv", b.wv);
  put("wo", b.wo);
  put("wgate", b.wgate);
  put("wup", b.wup);
  put("wdown", b.wdown);
  auto fp = abq::forward_fp(b, x);
  put("forward_fp", fp.first);
  std::printf("\"share_fp\": %.17g,\n", abq::first_token_attention_share(fp.second));
  // W4A4 / W8A8, init params
  for (unsigned bits : {4u, 8u}) {
    auto r = abq::forward_quant(b, x, abq::BlockSpecs::make(bits, bits), b.init_params());
    const std::string n = "quant_w" + std::to_string(bits) + "a" + std::to_string(bits);
    put(n.c_str(), r.first);
    std::printf("\"share_%s\": %.17g,\n", n.c_str(), abq::first_token_attention_share(r.second));
  }
  // W3A6 with balance vectors, alpha/beta and compensation on down_proj
  abq::BlockQuantParams p = b.init_params();
  abq::Rng prng(9);
  for (abq::Layer l : abq::kLayers) {
    for (auto& s : p.at(l).s) s = prng.uniform(0.5, 1.5);
    p.at(l).alpha = 0.9;
    p.at(l).beta = 0.95;
  }
  for (auto& v : p.comp_a) v = prng.uniform(0.9, 1.1);
  for (auto& v : p.comp_b) v = prng.uniform(-0.01, 0.01);
  p.gamma = 1;
  for (abq::Layer l : abq::kLayers) put_vec((std::string("s_") + abq::layer_name(l)).c_str(), p.at(l).s);
  put_vec("comp_a", p.comp_a);
  put_vec("comp_b", p.comp_b);
  auto r = abq::forward_quant(b, x, abq::BlockSpecs::make(3, 6), p);
  std::printf("\"share_quant_w3a6_params\": %.17g,\n", abq::first_token_attention_share(r.second));
  put("quant_w3a6_params", r.first, false);
  std::printf("}\n");
  return 0;
}
