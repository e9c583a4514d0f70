// CPU check of the C++ mirror's log2_rational replica (ckks32_b200.hpp
// scale_log2): prints %a of scale_log2 for scales given as
// "pow2 n1,n2,.. d1,d2,.." lines on stdin (empty lists as "-").
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>

#include "../../paper_2407_13055_b200/cpp/ckks32_b200.hpp"

using namespace ckks32::b200;

static std::vector<uint32_t> parse(const std::string& t) {
  std::vector<uint32_t> v;
  if (t == "-") return v;
  std::stringstream ss(t);
  std::string x;
  while (std::getline(ss, x, ',')) v.push_back((uint32_t)std::stoul(x));
  return v;
}

int main() {
  std::string line;
  while (std::getline(std::cin, line)) {
    std::stringstream ss(line);
    int p2;
    std::string a, b;
    ss >> p2 >> a >> b;
    Scale s = Scale::rational(p2, parse(a), parse(b));
    std::printf("%a\n", scale_log2(s));
  }
  return 0;
}
