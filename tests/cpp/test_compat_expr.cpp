// Expression front-end of the source-compatible layer (include/mcbatch/expr.hpp)
// dumped in the format of oracle/ref_shim.cpp's ref_expr_dump, one line per
// input line "dim|names|source|point...|params..." (';'-separated numbers), for
// tests/test_compat_expr.py to compare with the reference.  Host only: parse,
// compile (postfix + stack need), tree_eval and the print/parse round trip.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "mcbatch/expr.hpp"

using namespace mcbatch;

static std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  std::istringstream in(s);
  while (std::getline(in, cur, sep)) out.push_back(cur);
  if (!s.empty() && s.back() == sep) out.emplace_back();
  return out;
}

static std::string hex(double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, 8);
  char b[24];
  std::snprintf(b, sizeof b, "%016llx", (unsigned long long)u);
  return b;
}

int main() {
  std::string line;
  while (std::getline(std::cin, line)) {
    const std::vector<std::string> f = split(line, '|');
    const std::size_t dim = std::stoul(f[0]);
    std::vector<std::string> names = f[1].empty() ? std::vector<std::string>{} : split(f[1], ',');
    std::vector<double> point, params;
    for (const std::string& t : split(f[3], ';')) if (!t.empty()) point.push_back(std::stod(t));
    for (const std::string& t : split(f[4], ';')) if (!t.empty()) params.push_back(std::stod(t));
    std::string out;
    try {
      Expr e = parse(f[2]);
      CompiledProgram p = compile(e, dim, names);
      out = "OK " + std::to_string(p.stack_need()) + " ";
      for (const Instr& in : p.code())
        out += std::to_string(int(in.op)) + ":" + std::to_string(in.index) + ":" + hex(in.value) + ",";
      out += " " + hex(tree_eval(e, point, names, params));
      out += " " + std::to_string(parse(to_string(e)) == e);
    } catch (const SyntaxError&) {
      out = "ERR SyntaxError";
    } catch (const UnknownFunction&) {
      out = "ERR UnknownFunction";
    } catch (const ArityMismatch&) {
      out = "ERR ArityMismatch";
    } catch (const DimensionError&) {
      out = "ERR DimensionError";
    } catch (const UnboundParameter&) {
      out = "ERR UnboundParameter";
    } catch (const std::exception&) {
      out = "ERR other";
    }
    std::cout << out << "\n";
  }
  return 0;
}
