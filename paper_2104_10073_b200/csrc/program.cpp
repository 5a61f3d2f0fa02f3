// program.cpp — DSL parser/compiler for the GPU interpreter (see program.hpp).
#include "program.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numbers>

namespace mcb {
namespace prog {

namespace {

struct FnInfo {
  Op op;
  unsigned arity;
};

const std::map<std::string, FnInfo>& functions() {
  static const std::map<std::string, FnInfo> t = {
      {"sin", {kSin, 1}},   {"cos", {kCos, 1}},   {"tan", {kTan, 1}},     {"asin", {kAsin, 1}},
      {"acos", {kAcos, 1}}, {"atan", {kAtan, 1}}, {"exp", {kExp, 1}},     {"log", {kLog, 1}},
      {"sqrt", {kSqrt, 1}}, {"abs", {kAbs, 1}},   {"floor", {kFloor, 1}}, {"pow", {kPow, 2}},
      {"min", {kMin, 2}},   {"max", {kMax, 2}}};
  return t;
}

// ---- syntax tree -------------------------------------------------------------

struct Node {
  enum Kind { Num, Var, Param, Neg, Bin, Call } kind;
  double value = 0.0;
  uint32_t var = 0;
  std::string name;
  Op op = kAdd;
  std::vector<std::unique_ptr<Node>> kids;
};
using NodeP = std::unique_ptr<Node>;

NodeP make(Node::Kind k) {
  auto n = std::make_unique<Node>();
  n->kind = k;
  return n;
}

// ---- lexer -------------------------------------------------------------------

enum class Tok { Num, Ident, Plus, Minus, Star, Slash, Caret, LParen, RParen, Comma, End };

class Lexer {
 public:
  explicit Lexer(const std::string& s) : s_(s) { next(); }
  Tok tok = Tok::End;
  std::size_t at = 0;  // offset of the current token
  double num = 0.0;
  std::string ident;

  void next() {
    while (p_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[p_]))) ++p_;
    at = p_;
    if (p_ >= s_.size()) {
      tok = Tok::End;
      return;
    }
    const char c = s_[p_];
    static const std::string punct = "+-*/^(),";
    static const Tok ptok[] = {Tok::Plus,  Tok::Minus,  Tok::Star,   Tok::Slash,
                               Tok::Caret, Tok::LParen, Tok::RParen, Tok::Comma};
    if (auto k = punct.find(c); k != std::string::npos) {
      tok = ptok[k];
      ++p_;
      return;
    }
    if (std::isdigit(static_cast<unsigned char>(c))) {
      std::size_t q = p_;
      auto digits = [&] {
        while (q < s_.size() && std::isdigit(static_cast<unsigned char>(s_[q]))) ++q;
      };
      digits();
      if (q < s_.size() && s_[q] == '.') {
        ++q;
        digits();
      }
      if (q < s_.size() && (s_[q] == 'e' || s_[q] == 'E')) {
        std::size_t r = q + 1;
        if (r < s_.size() && (s_[r] == '+' || s_[r] == '-')) ++r;
        if (r < s_.size() && std::isdigit(static_cast<unsigned char>(s_[r]))) {
          q = r;
          digits();
        }  // otherwise the 'e' starts an identifier
      }
      num = std::strtod(s_.substr(p_, q - p_).c_str(), nullptr);
      p_ = q;
      tok = Tok::Num;
      return;
    }
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      std::size_t q = p_;
      while (q < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[q])) || s_[q] == '_')) ++q;
      ident = s_.substr(p_, q - p_);
      p_ = q;
      tok = Tok::Ident;
      return;
    }
    throw ParseError(p_, std::string("unexpected character '") + c + "'");
  }

 private:
  const std::string& s_;
  std::size_t p_ = 0;
};

// x followed by a decimal index without a leading zero -> 0-based variable
bool variable_index(const std::string& s, std::size_t at, uint32_t& out) {
  if (s.size() < 2 || s[0] != 'x' || s[1] < '1' || s[1] > '9') return false;
  uint64_t v = 0;
  for (std::size_t i = 1; i < s.size(); ++i) {
    if (!std::isdigit(static_cast<unsigned char>(s[i]))) return false;
    v = v * 10 + uint64_t(s[i] - '0');
    if (v > 1000000) throw ParseError(at, "variable index too large");
  }
  out = uint32_t(v - 1);
  return true;
}

// ---- recursive-descent parser ------------------------------------------------

class Parser {
 public:
  explicit Parser(const std::string& s) : lx_(s) {}

  NodeP parse_all() {
    NodeP e = expr();
    if (lx_.tok != Tok::End) throw ParseError(lx_.at, "unexpected trailing input");
    return e;
  }

 private:
  Lexer lx_;

  NodeP binary(Op op, NodeP l, NodeP r) {
    NodeP n = make(Node::Bin);
    n->op = op;
    n->kids.push_back(std::move(l));
    n->kids.push_back(std::move(r));
    return n;
  }

  NodeP expr() {
    NodeP l = term();
    while (lx_.tok == Tok::Plus || lx_.tok == Tok::Minus) {
      const Op op = lx_.tok == Tok::Plus ? kAdd : kSub;
      lx_.next();
      l = binary(op, std::move(l), term());
    }
    return l;
  }

  NodeP term() {
    NodeP l = factor();
    while (lx_.tok == Tok::Star || lx_.tok == Tok::Slash) {
      const Op op = lx_.tok == Tok::Star ? kMul : kDiv;
      lx_.next();
      l = binary(op, std::move(l), factor());
    }
    return l;
  }

  NodeP factor() {
    NodeP base = unary();
    if (lx_.tok != Tok::Caret) return base;
    lx_.next();
    return binary(kPow, std::move(base), factor());
  }

  NodeP unary() {
    if (lx_.tok != Tok::Minus) return primary();
    lx_.next();
    NodeP n = make(Node::Neg);
    n->kids.push_back(unary());
    return n;
  }

  void expect(Tok t, const char* what) {
    if (lx_.tok != t) throw ParseError(lx_.at, std::string("expected ") + what);
    lx_.next();
  }

  NodeP primary() {
    if (lx_.tok == Tok::Num) {
      NodeP n = make(Node::Num);
      n->value = lx_.num;
      lx_.next();
      return n;
    }
    if (lx_.tok == Tok::LParen) {
      lx_.next();
      NodeP n = expr();
      expect(Tok::RParen, "')'");
      return n;
    }
    if (lx_.tok != Tok::Ident) throw ParseError(lx_.at, "expected a number, identifier or '('");
    const std::string name = lx_.ident;
    const std::size_t at = lx_.at;
    lx_.next();
    auto fn = functions().find(name);
    if (lx_.tok == Tok::LParen) {
      if (fn == functions().end()) throw ParseError(at, "unknown function '" + name + "'");
      lx_.next();
      NodeP n = make(Node::Call);
      n->op = fn->second.op;
      n->kids.push_back(expr());
      while (lx_.tok == Tok::Comma) {
        lx_.next();
        n->kids.push_back(expr());
      }
      expect(Tok::RParen, "')'");
      if (n->kids.size() != fn->second.arity)
        throw ParseError(at, "function '" + name + "' expects " + std::to_string(fn->second.arity) +
                                 " argument(s), got " + std::to_string(n->kids.size()));
      return n;
    }
    if (fn != functions().end())
      throw ParseError(at, "expected '(' after function name '" + name + "'");
    if (name == "pi" || name == "e") {
      NodeP n = make(Node::Num);
      n->value = name == "pi" ? std::numbers::pi : std::numbers::e;
      return n;
    }
    uint32_t v;
    if (variable_index(name, at, v)) {
      NodeP n = make(Node::Var);
      n->var = v;
      return n;
    }
    NodeP n = make(Node::Param);
    n->name = name;
    return n;
  }
};

NodeP parse(const std::string& source) {
  if (source.empty()) throw ParseError(0, "empty expression");
  Parser p(source);
  return p.parse_all();
}

void collect(const Node& n, Symbols& out) {
  if (n.kind == Node::Var && std::find(out.vars.begin(), out.vars.end(), n.var) == out.vars.end())
    out.vars.push_back(n.var);
  if (n.kind == Node::Param &&
      std::find(out.params.begin(), out.params.end(), n.name) == out.params.end())
    out.params.push_back(n.name);
  for (const auto& k : n.kids) collect(*k, out);
}

// Postfix emission with explicit slots: `sp` is the depth before the node.
struct Emitter {
  Program& p;
  std::map<uint64_t, uint32_t> const_index;  // bit pattern -> pool slot

  uint32_t constant(double v) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    auto it = const_index.find(bits);
    if (it != const_index.end()) return it->second;
    const uint32_t k = uint32_t(p.consts.size());
    p.consts.push_back(v);
    const_index.emplace(bits, k);
    return k;
  }

  void push(Op op, uint32_t dst, uint32_t a, uint32_t b, uint32_t index) {
    p.code.push_back(Instr{op, dst, a, b, index});
    p.depth = std::max(p.depth, dst + 1);
  }

  void emit(const Node& n, uint32_t sp) {
    switch (n.kind) {
      case Node::Num:
        push(kPushConst, sp, 0, 0, constant(n.value));
        return;
      case Node::Var:
        if (n.var >= p.dim)
          throw CompileError("x" + std::to_string(n.var + 1) + " exceeds dim=" + std::to_string(p.dim));
        push(kLoadVar, sp, 0, 0, n.var);
        return;
      case Node::Param: {
        auto it = std::find(p.param_names.begin(), p.param_names.end(), n.name);
        if (it == p.param_names.end()) throw CompileError("unbound parameter '" + n.name + "'");
        push(kLoadParam, sp, 0, 0, uint32_t(it - p.param_names.begin()));
        return;
      }
      case Node::Neg:
        emit(*n.kids[0], sp);
        push(kNeg, sp, sp, 0, 0);
        return;
      case Node::Bin:
      case Node::Call:
        for (std::size_t i = 0; i < n.kids.size(); ++i) emit(*n.kids[i], sp + uint32_t(i));
        push(n.op, sp, sp, sp + 1, 0);
        return;
    }
  }
};

}  // namespace

std::vector<uint32_t> Program::words() const {
  std::vector<uint32_t> w;
  w.reserve(code.size());
  for (const Instr& i : code) w.push_back(encode(i.op, i.dst, i.a, i.b, i.index));
  return w;
}

Symbols symbols(const std::string& source) {
  NodeP root = parse(source);
  Symbols s;
  collect(*root, s);
  return s;
}

Program compile(const std::string& source, uint32_t dim,
                const std::vector<std::string>& sorted_param_names) {
  NodeP root = parse(source);
  Program p;
  p.source = source;
  p.dim = dim;
  p.param_names = sorted_param_names;
  Emitter em{p, {}};
  em.emit(*root, 0);
  if (p.depth > kMaxDepth)
    throw CompileError("expression needs " + std::to_string(p.depth) +
                       " stack slots; the GPU interpreter holds " + std::to_string(kMaxDepth));
  if (p.code.size() > kMaxCode)
    throw CompileError("expression compiles to " + std::to_string(p.code.size()) +
                       " instructions; the GPU interpreter takes at most " +
                       std::to_string(kMaxCode));
  if (p.consts.size() > kMaxConsts) throw CompileError("too many distinct constants");
  if (p.param_names.size() > kMaxParams)
    throw CompileError("more than " + std::to_string(kMaxParams) + " parameters");
  return p;
}

double evaluate(const Program& p, const double* x, const double* params) {
  double st[kMaxDepth] = {};
  for (const Instr& i : p.code) {
    double& d = st[i.dst];
    const double a = st[i.a], b = st[i.b];
    switch (i.op) {
      case kPushConst: d = p.consts[i.index]; break;
      case kLoadVar: d = x[i.index]; break;
      case kLoadParam: d = params[i.index]; break;
      case kNeg: d = -a; break;
      case kAdd: d = a + b; break;
      case kSub: d = a - b; break;
      case kMul: d = a * b; break;
      case kDiv: d = a / b; break;
      case kPow: d = std::pow(a, b); break;
      case kSin: d = std::sin(a); break;
      case kCos: d = std::cos(a); break;
      case kTan: d = std::tan(a); break;
      case kAsin: d = std::asin(a); break;
      case kAcos: d = std::acos(a); break;
      case kAtan: d = std::atan(a); break;
      case kExp: d = std::exp(a); break;
      case kLog: d = std::log(a); break;
      case kSqrt: d = std::sqrt(a); break;
      case kAbs: d = std::fabs(a); break;
      case kFloor: d = std::floor(a); break;
      case kMin: d = std::fmin(a, b); break;
      case kMax: d = std::fmax(a, b); break;
      default: d = NAN;
    }
  }
  return st[0];
}

}  // namespace prog
}  // namespace mcb
