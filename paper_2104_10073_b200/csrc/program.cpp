// program.cpp — DSL parser/compiler for the GPU interpreter (see program.hpp).
#include "program.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numbers>
#include <tuple>

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

// One operation with the host's libm (kSinCos: its sine result).
double host_op(Op op, double a, double b) {
  switch (op) {
    case kCopy: return a;
    case kSinCos: return std::sin(a);
    case kNeg: return -a;
    case kAdd: return a + b;
    case kSub: return a - b;
    case kMul: return a * b;
    case kDiv: return a / b;
    case kPow: return std::pow(a, b);
    case kSin: return std::sin(a);
    case kCos: return std::cos(a);
    case kTan: return std::tan(a);
    case kAsin: return std::asin(a);
    case kAcos: return std::acos(a);
    case kAtan: return std::atan(a);
    case kExp: return std::exp(a);
    case kLog: return std::log(a);
    case kSqrt: return std::sqrt(a);
    case kAbs: return std::fabs(a);
    case kFloor: return std::floor(a);
    case kMin: return std::fmin(a, b);
    case kMax: return std::fmax(a, b);
    case kCosPlusSin: return std::cos(a) + std::sin(a);
    default: return NAN;
  }
}

// ---- DAG + slot allocation ----------------------------------------------------

struct DagNode {
  bool leaf = false;
  Operand leaf_op;  // leaf: the operand
  Op op = kAdd;     // internal: the operation
  int a = -1, b = -1;
};

struct Lowering {
  Program& p;
  std::vector<DagNode> nodes;
  std::map<std::tuple<int, uint32_t, uint32_t, int, int>, int> index;  // hash-consing
  std::map<uint64_t, uint32_t> const_index;

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

  int intern(const DagNode& n) {
    const auto key = n.leaf ? std::make_tuple(-1, n.leaf_op.kind, n.leaf_op.index, -1, -1)
                            : std::make_tuple(int(n.op), 0u, 0u, n.a, n.b);
    auto it = index.find(key);
    if (it != index.end()) return it->second;
    nodes.push_back(n);
    index.emplace(key, int(nodes.size() - 1));
    return int(nodes.size() - 1);
  }

  const double* const_of(int node) const {
    const DagNode& n = nodes[size_t(node)];
    return n.leaf && n.leaf_op.kind == kConst ? &p.consts[n.leaf_op.index] : nullptr;
  }

  bool is_const(int node, double v) const {
    const double* c = const_of(node);
    return c && *c == v;
  }

  int leaf(uint32_t kind, uint32_t idx) {
    DagNode n;
    n.leaf = true;
    n.leaf_op = Operand{kind, idx};
    return intern(n);
  }

  // Tree -> DAG; counts the reference's postfix length on the way.
  int lower(const Node& n) {
    ++p.postfix_len;
    switch (n.kind) {
      case Node::Num:
        return leaf(kConst, constant(n.value));
      case Node::Var:
        if (n.var >= p.dim)
          throw CompileError("x" + std::to_string(n.var + 1) + " exceeds dim=" + std::to_string(p.dim));
        return leaf(kVar, n.var);
      case Node::Param: {
        auto it = std::find(p.param_names.begin(), p.param_names.end(), n.name);
        if (it == p.param_names.end()) throw CompileError("unbound parameter '" + n.name + "'");
        return leaf(kParam, uint32_t(it - p.param_names.begin()));
      }
      case Node::Neg: {
        DagNode d;
        d.op = kNeg;
        d.a = lower(*n.kids[0]);
        if (const double* v = const_of(d.a)) return leaf(kConst, constant(-*v));  // exact
        return intern(d);
      }
      case Node::Bin:
      case Node::Call: {
        DagNode d;
        d.op = n.op;
        d.a = lower(*n.kids[0]);
        if (n.kids.size() > 1) d.b = lower(*n.kids[1]);
        // E^2 / pow(E, 2) -> E*E: the correctly rounded square (glibc's pow
        // differs from it by one ulp in ~0.1 % of arguments, libdevice's pow
        // by up to 2 ulp; identical specials: ±inf, NaN, ±0, overflow).
        // A square is the common case in peak-shaped integrands and costs
        // one DMUL instead of a ~40-operation log/exp chain.
        if (d.op == kPow && is_const(d.b, 2.0)) {
          d.op = kMul;
          d.b = d.a;
        }
        // Other small integer exponents: E^1 = E and E^0 = 1 exactly (NaN
        // included, as C's pow); E^-1 = 1/E, correctly rounded; E^3 = (E*E)*E
        // and E^4 = (E*E)*(E*E), within 1.5 ulp — no worse than libdevice's
        // pow (2 ulp), far inside the 1e-12 per-sample bar, same specials.
        if (d.op == kPow) {
          if (is_const(d.b, 1.0)) return d.a;
          if (is_const(d.b, 0.0)) return leaf(kConst, constant(1.0));
          if (is_const(d.b, -1.0) && !const_of(d.a)) {
            d.op = kDiv;
            d.b = d.a;
            d.a = leaf(kConst, constant(1.0));
          } else if ((is_const(d.b, 3.0) || is_const(d.b, 4.0)) && !const_of(d.a)) {
            DagNode sq;
            sq.op = kMul;
            sq.a = sq.b = d.a;
            const int s2 = intern(sq);
            d.op = kMul;
            d.b = is_const(d.b, 3.0) ? d.a : s2;
            d.a = s2;
          }
        }
        // an operation on constants only is evaluated here, by the host's libm
        // — the library the reference evaluates it with at run time, so the
        // folded value is the reference's bit for bit (+ - * / are single
        // IEEE operations anyway): 2*pi*x1 = (2*pi)*x1, sin(1)*x1, 2^3*x1
        const double *ca = const_of(d.a), *cb = d.b >= 0 ? const_of(d.b) : nullptr;
        if (ca && (d.b < 0 || cb)) return leaf(kConst, constant(host_op(d.op, *ca, cb ? *cb : 0.0)));
        return intern(d);
      }
    }
    return -1;
  }
};

struct Scheduler {
  Program& p;
  const std::vector<DagNode>& nodes;
  std::vector<int> uses;       // remaining reads of each internal node
  std::vector<int> slot;       // assigned slot (-1 = not yet computed)
  std::vector<int> partner;    // sin <-> cos of the same argument
  std::vector<bool> busy;      // slot occupancy
  std::vector<int> need_;      // Sethi-Ullman register need (memoised)

  // Slots a subtree needs when leaves are operands (0) and the child with
  // the larger need is evaluated first; evaluation order does not change
  // any value (every operation is a pure function of its operands).
  int need(int id) {
    const DagNode& n = nodes[size_t(id)];
    if (n.leaf) return 0;
    if (need_.empty()) need_.assign(nodes.size(), -1);
    int& m = need_[size_t(id)];
    if (m >= 0) return m;
    const int a = need(n.a), b = n.b >= 0 ? need(n.b) : 0;
    if (n.a == n.b) return m = std::max(1, a);  // E*E: one evaluation of E
    m = std::max(1, a == b ? a + (n.b >= 0 && b > 0 ? 1 : 0) : std::max(a, b));
    return m;
  }

  uint32_t alloc() {
    for (uint32_t s = 0; s < busy.size(); ++s)
      if (!busy[s]) {
        busy[s] = true;
        p.depth = std::max(p.depth, s + 1);
        return s;
      }
    busy.push_back(true);
    p.depth = std::max(p.depth, uint32_t(busy.size()));
    return uint32_t(busy.size() - 1);
  }

  Operand operand(int id) {
    const DagNode& n = nodes[size_t(id)];
    if (n.leaf) return n.leaf_op;
    return Operand{kSlot, uint32_t(slot[size_t(id)])};
  }

  void release(int id) {
    if (nodes[size_t(id)].leaf) return;
    if (--uses[size_t(id)] == 0) busy[size_t(slot[size_t(id)])] = false;
  }

  void emit(int id) {
    const DagNode& n = nodes[size_t(id)];
    if (n.leaf || slot[size_t(id)] >= 0) return;
    if (n.b >= 0 && need(n.b) > need(n.a)) {
      emit(n.b);
      emit(n.a);
    } else {
      emit(n.a);
      if (n.b >= 0) emit(n.b);
    }
    Instr in;
    in.op = n.op;
    in.a = operand(n.a);
    if (n.b >= 0) in.b = operand(n.b);
    release(n.a);
    if (n.b >= 0) release(n.b);
    const int mate = partner[size_t(id)];
    if (mate >= 0 && slot[size_t(mate)] < 0) {  // sin and cos of one argument: one sincos
      const bool is_sin = n.op == kSin;
      in.op = kSinCos;
      const uint32_t s1 = alloc(), s2 = alloc();
      slot[size_t(id)] = int(is_sin ? s1 : s2);
      slot[size_t(mate)] = int(is_sin ? s2 : s1);
      in.dst = s1;   // sin
      in.dst2 = s2;  // cos
      // the partner's read of the argument happens here too
      release(n.a);
    } else {
      in.dst = alloc();
      slot[size_t(id)] = int(in.dst);
    }
    p.code.push_back(in);
  }
};

// Reads of every internal node reachable from `root` (one per operand
// position of each reachable parent, plus one for the root).
std::vector<int> reads_of(const std::vector<DagNode>& nodes, int root) {
  std::vector<int> reads(nodes.size(), 0);
  std::vector<bool> seen(nodes.size(), false);
  std::vector<int> stack{root};
  while (!stack.empty()) {
    const int id = stack.back();
    stack.pop_back();
    if (seen[size_t(id)]) continue;
    seen[size_t(id)] = true;
    const DagNode& n = nodes[size_t(id)];
    if (n.leaf) continue;
    ++reads[size_t(n.a)];
    stack.push_back(n.a);
    if (n.b >= 0) {
      ++reads[size_t(n.b)];
      stack.push_back(n.b);
    }
  }
  ++reads[size_t(root)];
  return reads;
}

// cos(E) + sin(E) / sin(E) + cos(E), each call read only by that sum, into
// one kCosPlusSin(E) (IEEE addition is commutative, so both orders are the
// reference's cos + sin).
void fuse_cos_plus_sin(std::vector<DagNode>& nodes, int root) {
  const std::vector<int> reads = reads_of(nodes, root);
  for (size_t id = 0; id < nodes.size(); ++id) {
    DagNode& n = nodes[id];
    if (!reads[id] || n.leaf || n.op != kAdd || n.b < 0) continue;
    const DagNode &l = nodes[size_t(n.a)], &r = nodes[size_t(n.b)];
    if (l.leaf || r.leaf || l.a != r.a || reads[size_t(n.a)] != 1 || reads[size_t(n.b)] != 1) continue;
    if (!((l.op == kCos && r.op == kSin) || (l.op == kSin && r.op == kCos))) continue;
    n.op = kCosPlusSin;
    n.a = l.a;
    n.b = -1;
  }
}

}  // namespace

std::vector<uint32_t> Program::words() const {
  std::vector<uint32_t> w(2 * code.size());
  for (size_t i = 0; i < code.size(); ++i) encode(code[i], &w[2 * i]);
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
  NodeP root_tree = parse(source);
  Program p;
  p.source = source;
  p.dim = dim;
  p.param_names = sorted_param_names;
  if (p.param_names.size() > kMaxParams)
    throw CompileError("more than " + std::to_string(kMaxParams) + " parameters");
  Lowering lw{p, {}, {}, {}};
  const int root = lw.lower(*root_tree);
  fuse_cos_plus_sin(lw.nodes, root);
  const auto& nodes = lw.nodes;
  Scheduler sc{p, nodes, std::vector<int>(nodes.size(), 0), std::vector<int>(nodes.size(), -1),
               std::vector<int>(nodes.size(), -1), {}};
  // reads: one per operand position of every reachable internal node, plus the root
  std::vector<bool> seen(nodes.size(), false);
  std::vector<int> stack{root};
  while (!stack.empty()) {
    const int id = stack.back();
    stack.pop_back();
    if (seen[size_t(id)]) continue;
    seen[size_t(id)] = true;
    const DagNode& n = nodes[size_t(id)];
    if (n.leaf) continue;
    ++sc.uses[size_t(n.a)];
    stack.push_back(n.a);
    if (n.b >= 0) {
      ++sc.uses[size_t(n.b)];
      stack.push_back(n.b);
    }
  }
  ++sc.uses[size_t(root)];
  for (size_t i = 0; i < nodes.size(); ++i)
    if (seen[i] && !nodes[i].leaf && (nodes[i].op == kSin || nodes[i].op == kCos))
      for (size_t j = 0; j < nodes.size(); ++j)
        if (j != i && seen[j] && !nodes[j].leaf && nodes[j].a == nodes[i].a &&
            nodes[j].op == (nodes[i].op == kSin ? kCos : kSin))
          sc.partner[i] = int(j);
  sc.emit(root);
  // the result must end in slot 0
  const Operand r = sc.operand(root);
  if (r.kind != kSlot || r.index != 0) {
    Instr cp;
    cp.op = kCopy;
    cp.a = r;
    cp.dst = 0;
    p.depth = std::max(p.depth, 1u);
    p.code.push_back(cp);
  }
  if (p.depth > kMaxDepth)
    throw CompileError("expression needs " + std::to_string(p.depth) +
                       " value slots; the GPU interpreter holds " + std::to_string(kMaxDepth));
  if (p.code.size() > kMaxCode)
    throw CompileError("expression compiles to " + std::to_string(p.code.size()) +
                       " instructions; the GPU interpreter takes at most " + std::to_string(kMaxCode));
  if (p.consts.size() > kMaxConsts) throw CompileError("too many distinct constants");
  return p;
}

double evaluate(const Program& p, const double* x, const double* params) {
  double st[kMaxDepth] = {};
  auto get = [&](const Operand& o) {
    switch (o.kind) {
      case kVar: return x[o.index];
      case kConst: return p.consts[o.index];
      case kParam: return params[o.index];
      default: return st[o.index];
    }
  };
  for (const Instr& i : p.code) {
    const double a = get(i.a), b = get(i.b);
    if (i.op == kSinCos) st[i.dst2] = std::cos(a);
    st[i.dst] = host_op(i.op, a, b);
  }
  return st[0];
}

std::string emit_cuda(const Program& p, const std::string& name) {
  auto opnd = [&](const Operand& o) -> std::string {
    char buf[64];
    switch (o.kind) {
      case kVar: std::snprintf(buf, sizeof buf, "x[%u]", o.index); break;
      case kParam: std::snprintf(buf, sizeof buf, "p[%u]", o.index); break;
      case kConst: {
        uint64_t bits;
        std::memcpy(&bits, &p.consts[o.index], 8);
        std::snprintf(buf, sizeof buf, "__longlong_as_double((long long)0x%016llxull)",
                      (unsigned long long)bits);
        break;
      }
      default: std::snprintf(buf, sizeof buf, "s%u", o.index); break;
    }
    return buf;
  };
  static const char* const unary[] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                      "sin", "cos", "tan", "asin", "acos", "atan", "mcb::dev::mcb_exp", "log",
                                      "__dsqrt_rn", "fabs", "floor"};
  std::string o = "struct " + name + " {\n  static __device__ __forceinline__ double eval(const double* x, "
                  "const double* p) {\n";
  const uint32_t slots = std::max<uint32_t>(p.depth, 1);
  o += "    double";
  for (uint32_t i = 0; i < slots; ++i) o += (i ? ", s" : " s") + std::to_string(i) + " = 0.0";
  o += ";\n    (void)x; (void)p;\n";
  for (const Instr& i : p.code) {
    const std::string d = "s" + std::to_string(i.dst), a = opnd(i.a), b = opnd(i.b);
    switch (i.op) {
      case kCopy: o += "    " + d + " = " + a + ";\n"; break;
      case kSinCos:  // second result first, as the interpreter stores it
        o += "    { double sn_, cs_; sincos(" + a + ", &sn_, &cs_); s" + std::to_string(i.dst2) + " = cs_; " + d +
             " = sn_; }\n";
        break;
      case kNeg: o += "    " + d + " = -(" + a + ");\n"; break;
      case kAdd: o += "    " + d + " = __dadd_rn(" + a + ", " + b + ");\n"; break;
      case kSub: o += "    " + d + " = __dsub_rn(" + a + ", " + b + ");\n"; break;
      case kMul: o += "    " + d + " = __dmul_rn(" + a + ", " + b + ");\n"; break;
      case kDiv: o += "    " + d + " = __ddiv_rn(" + a + ", " + b + ");\n"; break;
      case kPow: o += "    " + d + " = pow(" + a + ", " + b + ");\n"; break;
      case kMin: o += "    " + d + " = fmin(" + a + ", " + b + ");\n"; break;
      case kMax: o += "    " + d + " = fmax(" + a + ", " + b + ");\n"; break;
      case kCosPlusSin: o += "    " + d + " = mcb::dev::cos_plus_sin(" + a + ");\n"; break;
      default:
        if (i.op < kNumOps && i.op < sizeof(unary) / sizeof(unary[0]) && unary[i.op])
          o += "    " + d + " = " + unary[i.op] + "(" + a + ");\n";
        else
          o += "    " + d + " = __longlong_as_double(0x7FF8000000000000ll);\n";
    }
  }
  o += "    return s0;\n  }\n};\n";
  return o;
}

}  // namespace prog
}  // namespace mcb
