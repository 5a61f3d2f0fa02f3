// compat_mcbatch.cpp — the reference's C++ API (namespace mcbatch,
// include/mcbatch/{sampling,expr,estimator,batch,job_io}.hpp) over libmcb, so
// that code written against the reference compiles unchanged and runs on the
// GPU.  Reference behaviour restated here (file:line under
// /root/reference/proj): the DSL grammar and errors of src/expr.cpp:100-309
// (SPEC.md [MODULE] expr), postfix compilation of :442-518, the estimator
// signatures of include/mcbatch/estimator.hpp:87-125 and the batch layer of
// include/mcbatch/batch.hpp:19-93.  Everything numeric is delegated to the
// mcb:: layer (mcbatch.cpp), i.e. to the sm_100a kernels.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>
#include <numbers>
#include <stdexcept>

#include "mcbatch/batch.hpp"
#include "mcbatch/estimator.hpp"
#include "mcbatch/expr.hpp"
#include "mcbatch/job_io.hpp"
#include "mcbatch/sampling.hpp"

namespace mcbatch {

// ---- expression tree ------------------------------------------------------------

ParseError::ParseError(std::size_t at, const std::string& message)
    : std::runtime_error(message + " (at offset " + std::to_string(at) + ")"), offset(at) {}

Expr Expr::num(double v) {
  Expr e;
  e.kind = ExprKind::Number;
  e.number = v;
  return e;
}
Expr Expr::var(std::size_t index) {
  Expr e;
  e.kind = ExprKind::Variable;
  e.var_index = index;
  return e;
}
Expr Expr::param(std::string n) {
  Expr e;
  e.kind = ExprKind::Parameter;
  e.name = std::move(n);
  return e;
}
Expr Expr::neg(Expr child) {
  Expr e;
  e.kind = ExprKind::Unary;
  e.uop = UnaryOp::Neg;
  e.children = {std::move(child)};
  return e;
}
Expr Expr::binary(BinaryOp op, Expr lhs, Expr rhs) {
  Expr e;
  e.kind = ExprKind::Binary;
  e.bop = op;
  e.children.reserve(2);
  e.children.push_back(std::move(lhs));
  e.children.push_back(std::move(rhs));
  return e;
}
Expr Expr::call(std::string fn, std::vector<Expr> args) {
  Expr e;
  e.kind = ExprKind::Call;
  e.name = std::move(fn);
  e.children = std::move(args);
  return e;
}

bool Expr::operator==(const Expr& o) const {
  if (kind != o.kind || children.size() != o.children.size()) return false;
  bool head = true;
  switch (kind) {
    case ExprKind::Number: head = number == o.number; break;
    case ExprKind::Variable: head = var_index == o.var_index; break;
    case ExprKind::Parameter:
    case ExprKind::Call: head = name == o.name; break;
    case ExprKind::Unary: head = uop == o.uop; break;
    case ExprKind::Binary: head = bop == o.bop; break;
  }
  return head && std::equal(children.begin(), children.end(), o.children.begin());
}

namespace {

struct Builtin {
  std::string_view name;
  OpCode op;
  unsigned arity;
};
constexpr Builtin kBuiltins[] = {
    {"sin", OpCode::Sin, 1},   {"cos", OpCode::Cos, 1},     {"tan", OpCode::Tan, 1},
    {"asin", OpCode::Asin, 1}, {"acos", OpCode::Acos, 1},   {"atan", OpCode::Atan, 1},
    {"exp", OpCode::Exp, 1},   {"log", OpCode::Log, 1},     {"sqrt", OpCode::Sqrt, 1},
    {"abs", OpCode::Abs, 1},   {"floor", OpCode::Floor, 1}, {"pow", OpCode::Pow, 2},
    {"min", OpCode::Min, 2},   {"max", OpCode::Max, 2},
};
const Builtin* builtin(std::string_view name) {
  for (const Builtin& b : kBuiltins)
    if (b.name == name) return &b;
  return nullptr;
}

bool is_digit(char c) { return c >= '0' && c <= '9'; }
bool is_ident_start(char c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_'; }
bool is_ident_char(char c) { return is_ident_start(c) || is_digit(c); }

// Precedence climbing over the reference grammar: + - (1, left), * / (2,
// left), ^ (3, right; its operands are unary expressions, so -x^2 is (-x)^2
// and 2^-3 is 2^(-3)); unary minus; numbers, (expr), names and calls.
class Reader {
 public:
  explicit Reader(std::string_view s) : s_(s) {}

  Expr whole() {
    skip();
    if (pos_ == s_.size()) throw SyntaxError(0, "empty expression");
    Expr e = climb(1);
    skip();
    if (pos_ != s_.size()) {
      if (!strchr("+-*/^(),", s_[pos_]) && !is_digit(s_[pos_]) && !is_ident_start(s_[pos_]))
        throw SyntaxError(pos_, std::string("unexpected character '") + s_[pos_] + "'");
      throw SyntaxError(pos_, "unexpected trailing input");
    }
    return e;
  }

 private:
  std::string_view s_;
  std::size_t pos_ = 0;

  void skip() {
    while (pos_ < s_.size() && (s_[pos_] == ' ' || s_[pos_] == '\t' || s_[pos_] == '\n' || s_[pos_] == '\r' ||
                                s_[pos_] == '\f' || s_[pos_] == '\v'))
      ++pos_;
  }
  bool peek(char c) {
    skip();
    return pos_ < s_.size() && s_[pos_] == c;
  }

  Expr climb(int min_bp) {
    Expr lhs = unary();
    for (;;) {
      skip();
      if (pos_ == s_.size()) return lhs;
      int bp;
      BinaryOp op;
      switch (s_[pos_]) {
        case '+': bp = 1, op = BinaryOp::Add; break;
        case '-': bp = 1, op = BinaryOp::Sub; break;
        case '*': bp = 2, op = BinaryOp::Mul; break;
        case '/': bp = 2, op = BinaryOp::Div; break;
        case '^': bp = 3, op = BinaryOp::Pow; break;
        default: return lhs;
      }
      if (bp < min_bp) return lhs;
      ++pos_;
      Expr rhs = climb(op == BinaryOp::Pow ? bp : bp + 1);
      lhs = Expr::binary(op, std::move(lhs), std::move(rhs));
    }
  }

  Expr unary() {
    if (peek('-')) {
      ++pos_;
      return Expr::neg(unary());
    }
    return primary();
  }

  Expr primary() {
    skip();
    const std::size_t at = pos_;
    if (at == s_.size()) throw SyntaxError(at, "expected a number, identifier or '('");
    const char c = s_[at];
    if (c == '(') {
      ++pos_;
      Expr inner = climb(1);
      expect(')');
      return inner;
    }
    if (is_digit(c)) return number();
    if (is_ident_start(c)) return named();
    if (strchr("+*/^),", c)) throw SyntaxError(at, "expected a number, identifier or '('");
    throw SyntaxError(at, std::string("unexpected character '") + c + "'");
  }

  // digits [. digits] [(e|E) [+|-] digits]; an 'e' without digits after it
  // is not part of the number.
  Expr number() {
    const std::size_t start = pos_;
    auto digits = [&] {
      while (pos_ < s_.size() && is_digit(s_[pos_])) ++pos_;
    };
    digits();
    if (pos_ < s_.size() && s_[pos_] == '.') {
      ++pos_;
      digits();
    }
    if (pos_ < s_.size() && (s_[pos_] == 'e' || s_[pos_] == 'E')) {
      std::size_t q = pos_ + 1;
      if (q < s_.size() && (s_[q] == '+' || s_[q] == '-')) ++q;
      if (q < s_.size() && is_digit(s_[q])) {
        pos_ = q;
        digits();
      }
    }
    const std::string text(s_.substr(start, pos_ - start));
    return Expr::num(std::strtod(text.c_str(), nullptr));
  }

  Expr named() {
    const std::size_t at = pos_;
    while (pos_ < s_.size() && is_ident_char(s_[pos_])) ++pos_;
    std::string id(s_.substr(at, pos_ - at));
    const Builtin* fn = builtin(id);
    if (peek('(')) {
      if (!fn) throw UnknownFunction(at, "unknown function '" + id + "'");
      ++pos_;
      std::vector<Expr> args;
      args.push_back(climb(1));
      while (peek(',')) {
        ++pos_;
        args.push_back(climb(1));
      }
      expect(')');
      if (args.size() != fn->arity)
        throw ArityMismatch(at, "function '" + id + "' expects " + std::to_string(fn->arity) +
                                    " argument(s), got " + std::to_string(args.size()));
      return Expr::call(std::move(id), std::move(args));
    }
    if (fn) throw SyntaxError(at, "expected '(' after function name '" + id + "'");
    if (id == "pi") return Expr::num(std::numbers::pi);
    if (id == "e") return Expr::num(std::numbers::e);
    // x<k>, k a decimal without a leading zero: coordinate k-1
    if (id.size() >= 2 && id[0] == 'x' && id[1] != '0' &&
        std::all_of(id.begin() + 1, id.end(), [](char ch) { return is_digit(ch); })) {
      std::size_t k = 0;
      for (std::size_t i = 1; i < id.size(); ++i) {
        k = 10 * k + std::size_t(id[i] - '0');
        if (k > 1000000) throw std::out_of_range("variable index too large");
      }
      return Expr::var(k - 1);
    }
    return Expr::param(std::move(id));
  }

  void expect(char c) {
    if (!peek(c)) throw SyntaxError(pos_, std::string("expected '") + c + "'");
    ++pos_;
  }
};

char op_char(BinaryOp op) {
  switch (op) {
    case BinaryOp::Add: return '+';
    case BinaryOp::Sub: return '-';
    case BinaryOp::Mul: return '*';
    case BinaryOp::Div: return '/';
    case BinaryOp::Pow: return '^';
  }
  return '?';
}

void print(const Expr& e, std::string& out) {
  switch (e.kind) {
    case ExprKind::Number: {
      char buf[32];  // shortest text that parses back to the same double
      const auto r = std::to_chars(buf, buf + sizeof buf, std::fabs(e.number));
      if (std::signbit(e.number)) out += "(-";
      out.append(buf, r.ptr);
      if (std::signbit(e.number)) out += ')';
      return;
    }
    case ExprKind::Variable:
      out += 'x';
      out += std::to_string(e.var_index + 1);
      return;
    case ExprKind::Parameter:
      out += e.name;
      return;
    case ExprKind::Unary:
      out += "(-";
      print(e.children[0], out);
      out += ')';
      return;
    case ExprKind::Binary:
      out += '(';
      print(e.children[0], out);
      out += ' ';
      out += op_char(e.bop);
      out += ' ';
      print(e.children[1], out);
      out += ')';
      return;
    case ExprKind::Call:
      out += e.name;
      out += '(';
      for (std::size_t i = 0; i < e.children.size(); ++i) {
        if (i) out += ", ";
        print(e.children[i], out);
      }
      out += ')';
      return;
  }
}

template <class F>
void visit(const Expr& e, const F& f) {
  f(e);
  for (const Expr& c : e.children) visit(c, f);
}

std::string var_message(std::size_t index, std::size_t dim) {
  return "x" + std::to_string(index + 1) + " exceeds dim=" + std::to_string(dim);
}

}  // namespace

Expr parse(std::string_view source) { return Reader(source).whole(); }

std::string to_string(const Expr& e) {
  std::string out;
  print(e, out);
  return out;
}

std::set<std::size_t> free_variables(const Expr& e) {
  std::set<std::size_t> vars;
  visit(e, [&](const Expr& n) {
    if (n.kind == ExprKind::Variable) vars.insert(n.var_index);
  });
  return vars;
}

std::vector<std::string> free_parameters(const Expr& e) {
  std::vector<std::string> names;
  visit(e, [&](const Expr& n) {
    if (n.kind == ExprKind::Parameter && std::find(names.begin(), names.end(), n.name) == names.end())
      names.push_back(n.name);
  });
  return names;
}

double tree_eval(const Expr& e, std::span<const double> point, std::span<const std::string> param_names,
                 std::span<const double> params) {
  const std::function<double(const Expr&)> ev = [&](const Expr& n) -> double {
    switch (n.kind) {
      case ExprKind::Number: return n.number;
      case ExprKind::Variable:
        if (n.var_index >= point.size()) throw DimensionError(var_message(n.var_index, point.size()));
        return point[n.var_index];
      case ExprKind::Parameter: {
        const auto it = std::find(param_names.begin(), param_names.end(), n.name);
        if (it == param_names.end() || std::size_t(it - param_names.begin()) >= params.size())
          throw UnboundParameter("unbound parameter '" + n.name + "'");
        return params[std::size_t(it - param_names.begin())];
      }
      case ExprKind::Unary: return -ev(n.children[0]);
      case ExprKind::Binary: {
        const double a = ev(n.children[0]), b = ev(n.children[1]);
        switch (n.bop) {
          case BinaryOp::Add: return a + b;
          case BinaryOp::Sub: return a - b;
          case BinaryOp::Mul: return a * b;
          case BinaryOp::Div: return a / b;
          case BinaryOp::Pow: return std::pow(a, b);
        }
        return NAN;
      }
      case ExprKind::Call: {
        const Builtin* fn = builtin(n.name);
        if (!fn || fn->arity != n.children.size()) throw CompileError("bad call '" + n.name + "'");
        const double a = ev(n.children[0]);
        switch (fn->op) {
          case OpCode::Sin: return std::sin(a);
          case OpCode::Cos: return std::cos(a);
          case OpCode::Tan: return std::tan(a);
          case OpCode::Asin: return std::asin(a);
          case OpCode::Acos: return std::acos(a);
          case OpCode::Atan: return std::atan(a);
          case OpCode::Exp: return std::exp(a);
          case OpCode::Log: return std::log(a);
          case OpCode::Sqrt: return std::sqrt(a);
          case OpCode::Abs: return std::fabs(a);
          case OpCode::Floor: return std::floor(a);
          case OpCode::Pow: return std::pow(a, ev(n.children[1]));
          case OpCode::Min: return std::fmin(a, ev(n.children[1]));
          case OpCode::Max: return std::fmax(a, ev(n.children[1]));
          default: return NAN;
        }
      }
    }
    return NAN;
  };
  return ev(e);
}

// ---- compiled programs -----------------------------------------------------------

// The libmcb program behind a CompiledProgram: compiled once, on first use,
// from the program's DSL text; libmcb binds parameters in sorted-name order,
// `order[i]` is the caller's slot of the i-th bound name.
struct CompiledProgram::Device {
  std::once_flag once;
  mcb::CompiledSource handle;
  std::vector<std::size_t> order;
  std::string error;
};

CompiledProgram compile(const Expr& expr, std::size_t dim, std::span<const std::string> param_names) {
  CompiledProgram p;
  p.dim_ = dim;
  p.param_names_.assign(param_names.begin(), param_names.end());
  std::size_t depth = 0;
  const std::function<void(const Expr&)> emit = [&](const Expr& n) {
    for (const Expr& c : n.children) emit(c);  // operands left to right, then the operator
    Instr in{OpCode::PushConst};
    switch (n.kind) {
      case ExprKind::Number: in = {OpCode::PushConst, 0, n.number}; break;
      case ExprKind::Variable:
        if (n.var_index >= dim) throw DimensionError(var_message(n.var_index, dim));
        in = {OpCode::LoadVar, uint32_t(n.var_index), 0.0};
        break;
      case ExprKind::Parameter: {
        const auto it = std::find(param_names.begin(), param_names.end(), n.name);
        if (it == param_names.end()) throw UnboundParameter("unbound parameter '" + n.name + "'");
        in = {OpCode::LoadParam, uint32_t(it - param_names.begin()), 0.0};
        break;
      }
      case ExprKind::Unary: in.op = OpCode::Neg; break;
      case ExprKind::Binary: {
        constexpr OpCode ops[] = {OpCode::Add, OpCode::Sub, OpCode::Mul, OpCode::Div, OpCode::Pow};
        in.op = ops[int(n.bop)];
        break;
      }
      case ExprKind::Call: {
        const Builtin* fn = builtin(n.name);
        if (!fn || fn->arity != n.children.size()) throw CompileError("bad call '" + n.name + "'");
        in.op = fn->op;
        break;
      }
    }
    p.code_.push_back(in);
    // stack effect: leaves push one, an n-ary node pops n and pushes one
    depth = depth + 1 - n.children.size();
    p.stack_need_ = std::max(p.stack_need_, depth);
  };
  emit(expr);
  p.source_ = to_string(expr);
  p.device_ = std::make_shared<CompiledProgram::Device>();
  return p;
}

double CompiledProgram::evaluate(std::span<const double> point, std::span<const double> params,
                                 std::vector<double>&) const {
  Device& d = *device_;
  std::call_once(d.once, [&] {
    try {
      std::map<std::string, double> named;
      for (const std::string& n : param_names_) named[n] = 0.0;
      d.handle = mcb::compile_program(source_, dim_, named);
      for (const auto& [n, v] : named)
        d.order.push_back(std::size_t(std::find(param_names_.begin(), param_names_.end(), n) -
                                      param_names_.begin()));
    } catch (const std::exception& e) {
      d.error = e.what();
    }
  });
  if (!d.handle.handle) throw CompileError("program does not run on the GPU interpreter: " + d.error);
  if (point.size() < dim_) throw DimensionError("point has " + std::to_string(point.size()) + " coordinates, need " +
                                                std::to_string(dim_));
  std::vector<double> bound(d.order.size());
  for (std::size_t i = 0; i < bound.size(); ++i) {
    if (d.order[i] >= params.size()) throw UnboundParameter("unbound parameter '" + param_names_[d.order[i]] + "'");
    bound[i] = params[d.order[i]];
  }
  double out = 0.0;
  const mcb_status st =
      mcb_program_eval_points(d.handle.handle, bound.data(), bound.size(), point.data(), 1, 0, &out);
  if (st != MCB_OK) throw mcb::DeviceError(mcb_last_error());
  return out;
}

// ---- estimators -------------------------------------------------------------------

namespace {

// The program as a libmcb integrand spec: named parameters, the given domain.
mcb::IntegrandSpec program_spec(const CompiledProgram& program, std::span<const double> params,
                                const HyperRect& rect, std::uint64_t n_samples) {
  if (params.size() < program.param_names().size())
    throw std::invalid_argument("program binds " + std::to_string(program.param_names().size()) +
                                " parameter(s), got " + std::to_string(params.size()));
  std::map<std::string, double> named;
  for (std::size_t i = 0; i < program.param_names().size(); ++i) named[program.param_names()[i]] = params[i];
  return mcb::IntegrandSpec::from_source("program", program.source(), program.dim(), rect, std::move(named),
                                         n_samples);
}

StratumNode node_of(const mcb::StratumNode& n) { return StratumNode{n.cell, n.estimate, n.depth, {}}; }

}  // namespace

void ChunkAccum::add(double x) {
  mcb::ChunkAccum a{n, n_nonfinite, mean, m2};
  a.add(x);
  *this = ChunkAccum{a.n, a.n_nonfinite, a.mean, a.m2};
}

void ChunkAccum::merge(const ChunkAccum& other) {
  mcb::ChunkAccum a{n, n_nonfinite, mean, m2};
  a.merge(mcb::ChunkAccum{other.n, other.n_nonfinite, other.mean, other.m2});
  *this = ChunkAccum{a.n, a.n_nonfinite, a.mean, a.m2};
}

ChunkAccum accumulate_chunk(const CompiledProgram& program, std::span<const double> params,
                            const HyperRect& rect, const StreamKey& key, std::size_t count) {
  if (!rect.valid()) throw InvalidDomain("invalid hyperrectangle");
  const mcb::ChunkAccum a = mcb::accumulate_chunk(program_spec(program, params, rect, count < 2 ? 2 : count),
                                                  key, count, 0);
  return ChunkAccum{a.n, a.n_nonfinite, a.mean, a.m2};
}

McEstimate reduce_chunks(double volume, std::span<const ChunkAccum> chunks) {
  std::vector<mcb::ChunkAccum> c;
  c.reserve(chunks.size());
  for (const ChunkAccum& x : chunks) c.push_back(mcb::ChunkAccum{x.n, x.n_nonfinite, x.mean, x.m2});
  return mcb::reduce_chunks(volume, c);
}

UniformStream::UniformStream(const StreamKey& key) : key_(key) {
  if (key.chunk_index > 0xFFFFFFFFull) throw std::out_of_range("chunk_index exceeds 32 bits");
}

void UniformStream::refill() {
  // draws = the coordinates of 1-D points on [0, 1): low + 1 * u = u exactly
  const double lo = 0.0, hi = 1.0;
  const mcb_status st = mcb_debug_points(key_.global_seed, key_.integrand_index, key_.trial_index, key_.chunk_index,
                                         drawn_, kBatch, 1, &lo, &hi, 0, buf_.data());
  if (st != MCB_OK) throw mcb::DeviceError(mcb_last_error());
  drawn_ += kBatch;
  pos_ = 0;
}

McEstimate direct_mc(const CompiledProgram& program, std::span<const double> params, const HyperRect& rect,
                     std::uint64_t n_samples, const StreamKey& key_base) {
  return mcb::direct_mc(program_spec(program, params, rect, n_samples), n_samples, key_base, 0);
}

std::pair<McEstimate, std::vector<StratumNode>> stratified_mc(const CompiledProgram& program,
                                                              std::span<const double> params,
                                                              const HyperRect& rect, std::uint32_t cells_per_dim,
                                                              std::uint32_t samples_per_cell,
                                                              const StreamKey& key_base, std::uint64_t cell_cap) {
  auto [est, cells] = mcb::stratified_mc(program_spec(program, params, rect, samples_per_cell), cells_per_dim,
                                         samples_per_cell, key_base, cell_cap, 0);
  std::vector<StratumNode> out;
  out.reserve(cells.size());
  for (const mcb::StratumNode& c : cells) out.push_back(node_of(c));
  return {est, std::move(out)};
}

McEstimate tree_refine(const CompiledProgram& program, std::span<const double> params, const HyperRect& rect,
                       const RefineConfig& config, const StreamKey& key_base, std::vector<StratumNode>* leaves_out) {
  std::vector<mcb::StratumNode> leaves;
  const McEstimate est = mcb::tree_refine(program_spec(program, params, rect, config.total_budget), config,
                                          key_base, leaves_out ? &leaves : nullptr, 0);
  if (leaves_out) {
    leaves_out->clear();
    for (const mcb::StratumNode& l : leaves) leaves_out->push_back(node_of(l));
  }
  return est;
}

// ---- batch ----------------------------------------------------------------------------

std::optional<Method> method_from_name(std::string_view name) {
  for (Method m : {Method::Direct, Method::Stratified, Method::Tree})
    if (name == method_name(m)) return m;
  return std::nullopt;
}

mcb::IntegrandSpec to_mcb(const IntegrandSpec& s) {
  mcb::IntegrandSpec out = mcb::IntegrandSpec::from_source(s.name, s.source, s.dim, s.domain, s.params, s.n_samples);
  out.method = s.method;
  out.method_config = s.method_config;
  return out;
}

mcb::JobSpec to_mcb(const JobSpec& job) {
  mcb::JobSpec out;
  out.seed = job.seed;
  out.trials = job.trials;
  out.workers = job.workers;
  out.integrands.reserve(job.integrands.size());
  for (const IntegrandSpec& s : job.integrands) out.integrands.push_back(to_mcb(s));
  return out;
}

IntegrandSpec from_mcb(const mcb::IntegrandSpec& s) {
  return IntegrandSpec{s.name, s.source(), s.dim, s.domain, s.params, s.n_samples, s.method, s.method_config};
}

JobSpec from_mcb(const mcb::JobSpec& job) {
  JobSpec out{job.seed, job.trials, job.workers, {}};
  out.integrands.reserve(job.integrands.size());
  for (const mcb::IntegrandSpec& s : job.integrands) out.integrands.push_back(from_mcb(s));
  return out;
}

std::vector<Violation> validate(const JobSpec& job) { return mcb::validate(to_mcb(job)); }

BatchResult run_batch(const JobSpec& job) { return mcb::run_batch(to_mcb(job)); }

std::vector<TrialSummary> parameter_scan(const IntegrandSpec& tmpl, const std::string& param_name,
                                         std::span<const double> values, std::uint32_t trials,
                                         std::uint64_t seed, std::uint32_t workers) {
  return mcb::parameter_scan(to_mcb(tmpl), param_name, values, trials, seed, mcb::devices_for_workers(workers));
}

StratifiedPlan stratified_plan(const IntegrandSpec& spec) { return mcb::stratified_plan(to_mcb(spec)); }

std::uint32_t resolve_workers(std::uint32_t requested) {
  return requested ? requested : std::uint32_t(std::max(1, mcb_device_count()));
}

// ---- job files ---------------------------------------------------------------------

JobSpec read_job(const std::filesystem::path& path) { return from_mcb(mcb::read_job(path)); }
JobSpec job_from_json_text(const std::string& text) { return from_mcb(mcb::job_from_json_text(text)); }
void write_job(const JobSpec& job, const std::filesystem::path& path) { mcb::write_job(to_mcb(job), path); }
std::string job_to_json_text(const JobSpec& job) { return mcb::job_to_json_text(to_mcb(job)); }
std::vector<ResultsRow> make_results(const JobSpec& job, const BatchResult& br) {
  return mcb::make_results(to_mcb(job), br);
}
JobSpec make_harmonic_job(std::uint32_t n_count, std::uint64_t samples) {
  return from_mcb(mcb::make_harmonic_job(n_count, samples));
}

}  // namespace mcbatch
