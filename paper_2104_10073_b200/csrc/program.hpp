// program.hpp — the integrand DSL on the host: parser, postfix compiler and
// the register-slot ("3-address") form the GPU interpreter executes.
//
// Language and semantics follow the reference (ref/src/expr.cpp):
//   expr   := term (('+'|'-') term)*            left associative
//   term   := factor (('*'|'/') factor)*        left associative
//   factor := unary ('^' factor)?               right associative; -x^2 = (-x)^2
//   unary  := '-' unary | primary
//   primary:= number | '(' expr ')' | name | name '(' expr (',' expr)* ')'
// numbers: digits ['.' digits] [('e'|'E') ['+'|'-'] digits] (strtod);
// names: pi, e (constants), x1..xN (variables, no leading zero), functions
// sin cos tan asin acos atan exp log sqrt abs floor (1 arg), pow min max
// (2 args); any other name is a free parameter.  Compilation emits postfix
// in evaluation order (ref/src/expr.cpp:442-518): children left to right,
// then the operator; parameters bind by position in the sorted name list
// (ref/src/batch.cpp:129-140).
//
// For the GPU the tree is turned into a DAG (structurally identical pure
// subexpressions computed once — exact, since every operation is a pure
// function of its operands), sin/cos of the same argument fuse into one
// sincos, leaves become operand modes (slot | variable | constant |
// parameter) instead of load instructions, and values live in a small set
// of register slots freed at their last use.  `cos(E) + sin(E)` (either
// order, the two calls used nowhere else) becomes one cos_plus_sin(E): the
// Fig. 1 family's table form on the device (mcb_device.cuh), whose error,
// <= 2 ulp of 1, is that of the reference's two rounded libm values and
// rounded add.  The Fig. 1 integrand cos(k*(x1+x2+x3+x4)) +
// sin(k*(x1+x2+x3+x4)) is 21 postfix instructions in the reference and 5 here.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mcb {
namespace prog {

enum Op : uint8_t {
  kCopy = 0,  // dst = a
  kSinCos,    // dst = sin(a), dst2 = cos(a)
  kNeg,
  kAdd,
  kSub,
  kMul,
  kDiv,
  kPow,
  kSin,
  kCos,
  kTan,
  kAsin,
  kAcos,
  kAtan,
  kExp,
  kLog,
  kSqrt,
  kAbs,
  kFloor,
  kMin,
  kMax,
  kCosPlusSin,  // dst = cos(a) + sin(a): the compiler's fusion of `cos(E) + sin(E)`
  kNumOps
};

constexpr uint32_t kMaxDepth = 16;    // value slots the GPU interpreter holds
constexpr uint32_t kMaxCode = 1024;   // instructions per program (2 words each)
constexpr uint32_t kMaxConsts = 512;  // constant-pool entries per program
constexpr uint32_t kMaxParams = 8;    // parameter values carried per integrand

enum OperandKind : uint32_t { kSlot = 0, kVar = 1, kConst = 2, kParam = 3 };
struct Operand {
  uint32_t kind = kSlot, index = 0;
};

struct Instr {
  Op op;
  uint32_t dst = 0, dst2 = 0;  // result slot(s)
  Operand a, b;
};

// Device encoding, two words per instruction:
//   w0 = op (8) | dst (5) | dst2 (5) | a.kind (2) | b.kind (2)
//   w1 = a.index (16) | b.index (16)
inline void encode(const Instr& i, uint32_t w[2]) {
  w[0] = uint32_t(i.op) | (i.dst << 8) | (i.dst2 << 13) | (i.a.kind << 18) | (i.b.kind << 20);
  w[1] = (i.a.index & 0xFFFFu) | (i.b.index << 16);
}

struct ParseError : std::runtime_error {
  std::size_t offset;
  ParseError(std::size_t off, const std::string& msg)
      : std::runtime_error(msg + " (at offset " + std::to_string(off) + ")"), offset(off) {}
};

struct CompileError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Program {
  std::string source;
  uint32_t dim = 0;
  std::vector<std::string> param_names;  // sorted, as bound
  std::vector<Instr> code;
  std::vector<double> consts;
  uint32_t depth = 0;                    // value slots used (result in slot 0)
  uint32_t postfix_len = 0;              // the reference's postfix instruction count
  std::vector<uint32_t> words() const;   // device encoding (2 words / instruction)
};

// Names of the free variables (0-based indices) and parameters (first
// appearance order) of a source; throws ParseError.
struct Symbols {
  std::vector<uint32_t> vars;
  std::vector<std::string> params;
};
Symbols symbols(const std::string& source);

// Parse + compile; throws ParseError (syntax) or CompileError (x_i beyond
// dim, unbound parameter, program too large for the GPU interpreter).
Program compile(const std::string& source, uint32_t dim,
                const std::vector<std::string>& sorted_param_names);

// Scalar evaluation of a compiled program on the host (libm), used for
// shift constants; the tests use the oracle instead.
double evaluate(const Program& p, const double* x, const double* params);

// CUDA source of `struct <name> { static __device__ double eval(const double*
// x, const double* p); }` executing the scheduled instruction list as
// straight-line register code — the interpreter's operations in the
// interpreter's order (runtime specialisation, csrc/jit.cpp).
std::string emit_cuda(const Program& p, const std::string& name);

}  // namespace prog
}  // namespace mcb
