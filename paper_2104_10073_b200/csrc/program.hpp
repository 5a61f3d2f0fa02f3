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
// (ref/src/batch.cpp:129-140).  Each postfix instruction gets explicit
// stack-slot operands so the device never tracks a stack pointer.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mcb {
namespace prog {

enum Op : uint8_t {
  kPushConst = 0,
  kLoadVar,
  kLoadParam,
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
  kNumOps
};

constexpr uint32_t kMaxDepth = 16;    // stack slots the GPU interpreter holds
constexpr uint32_t kMaxCode = 1024;   // instructions per program
constexpr uint32_t kMaxConsts = 512;  // constant-pool entries per program
constexpr uint32_t kMaxParams = 8;    // parameter values carried per integrand

// Device word: op (8) | dst slot (4) | a slot (4) | b slot (4) | index (12).
inline uint32_t encode(Op op, uint32_t dst, uint32_t a, uint32_t b, uint32_t index) {
  return uint32_t(op) | (dst << 8) | (a << 12) | (b << 16) | (index << 20);
}

struct Instr {
  Op op;
  uint32_t dst, a, b;  // stack slots
  uint32_t index;      // var / param / constant index
};

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
  uint32_t depth = 0;                    // max stack depth
  std::vector<uint32_t> words() const;   // device encoding
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

// Reference-order scalar evaluation of a compiled program on the host (libm),
// used for shift constants; the tests use the oracle instead.
double evaluate(const Program& p, const double* x, const double* params);

}  // namespace prog
}  // namespace mcb
