// job_io.cpp — job files, results CSV and the Fig. 1 harness on the GPU
// backend (include/mcb/job_io.hpp).  Formats follow SPEC.md [MODULE] cli
// (strict JSON job files; the 17-digit results CSV; exit codes 0 / 2 / 3)
// so that the reference's own readers accept our files; the JSON reader is a
// small RFC 8259 parser, the CSV layer a column table (kColumns).
#include "mcb/job_io.hpp"

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <optional>
#include <string_view>
#include <memory>
#include <numbers>
#include <sstream>
#include <variant>

namespace mcb {

namespace {

// ---- minimal strict JSON ------------------------------------------------------

struct Json;
using JsonObject = std::map<std::string, Json>;
using JsonArray = std::vector<Json>;

struct Json {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0.0;
  bool is_integer = false;
  uint64_t u = 0;  // exact value of a non-negative integer literal
  bool negative = false;
  std::string str;
  std::shared_ptr<JsonArray> arr;
  std::shared_ptr<JsonObject> obj;
};

class JsonParser {
 public:
  explicit JsonParser(const std::string& s) : s_(s) {}

  Json parse_document() {
    Json v = value();
    ws();
    if (p_ != s_.size()) error("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  std::size_t p_ = 0;

  [[noreturn]] void error(const std::string& what) {
    throw JobFileError("invalid JSON: " + what + " at byte " + std::to_string(p_));
  }
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\t' || s_[p_] == '\n' || s_[p_] == '\r'))
      ++p_;
  }
  bool lit(const char* w) {
    const std::size_t n = std::char_traits<char>::length(w);
    if (s_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }

  Json value() {
    ws();
    if (p_ >= s_.size()) error("unexpected end of input");
    Json v;
    const char c = s_[p_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') {
      v.kind = Json::String;
      v.str = string();
      return v;
    }
    if (lit("true")) {
      v.kind = Json::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = Json::Bool;
      return v;
    }
    if (lit("null")) return v;
    return number();
  }

  Json number() {
    const std::size_t start = p_;
    Json v;
    v.kind = Json::Number;
    if (s_[p_] == '-') {
      v.negative = true;
      ++p_;
    }
    auto digits = [&] {
      const std::size_t d0 = p_;
      while (p_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[p_]))) ++p_;
      return p_ - d0;
    };
    const std::size_t int_start = p_;
    const std::size_t nd = digits();
    if (nd == 0) error("invalid number");
    if (nd > 1 && s_[int_start] == '0') error("leading zero in number");
    bool integral = true;
    if (p_ < s_.size() && s_[p_] == '.') {
      ++p_;
      if (digits() == 0) error("invalid fraction");
      integral = false;
    }
    if (p_ < s_.size() && (s_[p_] == 'e' || s_[p_] == 'E')) {
      ++p_;
      if (p_ < s_.size() && (s_[p_] == '+' || s_[p_] == '-')) ++p_;
      if (digits() == 0) error("invalid exponent");
      integral = false;
    }
    const std::string text = s_.substr(start, p_ - start);
    v.num = std::strtod(text.c_str(), nullptr);
    if (integral && !v.negative) {
      const auto r = std::from_chars(s_.data() + int_start, s_.data() + p_, v.u);
      v.is_integer = r.ec == std::errc();
    }
    return v;
  }

  std::string string() {
    ++p_;  // opening quote
    std::string out;
    while (true) {
      if (p_ >= s_.size()) error("unterminated string");
      const char c = s_[p_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) error("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p_ >= s_.size()) error("bad escape");
      const char e = s_[p_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          auto hex4 = [&] {
            if (p_ + 4 > s_.size()) error("bad \\u escape");
            unsigned v = 0;
            for (int i = 0; i < 4; ++i) {
              const char h = s_[p_++];
              v <<= 4;
              if (h >= '0' && h <= '9') v |= unsigned(h - '0');
              else if (h >= 'a' && h <= 'f') v |= unsigned(h - 'a' + 10);
              else if (h >= 'A' && h <= 'F') v |= unsigned(h - 'A' + 10);
              else error("bad \\u escape");
            }
            return v;
          };
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {
            if (!lit("\\u")) error("unpaired surrogate");
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo >= 0xE000) error("unpaired surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          if (cp < 0x80) {
            out += char(cp);
          } else if (cp < 0x800) {
            out += char(0xC0 | (cp >> 6));
            out += char(0x80 | (cp & 0x3F));
          } else if (cp < 0x10000) {
            out += char(0xE0 | (cp >> 12));
            out += char(0x80 | ((cp >> 6) & 0x3F));
            out += char(0x80 | (cp & 0x3F));
          } else {
            out += char(0xF0 | (cp >> 18));
            out += char(0x80 | ((cp >> 12) & 0x3F));
            out += char(0x80 | ((cp >> 6) & 0x3F));
            out += char(0x80 | (cp & 0x3F));
          }
        } break;
        default: error("bad escape");
      }
    }
  }

  Json array() {
    ++p_;
    Json v;
    v.kind = Json::Array;
    v.arr = std::make_shared<JsonArray>();
    ws();
    if (p_ < s_.size() && s_[p_] == ']') {
      ++p_;
      return v;
    }
    while (true) {
      v.arr->push_back(value());
      ws();
      if (p_ < s_.size() && s_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < s_.size() && s_[p_] == ']') {
        ++p_;
        return v;
      }
      error("expected ',' or ']'");
    }
  }

  Json object() {
    ++p_;
    Json v;
    v.kind = Json::Object;
    v.obj = std::make_shared<JsonObject>();
    ws();
    if (p_ < s_.size() && s_[p_] == '}') {
      ++p_;
      return v;
    }
    while (true) {
      ws();
      if (p_ >= s_.size() || s_[p_] != '"') error("expected a key");
      const std::string key = string();
      ws();
      if (p_ >= s_.size() || s_[p_] != ':') error("expected ':'");
      ++p_;
      (*v.obj)[key] = value();
      ws();
      if (p_ < s_.size() && s_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < s_.size() && s_[p_] == '}') {
        ++p_;
        return v;
      }
      error("expected ',' or '}'");
    }
  }
};

// typed accessors: "malformed job file: ..." like the reference's json::exception path
[[noreturn]] void malformed(const std::string& what) {
  throw JobFileError("malformed job file: " + what);
}
const Json& at(const Json& o, const char* key) {
  auto it = o.obj->find(key);
  if (it == o.obj->end()) malformed(std::string("missing field '") + key + "'");
  return it->second;
}
bool has(const Json& o, const char* key) { return o.obj->count(key) != 0; }
uint64_t as_u64(const Json& v, const char* what) {
  if (v.kind != Json::Number) malformed(std::string("'") + what + "' must be a number");
  if (v.is_integer) return v.u;
  if (v.negative || !(v.num >= 0.0) || v.num != std::floor(v.num) || v.num > 1.8446744073709552e19)
    malformed(std::string("'") + what + "' must be a non-negative integer");
  return uint64_t(v.num);
}
uint32_t as_u32(const Json& v, const char* what) {
  const uint64_t x = as_u64(v, what);
  if (x > 0xFFFFFFFFull) malformed(std::string("'") + what + "' out of range");
  return uint32_t(x);
}
double as_double(const Json& v, const char* what) {
  if (v.kind != Json::Number) malformed(std::string("'") + what + "' must be a number");
  return v.num;
}
std::string as_string(const Json& v, const char* what) {
  if (v.kind != Json::String) malformed(std::string("'") + what + "' must be a string");
  return v.str;
}
std::vector<double> as_doubles(const Json& v, const char* what) {
  if (v.kind != Json::Array) malformed(std::string("'") + what + "' must be an array");
  std::vector<double> out;
  for (const Json& e : *v.arr) out.push_back(as_double(e, what));
  return out;
}

void reject_unknown(const Json& obj, std::initializer_list<const char*> known, const std::string& where) {
  for (const auto& [k, v] : *obj.obj) {
    bool found = false;
    for (const char* n : known)
      if (k == n) found = true;
    if (!found) throw JobFileError("unknown field '" + k + "' in " + where);  // ref job_io.cpp:23-35
  }
}

RefineConfig refine_config_from_json(const Json& j, const std::string& where) {  // :37-52
  if (j.kind != Json::Object) malformed(where + " must be an object");
  reject_unknown(j, {"cells_per_dim", "samples_per_cell", "max_depth", "sigma_multiplier", "cell_cap"},
                 where);
  RefineConfig rc;
  if (has(j, "cells_per_dim")) rc.init_cells_per_dim = as_u32(at(j, "cells_per_dim"), "cells_per_dim");
  if (has(j, "samples_per_cell")) rc.samples_per_cell = as_u32(at(j, "samples_per_cell"), "samples_per_cell");
  if (has(j, "max_depth")) rc.max_depth = as_u32(at(j, "max_depth"), "max_depth");
  if (has(j, "sigma_multiplier"))
    rc.sigma_multiplier = as_double(at(j, "sigma_multiplier"), "sigma_multiplier");
  if (has(j, "cell_cap")) rc.cell_cap = as_u64(at(j, "cell_cap"), "cell_cap");
  return rc;
}

// ---- JSON writer (keys sorted, 2-space indent, like nlohmann::json::dump(2)) ---

std::string json_number(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);  // shortest round-trip
  std::string s(buf, r.ptr);
  if (s.find_first_of(".e") == std::string::npos) s += ".0";
  return s;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", unsigned(static_cast<unsigned char>(c)));
          o += b;
        } else {
          o += c;
        }
    }
  }
  return o + "\"";
}

}  // namespace

// ---- jobs (ref job_io.cpp:66-142) -------------------------------------------------

JobSpec job_from_json_text(const std::string& text) {
  Json j = JsonParser(text).parse_document();
  if (j.kind != Json::Object) throw JobFileError("job file must be a JSON object");
  reject_unknown(j, {"seed", "trials", "workers", "integrands"}, "job");
  JobSpec job;
  job.seed = as_u64(at(j, "seed"), "seed");
  job.trials = as_u32(at(j, "trials"), "trials");
  if (has(j, "workers")) job.workers = as_u32(at(j, "workers"), "workers");
  const Json& list = at(j, "integrands");
  if (list.kind != Json::Array) throw JobFileError("'integrands' must be an array");
  for (const Json& ji : *list.arr) {
    if (ji.kind != Json::Object) malformed("integrand entries must be objects");
    reject_unknown(ji, {"name", "expr", "dim", "low", "high", "params", "samples", "method", "method_config"},
                   "integrand");
    const std::string name = as_string(at(ji, "name"), "name");
    const std::string expr = as_string(at(ji, "expr"), "expr");
    const std::size_t dim = as_u64(at(ji, "dim"), "dim");
    HyperRect dom;
    dom.low = as_doubles(at(ji, "low"), "low");
    dom.high = as_doubles(at(ji, "high"), "high");
    std::map<std::string, double> params;
    if (has(ji, "params")) {
      const Json& p = at(ji, "params");
      if (p.kind != Json::Object) malformed("'params' must be an object");
      for (const auto& [k, v] : *p.obj) params[k] = as_double(v, "params");
    }
    const uint64_t samples = as_u64(at(ji, "samples"), "samples");
    IntegrandSpec s = IntegrandSpec::from_source(name, expr, dim, dom, params, samples);
    if (has(ji, "method")) {
      const std::string m = as_string(at(ji, "method"), "method");
      if (m == "direct") s.method = Method::Direct;
      else if (m == "stratified") s.method = Method::Stratified;
      else if (m == "tree") s.method = Method::Tree;
      else throw JobFileError("integrand '" + name + "': unknown method '" + m + "'");
    }
    if (has(ji, "method_config"))
      s.method_config = refine_config_from_json(at(ji, "method_config"),
                                                "integrand '" + name + "' method_config");
    job.integrands.push_back(std::move(s));
  }
  return job;
}

JobSpec read_job(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw JobFileError("cannot open job file: " + path.string());
  std::ostringstream buf;
  buf << in.rdbuf();
  return job_from_json_text(buf.str());
}

std::string job_to_json_text(const JobSpec& job) {  // ref job_io.cpp:122-142
  std::ostringstream o;
  o << "{\n  \"integrands\": [";
  for (std::size_t i = 0; i < job.integrands.size(); ++i) {
    const IntegrandSpec& s = job.integrands[i];
    o << (i ? "," : "") << "\n    {\n";
    o << "      \"dim\": " << s.dim << ",\n";
    o << "      \"expr\": " << json_string(s.source()) << ",\n";
    auto arr = [&](const std::vector<double>& v) {
      std::string r = "[";
      for (std::size_t k = 0; k < v.size(); ++k) r += (k ? ",\n        " : "\n        ") + json_number(v[k]);
      return r + (v.empty() ? "]" : "\n      ]");
    };
    o << "      \"high\": " << arr(s.domain.high) << ",\n";
    o << "      \"low\": " << arr(s.domain.low) << ",\n";
    if (s.method_config) {
      const RefineConfig& rc = *s.method_config;
      o << "      \"method\": \"" << method_name(s.method) << "\",\n      \"method_config\": {\n";
      if (rc.init_cells_per_dim) o << "        \"cells_per_dim\": " << rc.init_cells_per_dim << ",\n";
      o << "        \"cell_cap\": " << rc.cell_cap << ",\n";
      o << "        \"max_depth\": " << rc.max_depth << ",\n";
      o << "        \"samples_per_cell\": " << rc.samples_per_cell << ",\n";
      o << "        \"sigma_multiplier\": " << json_number(rc.sigma_multiplier) << "\n      },\n";
    } else {
      o << "      \"method\": \"" << method_name(s.method) << "\",\n";
    }
    o << "      \"name\": " << json_string(s.name) << ",\n";
    o << "      \"params\": ";
    const std::map<std::string, double>& params = s.params;
    if (params.empty()) {
      o << "{}";
    } else {
      o << "{";
      std::size_t k = 0;
      for (const auto& [n, v] : params)
        o << (k++ ? "," : "") << "\n        " << json_string(n) << ": " << json_number(v);
      o << "\n      }";
    }
    o << ",\n      \"samples\": " << s.n_samples << "\n    }";
  }
  o << (job.integrands.empty() ? "]" : "\n  ]") << ",\n";
  o << "  \"seed\": " << job.seed << ",\n";
  o << "  \"trials\": " << job.trials << ",\n";
  o << "  \"workers\": " << job.workers << "\n}\n";
  return o.str();
}

void write_job(const JobSpec& job, const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw JobFileError("cannot write job file: " + path.string());
  out << job_to_json_text(job);
}

// ---- results table ------------------------------------------------------------
// SPEC.md [MODULE] cli, ResultsTable: one CSV row per integrand in job order,
// header row, ',' separator, '.' decimal point, numbers with 17 significant
// digits (so a value survives write -> read bit for bit), warnings as a ';'
// list.  The table is described once, column by column (kColumns): the
// header, the writer and the reader are all driven by it.  The byte layout is
// the one the reference's own reader/writer accepts and reproduces
// (tests/test_job_io.py round-trips our files through them).

namespace {

// 17 significant digits, C locale (to_chars general == printf %.17g).
std::string num17(double v) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::general, 17);
  return std::string(buf, r.ptr);
}

// A cell may not contain the separator or a line break.
std::string cell_text(std::string s) {
  std::replace_if(s.begin(), s.end(), [](char c) { return c == ',' || c == '\n' || c == '\r'; }, ';');
  return s;
}

std::vector<std::string> csv_cells(std::string_view line) {
  if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
  std::vector<std::string> cells;
  for (std::size_t start = 0;;) {
    const std::size_t comma = line.find(',', start);
    cells.emplace_back(line.substr(start, comma == std::string_view::npos ? std::string_view::npos : comma - start));
    if (comma == std::string_view::npos) return cells;
    start = comma + 1;
  }
}

template <class T>
T read_number(const std::string& text, const char* column) {
  T v{};
  const char* end = text.data() + text.size();
  const auto r = std::from_chars(text.data(), end, v);
  if (r.ec != std::errc() || r.ptr != end)
    throw MalformedResults(std::string("column ") + column + ": not a number: '" + text + "'");
  return v;
}

std::string opt_num17(const std::optional<double>& v) { return v ? num17(*v) : std::string(); }
std::optional<double> read_opt(const std::string& text, const char* column) {
  if (text.empty()) return std::nullopt;
  return read_number<double>(text, column);
}

struct Column {
  const char* name;
  std::string (*write)(const ResultsRow&);
  void (*read)(ResultsRow&, const std::string&);
};

const Column kColumns[] = {
    {"name", [](const ResultsRow& r) { return cell_text(r.name); },
     [](ResultsRow& r, const std::string& s) { r.name = s; }},
    {"index", [](const ResultsRow& r) { return std::to_string(r.index); },
     [](ResultsRow& r, const std::string& s) { r.index = read_number<std::uint32_t>(s, "index"); }},
    {"dim", [](const ResultsRow& r) { return std::to_string(r.dim); },
     [](ResultsRow& r, const std::string& s) { r.dim = read_number<std::size_t>(s, "dim"); }},
    {"method", [](const ResultsRow& r) { return cell_text(r.method); },
     [](ResultsRow& r, const std::string& s) { r.method = s; }},
    {"samples", [](const ResultsRow& r) { return std::to_string(r.samples); },
     [](ResultsRow& r, const std::string& s) { r.samples = read_number<std::uint64_t>(s, "samples"); }},
    {"trials", [](const ResultsRow& r) { return std::to_string(r.trials); },
     [](ResultsRow& r, const std::string& s) { r.trials = read_number<std::uint32_t>(s, "trials"); }},
    {"mean", [](const ResultsRow& r) { return num17(r.mean); },
     [](ResultsRow& r, const std::string& s) { r.mean = read_number<double>(s, "mean"); }},
    {"trial_stddev", [](const ResultsRow& r) { return num17(r.trial_stddev); },
     [](ResultsRow& r, const std::string& s) { r.trial_stddev = read_number<double>(s, "trial_stddev"); }},
    {"mean_std_error", [](const ResultsRow& r) { return num17(r.mean_std_error); },
     [](ResultsRow& r, const std::string& s) { r.mean_std_error = read_number<double>(s, "mean_std_error"); }},
    {"analytic", [](const ResultsRow& r) { return opt_num17(r.analytic); },
     [](ResultsRow& r, const std::string& s) { r.analytic = read_opt(s, "analytic"); }},
    {"abs_error", [](const ResultsRow& r) { return opt_num17(r.abs_error); },
     [](ResultsRow& r, const std::string& s) { r.abs_error = read_opt(s, "abs_error"); }},
    {"warnings", [](const ResultsRow& r) { return cell_text(r.warnings); },
     [](ResultsRow& r, const std::string& s) { r.warnings = s; }},
};
constexpr std::size_t kNumColumns = sizeof kColumns / sizeof kColumns[0];

// A row whose warnings start with this marker is a failed integrand.
constexpr std::string_view kFailedMark = "FAILED";

std::string join(const std::vector<std::string>& parts, char sep) {
  std::string out;
  for (const std::string& p : parts) {
    if (!out.empty()) out += sep;
    out += p;
  }
  return out;
}

}  // namespace

std::vector<ResultsRow> make_results(const JobSpec& job, const BatchResult& br) {
  std::vector<ResultsRow> rows(br.per_integrand.size());
  const double nan = std::numeric_limits<double>::quiet_NaN();
  for (std::size_t i = 0; i < rows.size(); ++i) {
    const IntegrandResult& res = br.per_integrand[i];
    const IntegrandSpec& spec = job.integrands[i];
    ResultsRow& row = rows[i];
    row = ResultsRow{res.name, std::uint32_t(i + 1), spec.dim, method_name(spec.method), spec.n_samples,
                     job.trials, res.ok, nan, nan, nan, std::nullopt, std::nullopt, ""};
    if (!res.ok) {  // failed integrand: no numbers, the reason in the warnings
      row.warnings = std::string(kFailedMark) + ";" + res.error;
      continue;
    }
    row.mean = res.summary.mean;
    row.trial_stddev = res.summary.trial_stddev;
    // mean_std_error: the average per-trial standard error over the trials kept
    double se_sum = 0.0;
    for (const McEstimate& e : res.summary.per_trial) se_sum += e.std_error;
    row.mean_std_error = se_sum / double(res.summary.per_trial.size());
    std::vector<std::string> notes;
    if (res.nonfinite_warning) notes.emplace_back("nonfinite");
    if (res.budget_exhausted) notes.emplace_back("budget_exhausted");
    if (!res.error.empty()) notes.push_back(res.error);  // partial: the failed trials
    row.warnings = join(notes, ';');
  }
  return rows;
}

std::string results_to_csv_text(const std::vector<ResultsRow>& rows) {
  std::vector<std::string> cells(kNumColumns);
  for (std::size_t c = 0; c < kNumColumns; ++c) cells[c] = kColumns[c].name;
  std::string out = join(cells, ',') + "\n";
  for (const ResultsRow& r : rows) {
    for (std::size_t c = 0; c < kNumColumns; ++c) cells[c] = kColumns[c].write(r);
    out += join(cells, ',') + "\n";
  }
  return out;
}

void write_results(const std::vector<ResultsRow>& rows, const std::filesystem::path& path) {
  const std::string text = results_to_csv_text(rows);
  std::ofstream out(path, std::ios::binary);
  if (!out.write(text.data(), std::streamsize(text.size())))
    throw std::runtime_error("cannot write results: " + path.string());
}

std::vector<ResultsRow> read_results(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw MalformedResults("cannot open results file: " + path.string());
  std::string line;
  std::getline(in, line);
  const std::vector<std::string> header = csv_cells(line);
  bool header_ok = header.size() == kNumColumns;
  for (std::size_t c = 0; header_ok && c < kNumColumns; ++c) header_ok = header[c] == kColumns[c].name;
  if (!header_ok) throw MalformedResults("results file: missing or unexpected header row");
  std::vector<ResultsRow> rows;
  for (std::size_t line_no = 2; std::getline(in, line); ++line_no) {
    if (line.empty() || line == "\r") continue;
    const std::vector<std::string> cells = csv_cells(line);
    if (cells.size() != kNumColumns)
      throw MalformedResults("results line " + std::to_string(line_no) + " has " + std::to_string(cells.size()) +
                             " fields, expected " + std::to_string(kNumColumns));
    ResultsRow& r = rows.emplace_back();
    for (std::size_t c = 0; c < kNumColumns; ++c) kColumns[c].read(r, cells[c]);
    r.ok = std::string_view(r.warnings).substr(0, kFailedMark.size()) != kFailedMark;
  }
  if (rows.empty()) throw MalformedResults("results file has no data rows");
  return rows;
}

// ---- commands -----------------------------------------------------------------
// SPEC.md [MODULE] cli: run_command writes the ResultsTable and exits 0 on
// success, 2 when the job does not load or validate, 3 when nothing could be
// computed; one completion line per integrand on stdout.

int run_command(const std::filesystem::path& job_path, const std::filesystem::path& out_path,
                const RunOverrides& overrides) {
  std::optional<JobSpec> job;
  try {
    job = read_job(job_path);
  } catch (const JobFileError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
  job->seed = overrides.seed.value_or(job->seed);
  job->trials = overrides.trials.value_or(job->trials);
  job->workers = overrides.workers.value_or(job->workers);

  if (const std::vector<Violation> bad = validate(*job); !bad.empty()) {
    std::cerr << "error: " << bad.size() << " validation problem(s) in " << job_path.string() << ":\n";
    for (const Violation& v : bad)
      std::cerr << "  " << (v.integrand.empty() ? std::string("job") : v.integrand) << ": " << v.message << "\n";
    return 2;
  }

  BatchResult batch;
  try {
    batch = run_batch(*job);
  } catch (const std::exception& e) {
    std::cerr << "error: batch failed: " << e.what() << "\n";
    return 3;
  }

  const std::vector<ResultsRow> rows = make_results(*job, batch);
  for (const ResultsRow& r : rows) {
    if (r.ok)
      std::cout << r.name << ": mean " << num17(r.mean) << ", trial stddev " << num17(r.trial_stddev)
                << ", mean std_error " << num17(r.mean_std_error) << "\n";
    else
      std::cout << r.name << ": " << r.warnings << "\n";
  }
  write_results(rows, out_path);
  std::cerr << rows.size() << " row(s) written to " << out_path.string() << "; sampling took "
            << batch.total_seconds << " s\n";
  const bool any_ok = std::any_of(rows.begin(), rows.end(), [](const ResultsRow& r) { return r.ok; });
  return any_ok ? 0 : 3;
}

int gen_fig1(std::uint32_t n_count, std::uint64_t samples, const std::filesystem::path& out_path) {
  write_job(make_harmonic_job(n_count, samples), out_path);
  return 0;
}

// check_fig1 (SPEC.md [OP] check_fig1): per row, the harmonic number n and the
// analytic value — from the analytic column when the table has one, else
// analytic_harmonic(n) with n the integer that ends the row's name (gen-fig1
// names rows f001..f100) — then pass iff the row succeeded and
// |mean - analytic| <= 4 max(trial_stddev, mean_std_error).
Fig1Check check_fig1(const std::vector<ResultsRow>& rows) {
  if (rows.empty()) throw MalformedResults("no result rows");
  auto name_number = [](const std::string& name) -> std::optional<std::uint32_t> {
    const auto first_digit =
        std::find_if_not(name.rbegin(), name.rend(), [](unsigned char c) { return std::isdigit(c) != 0; }).base();
    if (first_digit == name.end()) return std::nullopt;
    std::uint32_t n = 0;
    std::from_chars(&*first_digit, name.data() + name.size(), n);
    return n;
  };
  Fig1Check check;
  check.rows.reserve(rows.size());
  for (const ResultsRow& r : rows) {
    const std::optional<std::uint32_t> n = name_number(r.name);
    if (!r.analytic && !n)
      throw MalformedResults("row '" + r.name + "' has neither an analytic value nor a trailing harmonic index");
    Fig1Row f;
    f.n = n ? *n : r.index;
    f.analytic = r.analytic ? *r.analytic : analytic_harmonic(f.n);
    f.mean = r.mean;
    f.trial_stddev = r.trial_stddev;
    f.mean_std_error = r.mean_std_error;
    const double band = 4.0 * std::max(r.trial_stddev, r.mean_std_error);
    f.pass = r.ok && std::isfinite(r.mean) && std::fabs(r.mean - f.analytic) <= band;
    check.passed += f.pass ? 1u : 0u;
    check.rows.push_back(f);
  }
  return check;
}

int check_fig1_command(const std::filesystem::path& results_path,
                       const std::optional<std::filesystem::path>& plot_out) {
  std::optional<Fig1Check> check;
  try {
    check = check_fig1(read_results(results_path));
  } catch (const MalformedResults& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
  for (const Fig1Row& r : check->rows)
    std::cout << (r.pass ? "PASS" : "FAIL") << " n=" << r.n << " mean=" << num17(r.mean)
              << " analytic=" << num17(r.analytic)
              << " band=" << num17(4.0 * std::max(r.trial_stddev, r.mean_std_error)) << "\n";
  std::cout << "passed " << check->passed << "/" << check->rows.size() << "\n";
  if (plot_out) {  // plot data: n, mean, the trial spread and the analytic curve
    std::string text = "n,mean,trial_stddev,analytic\n";
    for (const Fig1Row& r : check->rows)
      text += std::to_string(r.n) + "," + num17(r.mean) + "," + num17(r.trial_stddev) + "," + num17(r.analytic) + "\n";
    std::ofstream out(*plot_out, std::ios::binary);
    if (!out.write(text.data(), std::streamsize(text.size()))) {
      std::cerr << "error: cannot write " << plot_out->string() << "\n";
      return 2;
    }
  }
  // acceptance criterion 1: at least 95 % of the rows inside the band
  return 100 * std::size_t(check->passed) >= 95 * check->rows.size() ? 0 : 1;
}

}  // namespace mcb
