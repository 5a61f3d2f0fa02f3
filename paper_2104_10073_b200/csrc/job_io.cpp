// job_io.cpp — job files, results CSV and the Fig. 1 harness on the GPU
// backend (include/mcb/job_io.hpp).  Formats and messages follow the
// reference's src/job_io.cpp (file:line cited per function); the strict JSON
// reader is a small RFC 8259 parser of our own (the reference uses nlohmann).
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

std::string fmt17(double v) {  // ref job_io.cpp:144-148
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::string sanitize_field(std::string s) {  // ref job_io.cpp:150-155
  for (char& c : s)
    if (c == ',' || c == '\n' || c == '\r') c = ';';
  return s;
}

const char* kResultsHeader =
    "name,index,dim,method,samples,trials,mean,trial_stddev,mean_std_error,analytic,abs_error,"
    "warnings";

std::vector<std::string> split_csv_line(const std::string& line) {  // ref job_io.cpp:225-239
  std::vector<std::string> fields;
  std::string cur;
  for (char c : line) {
    if (c == ',') {
      fields.push_back(cur);
      cur.clear();
    } else if (c != '\r') {
      cur += c;
    }
  }
  fields.push_back(cur);
  return fields;
}

double parse_double(const std::string& s, const char* what) {
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (end == s.c_str()) throw MalformedResults(std::string("bad numeric field '") + s + "' for " + what);
  return v;
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

// ---- results (ref job_io.cpp:171-284) ------------------------------------------

std::vector<ResultsRow> make_results(const JobSpec& job, const BatchResult& br) {
  std::vector<ResultsRow> rows;
  rows.reserve(br.per_integrand.size());
  for (std::size_t i = 0; i < br.per_integrand.size(); ++i) {
    const IntegrandResult& r = br.per_integrand[i];
    const IntegrandSpec& s = job.integrands[i];
    ResultsRow row;
    row.name = r.name;
    row.index = uint32_t(i + 1);
    row.dim = s.dim;
    row.method = method_name(s.method);
    row.samples = s.n_samples;
    row.trials = job.trials;
    row.ok = r.ok;
    if (r.ok) {
      row.mean = r.summary.mean;
      row.trial_stddev = r.summary.trial_stddev;
      double se = 0.0;
      for (const McEstimate& e : r.summary.per_trial) se += e.std_error;
      row.mean_std_error = se / double(r.summary.per_trial.size());
      std::string w;
      if (r.nonfinite_warning) w += "nonfinite;";
      if (r.budget_exhausted) w += "budget_exhausted;";
      if (!r.error.empty()) w += sanitize_field(r.error) + ";";
      if (!w.empty()) w.pop_back();
      row.warnings = w;
    } else {
      row.mean = row.trial_stddev = row.mean_std_error = std::numeric_limits<double>::quiet_NaN();
      row.warnings = "FAILED;" + sanitize_field(r.error);
    }
    rows.push_back(std::move(row));
  }
  return rows;
}

std::string results_to_csv_text(const std::vector<ResultsRow>& rows) {
  std::ostringstream out;
  out << kResultsHeader << "\n";
  for (const ResultsRow& r : rows)
    out << sanitize_field(r.name) << ',' << r.index << ',' << r.dim << ',' << r.method << ','
        << r.samples << ',' << r.trials << ',' << fmt17(r.mean) << ',' << fmt17(r.trial_stddev) << ','
        << fmt17(r.mean_std_error) << ',' << (r.analytic ? fmt17(*r.analytic) : std::string()) << ','
        << (r.abs_error ? fmt17(*r.abs_error) : std::string()) << ',' << sanitize_field(r.warnings)
        << "\n";
  return out.str();
}

void write_results(const std::vector<ResultsRow>& rows, const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write results: " + path.string());
  out << results_to_csv_text(rows);
}

std::vector<ResultsRow> read_results(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw MalformedResults("cannot open results file: " + path.string());
  std::string line;
  if (!std::getline(in, line) || split_csv_line(line) != split_csv_line(kResultsHeader))
    throw MalformedResults("missing or wrong header row");
  std::vector<ResultsRow> rows;
  std::size_t lineno = 1;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    const std::vector<std::string> f = split_csv_line(line);
    if (f.size() != 12)
      throw MalformedResults("line " + std::to_string(lineno) + ": expected 12 fields, got " +
                             std::to_string(f.size()));
    ResultsRow r;
    r.name = f[0];
    r.index = uint32_t(std::strtoul(f[1].c_str(), nullptr, 10));
    r.dim = std::strtoul(f[2].c_str(), nullptr, 10);
    r.method = f[3];
    r.samples = std::strtoull(f[4].c_str(), nullptr, 10);
    r.trials = uint32_t(std::strtoul(f[5].c_str(), nullptr, 10));
    r.mean = parse_double(f[6], "mean");
    r.trial_stddev = parse_double(f[7], "trial_stddev");
    r.mean_std_error = parse_double(f[8], "mean_std_error");
    if (!f[9].empty()) r.analytic = parse_double(f[9], "analytic");
    if (!f[10].empty()) r.abs_error = parse_double(f[10], "abs_error");
    r.warnings = f[11];
    r.ok = r.warnings.rfind("FAILED", 0) != 0;
    rows.push_back(std::move(r));
  }
  if (rows.empty()) throw MalformedResults("results file has no data rows");
  return rows;
}

// ---- commands (ref job_io.cpp:286-455) --------------------------------------------

int run_command(const std::filesystem::path& job_path, const std::filesystem::path& out_path,
                const RunOverrides& overrides) {
  JobSpec job;
  try {
    job = read_job(job_path);
  } catch (const JobFileError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
  if (overrides.seed) job.seed = *overrides.seed;
  if (overrides.trials) job.trials = *overrides.trials;
  if (overrides.workers) job.workers = *overrides.workers;
  const std::vector<Violation> violations = validate(job);
  if (!violations.empty()) {
    std::cerr << "error: job does not validate:\n";
    for (const Violation& v : violations) {
      std::cerr << "  ";
      if (!v.integrand.empty()) std::cerr << v.integrand << ": ";
      std::cerr << v.message << "\n";
    }
    return 2;
  }
  BatchResult br;
  try {
    br = run_batch(job);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
  bool any_ok = false;
  for (const IntegrandResult& r : br.per_integrand) {
    if (r.ok) {
      any_ok = true;
      std::cout << r.name << ": " << fmt17(r.summary.mean) << " +- " << fmt17(r.summary.trial_stddev)
                << " (" << r.seconds << " s)\n";
    } else {
      std::cout << r.name << ": FAILED (" << r.error << ")\n";
    }
  }
  write_results(make_results(job, br), out_path);
  std::cerr << "wrote " << br.per_integrand.size() << " rows to " << out_path << " in "
            << br.total_seconds << " s\n";
  return any_ok ? 0 : 3;
}

int gen_fig1(std::uint32_t n_count, std::uint64_t samples, const std::filesystem::path& out_path) {
  write_job(make_harmonic_job(n_count, samples), out_path);
  return 0;
}

namespace {
std::optional<uint32_t> trailing_number(const std::string& name) {  // ref job_io.cpp:386-395
  std::size_t end = name.size(), begin = end;
  while (begin > 0 && std::isdigit(static_cast<unsigned char>(name[begin - 1]))) --begin;
  if (begin == end) return std::nullopt;
  return uint32_t(std::strtoul(name.c_str() + begin, nullptr, 10));
}
}  // namespace

Fig1Check check_fig1(const std::vector<ResultsRow>& rows) {
  if (rows.empty()) throw MalformedResults("no result rows");
  Fig1Check out;
  for (const ResultsRow& r : rows) {
    Fig1Row f;
    const auto n = trailing_number(r.name);
    if (r.analytic) {
      f.analytic = *r.analytic;
      f.n = n.value_or(r.index);
    } else {
      if (!n)
        throw MalformedResults("row '" + r.name +
                               "': no analytic column and no trailing index in the name");
      f.n = *n;
      f.analytic = analytic_harmonic(f.n);
    }
    f.mean = r.mean;
    f.trial_stddev = r.trial_stddev;
    f.mean_std_error = r.mean_std_error;
    const double band = 4.0 * std::max(f.trial_stddev, f.mean_std_error);
    f.pass = r.ok && std::isfinite(f.mean) && std::fabs(f.mean - f.analytic) <= band;
    if (f.pass) ++out.passed;
    out.rows.push_back(f);
  }
  return out;
}

int check_fig1_command(const std::filesystem::path& results_path,
                       const std::optional<std::filesystem::path>& plot_out) {
  Fig1Check check;
  try {
    check = check_fig1(read_results(results_path));
  } catch (const MalformedResults& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
  for (const Fig1Row& r : check.rows)
    std::cout << "n=" << r.n << " mean=" << fmt17(r.mean) << " analytic=" << fmt17(r.analytic)
              << " band=+-" << fmt17(4.0 * std::max(r.trial_stddev, r.mean_std_error))
              << (r.pass ? " PASS" : " FAIL") << "\n";
  std::cout << "passed " << check.passed << "/" << check.rows.size() << "\n";
  if (plot_out) {
    std::ofstream out(*plot_out);
    if (!out) {
      std::cerr << "error: cannot write " << *plot_out << "\n";
      return 2;
    }
    out << "n,mean,trial_stddev,analytic\n";
    for (const Fig1Row& r : check.rows)
      out << r.n << ',' << fmt17(r.mean) << ',' << fmt17(r.trial_stddev) << ',' << fmt17(r.analytic)
          << "\n";
  }
  const double frac = double(check.passed) / double(check.rows.size());
  return frac >= 0.95 ? 0 : 1;
}

}  // namespace mcb
