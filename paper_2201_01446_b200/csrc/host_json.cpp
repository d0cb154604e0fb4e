// JSON model files: write_model / read_model (model_io.cpp:226-283).
//
// The reference stores a DPModel as one JSON object {"format": "dpmd-model", "version": 1,
// "preset", "seed", "species", "masses", "r_cut", "r_smooth", "max_neighbors", "m_lt",
// "embedding": [{d1, w0, b0, w1, b1, w2, b2}], "fitting": [{input_width, width, layers:
// [{in, out, w, b}], w_out, b_out}]}. Doubles are written in shortest round-trip form, so a
// read after a write reproduces every weight bit for bit in both directions (ours <-> reference).
// Host-only code: a small recursive-descent parser, no third-party JSON library.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "host_common.hpp"

namespace dpb {
namespace {

struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  std::string text; // number token or string value
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;

  const JVal& at(const std::string& k) const {
    if (kind != Obj) throw InputErr("model file is missing fields: expected an object");
    auto it = obj.find(k);
    if (it == obj.end()) throw InputErr("model file is missing fields: key '" + k + "' not found");
    return it->second;
  }
  bool has(const std::string& k) const { return kind == Obj && obj.count(k); }
  double num() const {
    if (kind != Num) throw InputErr("model file is missing fields: expected a number");
    return std::strtod(text.c_str(), nullptr);
  }
  long long integer() const {
    if (kind != Num) throw InputErr("model file is missing fields: expected an integer");
    const double v = std::strtod(text.c_str(), nullptr);
    if (v != std::floor(v)) throw InputErr("model file is missing fields: expected an integer");
    return static_cast<long long>(v);
  }
  uint64_t u64() const {
    if (kind != Num || text.empty() || text[0] == '-') throw InputErr("model file is missing fields: expected a seed");
    return std::strtoull(text.c_str(), nullptr, 10);
  }
  const std::string& str() const {
    if (kind != Str) throw InputErr("model file is missing fields: expected a string");
    return text;
  }
  std::vector<double> nums() const {
    if (kind != Arr) throw InputErr("model file is missing fields: expected an array");
    std::vector<double> v;
    v.reserve(arr.size());
    for (const auto& x : arr) v.push_back(x.num());
    return v;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  JVal parse() {
    JVal v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;

  [[noreturn]] void fail(const char* what) {
    throw InputErr(std::string("model file is not valid JSON: ") + what + " at offset " + std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (s_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  JVal value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    const char c = s_[i_];
    JVal v;
    if (c == '{') {
      v.kind = JVal::Obj;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        if (i_ >= s_.size() || s_[i_] != '"') fail("expected a key");
        std::string k = string();
        ws();
        if (i_ >= s_.size() || s_[i_] != ':') fail("expected ':'");
        ++i_;
        v.obj[k] = value();
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == '}') {
          ++i_;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = JVal::Arr;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == ']') {
          ++i_;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::Str;
      v.text = string();
      return v;
    }
    if (lit("true")) {
      v.kind = JVal::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = JVal::Bool;
      return v;
    }
    if (lit("null")) return v;
    if (c == '-' || (c >= '0' && c <= '9')) {
      const size_t st = i_;
      if (s_[i_] == '-') ++i_;
      auto digits = [&] {
        const size_t d0 = i_;
        while (i_ < s_.size() && s_[i_] >= '0' && s_[i_] <= '9') ++i_;
        if (i_ == d0) fail("bad number");
      };
      digits();
      if (i_ < s_.size() && s_[i_] == '.') {
        ++i_;
        digits();
      }
      if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
        ++i_;
        if (i_ < s_.size() && (s_[i_] == '+' || s_[i_] == '-')) ++i_;
        digits();
      }
      v.kind = JVal::Num;
      v.text = s_.substr(st, i_ - st);
      return v;
    }
    fail("unexpected character");
  }
  std::string string() {
    ++i_; // opening quote
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) fail("bad escape");
        const char e = s_[i_++];
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
            if (i_ + 4 > s_.size()) fail("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::strtoul(s_.substr(i_, 4).c_str(), nullptr, 16));
            i_ += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
};

// ---- writer (compact, keys in lexicographic order like the reference's std::map-backed json)
void put_double(std::string& o, double x) {
  if (!std::isfinite(x)) {
    o += "null"; // what the reference's JSON library writes for non-finite numbers
    return;
  }
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, x);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eE") == std::string::npos && s.find("inf") == std::string::npos) s += ".0";
  o += s;
}
void put_str(std::string& o, const std::string& s) {
  o += '"';
  for (char c : s) {
    if (c == '"' || c == '\\') {
      o += '\\';
      o += c;
    } else if (static_cast<unsigned char>(c) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else {
      o += c;
    }
  }
  o += '"';
}
void put_arr(std::string& o, const double* v, size_t n) {
  o += '[';
  for (size_t k = 0; k < n; ++k) {
    if (k) o += ',';
    put_double(o, v[k]);
  }
  o += ']';
}

std::vector<std::string> split_csv(const char* csv, int n) {
  std::vector<std::string> out;
  if (csv && *csv) {
    std::stringstream ss(csv);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(item);
  }
  if (static_cast<int>(out.size()) != n) {
    if (!out.empty()) throw InputErr("species list does not match the number of types");
    for (int t = 0; t < n; ++t) out.push_back(std::string(1, static_cast<char>('A' + t)));
  }
  return out;
}

} // namespace
} // namespace dpb

using namespace dpb;

extern "C" {

int dp_write_model_json(const char* path, const dp_preset* s, const double* blob, const char* species_csv,
                        const char* preset, uint64_t seed) {
  return guard_call(nullptr, [&] {
    if (!path || !s || !blob) throw InputErr("null argument");
    if (s->n_types < 1 || s->n_types > 8 || s->d1 < 1 || s->fit_hidden < 1 || s->fit_width < 1)
      throw InputErr("model shape is inconsistent");
    const int nt = s->n_types, d1 = s->d1;
    const auto species = split_csv(species_csv, nt);
    std::string o;
    o.reserve(1 << 20);
    size_t at = 0;
    std::vector<std::string> emb(nt), fit(nt);
    for (int t = 0; t < nt; ++t) {
      std::string& e = emb[t];
      // keys sorted: b0 b1 b2 d1 w0 w1 w2 -> collect in blob order, emit sorted
      const double* w0 = blob + at;
      const double* b0 = w0 + d1;
      const double* w1 = b0 + d1;
      const double* b1 = w1 + 2 * d1 * d1;
      const double* w2 = b1 + 2 * d1;
      const double* b2 = w2 + 8 * d1 * d1;
      at = static_cast<size_t>(b2 + 4 * d1 - blob);
      e += '{';
      put_str(e, "b0"); e += ':'; put_arr(e, b0, d1); e += ',';
      put_str(e, "b1"); e += ':'; put_arr(e, b1, 2 * d1); e += ',';
      put_str(e, "b2"); e += ':'; put_arr(e, b2, 4 * d1); e += ',';
      put_str(e, "d1"); e += ':'; e += std::to_string(d1); e += ',';
      put_str(e, "w0"); e += ':'; put_arr(e, w0, d1); e += ',';
      put_str(e, "w1"); e += ':'; put_arr(e, w1, 2 * d1 * d1); e += ',';
      put_str(e, "w2"); e += ':'; put_arr(e, w2, 8 * d1 * d1);
      e += '}';
    }
    const int din = s->m_lt * 4 * d1;
    for (int t = 0; t < nt; ++t) {
      std::string& f = fit[t];
      f += '{';
      put_str(f, "b_out");
      f += ':';
      const double* cur = blob + at;
      // layers first (they precede w_out/b_out in the blob)
      std::string layers = "[";
      int in = din;
      for (int k = 0; k < s->fit_hidden; ++k) {
        const double* w = cur;
        const double* b = w + static_cast<size_t>(in) * s->fit_width;
        if (k) layers += ',';
        layers += '{';
        put_str(layers, "b"); layers += ':'; put_arr(layers, b, s->fit_width); layers += ',';
        put_str(layers, "in"); layers += ':'; layers += std::to_string(in); layers += ',';
        put_str(layers, "out"); layers += ':'; layers += std::to_string(s->fit_width); layers += ',';
        put_str(layers, "w"); layers += ':'; put_arr(layers, w, static_cast<size_t>(in) * s->fit_width);
        layers += '}';
        cur = b + s->fit_width;
        in = s->fit_width;
      }
      layers += ']';
      const double* wout = cur;
      const double bout = cur[in];
      at = static_cast<size_t>(cur + in + 1 - blob);
      put_double(f, bout);
      f += ',';
      put_str(f, "input_width"); f += ':'; f += std::to_string(din); f += ',';
      put_str(f, "layers"); f += ':'; f += layers; f += ',';
      put_str(f, "w_out"); f += ':'; put_arr(f, wout, in); f += ',';
      put_str(f, "width"); f += ':'; f += std::to_string(s->fit_width);
      f += '}';
    }
    o += '{';
    put_str(o, "embedding"); o += ":[";
    for (int t = 0; t < nt; ++t) { if (t) o += ','; o += emb[t]; }
    o += "],";
    put_str(o, "fitting"); o += ":[";
    for (int t = 0; t < nt; ++t) { if (t) o += ','; o += fit[t]; }
    o += "],";
    put_str(o, "format"); o += ':'; put_str(o, "dpmd-model"); o += ',';
    put_str(o, "m_lt"); o += ':'; o += std::to_string(s->m_lt); o += ',';
    put_str(o, "masses"); o += ':'; put_arr(o, s->masses, nt); o += ',';
    put_str(o, "max_neighbors"); o += ":[";
    for (int t = 0; t < nt; ++t) { if (t) o += ','; o += std::to_string(s->max_nbr[t]); }
    o += "],";
    put_str(o, "preset"); o += ':'; put_str(o, preset ? preset : ""); o += ',';
    put_str(o, "r_cut"); o += ':'; put_double(o, s->r_cut); o += ',';
    put_str(o, "r_smooth"); o += ':'; put_double(o, s->r_smooth); o += ',';
    put_str(o, "seed"); o += ':'; o += std::to_string(seed); o += ',';
    put_str(o, "species"); o += ":[";
    for (int t = 0; t < nt; ++t) { if (t) o += ','; put_str(o, species[t]); }
    o += "],";
    put_str(o, "version"); o += ":1}";
    o += '\n';
    std::ofstream os(path, std::ios::binary);
    if (!os) throw InputErr(std::string("cannot open model file for writing: ") + path);
    os << o;
    if (!os) throw InputErr(std::string("short write to model file: ") + path);
  });
}

int dp_read_model_json(const char* path, dp_preset* s, double* blob, int64_t blob_cap, char* species_csv,
                       int species_cap, char* preset, int preset_cap, uint64_t* seed) {
  return guard_call(nullptr, [&] {
    if (!path || !s) throw InputErr("null argument");
    std::ifstream is(path, std::ios::binary);
    if (!is) throw InputErr(std::string("cannot open model file: ") + path);
    std::stringstream ss;
    ss << is.rdbuf();
    const std::string txt = ss.str();
    const JVal j = Parser(txt).parse();
    if (j.kind != JVal::Obj) throw InputErr("model file is not valid JSON: top level is not an object");
    if (j.at("format").str() != "dpmd-model") throw InputErr(std::string("not a model file: ") + path);
    if (j.at("version").integer() != 1) throw InputErr("unsupported model file version");
    const std::string pname = j.has("preset") ? j.at("preset").str() : std::string();
    const uint64_t sd = j.has("seed") ? j.at("seed").u64() : 0;
    const auto& species = j.at("species");
    if (species.kind != JVal::Arr) throw InputErr("model file is missing fields: species");
    const int nt = static_cast<int>(species.arr.size());
    if (nt <= 0) throw InputErr("model has no species");                       // model.cpp:9
    if (nt > 8) throw InputErr("at most 8 species fit the dp_preset shape");
    const auto masses = j.at("masses").nums();
    const double r_cut = j.at("r_cut").num(), r_smooth = j.at("r_smooth").num();
    const auto mx = j.at("max_neighbors").nums();
    const int m_lt = static_cast<int>(j.at("m_lt").integer());
    const auto& emb = j.at("embedding");
    const auto& fit = j.at("fitting");
    if (emb.kind != JVal::Arr || fit.kind != JVal::Arr) throw InputErr("model file is missing fields: nets");
    // DPModel::validate (model.cpp:7-48)
    if (static_cast<int>(masses.size()) != nt) throw InputErr("model masses size mismatch");
    if (static_cast<int>(mx.size()) != nt) throw InputErr("model max_nbr size mismatch");
    if (static_cast<int>(emb.arr.size()) != nt) throw InputErr("model embedding count mismatch");
    if (static_cast<int>(fit.arr.size()) != nt) throw InputErr("model fitting count mismatch");
    if (!(r_cut > 0.0) || !(r_smooth >= 0.0) || !(r_smooth < r_cut))
      throw InputErr("model cutoffs must satisfy 0 <= r_smooth < r_cut");
    for (double c : mx)
      if (!(c > 0)) throw InputErr("model max_nbr entries must be positive");
    const int d1 = static_cast<int>(emb.arr[0].at("d1").integer());
    if (d1 <= 0) throw InputErr("embedding width must be positive");
    std::vector<double> out;
    for (const auto& e : emb.arr) {
      if (e.at("d1").integer() != d1) throw InputErr("all embedding nets must share d1");
      const auto w0 = e.at("w0").nums(), b0 = e.at("b0").nums(), w1 = e.at("w1").nums(), b1 = e.at("b1").nums(),
                 w2 = e.at("w2").nums(), b2 = e.at("b2").nums();
      if (static_cast<int>(w0.size()) != d1 || static_cast<int>(b0.size()) != d1 ||
          static_cast<int>(w1.size()) != d1 * 2 * d1 || static_cast<int>(b1.size()) != 2 * d1 ||
          static_cast<int>(w2.size()) != 2 * d1 * 4 * d1 || static_cast<int>(b2.size()) != 4 * d1)
        throw InputErr("embedding net parameter shapes are inconsistent");
      for (const auto* v : {&w0, &b0, &w1, &b1, &w2, &b2}) out.insert(out.end(), v->begin(), v->end());
    }
    if (m_lt <= 0 || m_lt > 4 * d1) throw InputErr("m_lt must lie in [1, 4*d1]");
    const int din = m_lt * 4 * d1;
    int width = -1, hidden = -1;
    for (const auto& f : fit.arr) {
      if (f.at("input_width").integer() != din) throw InputErr("fitting input width does not match descriptor");
      const auto& layers = f.at("layers");
      if (layers.kind != JVal::Arr || layers.arr.empty()) throw InputErr("fitting net needs at least one hidden layer");
      int cur = din;
      for (const auto& l : layers.arr) {
        const int in = static_cast<int>(l.at("in").integer()), o = static_cast<int>(l.at("out").integer());
        if (in != cur || o <= 0) throw InputErr("fitting layer widths are inconsistent");
        const auto w = l.at("w").nums(), b = l.at("b").nums();
        if (static_cast<int64_t>(w.size()) != static_cast<int64_t>(in) * o || static_cast<int>(b.size()) != o)
          throw InputErr("fitting layer parameter shapes are inconsistent");
        if (width < 0) width = o;
        if (o != width) throw InputErr("fitting layers of different widths do not fit the dp_preset shape");
        out.insert(out.end(), w.begin(), w.end());
        out.insert(out.end(), b.begin(), b.end());
        cur = o;
      }
      if (hidden < 0) hidden = static_cast<int>(layers.arr.size());
      if (static_cast<int>(layers.arr.size()) != hidden)
        throw InputErr("fitting nets of all types must share a shape");
      const auto wo = f.at("w_out").nums();
      if (static_cast<int>(wo.size()) != cur) throw InputErr("fitting output weights do not match last hidden width");
      out.insert(out.end(), wo.begin(), wo.end());
      out.push_back(f.at("b_out").num());
    }
    dp_preset shp{};
    shp.n_types = nt;
    shp.r_cut = r_cut;
    shp.r_smooth = r_smooth;
    shp.d1 = d1;
    shp.m_lt = m_lt;
    shp.fit_width = width;
    shp.fit_hidden = hidden;
    for (int t = 0; t < nt; ++t) {
      shp.masses[t] = masses[t];
      shp.max_nbr[t] = static_cast<int>(mx[t]);
    }
    *s = shp;
    if (seed) *seed = sd;
    if (preset && preset_cap > 0) {
      std::snprintf(preset, static_cast<size_t>(preset_cap), "%s", pname.c_str());
    }
    if (species_csv && species_cap > 0) {
      std::string csv;
      for (int t = 0; t < nt; ++t) {
        if (t) csv += ',';
        csv += species.arr[t].str();
      }
      std::snprintf(species_csv, static_cast<size_t>(species_cap), "%s", csv.c_str());
    }
    if (blob) {
      if (blob_cap < static_cast<int64_t>(out.size())) throw InputErr("model blob buffer too small");
      std::memcpy(blob, out.data(), out.size() * sizeof(double));
    }
  });
}

} // extern "C"
