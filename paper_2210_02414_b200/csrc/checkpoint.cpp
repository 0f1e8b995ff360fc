// checkpoint.cpp — loads a quantized GLM checkpoint written by the reference
// (`save_quantized_model`, quant.cpp:409-448; GLMT tensors, tensor_io.cpp:68-179) straight
// into the B200 model: the canonical payloads and FP64 scales go to the device layout
// without re-quantizing, so the GPU model holds exactly the reference's QuantizedModel.
//
// Directory layout (quant.cpp:409-448):
//   manifest.json           {"config": {...}, "policy": {"bits","scheme","axis"},
//                            "matrices": [{"name","bits","scheme","axis","rows","cols"}, ...]}
//   embedding.glmt          f64 [vocab, hidden]
//   layer<L>.<m>.codes.glmt i8  [payload bytes]   m in qkv, out_proj, ffn_w1, ffn_v, ffn_w2
//   layer<L>.<m>.scales.glmt f64 [groups]
//   layer<L>.ln{1,2}_{gain,bias}.glmt f64 [hidden]
// Every header, shape and file size is validated before any device work, so format errors
// surface as GLM_FORMAT (FormatError) even without a GPU; payloads then stream one matrix at a
// time (the embedding in 256 MB row chunks), so host memory stays at one matrix, not the model.
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "glm130b.h"
#include "kernels.h"

namespace glm {
namespace {

// ---- GLMT (tensor_io.cpp:12-13, 68-140): "GLMT", u8 version 1, u8 dtype (0 f64, 1 f32,
// 2 i8), u32 rank, u64 dims[rank] (little endian), then the raw payload -----------------
struct Glmt {
  int dtype = 0;
  std::vector<uint64_t> dims;
  std::vector<double> f64;
  std::vector<int8_t> i8;
  uint64_t count() const {
    uint64_t n = 1;
    for (uint64_t d : dims) n *= d;
    return n;
  }
};

// Header of a GLMT file and the byte offset of its payload; the file size is checked against
// the payload the header announces (a truncated file fails before any payload is read).
struct GlmtHeader {
  int dtype = 0;
  std::vector<uint64_t> dims;
  std::streamoff data = 0;
  uint64_t count() const {
    uint64_t n = 1;
    for (uint64_t d : dims) n *= d;
    return n;
  }
  size_t elem() const { return dtype == 0 ? 8 : dtype == 1 ? 4 : 1; }
};

GlmtHeader read_glmt_header(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) fail(GLM_FORMAT, "tensor_io", "cannot open " + path);
  const std::streamoff size = in.tellg();
  in.seekg(0);
  auto bytes = [&](void* dst, size_t n) {
    in.read(static_cast<char*>(dst), static_cast<std::streamsize>(n));
    if (static_cast<size_t>(in.gcount()) != n) fail(GLM_FORMAT, "tensor_io", "truncated file " + path);
  };
  char magic[4];
  bytes(magic, 4);
  if (std::memcmp(magic, "GLMT", 4) != 0) fail(GLM_FORMAT, "tensor_io", "bad magic in " + path);
  uint8_t version = 0, dtype = 0;
  bytes(&version, 1);
  if (version != 1) fail(GLM_FORMAT, "tensor_io", "unsupported version " + std::to_string(version));
  bytes(&dtype, 1);
  if (dtype > 2) fail(GLM_FORMAT, "tensor_io", "unknown dtype " + std::to_string(dtype));
  uint8_t b[8];
  bytes(b, 4);
  uint32_t rank = 0;
  for (int i = 3; i >= 0; --i) rank = (rank << 8) | b[i];
  if (rank > 64) fail(GLM_FORMAT, "tensor_io", "implausible rank " + std::to_string(rank));
  GlmtHeader h;
  h.dtype = dtype;
  h.dims.resize(rank);
  for (uint32_t r = 0; r < rank; ++r) {
    bytes(b, 8);
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
    h.dims[r] = v;
  }
  h.data = in.tellg();
  if (static_cast<uint64_t>(size - h.data) < h.count() * h.elem()) fail(GLM_FORMAT, "tensor_io", "truncated file " + path);
  return h;
}

// rows [row0, row0 + nrows) of an f64 / f32 GLMT matrix with `cols` columns, as doubles
void read_glmt_rows(const std::string& path, const GlmtHeader& h, uint64_t row0, uint64_t nrows, uint64_t cols,
                    std::vector<double>& out) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(GLM_FORMAT, "tensor_io", "cannot open " + path);
  out.resize(nrows * cols);
  in.seekg(h.data + static_cast<std::streamoff>(row0 * cols * h.elem()));
  if (h.dtype == 0) {
    in.read(reinterpret_cast<char*>(out.data()), static_cast<std::streamsize>(nrows * cols * 8));
    if (static_cast<uint64_t>(in.gcount()) != nrows * cols * 8) fail(GLM_FORMAT, "tensor_io", "truncated file " + path);
  } else {
    std::vector<float> f(nrows * cols);
    in.read(reinterpret_cast<char*>(f.data()), static_cast<std::streamsize>(f.size() * 4));
    if (static_cast<uint64_t>(in.gcount()) != f.size() * 4) fail(GLM_FORMAT, "tensor_io", "truncated file " + path);
    out.assign(f.begin(), f.end());
  }
}

Glmt read_glmt(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(GLM_FORMAT, "tensor_io", "cannot open " + path);
  auto bytes = [&](void* dst, size_t n) {
    in.read(static_cast<char*>(dst), static_cast<std::streamsize>(n));
    if (static_cast<size_t>(in.gcount()) != n) fail(GLM_FORMAT, "tensor_io", "truncated file " + path);
  };
  char magic[4];
  bytes(magic, 4);
  if (std::memcmp(magic, "GLMT", 4) != 0) fail(GLM_FORMAT, "tensor_io", "bad magic in " + path);
  uint8_t version = 0, dtype = 0;
  bytes(&version, 1);
  if (version != 1) fail(GLM_FORMAT, "tensor_io", "unsupported version " + std::to_string(version));
  bytes(&dtype, 1);
  if (dtype > 2) fail(GLM_FORMAT, "tensor_io", "unknown dtype " + std::to_string(dtype));
  uint8_t b[8];
  bytes(b, 4);
  uint32_t rank = 0;
  for (int i = 3; i >= 0; --i) rank = (rank << 8) | b[i];
  if (rank > 64) fail(GLM_FORMAT, "tensor_io", "implausible rank " + std::to_string(rank));
  Glmt t;
  t.dtype = dtype;
  t.dims.resize(rank);
  for (uint32_t r = 0; r < rank; ++r) {
    bytes(b, 8);
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
    t.dims[r] = v;
  }
  const uint64_t n = t.count();
  if (dtype == 0) {
    t.f64.resize(n);
    bytes(t.f64.data(), n * 8);
  } else if (dtype == 1) {
    std::vector<float> f(n);
    bytes(f.data(), n * 4);
    t.f64.assign(f.begin(), f.end());
    t.dtype = 0;
  } else {
    t.i8.resize(n);
    bytes(t.i8.data(), n);
  }
  return t;
}

// ---- minimal JSON (the manifest only needs objects, arrays, strings, numbers, bools) ----
struct Json {
  enum Kind { kNull, kBool, kNum, kStr, kArr, kObj } kind = kNull;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
  const Json& at(const std::string& k) const {
    auto it = obj.find(k);
    if (kind != kObj || it == obj.end()) fail(GLM_FORMAT, "quantlab", "manifest is missing \"" + k + "\"");
    return it->second;
  }
  int as_int() const {
    if (kind != kNum || num != std::floor(num)) fail(GLM_FORMAT, "quantlab", "manifest field is not an integer");
    return static_cast<int>(num);
  }
  double as_num() const {
    if (kind != kNum) fail(GLM_FORMAT, "quantlab", "manifest field is not a number");
    return num;
  }
  const std::string& as_str() const {
    if (kind != kStr) fail(GLM_FORMAT, "quantlab", "manifest field is not a string");
    return str;
  }
};

class JsonParser {
 public:
  explicit JsonParser(const std::string& s) : s_(s) {}
  Json parse() {
    Json v = value();
    ws();
    if (i_ != s_.size()) bad("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void bad(const char* what) {
    fail(GLM_FORMAT, "quantlab", std::string("manifest.json: ") + what + " at offset " + std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
  }
  char peek() {
    ws();
    if (i_ >= s_.size()) bad("unexpected end");
    return s_[i_];
  }
  void expect(char c) {
    if (peek() != c) bad("unexpected character");
    ++i_;
  }
  Json value() {
    const char c = peek();
    Json v;
    if (c == '{') {
      v.kind = Json::kObj;
      ++i_;
      if (peek() == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        Json k = value();
        if (k.kind != Json::kStr) bad("object key is not a string");
        expect(':');
        v.obj[k.str] = value();
        if (peek() == ',') {
          ++i_;
          continue;
        }
        expect('}');
        return v;
      }
    }
    if (c == '[') {
      v.kind = Json::kArr;
      ++i_;
      if (peek() == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        if (peek() == ',') {
          ++i_;
          continue;
        }
        expect(']');
        return v;
      }
    }
    if (c == '"') {
      v.kind = Json::kStr;
      ++i_;
      while (i_ < s_.size() && s_[i_] != '"') {
        if (s_[i_] == '\\') {
          if (++i_ >= s_.size()) bad("bad escape");
          const char e = s_[i_];
          if (e == 'u') {  // \uXXXX: keep ASCII, replace the rest
            if (i_ + 4 >= s_.size()) bad("bad escape");
            const int code = std::stoi(s_.substr(i_ + 1, 4), nullptr, 16);
            v.str.push_back(code < 128 ? static_cast<char>(code) : '?');
            i_ += 4;
          } else {
            v.str.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e == 'b' ? '\b' : e == 'f' ? '\f' : e);
          }
        } else {
          v.str.push_back(s_[i_]);
        }
        ++i_;
      }
      if (i_ >= s_.size()) bad("unterminated string");
      ++i_;
      return v;
    }
    if (s_.compare(i_, 4, "true") == 0) {
      v.kind = Json::kBool;
      v.b = true;
      i_ += 4;
      return v;
    }
    if (s_.compare(i_, 5, "false") == 0) {
      v.kind = Json::kBool;
      i_ += 5;
      return v;
    }
    if (s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
      return v;
    }
    const size_t start = i_;
    while (i_ < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[i_])) || std::strchr("+-.eE", s_[i_]))) ++i_;
    if (start == i_) bad("unexpected character");
    v.kind = Json::kNum;
    try {
      v.num = std::stod(s_.substr(start, i_ - start));
    } catch (...) {
      bad("bad number");
    }
    return v;
  }
  const std::string& s_;
  size_t i_ = 0;
};

int axis_from(const std::string& s) {  // to_string(GroupAxis), quant.cpp
  if (s == "row") return GLM_AXIS_ROW;
  if (s == "column") return GLM_AXIS_COLUMN;
  if (s == "whole") return GLM_AXIS_WHOLE;
  fail(GLM_FORMAT, "quantlab", "unknown group axis \"" + s + "\"");
}

}  // namespace
}  // namespace glm

using namespace glm;

extern "C" glm_status glm_model_load_quantized(const char* dir, int max_batch, int max_ctx, int head_bf16,
                                               int tp_rank, int tp_size, glm_model** out) {
  return guarded([&] {
    if (!dir || !out) fail(GLM_CONTRACT, "quantlab", "null argument");
    *out = nullptr;
    const std::string root(dir);
    std::ifstream in(root + "/manifest.json");
    if (!in) fail(GLM_FORMAT, "quantlab", "missing manifest.json in " + root);
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    const Json man = JsonParser(text).parse();
    const Json& jc = man.at("config");
    glm_config cfg{};
    cfg.num_layers = jc.at("num_layers").as_int();
    cfg.hidden = jc.at("hidden").as_int();
    cfg.num_heads = jc.at("num_heads").as_int();
    cfg.ffn_hidden = jc.at("ffn_hidden").as_int();
    cfg.vocab = jc.at("vocab").as_int();
    cfg.init_method_std = jc.at("init_method_std").as_num();
    cfg.layernorm_eps = jc.at("layernorm_eps").as_num();
    cfg.deepnorm_alpha = jc.at("deepnorm_alpha").as_num();
    const Json& jp = man.at("policy");
    const int bits = jp.at("bits").as_int();
    const std::string scheme_s = jp.at("scheme").as_str();  // to_string(QuantScheme), quant.cpp
    if (scheme_s != "absmax" && scheme_s != "zeropoint") fail(GLM_FORMAT, "quantlab", "unknown quantization scheme \"" + scheme_s + "\"");
    const bool zp = scheme_s == "zeropoint";
    const int axis = axis_from(jp.at("axis").as_str());
    std::map<std::string, const Json*> by_name;
    for (const Json& e : man.at("matrices").arr) by_name[e.at("name").as_str()] = &e;

    // pass 1: every header, shape and file size, before any payload is read or device work
    // starts (GLM_FORMAT on malformed input without a GPU)
    const int64_t d = cfg.hidden, f = cfg.ffn_hidden, L = cfg.num_layers;
    const int64_t shapes[5][2] = {{d, 3 * d}, {d, d}, {d, f}, {d, f}, {f, d}};
    const char* names[5] = {"qkv", "out_proj", "ffn_w1", "ffn_v", "ffn_w2"};
    const char* vecs[4] = {"ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias"};
    const std::string emb_path = root + "/embedding.glmt";
    const GlmtHeader emb = read_glmt_header(emb_path);
    if (emb.dtype == 2 || emb.count() != static_cast<uint64_t>(cfg.vocab) * d)
      fail(GLM_FORMAT, "quantlab", "embedding.glmt must be f64 [vocab, hidden]");
    for (int64_t l = 0; l < L; ++l) {
      const std::string p = root + "/layer" + std::to_string(l) + ".";
      for (int w = 0; w < 5; ++w) {
        const std::string nm = "layer" + std::to_string(l) + "." + names[w];
        auto it = by_name.find(nm);
        if (it == by_name.end()) fail(GLM_FORMAT, "quantlab", "manifest has no matrix " + nm);
        const Json& e = *it->second;
        if (e.at("bits").as_int() != bits || e.at("scheme").as_str() != scheme_s ||
            axis_from(e.at("axis").as_str()) != axis)
          fail(GLM_FORMAT, "quantlab", nm + " does not follow the manifest policy");
        if (e.at("rows").as_int() != shapes[w][0] || e.at("cols").as_int() != shapes[w][1])
          fail(GLM_FORMAT, "quantlab", nm + " has the wrong shape for the configured model");
        const GlmtHeader c = read_glmt_header(p + names[w] + ".codes.glmt");
        const GlmtHeader sc = read_glmt_header(p + names[w] + ".scales.glmt");
        const int64_t n = shapes[w][0] * shapes[w][1];
        const int64_t pb = bits == 4 ? (n + 1) / 2 : n;
        const int64_t ng = axis == GLM_AXIS_ROW ? shapes[w][0] : axis == GLM_AXIS_COLUMN ? shapes[w][1] : 1;
        if (c.dtype != 2 || static_cast<int64_t>(c.count()) != pb)
          fail(GLM_FORMAT, "quantlab", nm + ".codes.glmt payload length does not match");
        if (sc.dtype != 0 || static_cast<int64_t>(sc.count()) != ng)
          fail(GLM_FORMAT, "quantlab", nm + ".scales.glmt group count does not match");
        if (zp) {  // write_quantized_matrix adds .zeros.glmt for zeropoint matrices (quant.cpp:380-386)
          const GlmtHeader z = read_glmt_header(p + names[w] + ".zeros.glmt");
          if (z.dtype != 0 || static_cast<int64_t>(z.count()) != ng)
            fail(GLM_FORMAT, "quantlab", nm + ".zeros.glmt group count does not match");
        }
      }
      for (int v = 0; v < 4; ++v) {
        const GlmtHeader h = read_glmt_header(p + vecs[v] + ".glmt");
        if (h.dtype == 2 || static_cast<int64_t>(h.count()) != d)
          fail(GLM_FORMAT, "quantlab", std::string("layer LN vector ") + vecs[v] + " must be f64 [hidden]");
      }
    }

    // pass 2: stream. One matrix of host memory at a time (GLM-130B: <= 403 MB of INT8 codes);
    // the model keeps only this rank's shard on the device; codes and scales are validated
    // like glm_qweight_create (INT4 -8 / INT8 -128 are not absmax codes, scales finite >= 0).
    glm_model* m = nullptr;
    glm_status s = glm_model_create(&cfg, bits, static_cast<glm_axis>(axis), max_batch, max_ctx, head_bf16, tp_rank,
                                    tp_size, &m);
    if (s != GLM_OK) fail(s, "glmmodel", glm_last_error());
    std::unique_ptr<glm_model, glm_status (*)(glm_model*)> guard(m, glm_model_destroy);
    auto check = [&](glm_status st) {
      if (st != GLM_OK) fail(st, "glmmodel", glm_last_error());
    };
    if (zp) check(glm_model_set_scheme(m, GLM_ZEROPOINT));
    {
      std::vector<double> rows;
      const uint64_t chunk = std::max<uint64_t>(1, (uint64_t{256} << 20) / (8 * static_cast<uint64_t>(d)));
      for (uint64_t r0 = 0; r0 < static_cast<uint64_t>(cfg.vocab); r0 += chunk) {
        const uint64_t nr = std::min<uint64_t>(chunk, cfg.vocab - r0);
        read_glmt_rows(emb_path, emb, r0, nr, d, rows);
        check(glm_model_set_embedding_rows(m, static_cast<int64_t>(r0), static_cast<int64_t>(nr), rows.data()));
      }
    }
    for (int64_t l = 0; l < L; ++l) {
      const std::string p = root + "/layer" + std::to_string(l) + ".";
      for (int w = 0; w < 5; ++w) {
        const Glmt c = read_glmt(p + names[w] + ".codes.glmt");
        const Glmt sc = read_glmt(p + names[w] + ".scales.glmt");
        validate_absmax_payload(c.i8.data(), static_cast<int64_t>(c.i8.size()), shapes[w][0] * shapes[w][1], bits);
        if (zp) {
          const Glmt z = read_glmt(p + names[w] + ".zeros.glmt");
          check(glm_model_set_quantized_zp(m, static_cast<int>(l), w, c.i8.data(), static_cast<int64_t>(c.i8.size()),
                                           sc.f64.data(), z.f64.data(), static_cast<int64_t>(sc.f64.size())));
        } else {
          check(glm_model_set_quantized(m, static_cast<int>(l), w, c.i8.data(), static_cast<int64_t>(c.i8.size()),
                                        sc.f64.data(), static_cast<int64_t>(sc.f64.size())));
        }
      }
      for (int v = 0; v < 4; ++v) {
        const Glmt t = read_glmt(p + vecs[v] + ".glmt");
        check(glm_model_set_tensor(m, static_cast<int>(l), 5 + v, t.f64.data()));
      }
    }
    *out = guard.release();
  });
}
