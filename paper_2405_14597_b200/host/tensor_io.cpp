// QTNS container and JSON sidecars for the C++ drop-in layer.
//
// Byte layout, validation order and error types follow tensor_io.cpp:142-303 and
// quantize.cpp:175-270 (pinned by test_tensor_io.cpp:64-226 and
// test_quantize.cpp:284-328, transcribed in tests/cpp/test_api.cpp). The sidecar
// is written in the reference's key order and 2-space layout; the reader is a
// small strict JSON parser (the reference uses nlohmann::json; this library has no
// third-party dependencies).
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/intscale/quantize.hpp"
#include "../../include/intscale/tensor_io.hpp"

namespace intscale {
namespace {

constexpr std::uint64_t kMaxDim = std::uint64_t{1} << 32;       // tensor_io.cpp:15
constexpr std::uint64_t kMaxElements = std::uint64_t{1} << 40;  // tensor_io.cpp:16

void put_le(std::vector<std::uint8_t>& out, std::uint64_t v, int bytes) {
  for (int b = 0; b < bytes; ++b) out.push_back(static_cast<std::uint8_t>(v >> (8 * b)));
}

std::uint64_t get_le(const std::uint8_t* p, int bytes) {
  std::uint64_t v = 0;
  for (int b = 0; b < bytes; ++b) v |= std::uint64_t{p[b]} << (8 * b);
  return v;
}

std::vector<std::uint8_t> slurp(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path.string());
  std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(in)),
                                  std::istreambuf_iterator<char>());
  if (in.bad()) throw IoError("read failed on " + path.string());
  return bytes;
}

void spit(const std::filesystem::path& path, const std::vector<std::uint8_t>& bytes) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open " + path.string() + " for writing");
  out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
  if (!out) throw IoError("write failed on " + path.string());
}

Index require_rows(const TensorHeader& h) { return h.dims.size() == 1 ? 1 : static_cast<Index>(h.dims[0]); }
Index require_cols(const TensorHeader& h) { return static_cast<Index>(h.dims.back()); }

// ------------------------------------------------------------------ minimal JSON
struct Json {
  enum Kind { null, boolean, number, string, array, object } kind = null;
  double num = 0;
  bool integral = false;
  std::int64_t inum = 0;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;

  const Json& at(const std::string& key) const {
    if (kind != object) throw FormatError("expected an object");
    auto it = obj.find(key);
    if (it == obj.end()) throw FormatError("missing key '" + key + "'");
    return it->second;
  }
  std::int64_t as_int() const {
    if (kind != number || !integral) throw FormatError("expected an integer");
    return inum;
  }
  double as_double() const {
    if (kind != number) throw FormatError("expected a number");
    return num;
  }
  const std::string& as_string() const {
    if (kind != string) throw FormatError("expected a string");
    return str;
  }
  const std::vector<Json>& as_array() const {
    if (kind != array) throw FormatError("expected an array");
    return arr;
  }
};

struct Parser {
  const std::string& s;
  std::size_t i = 0;

  [[noreturn]] void fail(const std::string& what) const {
    throw FormatError(what + " at offset " + std::to_string(i));
  }
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\r' || s[i] == '\t')) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < s.size() && s[i] == c) return ++i, true;
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  bool word(const char* w) {
    const std::size_t n = std::strlen(w);
    if (s.compare(i, n, w) == 0) return i += n, true;
    return false;
  }
  std::string string_lit() {
    expect('"');
    std::string out;
    while (i < s.size() && s[i] != '"') {
      char c = s[i++];
      if (c == '\\') {
        if (i >= s.size()) fail("bad escape");
        const char e = s[i++];
        const char* map = "\"\"\\\\//b\bf\fn\nr\rt\t";
        const char* hit = nullptr;
        for (const char* m = map; *m; m += 2)
          if (*m == e) hit = m;
        if (!hit) fail("unsupported escape");
        c = hit[1];
      }
      out.push_back(c);
    }
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
  Json value() {
    ws();
    if (i >= s.size()) fail("unexpected end");
    Json v;
    const char c = s[i];
    if (c == '{') {
      ++i;
      v.kind = Json::object;
      if (eat('}')) return v;
      do {
        ws();
        std::string key = string_lit();
        expect(':');
        v.obj[key] = value();
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++i;
      v.kind = Json::array;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = Json::string;
      v.str = string_lit();
    } else if (word("true") || word("false")) {
      v.kind = Json::boolean;
    } else if (word("null")) {
      v.kind = Json::null;
    } else {
      const std::size_t start = i;
      while (i < s.size() && std::strchr("+-0123456789.eE", s[i])) ++i;
      if (start == i) fail("unexpected character");
      v.kind = Json::number;
      const char* b = s.data() + start;
      const char* e = s.data() + i;
      if (std::from_chars(b, e, v.num).ptr != e) fail("bad number");
      v.integral = std::from_chars(b, e, v.inum).ptr == e;
    }
    return v;
  }
};

std::string json_double(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eE") == std::string::npos && std::isfinite(v)) s += ".0";
  return s;
}

}  // namespace

// ------------------------------------------------------------------ header
std::uint64_t TensorHeader::element_count() const {
  std::uint64_t n = 1;
  for (auto d : dims) n *= d;
  return n;
}

std::size_t TensorHeader::payload_bytes() const {
  const std::uint64_t n = element_count();
  switch (dtype) {
    case DType::real32: return static_cast<std::size_t>(n * 4);
    case DType::signed8: return static_cast<std::size_t>(n);
    case DType::packed_signed4: return static_cast<std::size_t>((n + 1) / 2);
  }
  throw FormatError("unknown dtype");
}

std::vector<std::uint8_t> encode_header(const TensorHeader& h) {  // tensor_io.cpp:142-150
  std::vector<std::uint8_t> out(TensorHeader::kMagic, TensorHeader::kMagic + 4);
  put_le(out, h.version, 2);
  out.push_back(static_cast<std::uint8_t>(h.dtype));
  out.push_back(static_cast<std::uint8_t>(h.dims.size()));
  for (auto d : h.dims) put_le(out, d, 8);
  return out;
}

TensorHeader decode_header(const std::vector<std::uint8_t>& bytes, std::size_t& offset) {
  // tensor_io.cpp:152-177
  if (bytes.size() < offset + 8) throw FormatError("header truncated");
  const std::uint8_t* p = bytes.data() + offset;
  if (std::memcmp(p, TensorHeader::kMagic, 4) != 0) throw FormatError("bad magic, not a QTNS file");
  TensorHeader h;
  h.version = static_cast<std::uint16_t>(get_le(p + 4, 2));
  if (h.version != TensorHeader::kVersion)
    throw FormatError("unsupported version " + std::to_string(h.version));
  if (p[6] > 2) throw FormatError("unknown dtype code " + std::to_string(p[6]));
  h.dtype = static_cast<DType>(p[6]);
  const int ndim = p[7];
  if (ndim != 1 && ndim != 2) throw FormatError("ndim must be 1 or 2, got " + std::to_string(ndim));
  if (bytes.size() < offset + 8 + 8 * static_cast<std::size_t>(ndim)) throw FormatError("header truncated");
  std::uint64_t count = 1;
  for (int d = 0; d < ndim; ++d) {
    const std::uint64_t v = get_le(p + 8 + 8 * d, 8);
    if (v == 0) throw FormatError("zero dimension");
    if (v > kMaxDim) throw FormatError("dimension too large");
    count *= v;
    if (count > kMaxElements) throw FormatError("tensor too large");
    h.dims.push_back(v);
  }
  offset += 8 + 8 * static_cast<std::size_t>(ndim);
  return h;
}

// ------------------------------------------------------------------ tensors
TensorData read_tensor(const std::filesystem::path& path) {  // tensor_io.cpp:210-256
  const auto bytes = slurp(path);
  std::size_t off = 0;
  const TensorHeader h = decode_header(bytes, off);
  const std::size_t need = h.payload_bytes();
  if (bytes.size() - off < need) throw LengthError("payload truncated in " + path.string());
  if (bytes.size() - off > need) throw LengthError("trailing bytes after payload in " + path.string());
  const Index rows = require_rows(h), cols = require_cols(h);
  const std::uint8_t* p = bytes.data() + off;
  if (h.dtype == DType::real32) {
    MatF x(rows, cols);
    for (Index i = 0; i < x.size(); ++i) {
      const std::uint32_t bits = static_cast<std::uint32_t>(get_le(p + 4 * i, 4));
      float f;
      std::memcpy(&f, &bits, 4);
      if (!std::isfinite(f)) throw ValueError("non-finite value at element " + std::to_string(i));
      x.data()[i] = f;
    }
    return x;
  }
  QuantizedPayload q;
  if (h.dtype == DType::signed8) {
    q.bit_width = 8;
    q.values.resize(rows, cols);
    for (Index i = 0; i < q.values.size(); ++i) q.values.data()[i] = static_cast<std::int8_t>(p[i]);
  } else {
    q.bit_width = 4;
    q.values = unpack_signed4(std::vector<std::uint8_t>(p, p + need), rows, cols);
  }
  return q;
}

MatF read_float_tensor(const std::filesystem::path& path) {
  auto data = read_tensor(path);
  if (auto* x = std::get_if<MatF>(&data)) return std::move(*x);
  throw FormatError(path.string() + " holds integer codes, expected real32");
}

void write_tensor(const MatF& x, const std::filesystem::path& path) {  // tensor_io.cpp:264-279
  if (x.rows() < 1 || x.cols() < 1) throw ParamError("empty tensor");
  TensorHeader h;
  h.dtype = DType::real32;
  h.dims = {static_cast<std::uint64_t>(x.rows()), static_cast<std::uint64_t>(x.cols())};
  auto out = encode_header(h);
  for (Index i = 0; i < x.size(); ++i) {
    const float f = x.data()[i];
    if (!std::isfinite(f)) throw ValueError("refusing to write non-finite value at element " + std::to_string(i));
    std::uint32_t bits;
    std::memcpy(&bits, &f, 4);
    put_le(out, bits, 4);
  }
  spit(path, out);
}

void write_tensor(const MatQ& values, DType dtype, const std::filesystem::path& path) {
  // tensor_io.cpp:281-303
  if (dtype == DType::real32) throw ParamError("integer overload cannot write real32");
  if (values.rows() < 1 || values.cols() < 1) throw ParamError("empty tensor");
  TensorHeader h;
  h.dtype = dtype;
  h.dims = {static_cast<std::uint64_t>(values.rows()), static_cast<std::uint64_t>(values.cols())};
  auto out = encode_header(h);
  if (dtype == DType::signed8) {
    for (Index i = 0; i < values.size(); ++i) {
      const std::int16_t v = values.data()[i];
      if (v < -128 || v > 127) throw ValueError("value " + std::to_string(v) + " outside signed 8-bit range");
      out.push_back(static_cast<std::uint8_t>(v));
    }
  } else {
    for (Index i = 0; i < values.size(); ++i)
      if (values.data()[i] < -8 || values.data()[i] > 7)
        throw ValueError("value " + std::to_string(values.data()[i]) + " outside signed 4-bit range");
    const auto packed = pack_signed4(values);
    out.insert(out.end(), packed.begin(), packed.end());
  }
  spit(path, out);
}

// ------------------------------------------------------------------ names
std::string to_string(Scheme s) { return s == Scheme::symmetric ? "symmetric" : "asymmetric"; }

std::string to_string(GranKind k) {
  switch (k) {
    case GranKind::per_tensor: return "per_tensor";
    case GranKind::per_token: return "per_token";
    case GranKind::per_channel: return "per_channel";
    case GranKind::group: return "group";
  }
  throw ParamError("unknown granularity");
}

Scheme scheme_from_string(const std::string& s) {  // quantize.cpp:70-74
  if (s == "symmetric") return Scheme::symmetric;
  if (s == "asymmetric") return Scheme::asymmetric;
  throw ParamError("unknown scheme '" + s + "'");
}

GranKind gran_kind_from_string(const std::string& s) {  // quantize.cpp:76-82
  if (s == "per_tensor" || s == "tensor") return GranKind::per_tensor;
  if (s == "per_token" || s == "token") return GranKind::per_token;
  if (s == "per_channel" || s == "channel") return GranKind::per_channel;
  if (s == "group") return GranKind::group;
  throw ParamError("unknown granularity '" + s + "'");
}

// ------------------------------------------------------------------ sidecars
void write_quantized(const QuantizedTensor& q, const std::filesystem::path& values_path) {
  // quantize.cpp:194-220; unsigned codes stored as their two's-complement fold
  const int bits = q.params.bit_width;
  MatQ stored = q.values;
  if (q.params.scheme == Scheme::asymmetric)
    for (Index i = 0; i < stored.size(); ++i) {
      auto& v = stored.data()[i];
      if (v >= (1 << (bits - 1))) v = static_cast<std::int16_t>(v - (1 << bits));
    }
  write_tensor(stored, bits == 4 ? DType::packed_signed4 : DType::signed8, values_path);

  std::string js = "{\n  \"bit_width\": " + std::to_string(bits) + ",\n  \"scheme\": \"" +
                   to_string(q.params.scheme) + "\",\n  \"granularity\": {\n    \"kind\": \"" +
                   to_string(q.params.granularity.kind) + "\",\n    \"group_size\": " +
                   std::to_string(q.params.granularity.group_size) + "\n  },\n  \"scales\": ";
  auto list = [&](Index n, auto&& item) {
    if (n == 0) return std::string("[]");
    std::string s = "[\n";
    for (Index i = 0; i < n; ++i) s += "    " + item(i) + (i + 1 < n ? ",\n" : "\n");
    return s + "  ]";
  };
  js += list(q.params.scales.size(), [&](Index i) { return json_double(q.params.scales[i]); });
  js += ",\n  \"zero_points\": ";
  js += list(q.params.zero_points.size(), [&](Index i) { return std::to_string(q.params.zero_points[i]); });
  js += "\n}\n";
  std::filesystem::path side = values_path;
  side += ".json";
  spit(side, std::vector<std::uint8_t>(js.begin(), js.end()));
}

QuantizedTensor read_quantized(const std::filesystem::path& values_path) {  // quantize.cpp:222-270
  TensorData data = read_tensor(values_path);
  auto* payload = std::get_if<QuantizedPayload>(&data);
  if (!payload) throw FormatError(values_path.string() + " holds real values, expected codes");
  std::filesystem::path side_path = values_path;
  side_path += ".json";
  std::ifstream f(side_path);
  if (!f) throw IoError("cannot open sidecar " + side_path.string());
  const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());

  QuantizedTensor q;
  std::string scheme, kind;
  try {
    Parser p{text};
    const Json side = p.value();
    p.ws();
    if (p.i != text.size()) p.fail("trailing characters");
    q.params.bit_width = static_cast<int>(side.at("bit_width").as_int());
    scheme = side.at("scheme").as_string();
    const Json& gran = side.at("granularity");
    kind = gran.at("kind").as_string();
    q.params.granularity.group_size = gran.at("group_size").as_int();
    const auto& sc = side.at("scales").as_array();
    q.params.scales.resize(static_cast<Index>(sc.size()));
    for (std::size_t i = 0; i < sc.size(); ++i) q.params.scales[static_cast<Index>(i)] = sc[i].as_double();
    const auto& zp = side.at("zero_points").as_array();
    q.params.zero_points.resize(static_cast<Index>(zp.size()));
    for (std::size_t i = 0; i < zp.size(); ++i)
      q.params.zero_points[static_cast<Index>(i)] = static_cast<std::int32_t>(zp[i].as_int());
  } catch (const FormatError& e) {
    throw FormatError("bad sidecar " + side_path.string() + ": " + e.what());
  }
  q.params.scheme = scheme_from_string(scheme);
  q.params.granularity.kind = gran_kind_from_string(kind);
  if (q.params.bit_width != 4 && q.params.bit_width != 8)
    throw ParamError("bit width must be 4 or 8, got " + std::to_string(q.params.bit_width));
  if (q.params.bit_width != payload->bit_width)
    throw FormatError("sidecar bit width disagrees with container dtype");
  q.values = std::move(payload->values);
  if (q.params.scheme == Scheme::asymmetric)  // unfold_unsigned, quantize.cpp:186-190
    for (Index i = 0; i < q.values.size(); ++i) {
      auto& v = q.values.data()[i];
      if (v < 0) v = static_cast<std::int16_t>(v + (1 << q.params.bit_width));
    }
  q.params.granularity.validate(q.rows(), q.cols());
  if (q.params.scales.size() != q.params.granularity.unit_count(q.rows(), q.cols()))
    throw FormatError("sidecar scale count does not match shape");
  if (q.params.scheme == Scheme::asymmetric && q.params.zero_points.size() != q.params.scales.size())
    throw FormatError("sidecar zero point count does not match scale count");
  return q;
}

}  // namespace intscale
