// nolf_load.h -- native reader of the reference's ``.nolf`` asset container
// (assetio.py:1-7 container, 30-66 section table, 85-158 meta + arrays,
// 174-255 read_asset), host code compiled into libnolf_b200.so.
//
// Container: "NOLF", <HH version, count>, then per section name[16] + <QQI
// (offset, length, crc32)>, then the raw little-endian section bytes; array
// shapes and scalars live in the JSON ``meta`` section.  Gzip-compressed
// files are accepted (zlib).  Every failure is a DataError-class status
// (NOLF_EDATA) with a message, like assetio.read_asset.
#pragma once

#include <zlib.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace nolf_load {

// ---------------------------------------------------------------- JSON (the meta schema only needs
// objects, arrays, numbers, strings, true/false/null)
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;

  const Json *get(const char *k) const {
    if (kind != Obj) return nullptr;
    auto it = obj.find(k);
    return it == obj.end() ? nullptr : &it->second;
  }
};

class JsonParser {
 public:
  JsonParser(const char *s, size_t n) : p_(s), e_(s + n) {}
  bool parse(Json &out) {
    if (!value(out)) return false;
    ws();
    return p_ == e_;
  }

 private:
  const char *p_, *e_;
  int depth_ = 0;
  static constexpr int kMaxDepth = 64;     // the meta schema nests 4 deep; bound the recursion
  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }
  bool lit(const char *w) {
    const size_t n = strlen(w);
    if ((size_t)(e_ - p_) < n || memcmp(p_, w, n) != 0) return false;
    p_ += n;
    return true;
  }
  bool string(std::string &s) {
    if (p_ >= e_ || *p_ != '"') return false;
    ++p_;
    while (p_ < e_ && *p_ != '"') {
      if (*p_ == '\\') {
        if (++p_ >= e_) return false;
        const char c = *p_++;
        switch (c) {
          case 'n': s += '\n'; break;
          case 't': s += '\t'; break;
          case 'r': s += '\r'; break;
          case 'b': s += '\b'; break;
          case 'f': s += '\f'; break;
          case 'u': {                       // names are ASCII; keep BMP code points as UTF-8
            if (e_ - p_ < 4) return false;
            unsigned v = (unsigned)strtoul(std::string(p_, 4).c_str(), nullptr, 16);
            p_ += 4;
            if (v < 0x80) s += (char)v;
            else if (v < 0x800) { s += (char)(0xC0 | (v >> 6)); s += (char)(0x80 | (v & 0x3F)); }
            else { s += (char)(0xE0 | (v >> 12)); s += (char)(0x80 | ((v >> 6) & 0x3F)); s += (char)(0x80 | (v & 0x3F)); }
            break;
          }
          default: s += c;
        }
      } else {
        s += *p_++;
      }
    }
    if (p_ >= e_) return false;
    ++p_;
    return true;
  }
  bool value(Json &v) {
    if (++depth_ > kMaxDepth) return false;
    const bool ok = value_in(v);
    --depth_;
    return ok;
  }
  bool value_in(Json &v) {
    ws();
    if (p_ >= e_) return false;
    const char c = *p_;
    if (c == '{') {
      ++p_;
      v.kind = Json::Obj;
      ws();
      if (p_ < e_ && *p_ == '}') { ++p_; return true; }
      for (;;) {
        ws();
        std::string k;
        if (!string(k)) return false;
        ws();
        if (p_ >= e_ || *p_++ != ':') return false;
        if (!value(v.obj[k])) return false;
        ws();
        if (p_ < e_ && *p_ == ',') { ++p_; continue; }
        if (p_ < e_ && *p_ == '}') { ++p_; return true; }
        return false;
      }
    }
    if (c == '[') {
      ++p_;
      v.kind = Json::Arr;
      ws();
      if (p_ < e_ && *p_ == ']') { ++p_; return true; }
      for (;;) {
        v.arr.emplace_back();
        if (!value(v.arr.back())) return false;
        ws();
        if (p_ < e_ && *p_ == ',') { ++p_; continue; }
        if (p_ < e_ && *p_ == ']') { ++p_; return true; }
        return false;
      }
    }
    if (c == '"') { v.kind = Json::Str; return string(v.str); }
    if (lit("true")) { v.kind = Json::Bool; v.b = true; return true; }
    if (lit("false")) { v.kind = Json::Bool; v.b = false; return true; }
    if (lit("null")) { v.kind = Json::Null; return true; }
    if (lit("NaN")) { v.kind = Json::Num; v.num = NAN; return true; }           // Python json.dumps
    if (lit("Infinity")) { v.kind = Json::Num; v.num = INFINITY; return true; }
    if (lit("-Infinity")) { v.kind = Json::Num; v.num = -INFINITY; return true; }
    // number: strtod on the exact token (Python's repr round-trips)
    const char *q = p_;
    while (q < e_ && (strchr("+-0123456789.eE", *q) != nullptr)) ++q;
    if (q == p_) return false;
    std::string tok(p_, q);
    char *end = nullptr;
    v.kind = Json::Num;
    v.num = strtod(tok.c_str(), &end);
    if (end != tok.c_str() + tok.size()) return false;
    p_ = q;
    return true;
  }
};

// ---------------------------------------------------------------- container
struct Container {
  std::vector<uint8_t> raw;                                  // decompressed file
  std::map<std::string, std::pair<size_t, size_t>> sections;  // name -> (offset, length)
  Json meta;
};

inline bool gunzip(const uint8_t *src, size_t n, std::vector<uint8_t> &out, std::string &err) {
  z_stream zs;
  memset(&zs, 0, sizeof zs);
  if (inflateInit2(&zs, 16 + MAX_WBITS) != Z_OK) { err = "zlib init failed"; return false; }
  zs.next_in = const_cast<Bytef *>(src);
  zs.avail_in = (uInt)n;
  out.clear();
  std::vector<uint8_t> buf(1 << 20);
  int rc;
  do {
    zs.next_out = buf.data();
    zs.avail_out = (uInt)buf.size();
    rc = inflate(&zs, Z_NO_FLUSH);
    if (rc != Z_OK && rc != Z_STREAM_END) {
      inflateEnd(&zs);
      err = "corrupt gzip stream";
      return false;
    }
    out.insert(out.end(), buf.data(), buf.data() + (buf.size() - zs.avail_out));
  } while (rc != Z_STREAM_END);
  inflateEnd(&zs);
  return true;
}

// assetio.py:48-66 (unpack_sections): magic, version, bounds, crc32.
inline bool parse_container(std::vector<uint8_t> data, Container &c, std::string &err) {
  if (data.size() >= 2 && data[0] == 0x1f && data[1] == 0x8b) {
    std::vector<uint8_t> out;
    if (!gunzip(data.data(), data.size(), out, err)) return false;
    data.swap(out);
  }
  c.raw.swap(data);
  const std::vector<uint8_t> &d = c.raw;
  if (d.size() < 4 || memcmp(d.data(), "NOLF", 4) != 0) { err = "not an asset file (bad magic)"; return false; }
  if (d.size() < 8) { err = "asset header truncated"; return false; }
  uint16_t version, count;
  memcpy(&version, d.data() + 4, 2);
  memcpy(&count, d.data() + 6, 2);
  if (version != 1) { err = "unsupported asset version " + std::to_string(version); return false; }
  size_t pos = 8;
  for (int i = 0; i < count; ++i) {
    if (pos + 16 + 20 > d.size()) { err = "section table truncated"; return false; }
    char name[17] = {0};
    memcpy(name, d.data() + pos, 16);
    uint64_t off, len;
    uint32_t crc;
    memcpy(&off, d.data() + pos + 16, 8);
    memcpy(&len, d.data() + pos + 24, 8);
    memcpy(&crc, d.data() + pos + 32, 4);
    pos += 36;
    if (off > d.size() || len > d.size() - off) { err = std::string("section ") + name + " truncated"; return false; }
    if ((uint32_t)crc32(0L, d.data() + off, (uInt)len) != crc) {
      err = std::string("section ") + name + " failed its checksum";
      return false;
    }
    c.sections[name] = {(size_t)off, (size_t)len};
  }
  auto it = c.sections.find("meta");
  if (it == c.sections.end()) { err = "bad asset meta section: missing"; return false; }
  JsonParser jp(reinterpret_cast<const char *>(d.data() + it->second.first), it->second.second);
  if (!jp.parse(c.meta) || c.meta.kind != Json::Obj) { err = "bad asset meta section: invalid JSON"; return false; }
  return true;
}

// A typed view of one section with its element count checked (assetio.py:68-74).
template <class T>
inline const T *section(const Container &c, const std::string &name, size_t expect, std::string &err) {
  auto it = c.sections.find(name);
  if (it == c.sections.end()) { err = "missing section " + name; return nullptr; }
  if (it->second.second != expect * sizeof(T)) {
    err = "section " + name + " has " + std::to_string(it->second.second / sizeof(T)) + " elements, expected " +
          std::to_string(expect);
    return nullptr;
  }
  if (expect == 0) return reinterpret_cast<const T *>(c.raw.data());   // valid, never dereferenced
  return reinterpret_cast<const T *>(c.raw.data() + it->second.first);  // file offsets are not aligned:
}                                                                        // callers copy (see aligned())

// Section bytes copied into aligned storage (offsets in the file are arbitrary).
template <class T>
inline bool aligned(const Container &c, const std::string &name, size_t expect, std::vector<T> &out,
                    std::string &err) {
  const T *p = section<T>(c, name, expect, err);
  if (!p) return false;
  out.resize(expect);
  if (expect) memcpy(out.data(), p, expect * sizeof(T));
  return true;
}

inline bool num(const Json *j, double &v) {
  if (!j || j->kind != Json::Num) return false;
  v = j->num;
  return true;
}
inline bool inum(const Json *j, int64_t &v) {
  double d;
  if (!num(j, d) || d != std::floor(d)) return false;
  v = (int64_t)d;
  return true;
}
inline bool flag(const Json *j, bool dflt) {
  if (!j) return dflt;
  if (j->kind == Json::Bool) return j->b;
  if (j->kind == Json::Num) return j->num != 0.0;
  return dflt;
}

}  // namespace nolf_load
