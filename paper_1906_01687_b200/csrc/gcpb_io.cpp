// gcpb_io.cpp — tensor files for the device engine (host side of §8f item 3).
//
// read_tns follows the reference's text format and error behaviour
// (src/io.cpp:75-139) but parses in parallel: the file is memory-mapped, the
// prologue (comments, the '#shape:' header, the first entry that fixes d) is
// walked serially, and the rest is split at line boundaries across threads,
// each producing its slice of the entries in file order.  Files whose shape
// header is not in the prologue (a header after data, or several headers) are
// parsed serially by the same state machine, so the unusual cases keep the
// reference's exact semantics.  The first error in file order is reported
// with its 1-based line number.
//
// The binary "GCPBCOO1" format is this framework's own: a fixed header, the
// dims, the coordinates (u32 when every extent fits, else i64) and the f64
// values, read with mmap and widened in parallel — the fast path for feeding
// large tensors to gcpb_set_sparse.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gcpb.h"

namespace gcpb {
void set_global_error(const std::string& msg);
}

namespace {

constexpr int kMaxModes = 16;

struct io_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] void fail(const std::string& path, const std::string& msg) {
  throw io_error(path + ": " + msg);
}

template <typename F>
int io_guard(F&& f) {
  try {
    f();
    return GCPB_OK;
  } catch (const std::invalid_argument& e) {
    gcpb::set_global_error(e.what());
    return GCPB_ERR_USAGE;
  } catch (const std::out_of_range& e) {
    gcpb::set_global_error(e.what());
    return GCPB_ERR_RANGE;
  } catch (const std::bad_alloc&) {
    gcpb::set_global_error("out of host memory");
    return GCPB_ERR_RUNTIME;
  } catch (const std::exception& e) {
    gcpb::set_global_error(e.what());
    return GCPB_ERR_RUNTIME;
  }
}

// Read-only mapping of a whole file (empty files map to an empty range).
struct Mapped {
  const char* p = nullptr;
  size_t n = 0;
  int fd = -1;
  explicit Mapped(const std::string& path) {
    fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) fail(path, "cannot open for reading");
    struct stat st {};
    if (::fstat(fd, &st) != 0) fail(path, "read error");
    n = static_cast<size_t>(st.st_size);
    if (n > 0) {
      void* m = ::mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
      if (m == MAP_FAILED) fail(path, "read error");
      ::madvise(m, n, MADV_SEQUENTIAL);
      p = static_cast<const char*>(m);
    }
  }
  ~Mapped() {
    if (p) ::munmap(const_cast<char*>(p), n);
    if (fd >= 0) ::close(fd);
  }
  Mapped(const Mapped&) = delete;
  Mapped& operator=(const Mapped&) = delete;
};

int pick_threads(int threads) {
  if (threads > 0) return threads;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? static_cast<int>(std::min(h, 64u)) : 1;
}

// istringstream >> tokenisation splits on the C locale's isspace set.
inline bool is_ws(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

struct Token {
  const char* b;
  const char* e;
  std::string str() const { return std::string(b, e); }
};

// strtoll / strtod on a NUL-terminated copy: the same accept/reject rules
// as the reference's parse_int / parse_double (io.cpp:42-59).
bool parse_int(const Token& t, int64_t* out) {
  const size_t len = static_cast<size_t>(t.e - t.b);
  // fast path: plain decimal digits that cannot overflow
  if (len > 0 && len <= 18) {
    int64_t v = 0;
    const char* c = t.b;
    for (; c < t.e && *c >= '0' && *c <= '9'; ++c) v = v * 10 + (*c - '0');
    if (c == t.e) {
      *out = v;
      return true;
    }
  }
  char sbuf[64];
  std::string big;
  const char* s;
  if (len < sizeof(sbuf)) {
    std::memcpy(sbuf, t.b, len);
    sbuf[len] = '\0';
    s = sbuf;
  } else {
    big.assign(t.b, len);
    s = big.c_str();
  }
  errno = 0;
  char* end = nullptr;
  const long long v = std::strtoll(s, &end, 10);
  if (errno != 0 || end == s || *end != '\0') return false;
  *out = v;
  return true;
}

bool parse_double(const Token& t, double* out) {
  const size_t len = static_cast<size_t>(t.e - t.b);
  char sbuf[128];
  std::string big;
  const char* s;
  if (len < sizeof(sbuf)) {
    std::memcpy(sbuf, t.b, len);
    sbuf[len] = '\0';
    s = sbuf;
  } else {
    big.assign(t.b, len);
    s = big.c_str();
  }
  char* end = nullptr;
  const double v = std::strtod(s, &end);
  if (end == s || *end != '\0') return false;
  *out = v;
  return true;
}

// Parser state shared by the serial prologue and every chunk.
struct TnsState {
  int d = -1;
  std::vector<int64_t> header;  // declared extents (may be empty)
};

struct TnsOut {
  std::vector<int64_t> coords;   // row-major, `dl` entries per line
  std::vector<int> line_d;       // per-entry mode count when it varies (serial path)
  std::vector<double> values;
  int64_t maxima[kMaxModes];
  int maxima_n = 0;
  int64_t lines = 0;             // lines consumed
  bool has_err = false;
  int64_t err_line = 0;          // 1-based, relative to the chunk start
  std::string err_msg;
  bool saw_header = false;       // a '#shape:' line inside a parallel chunk
};

enum class LineResult { kOk, kError, kHeaderInChunk };

// One line (without its '\n') of the reference's read loop (io.cpp:86-129).
LineResult parse_line(const char* b, const char* e, TnsState& st, TnsOut& out, bool allow_header,
                      std::vector<Token>& tok) {
  const size_t len = static_cast<size_t>(e - b);
  if (len >= 7 && std::memcmp(b, "#shape:", 7) == 0) {
    if (!allow_header) return LineResult::kHeaderInChunk;
    tok.clear();
    for (const char* c = b + 7; c < e;) {
      while (c < e && is_ws(*c)) ++c;
      if (c == e) break;
      const char* t0 = c;
      while (c < e && !is_ws(*c)) ++c;
      tok.push_back({t0, c});
    }
    if (tok.empty()) {
      out.err_msg = "empty shape header";
      return LineResult::kError;
    }
    for (const Token& t : tok) {
      int64_t n = 0;
      if (!parse_int(t, &n)) {
        out.err_msg = "expected an integer, got '" + t.str() + "'";
        return LineResult::kError;
      }
      if (n < 1) {
        out.err_msg = "shape extent must be >= 1";
        return LineResult::kError;
      }
      st.header.push_back(n);
    }
    st.d = static_cast<int>(st.header.size());
    out.saw_header = true;
    return LineResult::kOk;
  }
  const char* f = b;
  while (f < e && (*f == ' ' || *f == '\t' || *f == '\r')) ++f;
  if (f == e || *f == '#') return LineResult::kOk;
  tok.clear();
  for (const char* c = b; c < e;) {
    while (c < e && is_ws(*c)) ++c;
    if (c == e) break;
    const char* t0 = c;
    while (c < e && !is_ws(*c)) ++c;
    tok.push_back({t0, c});
  }
  if (st.d < 0) {
    if (tok.size() < 2) {
      out.err_msg = "expected indices and a value";
      return LineResult::kError;
    }
    st.d = static_cast<int>(tok.size()) - 1;
  }
  const int d = st.d;
  if (tok.size() != static_cast<size_t>(d) + 1) {
    out.err_msg = "expected " + std::to_string(d + 1) + " tokens, got " + std::to_string(tok.size());
    return LineResult::kError;
  }
  const size_t at = out.coords.size();
  out.coords.resize(at + static_cast<size_t>(d));
  int64_t* idx = out.coords.data() + at;
  for (int k = 0; k < d; ++k) {
    int64_t v = 0;
    if (!parse_int(tok[static_cast<size_t>(k)], &v)) {
      out.coords.resize(at);
      out.err_msg = "expected an integer, got '" + tok[static_cast<size_t>(k)].str() + "'";
      return LineResult::kError;
    }
    if (v < 1) {
      out.coords.resize(at);
      out.err_msg = "indices are 1-based, got " + std::to_string(v);
      return LineResult::kError;
    }
    if (!st.header.empty() && k < static_cast<int>(st.header.size()) &&
        v > st.header[static_cast<size_t>(k)]) {
      out.coords.resize(at);
      out.err_msg = "index " + std::to_string(v) + " exceeds declared extent " +
                    std::to_string(st.header[static_cast<size_t>(k)]) + " in mode " +
                    std::to_string(k + 1);
      return LineResult::kError;
    }
    idx[k] = v - 1;
  }
  double val = 0.0;
  if (!parse_double(tok.back(), &val)) {
    out.coords.resize(at);
    out.err_msg = "expected a number, got '" + tok.back().str() + "'";
    return LineResult::kError;
  }
  out.values.push_back(val);
  if (allow_header) out.line_d.push_back(d);  // d can only change in the serial walk
  // maxima over the first min(d, 16) modes, starting at 1 (io.cpp:124-128)
  const int md = std::min(d, kMaxModes);
  while (out.maxima_n < md) out.maxima[out.maxima_n++] = 1;
  for (int k = 0; k < md; ++k) out.maxima[k] = std::max(out.maxima[k], idx[k] + 1);
  return LineResult::kOk;
}

// Parse [b, e) line by line; stops at the first error (or a header when not
// allowed).  Returns a pointer just past the last consumed line.
const char* parse_range(const char* b, const char* e, TnsState& st, TnsOut& out, bool allow_header,
                        bool stop_after_first_entry) {
  std::vector<Token> tok;
  tok.reserve(kMaxModes + 2);
  const char* c = b;
  while (c < e) {
    const char* nl = static_cast<const char*>(std::memchr(c, '\n', static_cast<size_t>(e - c)));
    const char* le = nl ? nl : e;
    const size_t before = out.values.size();
    const LineResult r = parse_line(c, le, st, out, allow_header, tok);
    if (r == LineResult::kHeaderInChunk) {
      out.saw_header = true;
      return c;
    }
    ++out.lines;
    if (r == LineResult::kError) {
      out.has_err = true;
      out.err_line = out.lines;
      return nl ? nl + 1 : e;
    }
    c = nl ? nl + 1 : e;
    if (stop_after_first_entry && out.values.size() > before) return c;
  }
  return c;
}

void coo_alloc(gcpb_coo* out, int d, int64_t nnz) {
  out->d = d;
  out->nnz = nnz;
  out->coords = static_cast<int64_t*>(std::malloc(std::max<size_t>(1, nnz * d) * sizeof(int64_t)));
  out->values = static_cast<double*>(std::malloc(std::max<int64_t>(1, nnz) * sizeof(double)));
  if (!out->coords || !out->values) {
    std::free(out->coords);
    std::free(out->values);
    out->coords = nullptr;
    out->values = nullptr;
    throw std::bad_alloc();
  }
}

template <typename F>
void parallel_for(int threads, int64_t n, F&& f) {
  if (threads <= 1 || n < 1 << 16) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const int64_t b = n * t / threads, e = n * (t + 1) / threads;
    pool.emplace_back([&f, b, e] { f(b, e); });
  }
  for (auto& th : pool) th.join();
}

void read_tns(const std::string& path, int threads, gcpb_coo* out) {
  Mapped m(path);
  const char* b = m.p;
  const char* e = m.p + m.n;
  TnsState st;
  std::vector<TnsOut> parts(1);
  // serial prologue: up to and including the first entry
  const char* c = parse_range(b, e, st, parts[0], true, true);
  bool serial = parts[0].has_err;
  const int nt = pick_threads(threads);
  if (!serial && c < e) {
    const int64_t rest = e - c;
    const int nchunks = rest < (1 << 20) ? 1 : nt;
    std::vector<const char*> cut(static_cast<size_t>(nchunks) + 1);
    cut[0] = c;
    cut[static_cast<size_t>(nchunks)] = e;
    for (int t = 1; t < nchunks; ++t) {
      const char* s = c + rest * t / nchunks;
      s = std::max(s, cut[static_cast<size_t>(t - 1)]);
      const char* nl = static_cast<const char*>(std::memchr(s, '\n', static_cast<size_t>(e - s)));
      cut[static_cast<size_t>(t)] = nl ? nl + 1 : e;
    }
    parts.resize(static_cast<size_t>(nchunks) + 1);
    std::vector<std::thread> pool;
    for (int t = 0; t < nchunks; ++t) {
      pool.emplace_back([&, t] {
        TnsState local = st;
        TnsOut& o = parts[static_cast<size_t>(t) + 1];
        const int64_t est = (cut[t + 1] - cut[t]) / (st.d * 3 + 4) + 16;
        o.coords.reserve(static_cast<size_t>(est * st.d));
        o.values.reserve(static_cast<size_t>(est));
        parse_range(cut[static_cast<size_t>(t)], cut[static_cast<size_t>(t) + 1], local, o, false,
                    false);
      });
    }
    for (auto& th : pool) th.join();
    for (size_t t = 1; t < parts.size(); ++t)
      if (parts[t].saw_header) serial = true;
    if (serial) {  // a shape header after the first entry: exact serial walk
      parts.resize(1);
      TnsState again;
      parts[0] = TnsOut();
      parse_range(b, e, again, parts[0], true, false);
      st = again;
    }
  }
  // the first error in file order
  int64_t line0 = 0;
  for (size_t t = 0; t < parts.size(); ++t) {
    const TnsOut& o = parts[t];
    if (o.has_err) {
      const int64_t base = (t == 0) ? 0 : line0;
      throw io_error(path + ":" + std::to_string(base + o.err_line) + ": " + o.err_msg);
    }
    line0 += o.lines;
  }

  // shape: the header, else the maxima (io.cpp:133-137)
  std::vector<int64_t> dims = st.header;
  int64_t nnz = 0;
  for (const TnsOut& o : parts) nnz += static_cast<int64_t>(o.values.size());
  if (dims.empty()) {
    if (nnz == 0) fail(path, "no shape header and no entries; shape unknown");
    dims.assign(static_cast<size_t>(st.d), 1);
    for (const TnsOut& o : parts)
      for (int k = 0; k < o.maxima_n && k < static_cast<int>(dims.size()); ++k)
        dims[static_cast<size_t>(k)] = std::max(dims[static_cast<size_t>(k)], o.maxima[k]);
  }
  // Shape(header_dims) and SparseTensor's check_index (shape.cpp:29-44,73-85)
  if (dims.size() > static_cast<size_t>(kMaxModes))
    throw std::invalid_argument("Shape: at most " + std::to_string(kMaxModes) +
                                " modes supported");
  const int d = static_cast<int>(dims.size());
  for (const TnsOut& o : parts)
    for (int ld : o.line_d)
      if (ld != d)
        throw std::out_of_range("index has " + std::to_string(ld) + " modes, shape has " +
                                std::to_string(d));
  for (const TnsOut& o : parts) {  // entries read before a later header
    if (!serial) break;  // parallel chunks were checked against the header while parsing
    for (size_t i = 0; i < o.values.size(); ++i)
      for (int k = 0; k < d; ++k) {
        const int64_t v = o.coords[i * static_cast<size_t>(d) + static_cast<size_t>(k)];
        if (v >= dims[static_cast<size_t>(k)])
          throw std::out_of_range("index " + std::to_string(v) + " out of range [0, " +
                                  std::to_string(dims[static_cast<size_t>(k)]) + ") in mode " +
                                  std::to_string(k));
      }
  }
  coo_alloc(out, d, nnz);
  for (int k = 0; k < d; ++k) out->dims[k] = dims[static_cast<size_t>(k)];
  // concatenate in file order
  std::vector<int64_t> at(parts.size() + 1, 0);
  for (size_t t = 0; t < parts.size(); ++t)
    at[t + 1] = at[t] + static_cast<int64_t>(parts[t].values.size());
  std::vector<std::thread> pool;
  for (size_t t = 0; t < parts.size(); ++t) {
    pool.emplace_back([&, t] {
      const TnsOut& o = parts[t];
      std::memcpy(out->coords + at[t] * d, o.coords.data(), o.coords.size() * sizeof(int64_t));
      std::memcpy(out->values + at[t], o.values.data(), o.values.size() * sizeof(double));
    });
  }
  for (auto& th : pool) th.join();
}

// %.17g, as fmt17 (io.cpp:18-22).
inline int fmt17(char* buf, double v) { return std::snprintf(buf, 40, "%.17g", v); }

inline char* put_i64(char* p, int64_t v) {
  char tmp[24];
  int n = 0;
  uint64_t u = v < 0 ? static_cast<uint64_t>(-(v + 1)) + 1 : static_cast<uint64_t>(v);
  do {
    tmp[n++] = static_cast<char>('0' + u % 10);
    u /= 10;
  } while (u);
  if (v < 0) *p++ = '-';
  while (n) *p++ = tmp[--n];
  return p;
}

void check_coo(const gcpb_coo* c) {
  if (!c) throw std::invalid_argument("null coordinate list");
  if (c->d < 1 || c->d > kMaxModes)
    throw std::invalid_argument("Shape: at most " + std::to_string(kMaxModes) +
                                " modes supported");
  if (c->nnz < 0 || (c->nnz > 0 && (!c->coords || !c->values)))
    throw std::invalid_argument("coordinate list: bad buffers");
}

void write_tns(const std::string& path, const gcpb_coo* c, int threads) {
  check_coo(c);
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) fail(path, "cannot open for writing");
  std::string head = "#shape:";
  for (int k = 0; k < c->d; ++k) head += " " + std::to_string(c->dims[k]);
  head += "\n";
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  // format blocks of lines in parallel, write them in order
  const int nt = pick_threads(threads);
  const int64_t block = 1 << 18;
  std::vector<std::string> bufs(static_cast<size_t>(nt));
  for (int64_t b0 = 0; ok && b0 < c->nnz; b0 += block * nt) {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) {
      pool.emplace_back([&, t] {
        std::string& s = bufs[static_cast<size_t>(t)];
        s.clear();
        const int64_t lo = b0 + block * t, hi = std::min(c->nnz, lo + block);
        if (lo >= hi) return;
        s.resize(static_cast<size_t>((hi - lo) * (c->d * 21 + 32)));
        char* p = s.data();
        for (int64_t e = lo; e < hi; ++e) {
          for (int k = 0; k < c->d; ++k) {
            p = put_i64(p, c->coords[e * c->d + k] + 1);
            *p++ = ' ';
          }
          p += fmt17(p, c->values[e]);
          *p++ = '\n';
        }
        s.resize(static_cast<size_t>(p - s.data()));
      });
    }
    for (auto& th : pool) th.join();
    for (const std::string& s : bufs)
      if (!s.empty()) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) fail(path, "write error");
}

struct CooHeader {
  char magic[8];
  uint32_t version;
  uint32_t d;
  int64_t nnz;
  uint32_t index_bytes;
  uint32_t flags;
  uint64_t reserved;
};
static_assert(sizeof(CooHeader) == 40, "binary COO header is 40 bytes");
constexpr char kMagic[8] = {'G', 'C', 'P', 'B', 'C', 'O', 'O', '1'};

void write_coo(const std::string& path, const gcpb_coo* c) {
  check_coo(c);
  bool narrow = true;
  for (int k = 0; k < c->d; ++k) narrow = narrow && c->dims[k] <= (int64_t{1} << 32);
  CooHeader h{};
  std::memcpy(h.magic, kMagic, 8);
  h.version = 1;
  h.d = static_cast<uint32_t>(c->d);
  h.nnz = c->nnz;
  h.index_bytes = narrow ? 4 : 8;
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) fail(path, "cannot open for writing");
  bool ok = std::fwrite(&h, sizeof(h), 1, f) == 1;
  ok = ok && std::fwrite(c->dims, sizeof(int64_t), static_cast<size_t>(c->d), f) ==
                 static_cast<size_t>(c->d);
  const int64_t n = c->nnz * c->d;
  if (narrow) {
    std::vector<uint32_t> buf(static_cast<size_t>(std::min<int64_t>(n, 1 << 22)));
    for (int64_t b0 = 0; ok && b0 < n; b0 += static_cast<int64_t>(buf.size())) {
      const int64_t m = std::min<int64_t>(n - b0, static_cast<int64_t>(buf.size()));
      for (int64_t i = 0; i < m; ++i) {
        const int64_t v = c->coords[b0 + i];
        if (v < 0 || v >= c->dims[(b0 + i) % c->d]) {
          std::fclose(f);
          throw std::out_of_range("index " + std::to_string(v) + " out of range [0, " +
                                  std::to_string(c->dims[(b0 + i) % c->d]) + ") in mode " +
                                  std::to_string((b0 + i) % c->d));
        }
        buf[static_cast<size_t>(i)] = static_cast<uint32_t>(v);
      }
      ok = std::fwrite(buf.data(), 4, static_cast<size_t>(m), f) == static_cast<size_t>(m);
    }
  } else if (n > 0) {
    ok = ok && std::fwrite(c->coords, 8, static_cast<size_t>(n), f) == static_cast<size_t>(n);
  }
  if (c->nnz > 0)
    ok = ok && std::fwrite(c->values, 8, static_cast<size_t>(c->nnz), f) ==
                   static_cast<size_t>(c->nnz);
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) fail(path, "write error");
}

void read_coo(const std::string& path, int threads, gcpb_coo* out) {
  Mapped m(path);
  CooHeader h{};
  if (m.n < sizeof(h)) fail(path, "not a GCPBCOO1 file (too short)");
  std::memcpy(&h, m.p, sizeof(h));
  if (std::memcmp(h.magic, kMagic, 8) != 0) fail(path, "not a GCPBCOO1 file (bad magic)");
  if (h.version != 1) fail(path, "unsupported GCPBCOO version " + std::to_string(h.version));
  if (h.d < 1 || h.d > static_cast<uint32_t>(kMaxModes)) fail(path, "bad mode count");
  if (h.index_bytes != 4 && h.index_bytes != 8) fail(path, "bad index width");
  if (h.nnz < 0) fail(path, "bad entry count");
  const int d = static_cast<int>(h.d);
  const size_t want = sizeof(h) + 8 * static_cast<size_t>(d) +
                      static_cast<size_t>(h.nnz) * (h.index_bytes * static_cast<size_t>(d) + 8);
  if (m.n < want)
    fail(path, "file shorter than the " + std::to_string(want) + " bytes its header implies");
  if (m.n > want) fail(path, "file longer than its header implies");
  int64_t dims[kMaxModes];
  std::memcpy(dims, m.p + sizeof(h), 8 * static_cast<size_t>(d));
  for (int k = 0; k < d; ++k)
    if (dims[k] < 1) fail(path, "shape extent must be >= 1");
  coo_alloc(out, d, h.nnz);
  for (int k = 0; k < d; ++k) out->dims[k] = dims[k];
  const char* cp = m.p + sizeof(h) + 8 * d;
  const char* vp = cp + static_cast<size_t>(h.nnz) * h.index_bytes * d;
  const int64_t n = h.nnz * d;
  const int nt = pick_threads(threads);
  if (h.index_bytes == 4) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(cp);
    parallel_for(nt, n, [&](int64_t b, int64_t e) {
      for (int64_t i = b; i < e; ++i) out->coords[i] = src[i];
    });
  } else {
    parallel_for(nt, n, [&](int64_t b, int64_t e) {
      std::memcpy(out->coords + b, cp + 8 * b, static_cast<size_t>(e - b) * 8);
    });
  }
  parallel_for(nt, h.nnz, [&](int64_t b, int64_t e) {
    std::memcpy(out->values + b, vp + 8 * b, static_cast<size_t>(e - b) * 8);
  });
}

std::vector<int64_t> dense_shape(const std::string& path) {
  const std::string sp = path + ".shape";
  FILE* f = std::fopen(sp.c_str(), "rb");
  if (!f) fail(sp, "cannot open for reading");
  std::string text;
  char buf[4096];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) text.append(buf, got);
  std::fclose(f);
  // `shape_in >> n` until extraction fails (io.cpp:199-203)
  std::vector<int64_t> dims;
  const char* c = text.c_str();
  for (;;) {
    while (*c && is_ws(*c)) ++c;
    if (!*c) break;
    errno = 0;
    char* end = nullptr;
    const long long v = std::strtoll(c, &end, 10);
    if (end == c || errno != 0) break;
    if (v < 1) fail(sp, "shape extent must be >= 1");
    dims.push_back(v);
    c = end;
  }
  if (dims.empty()) fail(sp, "empty shape sidecar");
  if (dims.size() > static_cast<size_t>(kMaxModes))
    throw std::invalid_argument("Shape: at most " + std::to_string(kMaxModes) +
                                " modes supported");
  return dims;
}

// ---- model text files (io.cpp:153-193) and the trace CSV (io.cpp:252-260) ----
// A cursor over a whole file with the two extraction rules read_model uses:
// `in >> int64` (skip whitespace, sign + digits, stop at the first non-digit)
// and `in >> string` (skip whitespace, read to the next whitespace).
struct Cursor {
  const char* p;
  const char* e;
  void skip() {
    while (p < e && is_ws(*p)) ++p;
  }
  bool int64(int64_t* out) {
    skip();
    const char* q = p;
    bool neg = false;
    if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
    const char* d0 = q;
    unsigned long long v = 0;
    bool overflow = false;
    for (; q < e && *q >= '0' && *q <= '9'; ++q) {
      const unsigned dig = static_cast<unsigned>(*q - '0');
      if (v > (0xffffffffffffffffull - dig) / 10) overflow = true;
      v = v * 10 + dig;
    }
    if (q == d0) return false;
    const unsigned long long lim = neg ? (1ull << 63) : (1ull << 63) - 1;
    if (overflow || v > lim) return false;
    *out = neg ? static_cast<int64_t>(0 - v) : static_cast<int64_t>(v);
    p = q;
    return true;
  }
  bool token(Token* t) {
    skip();
    if (p == e) return false;
    const char* q = p;
    while (q < e && !is_ws(*q)) ++q;
    *t = {p, q};
    p = q;
    return true;
  }
};

struct ModelHeader {
  int64_t d = 0, r = 0;
  std::vector<int64_t> dims;
};

ModelHeader read_model_header(const std::string& path, Cursor& c) {
  ModelHeader h;
  if (!c.int64(&h.d) || !c.int64(&h.r)) fail(path, "bad header: expected mode count and rank");
  if (h.d < 1 || h.r < 1) fail(path, "bad header: mode count and rank must be >= 1");
  if (h.d > kMaxModes)
    throw std::invalid_argument("Shape: at most " + std::to_string(kMaxModes) +
                                " modes supported");
  h.dims.resize(static_cast<size_t>(h.d));
  for (auto& n : h.dims)
    if (!c.int64(&n)) fail(path, "bad header: missing extents");
  for (int64_t n : h.dims)  // KruskalModel(factors) -> Shape (shape.cpp:38-39)
    if (n < 1) throw std::invalid_argument("Shape: every extent must be positive");
  return h;
}

}  // namespace

extern "C" {

int gcpb_tns_read(const char* path, int threads, gcpb_coo* out) {
  return io_guard([&] {
    if (!path || !out) throw std::invalid_argument("gcpb_tns_read: null argument");
    *out = gcpb_coo{};
    read_tns(path, threads, out);
  });
}

int gcpb_tns_write(const char* path, const gcpb_coo* coo) {
  return io_guard([&] {
    if (!path) throw std::invalid_argument("gcpb_tns_write: null path");
    write_tns(path, coo, 0);
  });
}

int gcpb_coo_write(const char* path, const gcpb_coo* coo) {
  return io_guard([&] {
    if (!path) throw std::invalid_argument("gcpb_coo_write: null path");
    write_coo(path, coo);
  });
}

int gcpb_coo_read(const char* path, int threads, gcpb_coo* out) {
  return io_guard([&] {
    if (!path || !out) throw std::invalid_argument("gcpb_coo_read: null argument");
    *out = gcpb_coo{};
    read_coo(path, threads, out);
  });
}

void gcpb_coo_free(gcpb_coo* coo) {
  if (!coo) return;
  std::free(coo->coords);
  std::free(coo->values);
  coo->coords = nullptr;
  coo->values = nullptr;
  coo->nnz = 0;
}

int gcpb_dense_shape(const char* path, int* d, int64_t* dims) {
  return io_guard([&] {
    if (!path || !d || !dims) throw std::invalid_argument("gcpb_dense_shape: null argument");
    const std::vector<int64_t> s = dense_shape(path);
    *d = static_cast<int>(s.size());
    for (size_t k = 0; k < s.size(); ++k) dims[k] = s[k];
  });
}

int gcpb_dense_read(const char* path, int64_t n, double* values) {
  return io_guard([&] {
    if (!path || (n > 0 && !values)) throw std::invalid_argument("gcpb_dense_read: null argument");
    Mapped m(path);
    const size_t want = static_cast<size_t>(n) * 8;
    if (m.n < want)
      fail(path, "file shorter than the " + std::to_string(want) +
                     " bytes implied by its shape sidecar");
    if (m.n > want) fail(path, "file longer than the shape sidecar implies");
    parallel_for(pick_threads(0), n, [&](int64_t b, int64_t e) {
      std::memcpy(values + b, m.p + 8 * b, static_cast<size_t>(e - b) * 8);
    });
  });
}

int gcpb_dense_write(const char* path, int d, const int64_t* dims, const double* values) {
  return io_guard([&] {
    if (!path || !dims || d < 1) throw std::invalid_argument("gcpb_dense_write: bad argument");
    const std::string sp = std::string(path) + ".shape";
    FILE* s = std::fopen(sp.c_str(), "wb");
    if (!s) fail(sp, "cannot open for writing");
    std::string line;
    int64_t n = 1;
    for (int k = 0; k < d; ++k) {
      line += std::to_string(dims[k]) + (k + 1 < d ? " " : "\n");
      n *= dims[k];
    }
    bool ok = std::fwrite(line.data(), 1, line.size(), s) == line.size();
    ok = (std::fclose(s) == 0) && ok;
    if (!ok) fail(sp, "write error");
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(path, "cannot open for writing");
    ok = n == 0 || std::fwrite(values, 8, static_cast<size_t>(n), f) == static_cast<size_t>(n);
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) fail(path, "write error");
  });
}

int gcpb_model_read_header(const char* path, int* d, int64_t* dims, int64_t* rank) {
  return io_guard([&] {
    if (!path || !d || !dims || !rank) throw std::invalid_argument("gcpb_model_read_header: null");
    Mapped m(path);
    Cursor c{m.p, m.p + m.n};
    const ModelHeader h = read_model_header(path, c);
    *d = static_cast<int>(h.d);
    *rank = h.r;
    for (int64_t k = 0; k < h.d; ++k) dims[k] = h.dims[static_cast<size_t>(k)];
  });
}

int gcpb_model_read(const char* path, double* factors) {
  return io_guard([&] {
    if (!path || !factors) throw std::invalid_argument("gcpb_model_read: null");
    Mapped m(path);
    Cursor c{m.p, m.p + m.n};
    const ModelHeader h = read_model_header(path, c);
    int64_t n = 0;
    for (int64_t k : h.dims) n += k * h.r;
    for (int64_t i = 0; i < n; ++i) {
      Token t{};
      if (!c.token(&t)) fail(path, "truncated factor data");
      if (!parse_double(t, factors + i))  // parse_double(tok, path, 0) (io.cpp:172)
        throw io_error(std::string(path) + ":0: expected a number, got '" + t.str() + "'");
    }
  });
}

int gcpb_model_write(const char* path, int d, const int64_t* dims, int64_t rank,
                     const double* factors) {
  return io_guard([&] {
    if (!path || !dims || !factors || d < 1 || rank < 1)
      throw std::invalid_argument("gcpb_model_write: bad argument");
    std::string out = std::to_string(d) + " " + std::to_string(rank) + "\n";
    for (int k = 0; k < d; ++k) out += std::to_string(dims[k]) + (k + 1 < d ? " " : "\n");
    char buf[40];
    const double* f = factors;
    for (int k = 0; k < d; ++k)
      for (int64_t i = 0; i < dims[k]; ++i)
        for (int64_t j = 0; j < rank; ++j) {
          out.append(buf, static_cast<size_t>(fmt17(buf, *f++)));
          out += j + 1 < rank ? ' ' : '\n';
        }
    FILE* fp = std::fopen(path, "wb");
    if (!fp) fail(path, "cannot open for writing");
    bool ok = std::fwrite(out.data(), 1, out.size(), fp) == out.size();
    ok = (std::fclose(fp) == 0) && ok;
    if (!ok) fail(path, "write error");
  });
}

int gcpb_trace_write_csv(const char* path, const gcpb_trace_record* recs, int64_t n) {
  return io_guard([&] {
    if (!path || (n > 0 && !recs)) throw std::invalid_argument("gcpb_trace_write_csv: null");
    std::string out = "epoch,loss_estimate,learning_rate,seconds,accepted\n";
    char buf[40];
    for (int64_t i = 0; i < n; ++i) {
      const gcpb_trace_record& t = recs[i];
      out += std::to_string(t.epoch) + ',';
      out.append(buf, static_cast<size_t>(fmt17(buf, t.loss_estimate)));
      out += ',';
      out.append(buf, static_cast<size_t>(fmt17(buf, t.learning_rate)));
      out += ',';
      out.append(buf, static_cast<size_t>(fmt17(buf, t.seconds)));
      out += t.accepted ? ",1\n" : ",0\n";
    }
    FILE* fp = std::fopen(path, "wb");
    if (!fp) fail(path, "cannot open for writing");
    bool ok = std::fwrite(out.data(), 1, out.size(), fp) == out.size();
    ok = (std::fclose(fp) == 0) && ok;
    if (!ok) fail(path, "write error");
  });
}

}  // extern "C"

