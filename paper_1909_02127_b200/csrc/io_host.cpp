// io_host.cpp -- host-side ingest of the reference's two on-disk formats
// (SURVEY.md 8f rows 1-2), same accept/reject behaviour and messages:
//   MatrixMarket coordinate  -> parse_matrix_market  (io.cpp:93-159)
//   TRIMCSR1 binary cache    -> read_csr_cache       (io.cpp:187-220)
// Tokenising text is byte-serial host work; the CSR produced here goes
// straight to the device (tc_graph_from_csr route, no sort).
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/tcb200.h"
#include "io_host.h"

namespace tcb {
namespace {

inline bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

std::string_view trim(std::string_view s) {
  while (!s.empty() && is_space(s.front())) s.remove_prefix(1);
  while (!s.empty() && is_space(s.back())) s.remove_suffix(1);
  return s;
}

bool iequals(std::string_view a, std::string_view b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    char x = a[i], y = b[i];
    if (x >= 'A' && x <= 'Z') x = char(x - 'A' + 'a');
    if (y >= 'A' && y <= 'Z') y = char(y - 'A' + 'a');
    if (x != y) return false;
  }
  return true;
}

// Whitespace split into at most `cap` tokens (returns the full count).
size_t split_ws(std::string_view s, std::string_view* out, size_t cap) {
  size_t n = 0, i = 0;
  while (i < s.size()) {
    while (i < s.size() && is_space(s[i])) ++i;
    size_t j = i;
    while (j < s.size() && !is_space(s[j])) ++j;
    if (j > i) {
      if (n < cap) out[n] = s.substr(i, j - i);
      ++n;
    }
    i = j;
  }
  return n;
}

[[noreturn]] void parse_error(const std::string& msg, uint64_t line) {
  throw IoFail(TC_EPARSE, msg + " (line " + std::to_string(line) + ")");
}

uint64_t parse_index(std::string_view tok, uint64_t line, const char* what) {
  uint64_t value = 0;
  auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), value);
  if (ec != std::errc{} || ptr != tok.data() + tok.size())
    parse_error(std::string("expected integer ") + what + ", got '" + std::string(tok) + "'", line);
  return value;
}

// std::getline over a byte buffer.
struct Lines {
  const char* p;
  const char* end;
  bool next(std::string_view& line) {
    if (p >= end) return false;
    const char* q = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
    if (!q) q = end;
    line = std::string_view(p, (size_t)(q - p));
    p = (q < end) ? q + 1 : end;
    return true;
  }
};

}  // namespace

void parse_mm_header(const char* text, uint64_t len, MmHeader& h) {
  Lines in{text, text + len};
  std::string_view raw;
  uint64_t line_no = 0;
  if (!in.next(raw)) parse_error("empty input", 1);
  ++line_no;
  std::string_view tok[4];
  const size_t nb = split_ws(trim(raw), tok, 4);
  if (nb < 3 || !iequals(tok[0], "%%MatrixMarket") || !iequals(tok[1], "matrix") ||
      !iequals(tok[2], "coordinate"))
    parse_error("malformed MatrixMarket banner", line_no);

  uint64_t rows = 0, cols = 0, nnz = 0;
  for (;;) {
    if (!in.next(raw)) parse_error("missing size line", line_no + 1);
    ++line_no;
    auto s = trim(raw);
    if (s.empty() || s.front() == '%') continue;
    if (split_ws(s, tok, 4) != 3) parse_error("size line must be 'rows cols nnz'", line_no);
    rows = parse_index(tok[0], line_no, "row count");
    cols = parse_index(tok[1], line_no, "column count");
    nnz = parse_index(tok[2], line_no, "entry count");
    break;
  }
  const uint64_t declared = std::max(rows, cols);
  if (declared > 0xFFFFFFFFull) parse_error("vertex count exceeds 32-bit id range", line_no);
  h.rows = rows;
  h.cols = cols;
  h.nnz = nnz;
  h.n_declared = (uint32_t)declared;
  h.line_no = line_no;
  h.body = (uint64_t)(in.p - text);
}

void parse_matrix_market(const char* text, uint64_t len, std::vector<uint32_t>& pairs, uint32_t& n_declared) {
  MmHeader hd;
  parse_mm_header(text, len, hd);
  Lines in{text + hd.body, text + len};
  std::string_view raw;
  std::string_view tok[4];
  uint64_t line_no = hd.line_no;
  const uint64_t rows = hd.rows, cols = hd.cols, nnz = hd.nnz;
  n_declared = hd.n_declared;
  pairs.clear();
  pairs.reserve(2 * std::min<uint64_t>(nnz, len / 4 + 1));

  uint64_t seen = 0;
  while (seen < nnz) {
    if (!in.next(raw))
      parse_error("expected " + std::to_string(nnz) + " entries, got " + std::to_string(seen), line_no + 1);
    ++line_no;
    auto s = trim(raw);
    if (s.empty() || s.front() == '%') continue;
    if (split_ws(s, tok, 2) < 2) parse_error("entry needs at least 'i j'", line_no);
    const uint64_t i = parse_index(tok[0], line_no, "row index");
    const uint64_t j = parse_index(tok[1], line_no, "column index");
    if (i < 1 || i > rows || j < 1 || j > cols) parse_error("entry index out of declared range", line_no);
    pairs.push_back((uint32_t)(i - 1));
    pairs.push_back((uint32_t)(j - 1));
    ++seen;
  }
  while (in.next(raw)) {
    ++line_no;
    auto s = trim(raw);
    if (!s.empty() && s.front() != '%')
      parse_error("unexpected content after " + std::to_string(nnz) + " entries", line_no);
  }
}

// TRIMCSR1 (io.cpp:18-19 magic/version, :187-205 reader header checks).
void parse_csr_cache(const void* bytes, uint64_t len, CsrView& out) {
  const unsigned char* b = static_cast<const unsigned char*>(bytes);
  static const char kMagic[8] = {'T', 'R', 'I', 'M', 'C', 'S', 'R', '1'};
  auto u64_at = [&](uint64_t off) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)b[off + i] << (8 * i);
    return v;
  };
  if (len < 8 || std::memcmp(b, kMagic, 8) != 0) parse_error("bad CSR cache magic", 1);
  if (len < 32) parse_error("corrupt CSR cache header", 1);
  if (u64_at(8) != 1) parse_error("unsupported CSR cache version", 1);
  const uint64_t nv = u64_at(16), ne = u64_at(24);
  if (nv > 0xFFFFFFFFull) parse_error("corrupt CSR cache header", 1);
  const uint64_t need = 32 + 8 * (nv + 1) + 4 * (2 * ne);
  if (ne > (len / 8) || len < need) parse_error("truncated CSR cache", 1);
  out.n = (uint32_t)nv;
  out.num_edges = ne;
  // little-endian host: the arrays are usable in place (8-/4-byte aligned
  // offsets 32 and 32+8(nv+1)); copy only when the buffer is misaligned.
  out.offsets = reinterpret_cast<const uint64_t*>(b + 32);
  out.nbrs = reinterpret_cast<const uint32_t*>(b + 32 + 8 * (nv + 1));
  // the O(|V|+|E|) invariant checks (io.cpp:206-218: offsets, then adjacency)
  // run on the device in the CSR build (build.cu build_from_csr, strict)
}

}  // namespace tcb
