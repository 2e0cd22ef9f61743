// io_host.h -- host ingest of MatrixMarket text and TRIMCSR1 caches.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tcb200.h"

namespace tcb {

struct IoFail : std::runtime_error {
  tc_status code;
  IoFail(tc_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct CsrView {
  uint32_t n = 0;
  uint64_t num_edges = 0;
  const uint64_t* offsets = nullptr;
  const uint32_t* nbrs = nullptr;
};

// MatrixMarket banner + comments + size line (io.cpp:93-122): the entry body
// starts at byte `body` of the text; `line_no` = the size line's number.
struct MmHeader {
  uint64_t rows = 0, cols = 0, nnz = 0, body = 0, line_no = 0;
  uint32_t n_declared = 0;
};
void parse_mm_header(const char* text, uint64_t len, MmHeader& h);
void parse_matrix_market(const char* text, uint64_t len, std::vector<uint32_t>& pairs, uint32_t& n_declared);
void parse_csr_cache(const void* bytes, uint64_t len, CsrView& out);

}  // namespace tcb
