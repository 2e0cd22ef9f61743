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

void parse_matrix_market(const char* text, uint64_t len, std::vector<uint32_t>& pairs, uint32_t& n_declared);
void parse_csr_cache(const void* bytes, uint64_t len, CsrView& out);

}  // namespace tcb
