// Ingest: Matrix Market reader, csr_from_triplets and the SHA-256-stamped binary
// CSR cache (ingest.cpp).
#pragma once

#include <string>
#include <vector>

#include "host_setup.hpp"

namespace rmg {

// matrix_market.cpp:34-148: coordinate / array, real / integer / pattern,
// general / symmetric; RuntimeError on malformed input
HostCsr read_matrix_market(const std::string& path);
// sparse.cpp:27-73: sorted by (row, column), duplicates summed in input order
HostCsr csr_from_triplets(int64_t n, int64_t f, const std::vector<int64_t>& rows, const std::vector<int64_t>& cols,
                          const std::vector<double>& vals);
// SHA-256 of (uint64 row offsets, uint64 column indices, fp64 values or 1.0)
std::string csr_sha256(const HostCsr& m);
void save_csr(const HostCsr& m, const std::string& path);
HostCsr load_csr(const std::string& path, bool verify, std::string* sha_hex);

}  // namespace rmg
