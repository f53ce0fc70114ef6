// On-disk formats of the reference, host only:
//  * CSCT tensors (include/dcsc/tensor_io.hpp): "CSCT", u32 version 1, u8 ndim,
//    ndim x u64 dims, float64 payload, all little-endian, row-major.
//  * convergence-trace CSV (include/dcsc/trace_io.hpp): fixed header, one row
//    per half-step, phase names "coding" / "learning", doubles at 17 digits.
// Byte-compatible with the reference's writers and readers (tests compare files).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "dcsc_cuda.h"

namespace {

thread_local std::string g_io_err;

int io_fail(const std::string& msg) {
  g_io_err = msg;
  return DCSC_ERR_IO;
}

void le_put(std::ostream& os, std::uint64_t v, int bytes) {
  char b[8];
  for (int i = 0; i < bytes; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
  os.write(b, bytes);
}

bool le_get(std::istream& is, std::uint64_t& v, int bytes) {
  unsigned char b[8];
  if (!is.read(reinterpret_cast<char*>(b), bytes)) return false;
  v = 0;
  for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | b[i];
  return true;
}

const char* kTraceHeader = "outer_iter,phase,objective,data_term,l1_term,admm_iters,cg_iters,elapsed_ms";

}  // namespace

extern "C" {

int dcsc_io_last_error(char* buf, size_t len) {
  if (buf && len) {
    std::strncpy(buf, g_io_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return static_cast<int>(g_io_err.size());
}

int dcsc_io_write_tensor(const char* path, int ndim, const uint64_t* dims, const double* values) {
  if (ndim < 1 || ndim > 255) return io_fail("tensor rank must be in [1, 255]");
  std::ofstream os(path, std::ios::binary);
  if (!os) return io_fail(std::string("cannot open '") + path + "' for writing");
  std::uint64_t count = 1;
  for (int a = 0; a < ndim; ++a) count *= dims[a];
  os.write("CSCT", 4);
  le_put(os, 1, 4);
  le_put(os, static_cast<std::uint64_t>(ndim), 1);
  for (int a = 0; a < ndim; ++a) le_put(os, dims[a], 8);
  for (std::uint64_t i = 0; i < count; ++i) {
    std::uint64_t bits;
    std::memcpy(&bits, values + i, 8);
    le_put(os, bits, 8);
  }
  if (!os) return io_fail(std::string("write failed for '") + path + "'");
  return DCSC_OK;
}

// Reads the header; dims must hold 255 entries. *count = product of dims.
int dcsc_io_read_tensor_header(const char* path, int* ndim, uint64_t* dims, uint64_t* count) {
  std::ifstream is(path, std::ios::binary);
  if (!is) return io_fail(std::string("cannot open '") + path + "'");
  char magic[4];
  if (!is.read(magic, 4) || std::memcmp(magic, "CSCT", 4) != 0)
    return io_fail(std::string("'") + path + "' is not a CSCT tensor");
  std::uint64_t v;
  if (!le_get(is, v, 4) || v != 1) return io_fail(std::string("unsupported CSCT version in '") + path + "'");
  if (!le_get(is, v, 1) || v == 0) return io_fail(std::string("bad tensor rank in '") + path + "'");
  *ndim = static_cast<int>(v);
  std::uint64_t c = 1;
  for (int a = 0; a < *ndim; ++a) {
    if (!le_get(is, dims[a], 8) || dims[a] == 0 || c > std::numeric_limits<std::uint64_t>::max() / dims[a])
      return io_fail(std::string("bad tensor dims in '") + path + "'");
    c *= dims[a];
  }
  *count = c;
  return DCSC_OK;
}

int dcsc_io_read_tensor(const char* path, double* values, uint64_t count) {
  int ndim = 0;
  std::uint64_t dims[255], c = 0;
  const int rc = dcsc_io_read_tensor_header(path, &ndim, dims, &c);
  if (rc) return rc;
  if (c != count) return io_fail("tensor element count mismatch");
  std::ifstream is(path, std::ios::binary);
  is.seekg(4 + 4 + 1 + 8 * static_cast<std::streamoff>(ndim));
  for (std::uint64_t i = 0; i < count; ++i) {
    std::uint64_t bits;
    if (!le_get(is, bits, 8)) return io_fail(std::string("truncated tensor payload in '") + path + "'");
    std::memcpy(values + i, &bits, 8);
  }
  is.peek();
  if (!is.eof()) return io_fail(std::string("trailing bytes after tensor payload in '") + path + "'");
  return DCSC_OK;
}

int dcsc_io_write_trace_csv(const char* path, const dcsc_trace_row* rows, int n) {
  std::ofstream os(path);
  if (!os) return io_fail(std::string("cannot open '") + path + "' for writing");
  os << kTraceHeader << "\n";
  os.precision(17);
  for (int i = 0; i < n; ++i) {
    const dcsc_trace_row& r = rows[i];
    os << r.outer_iter << ',' << (r.phase == 0 ? "coding" : "learning") << ',' << r.total << ','
       << r.data_term << ',' << r.l1_term << ',' << r.admm_iters << ',' << r.cg_iters << ','
       << r.elapsed_ms << "\n";
  }
  if (!os) return io_fail(std::string("write failed for '") + path + "'");
  return DCSC_OK;
}

int dcsc_io_read_trace_csv(const char* path, dcsc_trace_row* rows, int max_rows, int* n_rows) {
  std::ifstream is(path);
  if (!is) return io_fail(std::string("cannot open '") + path + "'");
  std::string line;
  if (!std::getline(is, line) || line != kTraceHeader)
    return io_fail(std::string("'") + path + "' does not carry the trace header");
  int n = 0, last = 0;
  while (std::getline(is, line)) {
    if (line.empty()) continue;
    if (n >= max_rows) return io_fail("trace has more rows than the buffer");
    std::istringstream row(line);
    std::string f[8];
    for (int i = 0; i < 8; ++i)
      if (!std::getline(row, f[i], ',')) return io_fail(std::string("short trace row in '") + path + "'");
    dcsc_trace_row r{};
    try {
      r.outer_iter = std::stoi(f[0]);
      if (f[1] == "coding")
        r.phase = 0;
      else if (f[1] == "learning")
        r.phase = 1;
      else
        return io_fail("unknown phase '" + f[1] + "' in '" + path + "'");
      r.total = std::stod(f[2]);
      r.data_term = std::stod(f[3]);
      r.l1_term = std::stod(f[4]);
      r.admm_iters = std::stol(f[5]);
      r.cg_iters = std::stol(f[6]);
      r.elapsed_ms = std::stod(f[7]);
    } catch (const std::exception&) {
      return io_fail(std::string("malformed trace row in '") + path + "'");
    }
    if (!std::isfinite(r.total)) return io_fail(std::string("non-finite objective value in '") + path + "'");
    if (r.outer_iter < last) return io_fail(std::string("trace rows out of order in '") + path + "'");
    last = r.outer_iter;
    rows[n++] = r;
  }
  *n_rows = n;
  return DCSC_OK;
}

}  // extern "C"
