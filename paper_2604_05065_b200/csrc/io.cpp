// Formats around the solve path: Matrix Market
// read/write (/root/reference/proj/include/aplicur/matrix_market.hpp:18-116),
// the per-iteration trace CSV and the solve report JSON
// (report_io.hpp:28-47, 49-110) written write-then-rename (report_io.hpp:112-122).
// Host code only; numbers are printed with %.17g so a read-back is bit-exact.
#include <algorithm>
#include <cctype>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "apc_internal.hpp"
#include "problem.hpp"

namespace apc {
int capi_guard(apc_ctx* ctx, const std::function<void()>& f);
}

namespace apc {
namespace {

std::string g17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

// lsqr.hpp:26-36
const char* reason_name(int r) {
  switch (r) {
    case 0: return "none";
    case 1: return "gradient-tol";
    case 2: return "dynamic-rate";
    case 3: return "dynamic-diff";
    case 4: return "iteration-cap";
    case 5: return "exact-zero-rhs";
  }
  return "unknown";
}

// solver.hpp:92-99
const char* status_name(int s) {
  switch (s) {
    case 0: return "converged";
    case 1: return "rank-exhausted";
    case 2: return "breakdown";
  }
  return "unknown";
}

void write_file_atomic(const std::string& path, const std::string& content) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream f(tmp, std::ios::binary);
    require(f.good(), APC_IO, "cannot open for writing: " + tmp);
    f << content;
    require(f.good(), APC_IO, "write failed: " + tmp);
  }
  require(std::rename(tmp.c_str(), path.c_str()) == 0, APC_IO, "rename failed: " + path);
}

void mm_write_csc(std::ostream& out, i64 m, i64 n, const std::int64_t* colptr, const std::int64_t* rowidx,
                  const double* vals) {
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << m << " " << n << " " << (n > 0 ? colptr[n] : 0) << "\n";
  for (i64 j = 0; j < n; ++j)
    for (i64 k = colptr[j]; k < colptr[j + 1]; ++k) out << (rowidx[k] + 1) << " " << (j + 1) << " " << g17(vals[k]) << "\n";
}

void mm_write_dense(std::ostream& out, i64 m, i64 n, const double* a) {
  out << "%%MatrixMarket matrix array real general\n";
  out << m << " " << n << "\n";
  for (i64 k = 0; k < m * n; ++k) out << g17(a[k]) << "\n";
}

struct Trip {
  i64 row, col;
  double v;
};

// read rules of matrix_market.hpp:48-116: general real/integer coordinate or
// array; '%' and blank lines skipped; coordinate entries sorted by (col, row),
// duplicates rejected, explicit zeros dropped (Matrix::sparse, matrix.hpp:68-94)
apc_problem* mm_read(std::istream& in) {
  std::string header;
  require(static_cast<bool>(std::getline(in, header)), APC_IO, "matrix market: empty stream");
  std::istringstream hs(header);
  std::string banner, object, format, field, symmetry;
  hs >> banner >> object >> format >> field >> symmetry;
  require(banner == "%%MatrixMarket" && object == "matrix", APC_IO, "matrix market: bad header: " + header);
  require(format == "coordinate" || format == "array", APC_IO, "matrix market: unsupported format: " + format);
  require(field == "real" || field == "integer", APC_IO, "matrix market: unsupported field: " + field);
  require(symmetry == "general", APC_IO, "matrix market: only general symmetry supported");
  std::string line;
  auto next_content = [&]() {
    while (std::getline(in, line)) {
      size_t i = 0;
      while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
      if (i == line.size() || line[i] == '%') continue;
      return true;
    }
    return false;
  };
  require(next_content(), APC_IO, "matrix market: missing size line");
  auto* p = new apc_problem();
  try {
    if (format == "coordinate") {
      i64 m = 0, n = 0, nz = 0;
      {
        std::istringstream ls(line);
        require(static_cast<bool>(ls >> m >> n >> nz), APC_IO, "matrix market: bad size line");
      }
      require(m >= 0 && n >= 0 && nz >= 0, APC_INVALID_ARGUMENT, "Matrix: negative dimension");
      std::vector<Trip> t;
      t.reserve(static_cast<size_t>(nz));
      for (i64 k = 0; k < nz; ++k) {
        require(next_content(), APC_IO, "matrix market: truncated entries");
        std::istringstream ls(line);
        i64 i = 0, j = 0;
        double v = 0.0;
        require(static_cast<bool>(ls >> i >> j >> v), APC_IO, "matrix market: bad entry line");
        t.push_back({i - 1, j - 1, v});
      }
      for (const auto& e : t)
        require(e.row >= 0 && e.row < m && e.col >= 0 && e.col < n, APC_INVALID_ARGUMENT,
                "Matrix::sparse: entry out of range");
      std::sort(t.begin(), t.end(),
                [](const Trip& a, const Trip& b) { return std::tie(a.col, a.row) < std::tie(b.col, b.row); });
      p->m = m;
      p->n = n;
      p->sparse = true;
      p->colptr.assign(static_cast<size_t>(n) + 1, 0);
      for (size_t k = 0; k < t.size(); ++k) {
        if (k > 0 && t[k].row == t[k - 1].row && t[k].col == t[k - 1].col)
          fail(APC_INVALID_ARGUMENT, "Matrix::sparse: duplicate entry");
        if (t[k].v == 0.0) continue;
        p->rowidx.push_back(t[k].row);
        p->vals.push_back(t[k].v);
        ++p->colptr[static_cast<size_t>(t[k].col) + 1];
      }
      for (i64 j = 0; j < n; ++j) p->colptr[j + 1] += p->colptr[j];
    } else {
      i64 m = 0, n = 0;
      {
        std::istringstream ls(line);
        require(static_cast<bool>(ls >> m >> n), APC_IO, "matrix market: bad size line");
      }
      require(m >= 0 && n >= 0, APC_INVALID_ARGUMENT, "Matrix: negative dimension");
      std::vector<double> vals;
      vals.reserve(static_cast<size_t>(m * n));
      while (static_cast<i64>(vals.size()) < m * n) {
        require(next_content(), APC_IO, "matrix market: truncated array");
        std::istringstream ls(line);
        double v;
        while (ls >> v) vals.push_back(v);
      }
      require(static_cast<i64>(vals.size()) == m * n, APC_IO, "matrix market: too many array values");
      p->m = m;
      p->n = n;
      p->sparse = false;
      p->dense = std::move(vals);
    }
    p->b.assign(static_cast<size_t>(p->m), 0.0);
  } catch (...) {
    delete p;
    throw;
  }
  return p;
}

// report_io.hpp:28-47: one row per trace row, reason on the last row of each
// phase (the phase report's reason when present, else the trace's)
std::string trace_csv(const apc_trace_row* rows, i64 nrows, const apc_phase_report* phases, i64 nph,
                      int trace_reason) {
  std::ostringstream out;
  out << "phase,iter,phibar,relres,matvecs,wall_ms,reason\n";
  for (i64 k = 0; k < nrows; ++k) {
    const apc_trace_row& r = rows[k];
    const bool last = (k + 1 == nrows) || (rows[k + 1].phase != r.phase);
    const char* reason = "";
    if (last) {
      reason = reason_name(trace_reason);
      for (i64 q = 0; q < nph; ++q)
        if (phases[q].phase == r.phase) reason = reason_name(phases[q].reason);
    }
    out << r.phase << "," << r.iter << "," << g17(r.phibar) << ",";
    if (!std::isnan(r.true_relres)) out << g17(r.true_relres);
    out << "," << r.matvecs << "," << g17(r.wall_ms) << "," << reason << "\n";
  }
  return out.str();
}

std::string jnum(double v) {
  if (std::isnan(v) || std::isinf(v)) return "null";  // JSON has no NaN / Inf
  return g17(v);
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (static_cast<unsigned char>(c) < 0x20) {
      char buf[8];
      std::snprintf(buf, sizeof buf, "\\u%04x", c);
      o += buf;
      continue;
    }
    o += c;
  }
  return o + "\"";
}

template <class T, class F>
std::string jarr(const T* a, i64 n, F f) {
  std::string o = "[";
  for (i64 k = 0; k < n; ++k) o += (k ? "," : "") + f(a[k]);
  return o + "]";
}

}  // namespace
}  // namespace apc

using namespace apc;

extern "C" {

int apc_mm_write_csc(const char* path, int64_t m, int64_t n, const int64_t* colptr, const int64_t* rowidx,
                     const double* vals) {
  return capi_guard(nullptr, [&] {
    require(path && colptr && m >= 0 && n >= 0, APC_INVALID_ARGUMENT, "apc_mm_write_csc: bad arguments");
    std::ostringstream out;
    mm_write_csc(out, m, n, colptr, rowidx, vals);
    std::ofstream f(path);
    require(f.good(), APC_IO, std::string("cannot open for writing: ") + path);
    f << out.str();
    require(f.good(), APC_IO, std::string("write failed: ") + path);
  });
}

int apc_mm_write_dense(const char* path, int64_t m, int64_t n, const double* a) {
  return capi_guard(nullptr, [&] {
    require(path && (a || m * n == 0) && m >= 0 && n >= 0, APC_INVALID_ARGUMENT, "apc_mm_write_dense: bad arguments");
    std::ostringstream out;
    mm_write_dense(out, m, n, a);
    std::ofstream f(path);
    require(f.good(), APC_IO, std::string("cannot open for writing: ") + path);
    f << out.str();
    require(f.good(), APC_IO, std::string("write failed: ") + path);
  });
}

int apc_mm_read(const char* path, apc_problem** out) {
  return capi_guard(nullptr, [&] {
    require(path && out, APC_INVALID_ARGUMENT, "apc_mm_read: bad arguments");
    std::ifstream f(path);
    require(f.good(), APC_IO, std::string("cannot open for reading: ") + path);
    *out = mm_read(f);
  });
}

int apc_trace_csv_write(const char* path, const apc_trace_row* rows, int64_t n_rows, const apc_phase_report* phases,
                        int64_t n_phases, int32_t trace_reason) {
  return capi_guard(nullptr, [&] {
    require(path && (rows || n_rows == 0) && (phases || n_phases == 0), APC_INVALID_ARGUMENT,
            "apc_trace_csv_write: bad arguments");
    write_file_atomic(path, trace_csv(rows, n_rows, phases, n_phases, trace_reason));
  });
}

int apc_report_json_write(const char* path, const apc_solver_config* cfg, int32_t status, double final_relres,
                          double final_rho, uint64_t sketch_applications, uint64_t system_matvecs,
                          const char* trace_path, const int64_t* row_indices, const int64_t* col_indices,
                          int64_t rank, const double* rho_history, int64_t n_rho, const apc_phase_report* phases,
                          int64_t n_phases, const double* const* spectra, const int64_t* n_spectra) {
  return capi_guard(nullptr, [&] {
    require(path && cfg, APC_INVALID_ARGUMENT, "apc_report_json_write: bad arguments");
    const auto i64s = [](int64_t v) { return std::to_string(v); };
    const auto dbl = [](double v) { return jnum(v); };
    std::string j = "{";
    // solver_config_to_json (report_io.hpp:67-83)
    j += "\"config\":{";
    j += "\"block\":" + std::to_string(cfg->block);
    j += ",\"eps_cur\":" + jnum(cfg->eps_cur);
    j += ",\"eps_lsqr\":" + jnum(cfg->eps_lsqr);
    j += ",\"nu_prec\":" + jnum(cfg->nu_prec);
    j += ",\"nu_lsqr\":" + jnum(cfg->nu_lsqr);
    j += ",\"mu\":" + jnum(cfg->mu);
    j += std::string(",\"variant\":") + (cfg->variant == 0 ? "\"svd\"" : "\"svd-free\"");
    j += ",\"sketch_xi\":" + std::to_string(cfg->sketch_xi);
    j += ",\"probe_count\":" + std::to_string(cfg->probe_count);
    j += ",\"lsqr_cap\":" + std::to_string(cfg->lsqr_cap);
    j += ",\"seed\":" + std::to_string(cfg->seed);
    j += std::string(",\"core\":") + (cfg->core == 0 ? "\"qr\"" : "\"lu\"");
    j += ",\"trace_sample_stride\":" + std::to_string(cfg->trace_sample_stride);
    j += "}";
    // solve_report_to_json (report_io.hpp:94-110)
    j += ",\"status\":" + jstr(status_name(status));
    j += ",\"final_relres\":" + jnum(final_relres);
    j += ",\"final_rho\":" + jnum(final_rho);
    j += ",\"sketch_applications\":" + std::to_string(sketch_applications);
    j += ",\"system_matvecs\":" + std::to_string(system_matvecs);
    j += ",\"trace\":" + jstr(trace_path ? trace_path : "");
    j += ",\"cur\":{\"row_indices\":" + jarr(row_indices, rank, i64s) + ",\"col_indices\":" +
         jarr(col_indices, rank, i64s) + ",\"rho_history\":" + jarr(rho_history, n_rho, dbl) + "}";
    j += ",\"phases\":[";
    for (int64_t k = 0; k < n_phases; ++k) {  // phase_report_to_json (report_io.hpp:49-65)
      const apc_phase_report& p = phases[k];
      j += k ? ",{" : "{";
      j += "\"phase\":" + std::to_string(p.phase);
      j += ",\"rank\":" + std::to_string(p.rank);
      j += ",\"rho\":" + jnum(p.rho);
      j += ",\"sigma_hat\":" + jnum(p.sigma_hat);
      j += ",\"mu\":" + jnum(p.mu);
      j += ",\"lsqr_iters\":" + std::to_string(p.lsqr_iters);
      j += ",\"reason\":" + jstr(reason_name(p.reason));
      j += ",\"relres_at_end\":" + jnum(p.relres_at_end);
      j += ",\"wall_ms\":{\"augment\":" + jnum(p.t_augment_ms) + ",\"factor\":" + jnum(p.t_factor_ms) +
           ",\"precond\":" + jnum(p.t_precond_ms) + ",\"lsqr\":" + jnum(p.t_lsqr_ms) + "}";
      if (spectra && n_spectra && n_spectra[k] > 0 && spectra[k])
        j += ",\"precond_spectrum\":" + jarr(spectra[k], n_spectra[k], dbl);
      j += "}";
    }
    j += "]}\n";
    write_file_atomic(path, j);
  });
}

}  // extern "C"
