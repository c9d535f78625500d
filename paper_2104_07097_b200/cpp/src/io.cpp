// Sample output: CSV / manifest / binary sidecar (host side, like the
// reference's src/io.cpp).  JSON is written by hand in the layout of
// nlohmann::json::dump(2) with sorted keys.
#include "mhar/io.hpp"

#include <charconv>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <vector>

namespace mhar {
namespace {

void write_text(const std::string& path, const std::string& text) {
  std::ofstream out(path, std::ios::binary);
  if (!out) raise(ErrorCode::io_failure, "cannot open " + path + " for writing");
  out << text;
  if (!out) raise(ErrorCode::io_failure, "write failed for " + path);
}

double parse_double(const std::string& token, const std::string& where) {
  double value = 0.0;
  const auto r = std::from_chars(token.data(), token.data() + token.size(), value);
  if (r.ec != std::errc{} || r.ptr != token.data() + token.size())
    raise(ErrorCode::io_failure, "bad number '" + token + "' in " + where);
  return value;
}

// JSON number for a double: shortest round trip, with ".0" on integral
// values so the field stays a float when parsed back.
std::string json_double(double v) {
  std::string s = format_double(v);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

std::string json_string(const std::string& s) {
  std::string out = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') {
      out += '\\';
      out += c;
    } else if (static_cast<unsigned char>(c) < 0x20) {
      char buf[8];
      std::snprintf(buf, sizeof(buf), "\\u%04x", c);
      out += buf;
    } else {
      out += c;
    }
  }
  return out + "\"";
}

}  // namespace

std::string format_double(double value) {
  char buffer[32];
  const auto result = std::to_chars(buffer, buffer + sizeof(buffer), value);
  return std::string(buffer, result.ptr);
}

std::string sample_csv_string(const Matrix& samples) {
  std::string out;
  out.reserve(static_cast<size_t>(samples.size()) * 20 + 16);
  for (Index j = 0; j < samples.cols(); ++j) {
    if (j > 0) out += ',';
    out += 'x';
    out += std::to_string(j + 1);
  }
  out += '\n';
  for (Index i = 0; i < samples.rows(); ++i) {
    for (Index j = 0; j < samples.cols(); ++j) {
      if (j > 0) out += ',';
      out += format_double(samples(i, j));
    }
    out += '\n';
  }
  return out;
}

void write_sample_csv(const std::string& path, const Matrix& samples) {
  write_text(path, sample_csv_string(samples));
}

Matrix read_sample_csv(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) raise(ErrorCode::io_failure, "cannot open " + path);
  std::string line;
  if (!std::getline(in, line)) raise(ErrorCode::io_failure, path + ": missing header");
  Index cols = 1;
  for (char c : line)
    if (c == ',') ++cols;
  std::vector<double> data;
  Index rows = 0;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::stringstream ss(line);
    std::string token;
    Index seen = 0;
    while (std::getline(ss, token, ',')) {
      data.push_back(parse_double(token, path + " row " + std::to_string(rows)));
      ++seen;
    }
    if (seen != cols)
      raise(ErrorCode::io_failure, path + ": row " + std::to_string(rows) + " has " +
                                       std::to_string(seen) + " fields, header has " +
                                       std::to_string(cols));
    ++rows;
  }
  Matrix out(rows, cols);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) out(i, j) = data[static_cast<size_t>(i * cols + j)];
  return out;
}

std::string manifest_string(const SampleSet& set, const std::string& polytope_source,
                            const std::string& samples_path) {
  const SamplerConfig& c = set.config;
  std::string s = "{\n";
  s += "  \"config\": {\n";
  s += "    \"burn_in\": " + std::to_string(c.burn_in) + ",\n";
  s += "    \"eps_dir\": " + json_double(c.eps_dir) + ",\n";
  s += "    \"eps_feas\": " + json_double(c.eps_feas) + ",\n";
  s += "    \"phi\": " + std::to_string(c.phi) + ",\n";
  s += "    \"reproject_every\": " + std::to_string(c.reproject_every) + ",\n";
  s += "    \"seed\": " + std::to_string(c.seed) + ",\n";
  s += "    \"t_target\": " + std::to_string(c.t_target) + ",\n";
  s += "    \"z\": " + std::to_string(c.z) + "\n";
  s += "  },\n";
  s += "  \"format_version\": 1,\n";
  s += "  \"iterate_count\": " + std::to_string(set.iterate_count) + ",\n";
  s += "  \"n\": " + std::to_string(set.samples.cols()) + ",\n";
  s += "  \"polytope\": " + json_string(polytope_source) + ",\n";
  s += "  \"redraw_count\": " + std::to_string(set.redraw_count) + ",\n";
  s += "  \"samples_file\": " + json_string(samples_path) + ",\n";
  s += "  \"samples_written\": " + std::to_string(set.samples.rows()) + ",\n";
  s += "  \"seconds\": " + json_double(set.seconds) + ",\n";
  s += "  \"start_radius\": " + json_double(set.start_radius) + ",\n";
  s += "  \"windows\": " + std::to_string(set.windows) + "\n";
  s += "}\n";
  return s;
}

void write_manifest(const std::string& path, const SampleSet& set,
                    const std::string& polytope_source, const std::string& samples_path) {
  write_text(path, manifest_string(set, polytope_source, samples_path));
}

void write_sample_bin(const std::string& path, const Matrix& samples) {
  std::ofstream out(path, std::ios::binary);
  if (!out) raise(ErrorCode::io_failure, "cannot open " + path + " for writing");
  const uint64_t rows = static_cast<uint64_t>(samples.rows());
  const uint64_t cols = static_cast<uint64_t>(samples.cols());
  out.write("MHARSMP1", 8);
  out.write(reinterpret_cast<const char*>(&rows), 8);
  out.write(reinterpret_cast<const char*>(&cols), 8);
  std::vector<double> row(cols);
  for (uint64_t i = 0; i < rows; ++i) {
    for (uint64_t j = 0; j < cols; ++j) row[j] = samples(static_cast<Index>(i), static_cast<Index>(j));
    out.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(8 * cols));
  }
  if (!out) raise(ErrorCode::io_failure, "write failed for " + path);
}

Matrix read_sample_bin(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) raise(ErrorCode::io_failure, "cannot open " + path);
  char magic[8];
  uint64_t rows = 0, cols = 0;
  in.read(magic, 8);
  in.read(reinterpret_cast<char*>(&rows), 8);
  in.read(reinterpret_cast<char*>(&cols), 8);
  if (!in || std::memcmp(magic, "MHARSMP1", 8) != 0)
    raise(ErrorCode::io_failure, path + ": not a sample sidecar");
  Matrix out(static_cast<Index>(rows), static_cast<Index>(cols));
  std::vector<double> row(cols);
  for (uint64_t i = 0; i < rows; ++i) {
    in.read(reinterpret_cast<char*>(row.data()), static_cast<std::streamsize>(8 * cols));
    if (!in) raise(ErrorCode::io_failure, path + ": truncated");
    for (uint64_t j = 0; j < cols; ++j) out(static_cast<Index>(i), static_cast<Index>(j)) = row[j];
  }
  return out;
}

// Throughput records (io.hpp bench writers): one CSV line per record,
// doubles as shortest round trips; JSON in dump(2) layout, sorted keys.
std::string bench_csv_string(const std::vector<BenchRecord>& records) {
  std::string s = "figure,n,z,phi,windows,total_samples,mean_sps,std_sps,runs\n";
  for (const BenchRecord& r : records)
    s += r.figure + "," + std::to_string(r.n) + "," + std::to_string(r.z) + "," +
         std::to_string(r.phi) + "," + std::to_string(r.windows) + "," +
         std::to_string(r.total_samples) + "," + format_double(r.mean_sps) + "," +
         format_double(r.std_sps) + "," + std::to_string(r.run_seconds.size()) + "\n";
  return s;
}

void write_bench_csv(const std::string& path, const std::vector<BenchRecord>& records) {
  write_text(path, bench_csv_string(records));
}

std::string bench_json_string(const std::vector<BenchRecord>& records) {
  auto array = [](const std::vector<double>& v, const std::string& pad) {
    if (v.empty()) return std::string("[]");
    std::string a = "[\n";
    for (size_t i = 0; i < v.size(); ++i)
      a += pad + "  " + json_double(v[i]) + (i + 1 < v.size() ? ",\n" : "\n");
    return a + pad + "]";
  };
  std::string s = "{\n  \"format_version\": 1,\n  \"records\": ";
  if (records.empty()) return s + "[]\n}\n";
  s += "[\n";
  for (size_t i = 0; i < records.size(); ++i) {
    const BenchRecord& r = records[i];
    const std::string p = "      ";
    s += "    {\n";
    s += p + "\"figure\": " + json_string(r.figure) + ",\n";
    s += p + "\"mean_sps\": " + json_double(r.mean_sps) + ",\n";
    s += p + "\"n\": " + std::to_string(r.n) + ",\n";
    s += p + "\"phi\": " + std::to_string(r.phi) + ",\n";
    s += p + "\"run_seconds\": " + array(r.run_seconds, p) + ",\n";
    s += p + "\"run_sps\": " + array(r.run_sps, p) + ",\n";
    s += p + "\"std_sps\": " + json_double(r.std_sps) + ",\n";
    s += p + "\"total_samples\": " + std::to_string(r.total_samples) + ",\n";
    s += p + "\"windows\": " + std::to_string(r.windows) + ",\n";
    s += p + "\"z\": " + std::to_string(r.z) + "\n";
    s += i + 1 < records.size() ? "    },\n" : "    }\n";
  }
  return s + "  ]\n}\n";
}

void write_bench_json(const std::string& path, const std::vector<BenchRecord>& records) {
  write_text(path, bench_json_string(records));
}

}  // namespace mhar
