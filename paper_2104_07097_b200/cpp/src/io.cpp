// Sample output: CSV / manifest / binary sidecar (host side, like the
// reference's src/io.cpp).  JSON is written by hand in the layout of
// nlohmann::json::dump(2) with sorted keys.
#include "mhar/io.hpp"

#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string_view>
#include <vector>

namespace mhar {
namespace {

// Whole-file output through C stdio; any short write or close failure is an
// IO_FAILURE naming the path and the errno text.
void save_bytes(const std::string& path, std::string_view bytes) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) raise(ErrorCode::io_failure, path + ": open for writing: " + std::strerror(errno));
  const size_t put = bytes.empty() ? 0 : std::fwrite(bytes.data(), 1, bytes.size(), f);
  const int closed = std::fclose(f);
  if (put != bytes.size() || closed != 0)
    raise(ErrorCode::io_failure, path + ": short write (" + std::to_string(put) + " of " +
                                     std::to_string(bytes.size()) + " bytes)");
}

std::string load_bytes(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) raise(ErrorCode::io_failure, path + ": open for reading: " + std::strerror(errno));
  std::string data;
  char chunk[1 << 16];
  size_t got = 0;
  while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) data.append(chunk, got);
  const bool bad = std::ferror(f) != 0;
  std::fclose(f);
  if (bad) raise(ErrorCode::io_failure, path + ": read error");
  return data;
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

// Appends the shortest round-trip text of v (std::to_chars without a format
// argument is specified to produce exactly that).
void append_number(std::string& out, double v) {
  char buf[32];
  char* end = std::to_chars(buf, buf + sizeof(buf), v).ptr;
  out.append(buf, end);
}

}  // namespace

std::string format_double(double value) {
  std::string s;
  append_number(s, value);
  return s;
}

// Header "x1,...,xn", then one line per collected point, cells separated by
// commas, numbers in shortest round-trip form.  Byte-identical output for
// identical matrices is what makes reruns comparable with cmp (acceptance #9).
std::string sample_csv_string(const Matrix& samples) {
  const Index rows = samples.rows(), cols = samples.cols();
  std::string text;
  text.reserve(static_cast<size_t>(rows * cols) * 20 + static_cast<size_t>(cols) * 6 + 1);
  for (Index j = 1; j <= cols; ++j) {
    text += j == 1 ? "x" : ",x";
    text += std::to_string(j);
  }
  text.push_back('\n');
  for (Index i = 0; i < rows; ++i) {
    for (Index j = 0; j < cols; ++j) {
      if (j) text.push_back(',');
      append_number(text, samples(i, j));
    }
    text.push_back('\n');
  }
  return text;
}

void write_sample_csv(const std::string& path, const Matrix& samples) {
  save_bytes(path, sample_csv_string(samples));
}

// One pass over the file image: the header fixes the column count, every
// non-empty line after it must carry exactly that many numbers that parse
// completely (from_chars) -- else IO_FAILURE with the 1-based line number.
Matrix read_sample_csv(const std::string& path) {
  const std::string text = load_bytes(path);
  const char* cur = text.data();
  const char* const stop = cur + text.size();
  const char* eol = static_cast<const char*>(std::memchr(cur, '\n', text.size()));
  const char* header_end = eol ? eol : stop;
  if (header_end == cur) raise(ErrorCode::io_failure, path + ": no header line");
  const Index width = 1 + std::count(cur, header_end, ',');
  cur = eol ? eol + 1 : stop;
  std::vector<double> cells;
  Index line_no = 1;
  while (cur < stop) {
    ++line_no;
    const char* line_end = static_cast<const char*>(std::memchr(cur, '\n', stop - cur));
    if (!line_end) line_end = stop;
    if (line_end != cur) {
      Index fields = 0;
      const char* field = cur;
      for (;;) {
        const char* comma = std::find(field, line_end, ',');
        double v = 0.0;
        const auto r = std::from_chars(field, comma, v);
        if (r.ec != std::errc{} || r.ptr != comma || field == comma)
          raise(ErrorCode::io_failure, path + ":" + std::to_string(line_no) + ": '" +
                                           std::string(field, comma) + "' is not a number");
        cells.push_back(v);
        ++fields;
        if (comma == line_end) break;
        field = comma + 1;
      }
      if (fields != width)
        raise(ErrorCode::io_failure, path + ":" + std::to_string(line_no) + ": " +
                                         std::to_string(fields) + " values where the header names " +
                                         std::to_string(width) + " columns");
    }
    cur = line_end == stop ? stop : line_end + 1;
  }
  const Index rows = static_cast<Index>(cells.size()) / width;
  Matrix out(rows, width);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < width; ++j) out(i, j) = cells[static_cast<size_t>(i * width + j)];
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
  save_bytes(path, manifest_string(set, polytope_source, samples_path));
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
  save_bytes(path, bench_csv_string(records));
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
  save_bytes(path, bench_json_string(records));
}

}  // namespace mhar
