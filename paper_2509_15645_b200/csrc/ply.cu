// PLY point-cloud ingestion (reference: src/ply.cpp:53-199 load_ply, 201-225 save_ply; SURVEY.md
// §8f f4): the input side of init_gaussians (scene.hpp:146-195) for real scenes.
//
// The header is parsed on the host (it is text). A binary_little_endian vertex body is not parsed
// on the host at all: it streams from the file into two pinned 32 MB staging buffers (file read of
// chunk k+1 overlapping the H2D copy of chunk k) into HBM, and one decode kernel turns every
// fixed-size vertex record into x,y,z + colour floats in place, with the reference's conversions
// (value read as double, float(v) for coordinates, float(v / 255.0) for byte colours,
// float(clamp(v, 0, 1)) otherwise) and its first-non-finite-vertex error. ASCII bodies are
// tokenised on the host with strtod, as the reference does (nan/inf accepted by the tokenizer,
// rejected as coordinates). Errors carry the reference's ParseError messages (status
// GSS_ERR_PARSE).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "common.cuh"

struct gss_ply {
  std::string path;
  bool binary = false;
  int64_t body_offset = 0;  // byte offset of the first element's data (binary) / line number (ascii)
  int line_no = 0;
  struct Prop {
    std::string name, type;
    bool list = false;
    int size = 0;
  };
  struct Elem {
    std::string name;
    long count = 0;
    std::vector<Prop> props;
  };
  std::vector<Elem> elems;
  int vertex = -1;
  int ix = -1, iy = -1, iz = -1, ir = -1, ig = -1, ib = -1;
};

namespace gssd {
namespace {

// Scalar type codes shared by host and device (ply.cpp:26-51).
enum PlyType : int { kU8 = 0, kI8, kU16, kI16, kU32, kI32, kF32, kF64, kBad };

PlyType type_code(const std::string& t) {
  if (t == "uchar" || t == "uint8") return kU8;
  if (t == "char" || t == "int8") return kI8;
  if (t == "ushort" || t == "uint16") return kU16;
  if (t == "short" || t == "int16") return kI16;
  if (t == "uint" || t == "uint32") return kU32;
  if (t == "int" || t == "int32") return kI32;
  if (t == "float" || t == "float32") return kF32;
  if (t == "double" || t == "float64") return kF64;
  return kBad;
}
int type_bytes(PlyType c) {
  switch (c) {
    case kU8: case kI8: return 1;
    case kU16: case kI16: return 2;
    case kU32: case kI32: case kF32: return 4;
    case kF64: return 8;
    default: return -1;
  }
}
bool byte_colour(const std::string& t) { return t == "uchar" || t == "uint8" || t == "char" || t == "int8"; }

[[noreturn]] void parse_error(const std::string& m) { throw Error(GSS_ERR_PARSE, m); }

struct Field {
  int32_t offset;  // byte offset inside the record
  int32_t type;    // PlyType
};
struct DecodeArgs {
  Field f[6];        // x y z r g b
  int32_t byte_col[3];  // per channel: 1 byte-typed (v / 255), 0 otherwise (clamp to [0, 1])
  int32_t has_col;
  int64_t rec;       // record bytes
};

__device__ __forceinline__ double load_le(const unsigned char* p, int type) {
  // Little-endian scalar at an arbitrary byte address (records are packed; no alignment).
  uint64_t u = 0;
  const int nb = type == kU8 || type == kI8 ? 1 : type == kU16 || type == kI16 ? 2 : type == kF64 ? 8 : 4;
  for (int k = 0; k < nb; ++k) u |= (uint64_t)p[k] << (8 * k);
  switch (type) {
    case kU8: return (double)(uint8_t)u;
    case kI8: return (double)(int8_t)u;
    case kU16: return (double)(uint16_t)u;
    case kI16: return (double)(int16_t)u;
    case kU32: return (double)(uint32_t)u;
    case kI32: return (double)(int32_t)u;
    case kF32: return (double)__uint_as_float((uint32_t)u);
    default: return __longlong_as_double((long long)u);
  }
}

// One thread per vertex record: coordinates (checked finite, ply.cpp:157-161) and colours
// (ply.cpp:162-164). bad_idx receives the smallest vertex index with a non-finite coordinate.
__global__ void ply_decode_kernel(const unsigned char* body, int64_t m, DecodeArgs a, float* pos, float* col,
                                  unsigned long long* bad_idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned char* r = body + i * a.rec;
    bool fin = true;
    for (int c = 0; c < 3; ++c) {
      const double v = load_le(r + a.f[c].offset, a.f[c].type);
      fin = fin && isfinite(v);
      pos[i * 3 + c] = (float)v;
    }
    if (!fin) atomicMin(bad_idx, (unsigned long long)i);
    if (a.has_col && col) {
      for (int c = 0; c < 3; ++c) {
        const double v = load_le(r + a.f[3 + c].offset, a.f[3 + c].type);
        col[i * 3 + c] = a.byte_col[c] ? (float)(v / 255.0) : (float)(v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v));
      }
    }
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

// load_ply header (ply.cpp:53-143).
gss_ply* ply_open(const char* path, int64_t* count, int32_t* has_color) {
  require(path != nullptr, "ply: null path");
  std::ifstream in(path, std::ios::binary);
  if (!in) parse_error(std::string("ply: cannot open file: ") + path);
  auto p = std::make_unique<gss_ply>();
  p->path = path;
  std::string line;
  auto next = [&]() -> std::string {
    if (!std::getline(in, line)) parse_error("ply: unexpected end of header at line " + std::to_string(p->line_no));
    ++p->line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    return line;
  };
  if (next() != "ply") parse_error("ply: line 1: missing 'ply' magic, got '" + line + "'");
  bool have_format = false;
  for (;;) {
    const std::string l = next();
    const std::string at = "ply: line " + std::to_string(p->line_no) + ": ";
    std::istringstream ss(l);
    std::string kw;
    ss >> kw;
    if (kw.empty() || kw == "comment" || kw == "obj_info") continue;
    if (kw == "end_header") break;
    if (kw == "format") {
      std::string fmt, ver;
      ss >> fmt >> ver;
      if (fmt == "ascii") p->binary = false;
      else if (fmt == "binary_little_endian") p->binary = true;
      else parse_error(at + "unsupported format '" + l + "'");
      have_format = true;
    } else if (kw == "element") {
      gss_ply::Elem e;
      if (!(ss >> e.name >> e.count) || e.count < 0) parse_error(at + "bad element declaration '" + l + "'");
      p->elems.push_back(e);
    } else if (kw == "property") {
      if (p->elems.empty()) parse_error(at + "property before any element: '" + l + "'");
      gss_ply::Prop pr;
      std::string t;
      ss >> t;
      if (t == "list") {
        std::string ct, it;
        ss >> ct >> it >> pr.name;
        pr.list = true;
        pr.type = it;
        if (type_code(ct) == kBad || type_code(it) == kBad) parse_error(at + "bad list property '" + l + "'");
      } else {
        pr.type = t;
        ss >> pr.name;
        if (type_code(t) == kBad || pr.name.empty()) parse_error(at + "bad property '" + l + "'");
      }
      pr.size = type_bytes(type_code(pr.type));
      p->elems.back().props.push_back(pr);
    } else {
      parse_error(at + "unknown header keyword '" + l + "'");
    }
  }
  if (!have_format) parse_error("ply: header has no format line");
  for (size_t k = 0; k < p->elems.size(); ++k)
    if (p->elems[k].name == "vertex") {
      p->vertex = (int)k;
      break;
    }
  if (p->vertex < 0) parse_error("ply: no 'vertex' element in header");
  const auto& v = p->elems[p->vertex];
  if (v.count < 1) parse_error("ply: vertex element is empty");
  for (size_t k = 0; k < v.props.size(); ++k) {
    const std::string& n = v.props[k].name;
    if (n == "x") p->ix = (int)k;
    else if (n == "y") p->iy = (int)k;
    else if (n == "z") p->iz = (int)k;
    else if (n == "red" || n == "r") p->ir = (int)k;
    else if (n == "green" || n == "g") p->ig = (int)k;
    else if (n == "blue" || n == "b") p->ib = (int)k;
  }
  if (p->ix < 0 || p->iy < 0 || p->iz < 0) parse_error("ply: vertex element lacks x,y,z properties");
  p->body_offset = (int64_t)in.tellg();
  if (count) *count = v.count;
  if (has_color) *has_color = (p->ir >= 0 && p->ig >= 0 && p->ib >= 0) ? 1 : 0;
  return p.release();
}

void ply_close(gss_ply* p) { delete p; }

namespace {

// ASCII body (ply.cpp:175-193): whitespace-separated tokens, one item per non-blank line.
void read_ascii(const gss_ply* p, float* pos, float* col) {
  std::ifstream in(p->path, std::ios::binary);
  if (!in) parse_error("ply: cannot open file: " + p->path);
  in.seekg(p->body_offset);
  int line_no = p->line_no;
  const bool has_col = p->ir >= 0 && p->ig >= 0 && p->ib >= 0;
  const auto& vx = p->elems[p->vertex];
  std::vector<double> vals;
  std::string row, tok;
  for (int ei = 0; ei <= p->vertex; ++ei) {
    const auto& e = p->elems[ei];
    const bool is_vertex = ei == p->vertex;
    vals.assign(e.props.size(), 0.0);
    for (long i = 0; i < e.count; ++i) {
      do {
        if (!std::getline(in, row))
          parse_error("ply: truncated body at element '" + e.name + "' item " + std::to_string(i));
        ++line_no;
      } while (row.find_first_not_of(" \t\r\n") == std::string::npos);
      std::istringstream ss(row);
      for (size_t k = 0; k < e.props.size(); ++k) {
        if (e.props[k].list) parse_error("ply: list properties are not supported (element '" + e.name + "')");
        if (!(ss >> tok))
          parse_error("ply: line " + std::to_string(line_no) + ": expected " + std::to_string(e.props.size()) +
                      " values, got fewer");
        char* end = nullptr;
        vals[k] = std::strtod(tok.c_str(), &end);
        if (end == tok.c_str()) parse_error("ply: line " + std::to_string(line_no) + ": bad numeric token '" + tok + "'");
      }
      if (!is_vertex) continue;
      const int ci[3] = {p->ix, p->iy, p->iz};
      for (int c = 0; c < 3; ++c) {
        const double v = vals[ci[c]];
        if (!std::isfinite(v)) parse_error("ply: non-finite coordinate at vertex " + std::to_string(i));
        pos[i * 3 + c] = (float)v;
      }
      if (has_col && col) {
        const int cc[3] = {p->ir, p->ig, p->ib};
        for (int c = 0; c < 3; ++c) {
          const double v = vals[cc[c]];
          col[i * 3 + c] = byte_colour(vx.props[cc[c]].type) ? (float)(v / 255.0) : (float)std::clamp(v, 0.0, 1.0);
        }
      }
    }
  }
}

}  // namespace

// load_ply body. positions (m x 3) and colors (m x 3, may be NULL; ignored without colour
// properties) may be device or host pointers.
void ply_read(gss_ply* p, float* pos, float* col, cudaStream_t st) {
  require(p != nullptr && pos != nullptr, "ply: null argument");
  const auto& vx = p->elems[p->vertex];
  const int64_t m = vx.count;
  const bool has_col = p->ir >= 0 && p->ig >= 0 && p->ib >= 0;
  if (!has_col) col = nullptr;
  if (!p->binary) {
    // host tokenizer; device destinations receive one copy
    const bool dpos = is_device_ptr(pos), dcol = col && is_device_ptr(col);
    std::vector<float> hp(dpos ? (size_t)m * 3 : 0), hc(dcol ? (size_t)m * 3 : 0);
    read_ascii(p, dpos ? hp.data() : pos, col ? (dcol ? hc.data() : col) : nullptr);
    if (dpos) GSS_CUDA(cudaMemcpyAsync(pos, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice, st));
    if (dcol) GSS_CUDA(cudaMemcpyAsync(col, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice, st));
    if (dpos || dcol) GSS_CUDA(cudaStreamSynchronize(st));
    return;
  }
  // Binary: byte offset of the vertex records = header end + the fixed-size elements before it
  // (ply.cpp:166-174 reads and discards them; lists there are unsupported).
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw Error(GSS_ERR_CUDA, "no CUDA device: the binary PLY body is decoded on the GPU (no CPU fallback)");
  }
  std::FILE* f = std::fopen(p->path.c_str(), "rb");
  if (!f) parse_error("ply: cannot open file: " + p->path);
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, std::fclose);
  std::fseek(f, 0, SEEK_END);
  const int64_t fsize = std::ftell(f);
  int64_t off = p->body_offset;
  auto rec_bytes = [&](const gss_ply::Elem& e) {
    int64_t r = 0;
    for (const auto& pr : e.props) {
      if (pr.list && e.count > 0) parse_error("ply: list properties are not supported (element '" + e.name + "')");
      r += pr.size;
    }
    return r;
  };
  for (int ei = 0; ei < p->vertex; ++ei) {
    const auto& e = p->elems[ei];
    const int64_t r = rec_bytes(e);
    if (off + r * e.count > fsize)
      parse_error("ply: truncated body at element '" + e.name + "' item " +
                  std::to_string(r > 0 ? (fsize - off) / r : 0));
    off += r * e.count;
  }
  const int64_t rec = rec_bytes(vx);
  if (off + rec * m > fsize)
    parse_error("ply: truncated body at element 'vertex' item " + std::to_string(rec > 0 ? (fsize - off) / rec : 0));
  DecodeArgs a{};
  const int idx[6] = {p->ix, p->iy, p->iz, p->ir, p->ig, p->ib};
  for (int c = 0; c < 6; ++c) {
    if (idx[c] < 0) continue;
    int32_t o = 0;
    for (int k = 0; k < idx[c]; ++k) o += vx.props[k].size;
    a.f[c] = Field{o, (int32_t)type_code(vx.props[idx[c]].type)};
  }
  a.has_col = has_col ? 1 : 0;
  // ply.cpp:150-152: byte or float normalisation by each colour property's own type
  for (int c = 0; c < 3; ++c) a.byte_col[c] = has_col && byte_colour(vx.props[idx[3 + c]].type) ? 1 : 0;
  a.rec = rec;
  // Stream the body into HBM through two pinned chunks (file read of k+1 overlaps the copy of k).
  const int64_t body = rec * m;
  unsigned char* dbody = nullptr;
  GSS_CUDA(cudaMalloc(&dbody, (size_t)std::max<int64_t>(body, 1)));
  std::unique_ptr<unsigned char, cudaError_t (*)(void*)> dguard(dbody, cudaFree);
  const int64_t chunk = int64_t(32) << 20;
  unsigned char* stage[2] = {nullptr, nullptr};
  cudaEvent_t done[2];
  for (int b = 0; b < 2; ++b) {
    GSS_CUDA(cudaHostAlloc((void**)&stage[b], (size_t)chunk, cudaHostAllocDefault));
    GSS_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
  }
  auto free_stage = [&]() {
    for (int b = 0; b < 2; ++b) {
      cudaEventSynchronize(done[b]);
      cudaEventDestroy(done[b]);
      cudaFreeHost(stage[b]);
    }
  };
  try {
    std::fseek(f, (long)off, SEEK_SET);
    for (int64_t at = 0, k = 0; at < body; at += chunk, ++k) {
      const int b = (int)(k & 1);
      const int64_t nb = std::min(chunk, body - at);
      GSS_CUDA(cudaEventSynchronize(done[b]));  // the copy that last used this buffer is done
      if ((int64_t)std::fread(stage[b], 1, (size_t)nb, f) != nb) parse_error("ply: read error in body of " + p->path);
      GSS_CUDA(cudaMemcpyAsync(dbody + at, stage[b], (size_t)nb, cudaMemcpyHostToDevice, st));
      GSS_CUDA(cudaEventRecord(done[b], st));
    }
  } catch (...) {
    free_stage();
    throw;
  }
  free_stage();
  const bool dpos = is_device_ptr(pos), dcol = col && is_device_ptr(col);
  float* dp = pos;
  float* dc = col;
  std::unique_ptr<float, cudaError_t (*)(void*)> tp(nullptr, cudaFree), tc(nullptr, cudaFree);
  if (!dpos) {
    GSS_CUDA(cudaMalloc(&dp, (size_t)m * 12));
    tp.reset(dp);
  }
  if (col && !dcol) {
    GSS_CUDA(cudaMalloc(&dc, (size_t)m * 12));
    tc.reset(dc);
  }
  unsigned long long* bad = nullptr;
  GSS_CUDA(cudaMalloc(&bad, 8));
  std::unique_ptr<unsigned long long, cudaError_t (*)(void*)> bguard(bad, cudaFree);
  GSS_CUDA(cudaMemsetAsync(bad, 0xff, 8, st));
  const int blocks = (int)std::min<int64_t>(ceil_div(m, 256), (int64_t)sm_count() * 8);
  ply_decode_kernel<<<blocks, 256, 0, st>>>(dbody, m, a, dp, dc, bad);
  GSS_LAUNCHED();
  unsigned long long first_bad = 0;
  GSS_CUDA(cudaMemcpyAsync(&first_bad, bad, 8, cudaMemcpyDeviceToHost, st));
  if (!dpos) GSS_CUDA(cudaMemcpyAsync(pos, dp, (size_t)m * 12, cudaMemcpyDeviceToHost, st));
  if (col && !dcol) GSS_CUDA(cudaMemcpyAsync(col, dc, (size_t)m * 12, cudaMemcpyDeviceToHost, st));
  GSS_CUDA(cudaStreamSynchronize(st));
  if (first_bad != ~0ull) parse_error("ply: non-finite coordinate at vertex " + std::to_string(first_bad));
}

// save_ply (ply.cpp:201-225): host writer (positions / colours are host arrays).
void save_ply(const char* path, const float* pos, const float* col, int64_t m, bool binary) {
  require(path && (m == 0 || pos), "ply: null argument");
  std::ofstream out(path, std::ios::binary);
  if (!out) parse_error(std::string("ply: cannot open for writing: ") + path);
  out << "ply\nformat " << (binary ? "binary_little_endian" : "ascii") << " 1.0\n";
  out << "element vertex " << m << "\n";
  out << "property float x\nproperty float y\nproperty float z\n";
  out << "property uchar red\nproperty uchar green\nproperty uchar blue\n";
  out << "end_header\n";
  auto cb = [&](int64_t i, int c) -> uint8_t {
    const float v = col ? col[i * 3 + c] : 0.5f;
    return (uint8_t)std::clamp((int)std::lround(v * 255.0f), 0, 255);
  };
  for (int64_t i = 0; i < m; ++i) {
    if (binary) {
      out.write(reinterpret_cast<const char*>(pos + i * 3), 12);
      const uint8_t rgb[3] = {cb(i, 0), cb(i, 1), cb(i, 2)};
      out.write(reinterpret_cast<const char*>(rgb), 3);
    } else {
      out << pos[i * 3] << " " << pos[i * 3 + 1] << " " << pos[i * 3 + 2] << " " << int(cb(i, 0)) << " "
          << int(cb(i, 1)) << " " << int(cb(i, 2)) << "\n";
    }
  }
}

}  // namespace gssd
