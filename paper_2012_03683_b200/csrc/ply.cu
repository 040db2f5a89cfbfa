// PLY ingest straight into a device cloud.
//
// Reference: read_ply, /root/reference/proj/src/cloud_io.cpp:141-297 (header
// grammar, schema inference, error texts) and assemble() :102-138 (feature
// order colour, intensity, semantic_0..K-1; 8/16-bit values / 255 / 65535).
//
// B200 path: the host parses the header and reads the vertex block with one
// read into pinned memory (binary_little_endian), or parses ASCII rows into
// FP64 columns; one copy to the device; a decode kernel turns the records into
// FP64 positions and padded FP32 feature rows; the bbox, the 63-bit Morton
// keys (the same formula as the host staging path, cloud_stage) and a CUB
// radix sort (stable: ties by point index) give the engine's spatial order,
// and a gather writes the device cloud layout. A cloud read this way is
// bitwise the cloud kreg_cloud_create makes from read_ply's PointCloud.
#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "engine_host.hpp"

namespace kreg_host {

struct ParseError : Error {
  ParseError(const std::string& path, int line, const std::string& what)
      : Error(KREG_PARSE_ERROR, path + ":" + std::to_string(line) + ": " + what) {}
};

namespace {

enum PlyType : int { kI8, kU8, kI16, kU16, kI32, kU32, kF32, kF64 };

std::optional<PlyType> parse_type(const std::string& s) {
  if (s == "char" || s == "int8") return kI8;
  if (s == "uchar" || s == "uint8") return kU8;
  if (s == "short" || s == "int16") return kI16;
  if (s == "ushort" || s == "uint16") return kU16;
  if (s == "int" || s == "int32") return kI32;
  if (s == "uint" || s == "uint32") return kU32;
  if (s == "float" || s == "float32") return kF32;
  if (s == "double" || s == "float64") return kF64;
  return std::nullopt;
}

int type_size(int t) {
  switch (t) {
    case kI8: case kU8: return 1;
    case kI16: case kU16: return 2;
    case kI32: case kU32: case kF32: return 4;
    default: return 8;
  }
}

double int_norm(int t) { return t == kU8 ? 255.0 : t == kU16 ? 65535.0 : 1.0; }

struct Prop {
  std::string name;
  int type = kF32;
};
struct Element {
  std::string name;
  size_t count = 0;
  std::vector<Prop> props;
  bool has_list = false;
};

constexpr int kMaxPlyFeat = 64;
// Decode description (kernel argument): record layout of x, y, z and of each
// feature value, its type, normalisation and padded row position.
struct PlyDecode {
  int n;
  int record;  // bytes per vertex record
  int xyz_off[3], xyz_type[3];
  int n_feat;
  int f_off[kMaxPlyFeat], f_type[kMaxPlyFeat], f_dst[kMaxPlyFeat];
  double f_norm[kMaxPlyFeat];
  int fstride;
};

__device__ __forceinline__ double decode(const unsigned char* p, int t) {
  switch (t) {
    case kI8: return (double)*reinterpret_cast<const signed char*>(p);
    case kU8: return (double)*p;
    case kI16: { short v; memcpy(&v, p, 2); return (double)v; }
    case kU16: { unsigned short v; memcpy(&v, p, 2); return (double)v; }
    case kI32: { int v; memcpy(&v, p, 4); return (double)v; }
    case kU32: { unsigned v; memcpy(&v, p, 4); return (double)v; }
    case kF32: { float v; memcpy(&v, p, 4); return (double)v; }
    default: { double v; memcpy(&v, p, 8); return v; }
  }
}

// bit patterns of doubles that order like the values (bbox by integer atomics)
__device__ __forceinline__ unsigned long long ordered(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double unordered(unsigned long long o) {
  const unsigned long long b = (o >> 63) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o;
  double v;
  memcpy(&v, &b, 8);
  return v;
}

// records -> FP64 positions (x, y, z arrays, input order), padded FP32 feature
// rows, bbox (ordered bits: lo[3] as max of the complement, hi[3])
__global__ void k_ply_decode(const unsigned char* __restrict__ raw, PlyDecode D, double* px, double* py, double* pz,
                             float* feat, unsigned long long* box) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double v[3] = {0.0, 0.0, 0.0};
  const bool ok = i < D.n;
  if (ok) {
    const unsigned char* r = raw + (size_t)i * D.record;
    for (int k = 0; k < 3; ++k) v[k] = decode(r + D.xyz_off[k], D.xyz_type[k]);
    px[i] = v[0];
    py[i] = v[1];
    pz[i] = v[2];
    float* row = feat + (size_t)i * D.fstride;
    for (int d = 0; d < D.fstride; ++d) row[d] = 0.0f;
    for (int d = 0; d < D.n_feat; ++d) row[D.f_dst[d]] = (float)(decode(r + D.f_off[d], D.f_type[d]) / D.f_norm[d]);
  }
  // block bbox, then one atomic per block and bound
  __shared__ unsigned long long s_lo[3], s_hi[3];
  if (threadIdx.x < 3) s_lo[threadIdx.x] = 0ull, s_hi[threadIdx.x] = 0ull;
  __syncthreads();
  if (ok)
    for (int k = 0; k < 3; ++k) {
      atomicMax(&s_lo[k], ~ordered(v[k]));
      atomicMax(&s_hi[k], ordered(v[k]));
    }
  __syncthreads();
  if (threadIdx.x < 3) {
    atomicMax(&box[threadIdx.x], s_lo[threadIdx.x]);
    atomicMax(&box[3 + threadIdx.x], s_hi[threadIdx.x]);
  }
}

__device__ __forceinline__ unsigned long long spread3_d(unsigned long long v) {
  v &= 0x1FFFFF;
  v = (v | v << 32) & 0x1F00000000FFFFULL;
  v = (v | v << 16) & 0x1F0000FF0000FFULL;
  v = (v | v << 8) & 0x100F00F00F00F00FULL;
  v = (v | v << 4) & 0x10C30C30C30C30C3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}

// Morton key of point i (engine_host.cu cloud_stage, same FP64 arithmetic)
__global__ void k_ply_keys(const double* px, const double* py, const double* pz, int n, const unsigned long long* box,
                           unsigned long long* keys, int* idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = unordered(~box[k]);
    hi[k] = unordered(box[3 + k]);
  }
  double span = 0.0;
  for (int k = 0; k < 3; ++k) span = fmax(span, hi[k] - lo[k]);
  const double s = span > 0 ? (double)((1 << 21) - 1) / span : 0.0;
  const double p[3] = {px[i], py[i], pz[i]};
  unsigned long long m = 0;
  for (int k = 0; k < 3; ++k) {
    const double f = __dmul_rn(p[k] - lo[k], s);
    const unsigned long long q = isfinite(f) ? (unsigned long long)fmin(fmax(f, 0.0), 2097151.0) : 0ull;
    m |= spread3_d(q) << k;
  }
  keys[i] = m;
  idx[i] = i;
}

__global__ void k_ply_gather(const double* px, const double* py, const double* pz, const float* feat, int fstride,
                             const int* order, int n, double* x, double* y, double* z, double4* xw, float* frow) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = order[r];
  x[r] = px[i];
  y[r] = py[i];
  z[r] = pz[i];
  xw[r] = make_double4(px[i], py[i], pz[i], 0.0);
  for (int d = 0; d < fstride; ++d) frow[(size_t)r * fstride + d] = feat[(size_t)i * fstride + d];
}

}  // namespace

kreg_cloud* cloud_read_ply(kreg_ctx* ctx, const std::string& path, std::string* warnings) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(KREG_RUNTIME_ERROR, "cannot open " + path);
  int line_no = 0;
  std::string line;
  auto next_line = [&]() {
    if (!std::getline(in, line)) throw ParseError(path, line_no, "unexpected end of header");
    if (!line.empty() && line.back() == '\r') line.pop_back();
    ++line_no;
  };
  // header (cloud_io.cpp:152-197)
  next_line();
  if (line != "ply") throw ParseError(path, 1, "missing 'ply' magic");
  bool binary = false, format_seen = false;
  std::vector<Element> elements;
  for (;;) {
    next_line();
    std::istringstream ls(line);
    std::string word;
    ls >> word;
    if (word == "comment" || word == "obj_info" || word.empty()) continue;
    if (word == "format") {
      std::string fmt, version;
      ls >> fmt >> version;
      if (fmt == "ascii") binary = false;
      else if (fmt == "binary_little_endian") binary = true;
      else throw ParseError(path, line_no, "unsupported format '" + fmt + "'");
      format_seen = true;
    } else if (word == "element") {
      Element el;
      if (!(ls >> el.name >> el.count)) throw ParseError(path, line_no, "malformed element line");
      elements.push_back(el);
    } else if (word == "property") {
      if (elements.empty()) throw ParseError(path, line_no, "property before any element");
      std::string tw;
      ls >> tw;
      if (tw == "list") {
        elements.back().has_list = true;
        continue;
      }
      const auto t = parse_type(tw);
      if (!t) throw ParseError(path, line_no, "unknown property type '" + tw + "'");
      std::string name;
      if (!(ls >> name)) throw ParseError(path, line_no, "property without a name");
      elements.back().props.push_back({name, *t});
    } else if (word == "end_header") {
      break;
    } else {
      throw ParseError(path, line_no, "unrecognized header keyword '" + word + "'");
    }
  }
  if (!format_seen) throw ParseError(path, line_no, "missing format line");
  size_t vi = 0;
  while (vi < elements.size() && elements[vi].name != "vertex") ++vi;
  if (vi == elements.size()) throw ParseError(path, line_no, "no vertex element");
  const Element& vertex = elements[vi];
  if (vertex.has_list) throw ParseError(path, line_no, "list properties on vertices unsupported");
  for (size_t e = 0; e < vi; ++e)
    if (elements[e].has_list)
      throw ParseError(path, line_no, "cannot skip list element '" + elements[e].name + "' before vertex");

  // vertex layout and schema (cloud_io.cpp:224-257, assemble :102-138)
  int cx = -1, cy = -1, cz = -1, rgb[3] = {-1, -1, -1}, inten = -1;
  std::map<int, int> sem_cols;
  for (size_t p = 0; p < vertex.props.size(); ++p) {
    const std::string& nm = vertex.props[p].name;
    const int col = static_cast<int>(p);
    if (nm == "x") cx = col;
    else if (nm == "y") cy = col;
    else if (nm == "z") cz = col;
    else if (nm == "red") rgb[0] = col;
    else if (nm == "green") rgb[1] = col;
    else if (nm == "blue") rgb[2] = col;
    else if (nm == "intensity") inten = col;
    else if (nm.rfind("semantic_", 0) == 0) {
      try {
        sem_cols[std::stoi(nm.substr(9))] = col;
      } catch (const std::exception&) {
        throw ParseError(path, line_no, "malformed semantic property '" + nm + "'");
      }
    } else if (warnings) {
      *warnings += "property '" + nm + "' skipped\n";
    }
  }
  if (cx < 0 || cy < 0 || cz < 0) throw ParseError(path, line_no, "vertex element lacks x/y/z properties");
  const bool any_rgb = rgb[0] >= 0 || rgb[1] >= 0 || rgb[2] >= 0;
  if (any_rgb && (rgb[0] < 0 || rgb[1] < 0 || rgb[2] < 0))
    throw ParseError(path, line_no, "incomplete red/green/blue property triple");
  std::vector<int> sem;
  for (const auto& [cls, col] : sem_cols) {
    if (cls != static_cast<int>(sem.size()))
      throw ParseError(path, line_no, "semantic properties must be contiguous from semantic_0");
    sem.push_back(col);
  }
  std::vector<kreg_channel> chans;
  std::vector<int> feat_cols;
  if (any_rgb) {
    chans.push_back({"color", 3, KREG_KIND_COLOR});
    feat_cols.insert(feat_cols.end(), rgb, rgb + 3);
  }
  if (inten >= 0) {
    chans.push_back({"intensity", 1, KREG_KIND_INTENSITY});
    feat_cols.push_back(inten);
  }
  if (!sem.empty()) {
    chans.push_back({"semantic", static_cast<int>(sem.size()), KREG_KIND_SEMANTIC});
    feat_cols.insert(feat_cols.end(), sem.begin(), sem.end());
  }
  if (vertex.count > static_cast<size_t>(INT32_MAX)) throw Error(KREG_INVALID_ARGUMENT, "read_ply: too many vertices");
  const int n = static_cast<int>(vertex.count);

  // metadata (schema validation, padded rows) through the common path
  kreg_cloud_view view{};
  view.n = 0;
  view.dim = static_cast<int>(feat_cols.size());
  view.channels = chans.data();
  view.n_channels = static_cast<int>(chans.size());
  std::unique_ptr<kreg_cloud> c(cloud_describe(ctx, &view));
  c->n = n;

  // vertex block -> pinned memory (one read), record layout for the decoder
  PlyDecode D{};
  D.n = n;
  D.fstride = c->fstride;
  std::vector<int> col_off(vertex.props.size()), col_type(vertex.props.size());
  PinnedBuf<unsigned char> pin;
  if (binary) {
    for (size_t e = 0; e < vi; ++e) {  // skip fixed-size elements before the vertices
      size_t rec = 0;
      for (const auto& pr : elements[e].props) rec += static_cast<size_t>(type_size(pr.type));
      in.seekg(static_cast<std::streamoff>(rec * elements[e].count), std::ios::cur);
    }
    int off = 0;
    for (size_t p = 0; p < vertex.props.size(); ++p) {
      col_off[p] = off;
      col_type[p] = vertex.props[p].type;
      off += type_size(vertex.props[p].type);
    }
    D.record = off;
    const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(off);
    pin.ensure(bytes + 16);
    in.read(reinterpret_cast<char*>(pin.ptr), static_cast<std::streamsize>(bytes));
    if (static_cast<size_t>(in.gcount()) != bytes) throw ParseError(path, line_no, "truncated binary vertex data");
  } else {
    for (size_t e = 0; e < vi; ++e)
      for (size_t r = 0; r < elements[e].count; ++r) next_line();
    const size_t P = vertex.props.size();
    for (size_t p = 0; p < P; ++p) {
      col_off[p] = static_cast<int>(8 * p);
      col_type[p] = kF64;
    }
    D.record = static_cast<int>(8 * P);
    pin.ensure(static_cast<size_t>(n) * 8 * P + 16);
    double* vals = reinterpret_cast<double*>(pin.ptr);
    for (int r = 0; r < n; ++r) {
      next_line();
      std::istringstream ls(line);
      for (size_t p = 0; p < P; ++p)
        if (!(ls >> vals[static_cast<size_t>(r) * P + p])) throw ParseError(path, line_no, "vertex line has too few values");
      std::string extra;
      if (ls >> extra) throw ParseError(path, line_no, "trailing data '" + extra + "' on vertex line");
    }
  }
  const int pcols[3] = {cx, cy, cz};
  for (int k = 0; k < 3; ++k) {
    D.xyz_off[k] = col_off[static_cast<size_t>(pcols[k])];
    D.xyz_type[k] = col_type[static_cast<size_t>(pcols[k])];
  }
  D.n_feat = static_cast<int>(feat_cols.size());
  if (D.n_feat > kMaxPlyFeat) throw Error(KREG_INVALID_ARGUMENT, "read_ply: too many feature properties");
  {
    int d = 0;
    for (int k = 0; k < view.n_channels; ++k)
      for (int e = 0; e < chans[static_cast<size_t>(k)].dim; ++e, ++d) {
        const int col = feat_cols[static_cast<size_t>(d)];
        D.f_off[d] = col_off[static_cast<size_t>(col)];
        D.f_type[d] = col_type[static_cast<size_t>(col)];
        // colour and intensity integers are normalised, semantic values kept (assemble)
        D.f_norm[d] = chans[static_cast<size_t>(k)].kind == KREG_KIND_SEMANTIC ? 1.0 : int_norm(D.f_type[d]);
        D.f_dst[d] = c->chan_off[static_cast<size_t>(k)] + e;
      }
  }

  // device: decode, bbox, Morton keys, radix sort, gather
  KREG_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t raw_bytes = static_cast<size_t>(n) * static_cast<size_t>(D.record);
  DevBuf<unsigned char> d_raw;
  DevBuf<double> d_pos;
  DevBuf<float> d_feat;
  DevBuf<unsigned long long> d_box, d_keys, d_keys2;
  DevBuf<int> d_idx, d_order;
  d_raw.ensure(raw_bytes + 16, false, 1.0);
  d_pos.ensure(3 * static_cast<size_t>(n) + 3, false, 1.0);
  d_feat.ensure(static_cast<size_t>(n) * c->fstride + 4, false, 1.0);
  d_box.ensure(6, true, 1.0);
  c->x.ensure(static_cast<size_t>(n) + 1, false, 1.0);
  c->y.ensure(static_cast<size_t>(n) + 1, false, 1.0);
  c->z.ensure(static_cast<size_t>(n) + 1, false, 1.0);
  c->xw.ensure(static_cast<size_t>(n) + 1, false, 1.0);
  c->feat.ensure(cloud_stage_floats(c.get()), false, 1.0);
  c->order.resize(static_cast<size_t>(n));
  c->rank.resize(static_cast<size_t>(n));
  if (n > 0) {
    ctx->h2d_bytes += static_cast<long long>(raw_bytes);
    KREG_CUDA(cudaMemcpyAsync(d_raw.ptr, pin.ptr, raw_bytes, cudaMemcpyHostToDevice, st));
    double* px = d_pos.ptr;
    double* py = px + n;
    double* pz = py + n;
    const int T = 256, B = (n + T - 1) / T;
    k_ply_decode<<<B, T, 0, st>>>(d_raw.ptr, D, px, py, pz, d_feat.ptr, d_box.ptr);
    d_keys.ensure(static_cast<size_t>(n), false, 1.0);
    d_keys2.ensure(static_cast<size_t>(n), false, 1.0);
    d_idx.ensure(static_cast<size_t>(n), false, 1.0);
    d_order.ensure(static_cast<size_t>(n), false, 1.0);
    k_ply_keys<<<B, T, 0, st>>>(px, py, pz, n, d_box.ptr, d_keys.ptr, d_idx.ptr);
    size_t tmp_bytes = 0;
    KREG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_keys.ptr, d_keys2.ptr, d_idx.ptr, d_order.ptr, n,
                                              0, 63, st));
    DevBuf<unsigned char> d_tmp;
    d_tmp.ensure(tmp_bytes + 16, false, 1.0);
    KREG_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp.ptr, tmp_bytes, d_keys.ptr, d_keys2.ptr, d_idx.ptr, d_order.ptr,
                                              n, 0, 63, st));
    k_ply_gather<<<B, T, 0, st>>>(px, py, pz, d_feat.ptr, c->fstride, d_order.ptr, n, c->x.ptr, c->y.ptr, c->z.ptr,
                                  c->xw.ptr, c->feat.ptr);
    kreg_dev::note_launches(3);
    unsigned long long box[6];
    KREG_CUDA(cudaMemcpyAsync(box, d_box.ptr, sizeof(box), cudaMemcpyDeviceToHost, st));
    KREG_CUDA(cudaMemcpyAsync(c->order.data(), d_order.ptr, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    std::vector<double> small;
    if (n <= 2000) {  // the exact O(N^2) diameter needs the positions (point_cloud.cpp:69-87)
      small.resize(3 * static_cast<size_t>(n));
      KREG_CUDA(cudaMemcpyAsync(small.data(), px, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
    }
    KREG_CUDA(cudaGetLastError());
    KREG_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < 3; ++k) {
      c->lo[k] = unordered(~box[k]);
      c->hi[k] = unordered(box[3 + k]);
    }
    for (int r = 0; r < n; ++r) c->rank[static_cast<size_t>(c->order[static_cast<size_t>(r)])] = r;
    if (n <= 2000) {
      std::vector<double> xyz(3 * static_cast<size_t>(n));
      for (int i = 0; i < n; ++i) {
        xyz[3 * static_cast<size_t>(i)] = small[static_cast<size_t>(i)];
        xyz[3 * static_cast<size_t>(i) + 1] = small[static_cast<size_t>(n + i)];
        xyz[3 * static_cast<size_t>(i) + 2] = small[static_cast<size_t>(2 * n + i)];
      }
      c->diam = diameter_host(xyz.data(), n);
    } else {
      const double d0 = c->hi[0] - c->lo[0], d1 = c->hi[1] - c->lo[1], d2 = c->hi[2] - c->lo[2];
      c->diam = std::sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    }
  }
  return c.release();
}

// Positions (FP64, exact) and features (the device's FP32 values) back in the
// original point order.
void cloud_download(const kreg_cloud* c, double* xyz, double* features) {
  const int n = c->n, fs = c->fstride;
  std::vector<double> x(static_cast<size_t>(n)), y(static_cast<size_t>(n)), z(static_cast<size_t>(n));
  std::vector<float> f(static_cast<size_t>(n) * fs);
  KREG_CUDA(cudaSetDevice(c->ctx->device));
  if (n) {
    KREG_CUDA(cudaMemcpyAsync(x.data(), c->x.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, c->ctx->stream));
    KREG_CUDA(cudaMemcpyAsync(y.data(), c->y.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, c->ctx->stream));
    KREG_CUDA(cudaMemcpyAsync(z.data(), c->z.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, c->ctx->stream));
    if (fs)
      KREG_CUDA(cudaMemcpyAsync(f.data(), c->feat.ptr, sizeof(float) * f.size(), cudaMemcpyDeviceToHost, c->ctx->stream));
    KREG_CUDA(cudaStreamSynchronize(c->ctx->stream));
  }
  for (int r = 0; r < n; ++r) {
    const int i = c->order[static_cast<size_t>(r)];
    if (xyz) {
      xyz[3 * static_cast<size_t>(i)] = x[static_cast<size_t>(r)];
      xyz[3 * static_cast<size_t>(i) + 1] = y[static_cast<size_t>(r)];
      xyz[3 * static_cast<size_t>(i) + 2] = z[static_cast<size_t>(r)];
    }
    if (features) {
      int at = 0;
      for (size_t k = 0; k < c->schema.size(); ++k)
        for (int d = 0; d < c->schema[k].dim; ++d)
          features[static_cast<size_t>(i) * c->dim + at++] = f[static_cast<size_t>(r) * fs + c->chan_off[k] + d];
    }
  }
}

}  // namespace kreg_host
