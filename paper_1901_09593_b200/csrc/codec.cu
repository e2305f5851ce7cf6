// Wire formats either side of the disparity path:
// PGM/PPM decode (host, and binary payloads on the device), PFM decode and
// encode, binary PGM encode.  Semantics follow the reference's formats.py
// (file:line cited per function); error classes map to its exception
// hierarchy through the MSHBM_ERR_* decode codes, with the same messages.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/mshbm.h"

namespace mshbm {
void set_global_error(const std::string& msg);   // api.cu
}

namespace {

using mshbm::set_global_error;

int decode_fail(int code, const char* fmt, ...) {
  char buf[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  set_global_error(buf);
  return code;
}

// formats.py:35 whitespace set
bool is_ws(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == 0x0b || c == 0x0c;
}

// Python-style repr of a short byte token, for messages: b'...'
std::string brepr(const uint8_t* p, int64_t n) {
  std::string s = "b'";
  for (int64_t i = 0; i < n && i < 40; ++i) {
    const uint8_t c = p[i];
    if (c == '\\' || c == '\'') {
      s += '\\';
      s += (char)c;
    } else if (c >= 32 && c < 127) {
      s += (char)c;
    } else {
      char h[8];
      snprintf(h, sizeof h, "\\x%02x", c);
      s += h;
    }
  }
  return s + "'";
}

// formats.py:95-112: next whitespace-delimited token, '#' comments skipped.
// Returns MSHBM_OK or MSHBM_ERR_MALFORMED at end of input.
int next_token(const uint8_t* buf, int64_t n, int64_t* pos, int64_t* start, int64_t* len) {
  int64_t p = *pos;
  while (p < n) {
    if (is_ws(buf[p])) {
      ++p;
    } else if (buf[p] == '#') {
      while (p < n && buf[p] != '\r' && buf[p] != '\n') ++p;
    } else {
      break;
    }
  }
  if (p >= n) return decode_fail(MSHBM_ERR_MALFORMED, "unexpected end of file in header");
  *start = p;
  while (p < n && !is_ws(buf[p]) && buf[p] != '#') ++p;
  *len = p - *start;
  *pos = p;
  return MSHBM_OK;
}

// int(token) for the header fields: optional sign, decimal digits
// (saturating; out-of-range values fail the later range checks)
bool parse_int(const uint8_t* p, int64_t n, int64_t* out) {
  int64_t i = 0;
  bool neg = false;
  if (i < n && (p[i] == '+' || p[i] == '-')) neg = p[i++] == '-';
  if (i >= n) return false;
  int64_t v = 0;
  for (; i < n; ++i) {
    if (p[i] < '0' || p[i] > '9') return false;
    v = v > (INT64_MAX - 9) / 10 ? INT64_MAX : v * 10 + (p[i] - '0');
  }
  *out = neg ? -v : v;
  return true;
}

int token_int(const uint8_t* buf, int64_t n, int64_t* pos, const char* what, int64_t* out) {
  int64_t s, l;
  int st = next_token(buf, n, pos, &s, &l);
  if (st) return st;
  if (!parse_int(buf + s, l, out))
    return decode_fail(MSHBM_ERR_MALFORMED, "non-numeric %s: %s", what, brepr(buf + s, l).c_str());
  return MSHBM_OK;
}

// BT.601 luma (formats.py:38)
constexpr double kLuma[3] = {0.299, 0.587, 0.114};

__global__ void pnm_decode_kernel(const uint8_t* payload, int h, int w, int channels,
                                  int itemsize, int maxval, float* out, int64_t ld, int* bad) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  const int64_t base = ((int64_t)y * w + x) * channels;
  double s[3];
  for (int c = 0; c < channels; ++c) {
    const int64_t o = (base + c) * itemsize;
    const int v = itemsize == 2 ? (payload[o] << 8) | payload[o + 1] : payload[o];
    if (v > maxval) atomicExch(bad, 1);
    s[c] = (double)v;
  }
  const double g = channels == 3 ? (s[0] * 0.299 + s[1] * 0.587) + s[2] * 0.114 : s[0];
  out[(int64_t)y * ld + x] = (float)(g / (double)maxval);
}

}  // namespace

extern "C" {

// formats.py:123-190 (header part)
int mshbm_pnm_parse(const uint8_t* buf, int64_t len, mshbm_pnm_header* hdr) {
  if (!buf || !hdr || len < 0) return decode_fail(MSHBM_ERR_VALUE, "null buffer");
  int64_t pos = 0, s, l;
  int st = next_token(buf, len, &pos, &s, &l);
  if (st) return st;
  const bool p2 = l == 2 && buf[s] == 'P' && buf[s + 1] == '2';
  const bool p3 = l == 2 && buf[s] == 'P' && buf[s + 1] == '3';
  const bool p5 = l == 2 && buf[s] == 'P' && buf[s + 1] == '5';
  const bool p6 = l == 2 && buf[s] == 'P' && buf[s + 1] == '6';
  if (!(p2 || p3 || p5 || p6))
    return decode_fail(MSHBM_ERR_MALFORMED, "unsupported PNM magic %s", brepr(buf + s, l).c_str());
  int64_t width, height, maxval;
  if ((st = token_int(buf, len, &pos, "width", &width))) return st;
  if ((st = token_int(buf, len, &pos, "height", &height))) return st;
  if ((st = token_int(buf, len, &pos, "maxval", &maxval))) return st;
  if (width <= 0 || height <= 0)
    return decode_fail(MSHBM_ERR_MALFORMED, "bad dimensions %lldx%lld", (long long)width,
                       (long long)height);
  if (maxval < 1 || maxval > 65535)
    return decode_fail(MSHBM_ERR_MAXVAL, "maxval %lld outside [1, 65535]", (long long)maxval);
  if (width > INT32_MAX || height > INT32_MAX || width * height > ((int64_t)1 << 40))
    return decode_fail(MSHBM_ERR_TRUNCATED, "payload too short for %lldx%lld samples",
                       (long long)width, (long long)height);
  hdr->width = (int32_t)width;
  hdr->height = (int32_t)height;
  hdr->maxval = (int32_t)maxval;
  hdr->channels = (p3 || p6) ? 3 : 1;
  hdr->ascii = (p2 || p3) ? 1 : 0;
  hdr->itemsize = maxval > 255 ? 2 : 1;
  if (!hdr->ascii) {
    if (pos >= len || !is_ws(buf[pos]))
      return decode_fail(MSHBM_ERR_MALFORMED, "missing whitespace before binary payload");
    pos += 1;
    const int64_t need = width * height * hdr->channels * hdr->itemsize;
    if (len - pos < need)
      return decode_fail(MSHBM_ERR_TRUNCATED, "payload holds %lld bytes, need %lld",
                         (long long)(len - pos), (long long)need);
  }
  hdr->payload_offset = pos;
  return MSHBM_OK;
}

// formats.py:150-190: samples -> grayscale in [0, 1] (fp64, host)
int mshbm_pnm_decode(const uint8_t* buf, int64_t len, const mshbm_pnm_header* hdr,
                     double* gray, int64_t ld) {
  if (!buf || !hdr || !gray || ld < hdr->width) return decode_fail(MSHBM_ERR_VALUE, "bad arguments");
  const int64_t w = hdr->width, h = hdr->height, ch = hdr->channels;
  const int64_t count = w * h * ch;
  std::vector<int64_t> v((size_t)count);
  if (hdr->ascii) {
    int64_t pos = hdr->payload_offset;
    for (int64_t k = 0; k < count; ++k) {
      int64_t s, l;
      if (next_token(buf, len, &pos, &s, &l))
        return decode_fail(MSHBM_ERR_TRUNCATED, "expected %lld samples, found %lld",
                           (long long)count, (long long)k);
      if (!parse_int(buf + s, l, &v[(size_t)k]))
        return decode_fail(MSHBM_ERR_DECODE, "non-numeric ASCII sample");
    }
  } else {
    const uint8_t* p = buf + hdr->payload_offset;
    if (hdr->itemsize == 2)
      for (int64_t k = 0; k < count; ++k) v[(size_t)k] = (p[2 * k] << 8) | p[2 * k + 1];
    else
      for (int64_t k = 0; k < count; ++k) v[(size_t)k] = p[k];
  }
  int64_t lo = INT64_MAX, hi = INT64_MIN;
  for (int64_t x : v) lo = x < lo ? x : lo, hi = x > hi ? x : hi;
  if (count && (lo < 0 || hi > hdr->maxval))
    return decode_fail(MSHBM_ERR_DECODE, "sample value %lld outside [0, %d]",
                       (long long)(hi > hdr->maxval ? hi : lo), hdr->maxval);
  const double mv = (double)hdr->maxval;
  for (int64_t y = 0; y < h; ++y)
    for (int64_t x = 0; x < w; ++x) {
      const int64_t b = (y * w + x) * ch;
      const double g = ch == 3 ? ((double)v[(size_t)b] * kLuma[0] + (double)v[(size_t)b + 1] * kLuma[1]) +
                                     (double)v[(size_t)b + 2] * kLuma[2]
                               : (double)v[(size_t)b];
      gray[y * ld + x] = g / mv;
    }
  return MSHBM_OK;
}

// Binary (P5/P6) payload -> fp32 grayscale on the device: the raw samples
// (1-2 bytes per channel) cross PCIe instead of 4-8 byte floats.
int mshbm_pnm_upload(const uint8_t* buf, int64_t len, const mshbm_pnm_header* hdr,
                     float* d_gray, int64_t ld, void* stream) {
  if (!buf || !hdr || !d_gray || ld < hdr->width) return decode_fail(MSHBM_ERR_VALUE, "bad arguments");
  if (hdr->ascii) return decode_fail(MSHBM_ERR_UNSUPPORTED, "ASCII PNM: decode on the host");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t bytes = (int64_t)hdr->width * hdr->height * hdr->channels * hdr->itemsize;
  if (len - hdr->payload_offset < bytes) return decode_fail(MSHBM_ERR_TRUNCATED, "short payload");
  uint8_t* dev = nullptr;
  int* bad = nullptr;
  if (cudaMallocAsync((void**)&dev, bytes + 16, s) != cudaSuccess ||
      cudaMallocAsync((void**)&bad, sizeof(int), s) != cudaSuccess)
    return decode_fail(MSHBM_ERR_CUDA, "device allocation failed");
  cudaMemsetAsync(bad, 0, sizeof(int), s);
  cudaMemcpyAsync(dev, buf + hdr->payload_offset, bytes, cudaMemcpyHostToDevice, s);
  dim3 blk(32, 8), grid((hdr->width + 31) / 32, (hdr->height + 7) / 8);
  pnm_decode_kernel<<<grid, blk, 0, s>>>(dev, hdr->height, hdr->width, hdr->channels,
                                         hdr->itemsize, hdr->maxval, d_gray, ld, bad);
  int hbad = 0;
  cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(dev, s);
  cudaFreeAsync(bad, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return decode_fail(MSHBM_ERR_CUDA, "%s", cudaGetErrorString(e));
  if (hbad) return decode_fail(MSHBM_ERR_DECODE, "sample value outside [0, %d]", hdr->maxval);
  return MSHBM_OK;
}

// formats.py:193-232 (header part)
int mshbm_pfm_parse(const uint8_t* buf, int64_t len, mshbm_pfm_header* hdr) {
  if (!buf || !hdr || len < 0) return decode_fail(MSHBM_ERR_VALUE, "null buffer");
  int64_t pos = 0, s, l;
  int st = next_token(buf, len, &pos, &s, &l);
  if (st) return st;
  if (!(l == 2 && buf[s] == 'P' && buf[s + 1] == 'f'))
    return decode_fail(MSHBM_ERR_MALFORMED, "bad PFM magic %s (expected grayscale 'Pf')",
                       brepr(buf + s, l).c_str());
  int64_t width, height;
  if ((st = token_int(buf, len, &pos, "width", &width))) return st;
  if ((st = token_int(buf, len, &pos, "height", &height))) return st;
  if ((st = next_token(buf, len, &pos, &s, &l))) return st;
  std::string tok((const char*)buf + s, (size_t)l);
  char* end = nullptr;
  const double scale = strtod(tok.c_str(), &end);
  if (tok.empty() || end != tok.c_str() + tok.size())
    return decode_fail(MSHBM_ERR_MALFORMED, "non-numeric scale %s", brepr(buf + s, l).c_str());
  if (scale == 0.0) return decode_fail(MSHBM_ERR_MALFORMED, "zero scale");
  if (width <= 0 || height <= 0)
    return decode_fail(MSHBM_ERR_MALFORMED, "bad dimensions %lldx%lld", (long long)width,
                       (long long)height);
  if (pos >= len || !is_ws(buf[pos]))
    return decode_fail(MSHBM_ERR_MALFORMED, "missing whitespace before binary payload");
  pos += 1;
  if (width > INT32_MAX || height > INT32_MAX || width * height > ((int64_t)1 << 40) ||
      len - pos < 4 * width * height)
    return decode_fail(MSHBM_ERR_TRUNCATED, "payload holds %lld bytes, need %lld",
                       (long long)(len - pos), (long long)(4 * width * height));
  hdr->width = (int32_t)width;
  hdr->height = (int32_t)height;
  hdr->scale = scale;
  hdr->payload_offset = pos;
  return MSHBM_OK;
}

// formats.py:224-232: rows bottom-up on disk, endianness from the scale
// sign, non-finite samples -> NaN values + invalid mask
int mshbm_pfm_decode(const uint8_t* buf, int64_t len, const mshbm_pfm_header* hdr,
                     double* values, uint8_t* invalid, int64_t ld) {
  if (!buf || !hdr || !values || !invalid || ld < hdr->width)
    return decode_fail(MSHBM_ERR_VALUE, "bad arguments");
  const int64_t w = hdr->width, h = hdr->height;
  if (len - hdr->payload_offset < 4 * w * h) return decode_fail(MSHBM_ERR_TRUNCATED, "short payload");
  const uint8_t* p = buf + hdr->payload_offset;
  const bool little = hdr->scale < 0;
  for (int64_t r = 0; r < h; ++r) {
    const int64_t y = h - 1 - r;   // flipud
    for (int64_t x = 0; x < w; ++x) {
      const uint8_t* q = p + 4 * (r * w + x);
      uint32_t u = little ? (uint32_t)q[0] | (uint32_t)q[1] << 8 | (uint32_t)q[2] << 16 |
                                (uint32_t)q[3] << 24
                          : (uint32_t)q[3] | (uint32_t)q[2] << 8 | (uint32_t)q[1] << 16 |
                                (uint32_t)q[0] << 24;
      float f;
      memcpy(&f, &u, 4);
      const bool bad = !isfinite(f);
      values[y * ld + x] = bad ? NAN : (double)f;
      invalid[y * ld + x] = bad ? 1 : 0;
    }
  }
  return MSHBM_OK;
}

// formats.py:235-254.  Returns the encoded size; writes only if cap suffices.
int64_t mshbm_pfm_encode(const double* values, int32_t h, int32_t w, int64_t ld, double scale,
                         uint8_t* out, int64_t cap) {
  if (!values || h <= 0 || w <= 0 || ld < w) {
    decode_fail(MSHBM_ERR_VALUE, "expected a non-empty 2-D array");
    return -MSHBM_ERR_VALUE;
  }
  if (scale == 0.0) {
    decode_fail(MSHBM_ERR_VALUE, "scale must be nonzero");
    return -MSHBM_ERR_VALUE;
  }
  char head[96];
  const int hl = snprintf(head, sizeof head, "Pf\n%d %d\n%.6f\n", w, h, scale);
  const int64_t total = hl + (int64_t)4 * w * h;
  if (!out || cap < total) return total;
  memcpy(out, head, (size_t)hl);
  uint8_t* p = out + hl;
  const bool little = scale < 0;
  for (int64_t r = 0; r < h; ++r) {
    const double* row = values + (int64_t)(h - 1 - r) * ld;   // flipud
    for (int64_t x = 0; x < w; ++x) {
      const double v = isnan(row[x]) ? INFINITY : row[x];
      const float f = (float)v;
      uint32_t u;
      memcpy(&u, &f, 4);
      uint8_t* q = p + 4 * (r * w + x);
      if (little) q[0] = u, q[1] = u >> 8, q[2] = u >> 16, q[3] = u >> 24;
      else q[3] = u, q[2] = u >> 8, q[1] = u >> 16, q[0] = u >> 24;
    }
  }
  return total;
}

// formats.py:257-278 (binary P5; round half to even, NaN -> 0, clip)
int64_t mshbm_pgm_encode(const double* values, int32_t h, int32_t w, int64_t ld, int32_t maxval,
                         double scale_max, uint8_t* out, int64_t cap) {
  if (!values || h <= 0 || w <= 0 || ld < w) {
    decode_fail(MSHBM_ERR_VALUE, "expected a non-empty 2-D array");
    return -MSHBM_ERR_VALUE;
  }
  if (maxval < 1 || maxval > 65535) {
    decode_fail(MSHBM_ERR_VALUE, "maxval %d outside [1, 65535]", maxval);
    return -MSHBM_ERR_VALUE;
  }
  if (!(scale_max > 0)) {
    decode_fail(MSHBM_ERR_VALUE, "scale_max must be positive");
    return -MSHBM_ERR_VALUE;
  }
  char head[64];
  const int hl = snprintf(head, sizeof head, "P5\n%d %d\n%d\n", w, h, maxval);
  const int isz = maxval > 255 ? 2 : 1;
  const int64_t total = hl + (int64_t)isz * w * h;
  if (!out || cap < total) return total;
  memcpy(out, head, (size_t)hl);
  uint8_t* p = out + hl;
  for (int64_t y = 0; y < h; ++y)
    for (int64_t x = 0; x < w; ++x) {
      double v = values[y * ld + x];
      if (isnan(v)) v = 0.0;
      else if (isinf(v)) v = v > 0 ? 1.7976931348623157e308 : -1.7976931348623157e308;
      double q = nearbyint(v / scale_max * (double)maxval);   // numpy round: half to even
      q = q < 0 ? 0 : (q > maxval ? maxval : q);
      const int iv = (int)q;
      const int64_t k = y * w + x;
      if (isz == 2) p[2 * k] = (uint8_t)(iv >> 8), p[2 * k + 1] = (uint8_t)iv;
      else p[k] = (uint8_t)iv;
    }
  return total;
}

}  // extern "C"
