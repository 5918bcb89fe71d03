// codec.cuh -- frame codecs on the device: PNG encoding of
// depth / RGB / semantic frames, the teleop wire format (sensors.py:211-246,
// teleop.py:75-110).
//
// The reference quantises (depth: round(d / max_range * 65535) clipped to u16;
// rgb: round(rgb * 255) clipped to u8; semantic: u16 as is) and compresses
// with PIL/zlib.  Here every env's frame becomes a complete PNG on the device
// with zlib *stored* (uncompressed) deflate blocks -- a valid PNG any decoder
// reads back to exactly the quantised samples -- so the D2H copy is the
// finished byte stream and no host pass touches the pixels:
//   k_png_emit   one thread per 4 raw scanline bytes: filter byte 0 + the
//                big-endian samples, scattered into the stored blocks; CTA
//                (0, n) writes signature, IHDR (+CRC), IDAT/zlib/block
//                headers and IEND;
//   k_png_sums   one CTA per frame: Adler-32 of the raw data and CRC-32 of the
//                IDAT chunk from per-thread partial sums, combined exactly
//                (Adler: positional weights mod 65521; CRC: each chunk's CRC
//                shifted by x^(8 * bytes after it) mod P, zlib's multmodp).
#pragma once

#include <stdint.h>

namespace nvk {

#define NV_CRC_POLY 0xedb88320u

// a * b mod P (bit-reflected CRC-32 polynomial arithmetic, zlib's multmodp)
__host__ __device__ inline uint32_t crc_multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ NV_CRC_POLY : b >> 1;
  }
  return p;
}

// x^(8 n) mod P: the operator that advances a CRC register over n zero bytes
__host__ __device__ inline uint32_t crc_x8n(unsigned long long n) {
  uint32_t p = 1u << 31;     // x^0
  uint32_t sq = 1u << 23;    // x^8
  while (n) {
    if (n & 1) p = crc_multmodp(sq, p);
    sq = crc_multmodp(sq, sq);
    n >>= 1;
  }
  return p;
}

// CRC register update over bytes (init c, no conditioning), bitwise
__host__ __device__ inline uint32_t crc_raw_bits(uint32_t c, const uint8_t *p, long long n) {
  for (long long i = 0; i < n; ++i) {
    c ^= p[i];
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ NV_CRC_POLY : c >> 1;
  }
  return c;
}

struct PngGeom {
  int W, H, bpp;         // bytes per pixel in the PNG (2: 16-bit gray, 3: RGB8)
  long long rl;          // raw scanline bytes (1 + W * bpp)
  long long raw;         // H * rl
  long long nblk;        // stored blocks of <= 65535 bytes
  long long zlen;        // zlib stream: 2 + raw + 5 nblk + 4
  long long total;       // whole PNG
  long long idat_data;   // offset of the zlib stream in the PNG
};

__host__ __device__ inline PngGeom png_geom(int kind, int W, int H) {
  PngGeom g;
  g.W = W;
  g.H = H;
  g.bpp = kind == 1 ? 3 : 2;
  g.rl = 1 + (long long)W * g.bpp;
  g.raw = (long long)H * g.rl;
  g.nblk = (g.raw + 65534) / 65535;
  g.zlen = 2 + g.raw + 5 * g.nblk + 4;
  g.idat_data = 8 + 25 + 8;
  g.total = g.idat_data + g.zlen + 4 + 12;
  return g;
}

// PNG offset of raw byte r (inside stored block r / 65535)
__device__ __forceinline__ long long png_raw_pos(const PngGeom &g, long long r) {
  const long long b = r / 65535;
  return g.idat_data + 2 + b * (65535 + 5) + 5 + (r - b * 65535);
}

struct PngArgs {
  int kind;        // 0 depth (16-bit gray), 1 rgb (8-bit RGB), 2 semantic (16-bit gray)
  int src_f64;     // 1: the reference's f64 arrays (depth metres / rgb in [0, 1])
  const void *src; // n frames [H, W(, 3)]: f32|f64 depth, u8|f64 rgb, u16 semantic
  double max_range;
  uint8_t *out;    // n x stride
  long long stride;
};

__device__ __forceinline__ void put_be32(uint8_t *p, uint32_t v) {
  p[0] = (uint8_t)(v >> 24);
  p[1] = (uint8_t)(v >> 16);
  p[2] = (uint8_t)(v >> 8);
  p[3] = (uint8_t)v;
}

// sample value of pixel px (channel ch) of frame n, quantised like the reference
__device__ __forceinline__ uint32_t png_sample(const PngArgs &a, const PngGeom &g, int n,
                                               long long px, int ch) {
  const long long npx = (long long)g.W * g.H;
  if (a.kind == 0) {  // depth_to_png: clip(round(d / max_range * 65535), 0, 65535)
    const double d = a.src_f64 ? static_cast<const double *>(a.src)[n * npx + px]
                               : (double)static_cast<const float *>(a.src)[n * npx + px];
    double q = rint(__dmul_rn(__ddiv_rn(d, a.max_range), 65535.0));
    q = fmin(fmax(q, 0.0), 65535.0);
    return (uint32_t)q;
  }
  if (a.kind == 1) {  // rgb_to_png: clip(round(rgb * 255), 0, 255)
    if (!a.src_f64) return static_cast<const uint8_t *>(a.src)[(n * npx + px) * 3 + ch];
    double q = rint(__dmul_rn(static_cast<const double *>(a.src)[(n * npx + px) * 3 + ch], 255.0));
    return (uint32_t)fmin(fmax(q, 0.0), 255.0);
  }
  return static_cast<const uint16_t *>(a.src)[n * npx + px];
}

__global__ void k_png_emit(PngArgs a, PngGeom g) {
  const int n = blockIdx.y;
  uint8_t *o = a.out + (size_t)n * a.stride;
  const long long r0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  for (long long r = r0; r < min(r0 + 4, g.raw); ++r) {
    const long long row = r / g.rl, k = r - row * g.rl;
    uint8_t byte = 0;  // filter type 0 (None) at k == 0
    if (k > 0) {
      const long long col = (k - 1) / g.bpp;
      const int sub = (int)((k - 1) - col * g.bpp);
      const long long px = row * g.W + col;
      if (g.bpp == 3) {
        byte = (uint8_t)png_sample(a, g, n, px, sub);
      } else {
        const uint32_t v = png_sample(a, g, n, px, 0);
        byte = (uint8_t)(sub == 0 ? v >> 8 : v);  // big-endian 16-bit samples
      }
    }
    o[png_raw_pos(g, r)] = byte;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
    for (int i = 0; i < 8; ++i) o[i] = sig[i];
    // IHDR: length 13, type, width, height, depth, colour type, 0, 0, 0, CRC
    uint8_t *h = o + 8;
    put_be32(h, 13);
    h[4] = 'I'; h[5] = 'H'; h[6] = 'D'; h[7] = 'R';
    put_be32(h + 8, (uint32_t)g.W);
    put_be32(h + 12, (uint32_t)g.H);
    h[16] = g.bpp == 3 ? 8 : 16;
    h[17] = g.bpp == 3 ? 2 : 0;
    h[18] = h[19] = h[20] = 0;
    put_be32(h + 21, crc_raw_bits(0xffffffffu, h + 4, 17) ^ 0xffffffffu);
    // IDAT header, zlib header (deflate, 32K window, no dictionary, level 0)
    uint8_t *d = o + 33;
    put_be32(d, (uint32_t)g.zlen);
    d[4] = 'I'; d[5] = 'D'; d[6] = 'A'; d[7] = 'T';
    d[8] = 0x78;
    d[9] = 0x01;
    // IEND
    uint8_t *e = o + g.idat_data + g.zlen + 4;
    put_be32(e, 0);
    e[4] = 'I'; e[5] = 'E'; e[6] = 'N'; e[7] = 'D';
    put_be32(e + 8, 0xae426082u);
  }
  // stored-block headers: BFINAL on the last, LEN, ~LEN (little-endian)
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < g.nblk) {
    const long long len = min(65535LL, g.raw - b * 65535);
    uint8_t *p = o + g.idat_data + 2 + b * (65535 + 5);
    p[0] = b == g.nblk - 1 ? 1 : 0;
    p[1] = (uint8_t)len;
    p[2] = (uint8_t)(len >> 8);
    p[3] = (uint8_t)~len;
    p[4] = (uint8_t)(~len >> 8);
  }
}

// Adler-32 of the raw data and CRC-32 of the IDAT chunk of every frame.
__global__ void __launch_bounds__(256) k_png_sums(PngArgs a, PngGeom g) {
  __shared__ uint32_t tab[256];
  __shared__ unsigned long long sa[256], sb[256];
  __shared__ uint32_t sc[256];
  const int n = blockIdx.x, t = threadIdx.x, T = blockDim.x;
  uint8_t *o = a.out + (size_t)n * a.stride;
  for (int i = t; i < 256; i += T) {
    uint32_t c = (uint32_t)i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ NV_CRC_POLY : c >> 1;
    tab[i] = c;
  }
  // --- Adler-32: a = 1 + sum d_i, b = L + sum (L - i) d_i  (mod 65521)
  const long long L = g.raw;
  const long long per = (L + T - 1) / T;
  const long long lo = min(L, t * per), hi = min(L, lo + per);
  unsigned long long s = 0, w = 0;
  for (long long r = lo; r < hi; ++r) {
    const uint32_t d = o[png_raw_pos(g, r)];
    s += d;
    w += (unsigned long long)(hi - r) * d;  // (len - j) weights inside the chunk
  }
  sa[t] = s % 65521;
  sb[t] = (w + (unsigned long long)((L - hi) % 65521) * (s % 65521)) % 65521;
  __syncthreads();
  if (t == 0) {
    unsigned long long A = 1, B = (unsigned long long)(L % 65521);
    for (int k = 0; k < T; ++k) {
      A = (A + sa[k]) % 65521;
      B = (B + sb[k]) % 65521;
    }
    put_be32(o + g.idat_data + g.zlen - 4, (uint32_t)((B << 16) | A));
  }
  __syncthreads();
  // --- CRC-32 over "IDAT" + the zlib stream: per-thread raw CRCs of equal
  // chunks, each shifted over the bytes after it, plus the init term
  const uint8_t *c0 = o + g.idat_data - 4;
  const long long CL = 4 + g.zlen;
  const long long cper = (CL + T - 1) / T;
  const long long clo = min(CL, t * cper), chi = min(CL, clo + cper);
  uint32_t c = 0;
  for (long long i = clo; i < chi; ++i) c = tab[(c ^ c0[i]) & 0xff] ^ (c >> 8);
  sc[t] = crc_multmodp(crc_x8n((unsigned long long)(CL - chi)), c);
  __syncthreads();
  if (t == 0) {
    uint32_t crc = crc_multmodp(crc_x8n((unsigned long long)CL), 0xffffffffu);
    for (int k = 0; k < T; ++k) crc ^= sc[k];
    put_be32(o + g.idat_data + g.zlen, crc ^ 0xffffffffu);
  }
}

}  // namespace nvk
