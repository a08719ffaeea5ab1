/*
 * TEST INFRASTRUCTURE ONLY — independent fp64 C restatement of the C1 (toy
 * MLP) forward, used to pin oracle/plan_ref.py and the converter.
 *
 * Parses the reference's toy-binary layout exactly as
 * pkg/src/modelci/converter/toyformat.py:99-149 writes/reads it
 * ("TOYB" | u32 n | per layer u16 oplen op u32 in u32 out u32 nw f64[nw] |
 * u32 crc32(payload)) and executes the op semantics this repo defines for toy
 * graphs (paper_2006_05096_b200/zoo.py docstring; the reference itself never
 * computes, mockserve/server.py:117-127):
 *   linear  y = W x (+ b), W row-major [out][in], optional out biases
 *   relu    max(x, 0);  gelu  0.5 x (1 + erf(x / sqrt 2))
 *   norm    LayerNorm over the features, eps 1e-5, optional gamma+beta
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint32_t crc_table[256];
static int crc_ready = 0;

static uint32_t crc32_buf(const uint8_t* p, size_t n) {
  if (!crc_ready) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      crc_table[i] = c;
    }
    crc_ready = 1;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = crc_table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

static uint32_t rd_u32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

/* returns 0 on success; 1 bad magic, 2 CRC, 3 truncated, 4 unsupported op, 5 shape */
int toyref_forward(const uint8_t* blob, size_t len, const double* x, int batch, int in_dim,
                   double* y, int y_cap, int* out_dim) {
  if (len < 12 || memcmp(blob, "TOYB", 4) != 0) return 1;
  const uint8_t* pay = blob + 4;
  size_t plen = len - 8;
  if (crc32_buf(pay, plen) != rd_u32(blob + len - 4)) return 2;
  size_t pos = 0;
  if (plen < 4) return 3;
  uint32_t nl = rd_u32(pay);
  pos = 4;
  int width = in_dim;
  double* cur = (double*)malloc(sizeof(double) * (size_t)batch * (width > 0 ? width : 1));
  memcpy(cur, x, sizeof(double) * (size_t)batch * width);
  for (uint32_t l = 0; l < nl; ++l) {
    if (pos + 2 > plen) { free(cur); return 3; }
    uint16_t oplen = (uint16_t)(pay[pos] | (pay[pos + 1] << 8));
    pos += 2;
    if (pos + oplen + 12 > plen) { free(cur); return 3; }
    char op[64] = {0};
    memcpy(op, pay + pos, oplen < 63 ? oplen : 63);
    pos += oplen;
    uint32_t din = rd_u32(pay + pos), dout = rd_u32(pay + pos + 4), nw = rd_u32(pay + pos + 8);
    pos += 12;
    if (pos + (size_t)nw * 8 > plen) { free(cur); return 3; }
    double* w = (double*)malloc(sizeof(double) * (nw ? nw : 1));
    memcpy(w, pay + pos, (size_t)nw * 8);   /* little-endian f64, host order */
    pos += (size_t)nw * 8;
    if ((int)din != width) { free(w); free(cur); return 5; }
    double* nxt = (double*)calloc((size_t)batch * dout, sizeof(double));
    if (strcmp(op, "linear") == 0) {
      int has_b = nw == din * dout + dout;
      if (!has_b && nw != din * dout) { free(w); free(nxt); free(cur); return 5; }
      for (int b = 0; b < batch; ++b)
        for (uint32_t o = 0; o < dout; ++o) {
          double s = has_b ? w[din * dout + o] : 0.0;
          for (uint32_t i = 0; i < din; ++i) s += w[(size_t)o * din + i] * cur[(size_t)b * din + i];
          nxt[(size_t)b * dout + o] = s;
        }
    } else if (strcmp(op, "relu") == 0 || strcmp(op, "gelu") == 0) {
      if (din != dout) { free(w); free(nxt); free(cur); return 5; }
      for (size_t i = 0; i < (size_t)batch * dout; ++i) {
        double v = cur[i];
        nxt[i] = op[0] == 'r' ? (v > 0 ? v : 0) : 0.5 * v * (1.0 + erf(v / sqrt(2.0)));
      }
    } else if (strcmp(op, "norm") == 0) {
      if (din != dout || (nw != 0 && nw != 2 * dout)) { free(w); free(nxt); free(cur); return 5; }
      for (int b = 0; b < batch; ++b) {
        const double* r = cur + (size_t)b * din;
        double mu = 0, var = 0;
        for (uint32_t i = 0; i < din; ++i) mu += r[i];
        mu /= din;
        for (uint32_t i = 0; i < din; ++i) var += (r[i] - mu) * (r[i] - mu);
        var /= din;
        for (uint32_t i = 0; i < din; ++i) {
          double v = (r[i] - mu) / sqrt(var + 1e-5);
          if (nw) v = v * w[i] + w[dout + i];
          nxt[(size_t)b * dout + i] = v;
        }
      }
    } else {
      free(w); free(nxt); free(cur);
      return 4;
    }
    free(w);
    free(cur);
    cur = nxt;
    width = (int)dout;
  }
  if (pos != plen) { free(cur); return 3; }
  *out_dim = width;
  if ((long)batch * width > y_cap) { free(cur); return 5; }
  memcpy(y, cur, sizeof(double) * (size_t)batch * width);
  free(cur);
  return 0;
}
