/* philox_grid.c -- C restatement of oracle/philox.py's keep masks (TEST INFRASTRUCTURE ONLY).
 *
 * Same algorithm as oracle/philox.py (Philox4x32-10, Random123 constants; counter
 * (col >> 3, row, layer, site); 16 bits per element; keep iff u16 >= threshold), used by the
 * oracle only to make large dropout masks (24-layer BERT-large stacks) cheap to draw.
 * tests/test_philox.py checks it against the numpy restatement and the Random123 known-answer
 * vectors.  Built by oracle/Makefile (gcc -O2 -shared) from __graft_entry__.build(). */
#include <stdint.h>

static void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t x = hi1 ^ c[1] ^ k0, z = hi0 ^ c[3] ^ k1;
    c[0] = x;
    c[1] = lo1;
    c[2] = z;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

/* out[i * n_cols + col] = keep(rows[i], col) for col in [0, n_cols) */
void philox_keep_grid(const int64_t* rows, int64_t n_rows, int64_t n_cols, uint32_t layer, uint32_t site,
                      uint64_t seed, uint32_t thresh, uint8_t* out) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t i = 0; i < n_rows; ++i) {
    uint8_t* o = out + i * n_cols;
    for (int64_t c8 = 0; c8 < n_cols; c8 += 8) {
      uint32_t c[4] = {(uint32_t)(c8 >> 3), (uint32_t)rows[i], layer, site};
      philox4x32_10(c, k0, k1);
      for (int64_t e = 0; e < 8 && c8 + e < n_cols; ++e) {
        const uint32_t word = c[e >> 1];
        const uint32_t u16 = (e & 1) ? (word >> 16) : (word & 0xFFFFu);
        o[c8 + e] = u16 >= thresh;
      }
    }
  }
}
