// Client tokenized mode on the device (ChunkStreamer.tokenized
// client.py:451-506): a token store built once from the JSON-lines records and
// the packing of a chunk's samples into fixed-length sequences with per-token
// mixture-key tags, the tags being stage 3's domain ids (per_domain_loss).
//
//  * jsonl_tokenize_kernel<WRITE> -- one thread per record: the top-level
//    `text_field` string (the last occurrence, as json.loads keeps it) is
//    decoded from its JSON escapes to UTF-8 on the fly and tokenized
//      ByteTokenizer:       the UTF-8 bytes            (tokenizers.py:33-40)
//      WhitespaceTokenizer: str.split() on Python's whitespace code points,
//                           stable_hash("tok", piece) % vocab (BLAKE2b-128,
//                           seeding.py:18-28; tokenizers.py:20-30)
//    pass 1 counts, pass 2 writes at the scanned offsets. Records outside
//    this path (no string value / non-object record / escaped key / lone
//    surrogate) are flagged for the host tokenizer.
//  * pack_tokens_kernel -- one thread per output token: window w, key slot
//    and sequence within the window, stream position, sample by binary
//    search in the key's token prefix, token gather.
#include <stdint.h>

#include "blake2b.cuh"
#include "common.cuh"
#include "mixtera_internal.cuh"

namespace mx {

__device__ __forceinline__ bool tk_ws(uint8_t c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }

// Python str.isspace() code points (str.split() separators)
__device__ __forceinline__ bool py_space(u32 cp) {
  if (cp <= 0x20) return cp == 0x20 || (cp >= 0x09 && cp <= 0x0d) || (cp >= 0x1c && cp <= 0x1f);
  if (cp < 0x85) return false;
  return cp == 0x85 || cp == 0xa0 || cp == 0x1680 || (cp >= 0x2000 && cp <= 0x200a) || cp == 0x2028 ||
         cp == 0x2029 || cp == 0x202f || cp == 0x205f || cp == 0x3000;
}

__device__ __forceinline__ int hexv(uint8_t h) {
  return h <= '9' ? h - '0' : (h | 0x20) - 'a' + 10;
}

// Decoder over a JSON string body [p, e) (after the opening quote): next code
// point and its UTF-8 bytes. Returns 0 at the closing quote, -1 on a lone
// surrogate / malformed input (host), else the number of UTF-8 bytes.
struct JStr {
  const uint8_t* p;
  const uint8_t* e;
  __device__ int next(u32* cp, uint8_t out[4]) {
    if (p >= e) return -1;
    uint8_t c = *p;
    if (c == '"') return 0;
    if (c != '\\') {
      int n = c < 0x80 ? 1 : (c >= 0xf0 ? 4 : (c >= 0xe0 ? 3 : 2));
      if (p + n > e) return -1;
      u32 v = n == 1 ? c : (c & (0x7f >> n));
      out[0] = c;
      for (int k = 1; k < n; ++k) {
        out[k] = p[k];
        v = (v << 6) | (p[k] & 0x3f);
      }
      if (n == 3 && v >= 0xd800 && v <= 0xdfff) return -1;  // encoded surrogate: encode('utf-8') raises
      p += n;
      *cp = v;
      return n;
    }
    if (p + 1 >= e) return -1;
    const uint8_t d = p[1];
    u32 v;
    if (d == 'u') {
      if (p + 6 > e) return -1;
      v = (hexv(p[2]) << 12) | (hexv(p[3]) << 8) | (hexv(p[4]) << 4) | hexv(p[5]);
      p += 6;
      if (v >= 0xd800 && v <= 0xdbff) {  // high surrogate: a low one must follow
        if (p + 6 > e || p[0] != '\\' || p[1] != 'u') return -1;
        const u32 lo = (hexv(p[2]) << 12) | (hexv(p[3]) << 8) | (hexv(p[4]) << 4) | hexv(p[5]);
        if (lo < 0xdc00 || lo > 0xdfff) return -1;
        p += 6;
        v = 0x10000 + ((v - 0xd800) << 10) + (lo - 0xdc00);
      } else if (v >= 0xdc00 && v <= 0xdfff) {
        return -1;  // lone low surrogate: str.encode('utf-8') raises in the reference
      }
    } else {
      p += 2;
      v = d == 'b' ? 8 : d == 'f' ? 12 : d == 'n' ? 10 : d == 'r' ? 13 : d == 't' ? 9 : d;
    }
    *cp = v;
    if (v < 0x80) {
      out[0] = (uint8_t)v;
      return 1;
    }
    if (v < 0x800) {
      out[0] = (uint8_t)(0xc0 | (v >> 6));
      out[1] = (uint8_t)(0x80 | (v & 0x3f));
      return 2;
    }
    if (v < 0x10000) {
      out[0] = (uint8_t)(0xe0 | (v >> 12));
      out[1] = (uint8_t)(0x80 | ((v >> 6) & 0x3f));
      out[2] = (uint8_t)(0x80 | (v & 0x3f));
      return 3;
    }
    out[0] = (uint8_t)(0xf0 | (v >> 18));
    out[1] = (uint8_t)(0x80 | ((v >> 12) & 0x3f));
    out[2] = (uint8_t)(0x80 | ((v >> 6) & 0x3f));
    out[3] = (uint8_t)(0x80 | (v & 0x3f));
    return 4;
  }
};

// skip one JSON value (already validated at registration); nullptr if the
// structure is broken
__device__ const uint8_t* tk_skip(const uint8_t* p, const uint8_t* e) {
  int depth = 0;
  bool instr = false;
  for (; p < e; ++p) {
    const uint8_t c = *p;
    if (instr) {
      if (c == '\\') ++p;
      else if (c == '"') {
        instr = false;
        if (depth == 0) return p + 1;
      }
      continue;
    }
    if (c == '"') {
      instr = true;
    } else if (c == '{' || c == '[') {
      ++depth;
    } else if (c == '}' || c == ']') {
      if (depth == 0) return p;  // end of the enclosing container
      if (--depth == 0) return p + 1;
    } else if (c == ',') {
      if (depth == 0) return p;
    }
  }
  return depth == 0 ? p : nullptr;
}

template <bool WRITE>
__global__ void jsonl_tokenize_kernel(const uint8_t* __restrict__ buf, const long long* __restrict__ rs,
                                      const long long* __restrict__ re, long long n_rec, const uint8_t* field,
                                      int field_len, int kind, u32 vocab, const long long* off, long long* cnt,
                                      int32_t* out, uint8_t* host) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= n_rec) return;
  if (WRITE && host[r]) return;
  const uint8_t* p = buf + rs[r];
  const uint8_t* e = buf + re[r];
  bool bad = false;
  const uint8_t* val = nullptr;  // the text field's value (last occurrence)
  while (p < e && tk_ws(*p)) ++p;
  if (p >= e || *p != '{') bad = true;
  else ++p;
  while (!bad) {
    while (p < e && tk_ws(*p)) ++p;
    if (p < e && *p == '}') break;
    if (p < e && *p == ',') {
      ++p;
      continue;
    }
    if (p >= e || *p != '"') {
      bad = true;
      break;
    }
    const uint8_t* ks = ++p;
    bool esc = false;
    while (p < e && *p != '"') {
      if (*p == '\\') {
        esc = true;
        ++p;
      }
      ++p;
    }
    if (p >= e || esc) {
      bad = true;
      break;
    }
    const long long klen = p - ks;
    ++p;
    while (p < e && tk_ws(*p)) ++p;
    if (p >= e || *p != ':') {
      bad = true;
      break;
    }
    ++p;
    while (p < e && tk_ws(*p)) ++p;
    bool match = klen == field_len;
    for (int t = 0; match && t < field_len; ++t) match = ks[t] == field[t];
    if (match) val = p;
    p = tk_skip(p, e);
    if (!p) bad = true;
  }
  long long n = 0;
  if (!bad && val) {
    if (*val != '"') {
      bad = true;  // null / number / list: the reference's tokenizer decides (or fails)
    } else {
      JStr js{val + 1, e};
      int32_t* o = WRITE ? out + off[r] : nullptr;
      if (kind == 0) {  // ByteTokenizer
        while (true) {
          u32 cp;
          uint8_t b[4];
          const int k = js.next(&cp, b);
          if (k <= 0) {
            bad = k < 0;
            break;
          }
          for (int t = 0; t < k; ++t) {
            if (WRITE) o[n] = b[t];
            ++n;
          }
        }
      } else {  // WhitespaceTokenizer: pieces between whitespace code points
        while (!bad) {
          u32 cp;
          uint8_t b[4];
          JStr at = js;  // piece start
          int k;
          while ((k = js.next(&cp, b)) > 0 && py_space(cp)) at = js;
          if (k < 0) {
            bad = true;
            break;
          }
          if (k == 0) break;
          // piece: this code point and the following non-space ones
          long long len = k;
          JStr scan = js;
          JStr endp = js;
          while ((k = scan.next(&cp, b)) > 0 && !py_space(cp)) {
            len += k;
            endp = scan;
          }
          if (k < 0) {
            bad = true;
            break;
          }
          if (WRITE) {
            Blake2b h;
            h.init();
            h.len8(3);
            h.byte('t');
            h.byte('o');
            h.byte('k');
            h.len8((unsigned long long)len);
            JStr f2 = at;
            long long fed = 0;
            while (fed < len) {
              const int kk = f2.next(&cp, b);
              for (int t = 0; t < kk; ++t) h.byte(b[t]);
              fed += kk;
            }
            o[n] = (int32_t)(h.seed63() % vocab);
          }
          ++n;
          js = endp;
        }
      }
    }
  }
  if (!WRITE) {
    cnt[r] = bad ? 0 : n;
    host[r] = bad ? 1 : 0;
  }
}

// Packing. Key m (slot order of the chunk's sorted keys) has samples
// [key_off[m], key_off[m+1]) of `samples` (global sample ids in iterator
// order) with token prefix sprefix (per sample, exclusive, per key) ...
struct PackArgs {
  long long n_out;     // total tokens = W * S * L
  int L;
  int S;               // sequences per window
  int n_slots;         // keys in the window order
  const int* slot_key;     // [n_slots] key of each order slot
  const int* slot_first;   // [n_slots + 1] first sequence of each slot within a window
  const int* key_count;    // [keys] sequences per window
  const long long* key_off;    // [keys + 1] into samples / sprefix
  const long long* samples;    // global sample ids
  const long long* sprefix;    // token prefix within the key's stream (exclusive, per sample)
  const long long* tok_off;    // token store offsets [n_records + 1]
  const int32_t* tokens;
  const int* key_tag;          // tag written for key m (e.g. a domain id)
  int32_t* out_tokens;
  int32_t* out_tags;
};

__global__ void pack_tokens_kernel(PackArgs a) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= a.n_out) return;
  const long long q = i / a.L;
  const int t = (int)(i - q * a.L);
  const long long w = q / a.S;
  const int r = (int)(q - w * a.S);
  int s = 0;
  while (a.slot_first[s + 1] <= r) ++s;
  const int m = a.slot_key[s];
  const int j = r - a.slot_first[s];
  const long long pos = (w * a.key_count[m] + j) * (long long)a.L + t;
  long long lo = a.key_off[m], hi = a.key_off[m + 1];  // last sample with prefix <= pos
  while (hi - lo > 1) {
    const long long mid = (lo + hi) >> 1;
    if (a.sprefix[mid] <= pos) lo = mid; else hi = mid;
  }
  const long long g = a.samples[lo];
  a.out_tokens[i] = a.tokens[a.tok_off[g] + (pos - a.sprefix[lo])];
  a.out_tags[i] = a.key_tag[m];
}

}  // namespace mx

using namespace mx;

extern "C" {

int mx_jsonl_tokenize(const uint8_t* buf, const int64_t* rec_start, const int64_t* rec_end, int64_t n_records,
                      const uint8_t* field, int32_t field_len, int32_t tokenizer, uint32_t vocab_size,
                      const int64_t* offsets, int64_t* counts, int32_t* tokens, uint8_t* host, void* stream) {
  if (tokenizer != 0 && tokenizer != 1) return mx_fail(MX_ERR_INVALID, "tokenizer %d (0 byte, 1 whitespace)", tokenizer);
  if (tokenizer == 1 && vocab_size == 0) return mx_fail(MX_ERR_INVALID, "whitespace tokenizer needs vocab_size > 0");
  if (n_records == 0) return MX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)((n_records + 127) / 128);
  const long long* rs = reinterpret_cast<const long long*>(rec_start);
  const long long* re = reinterpret_cast<const long long*>(rec_end);
  if (!tokens) {
    jsonl_tokenize_kernel<false><<<grid, 128, 0, s>>>(buf, rs, re, n_records, field, field_len, tokenizer,
                                                       vocab_size, nullptr, reinterpret_cast<long long*>(counts),
                                                       nullptr, host);
  } else {
    jsonl_tokenize_kernel<true><<<grid, 128, 0, s>>>(buf, rs, re, n_records, field, field_len, tokenizer,
                                                      vocab_size, reinterpret_cast<const long long*>(offsets),
                                                      nullptr, tokens, host);
  }
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

int mx_pack_tokens(int64_t n_windows, int32_t sequence_length, int32_t n_slots, const int32_t* slot_key,
                   const int32_t* slot_first, const int32_t* key_count, const int64_t* key_off,
                   const int64_t* samples, const int64_t* sample_prefix, const int64_t* token_offsets,
                   const int32_t* tokens, const int32_t* key_tag, int32_t seqs_per_window, int32_t* out_tokens,
                   int32_t* out_tags, void* stream) {
  if (sequence_length < 1 || n_windows < 0 || seqs_per_window < 0)
    return mx_fail(MX_ERR_INVALID, "bad packing sizes");
  PackArgs a{};
  a.n_out = n_windows * (long long)seqs_per_window * sequence_length;
  if (a.n_out == 0) return MX_OK;
  a.L = sequence_length;
  a.S = seqs_per_window;
  a.n_slots = n_slots;
  a.slot_key = slot_key;
  a.slot_first = slot_first;
  a.key_count = key_count;
  a.key_off = reinterpret_cast<const long long*>(key_off);
  a.samples = reinterpret_cast<const long long*>(samples);
  a.sprefix = reinterpret_cast<const long long*>(sample_prefix);
  a.tok_off = reinterpret_cast<const long long*>(token_offsets);
  a.tokens = tokens;
  a.key_tag = key_tag;
  a.out_tokens = out_tokens;
  a.out_tags = out_tags;
  cudaStream_t s = (cudaStream_t)stream;
  pack_tokens_kernel<<<(unsigned)((a.n_out + 255) / 256), 256, 0, s>>>(a);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

}  // extern "C"
