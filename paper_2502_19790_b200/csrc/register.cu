// Metadata registration on the device: JSON-lines bytes ->
// per-sample, per-field value hashes, the input of code interning.
//
// The reference parses every record with json.loads + JsonFieldParser.parse +
// _normalize_values (catalog.py:186-262, formats.py:47-56) in Python. Here
// the file bytes are resident in HBM and
//   1. newline positions are found with a reduce-then-scan over 16-byte words
//      (mx_jsonl_records; files are newline-terminated by the caller) and the
//      non-empty lines -- the records, in file order -- compacted with their
//      physical line numbers (error messages cite them);
//   2. one thread per record runs a JSON validator / extractor
//      (mx_jsonl_extract): the full RFC 8259 grammar, UTF-8 validity as
//      Python decodes it (surrogates pass, json.loads(bytes) decodes with
//      'surrogatepass'), duplicate keys (the last one wins, as in json.loads),
//      and for every requested top-level field the NORMALISED value of
//      _normalize_values -- missing (kind 0), null / [] (kind 3: present, no
//      value), a string = the 1-tuple, a list of strings = the sorted set
//      (kind 1) -- as a 128-bit hash of the sorted distinct element hashes,
//      the distinct element count and the value's byte span (a string's
//      content, or ~offset of a whole [...] list) for the representative
//      records whose strings become the vocabulary.
//      Records the fast path does not cover (numbers / booleans / nested
//      values in a requested field, escapes in a requested value or any
//      top-level key, more than LIST_MAX list elements, NaN / Infinity
//      literals, NUL bytes, BOM, invalid JSON) are flagged: the host runs the
//      reference semantics on exactly those records (and raises its errors).
// Interning (hash -> code in first-appearance order) and the column layout
// are in register.py; the value strings of each distinct hash come from one
// representative record.
#include <stdint.h>

#include "common.cuh"
#include "mixtera_internal.cuh"
#include "scan.cuh"

namespace mx {

constexpr int JL_MAX_FIELDS = 32;
constexpr int LIST_MAX = 8;

struct JsonlFields {
  int n;
  const uint8_t* names;      // field name bytes (device)
  const long long* off;      // [n + 1]
};

// ---------------------------------------------------------------- lines
struct NewlineF {  // newline bytes per 16-byte word; positions in order
  const uint4* w;
  long long* nl;
  __device__ static u32 mask(uint4 v) {
    u32 m = 0;
    const u32 x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int b = 0; b < 4; ++b) m |= (((x[k] >> (8 * b)) & 0xffu) == 0x0au ? 1u : 0u) << (4 * k + b);
    return m;
  }
  __device__ u64 value(long long i) const { return __popc(mask(w[i])); }
  __device__ void apply(long long i, u64 ex, u64 v) const {
    if (!v) return;
    u32 m = mask(w[i]);
    u64 o = ex;
    while (m) {
      nl[o++] = i * 16 + (__ffs(m) - 1);
      m &= m - 1;
    }
  }
  __device__ void total(u64) const {}
};

struct RecordF {  // non-empty lines -> records (start, end, physical line)
  const long long* nl;
  long long* rs;
  long long* re;
  long long* rline;
  __device__ u64 value(long long k) const {
    const long long s = k == 0 ? 0 : nl[k - 1] + 1;
    return nl[k] > s ? 1 : 0;
  }
  __device__ void apply(long long k, u64 ex, u64 v) const {
    if (!v) return;
    rs[ex] = k == 0 ? 0 : nl[k - 1] + 1;
    re[ex] = nl[k];
    rline[ex] = k;
  }
  __device__ void total(u64) const {}
};

struct CountF {  // newlines in the buffer
  const uint4* w;
  u64* t;
  __device__ u64 value(long long i) const { return __popc(NewlineF::mask(w[i])); }
  __device__ void apply(long long, u64, u64) const {}
  __device__ void total(u64 x) const { *t = x; }
};

struct NonEmptyF {  // non-empty lines (records)
  const long long* nl;
  u64* t;
  __device__ u64 value(long long k) const { return nl[k] > (k == 0 ? 0 : nl[k - 1] + 1) ? 1 : 0; }
  __device__ void apply(long long, u64, u64) const {}
  __device__ void total(u64 x) const { *t = x; }
};

struct RecCountF {
  RecordF r;
  u64* t;
  __device__ u64 value(long long k) const { return r.value(k); }
  __device__ void apply(long long k, u64 ex, u64 v) const { r.apply(k, ex, v); }
  __device__ void total(u64 x) const { *t = x; }
};

// ---------------------------------------------------------------- hashing
__device__ __forceinline__ u64 mix64(u64 z) {  // splitmix64 finaliser
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct H128 {
  u64 a, b;
};

// hash of one element's bytes (register.py: element_hash)
__device__ __forceinline__ H128 elem_hash(const uint8_t* p, long long n) {
  u64 a = 0x9e3779b97f4a7c15ull ^ (u64)n, b = 0xc2b2ae3d27d4eb4full + (u64)n;
  for (long long i = 0; i < n; ++i) {
    a = (a ^ p[i]) * 0x100000001b3ull;
    b = (b ^ p[i]) * 0x00000100000001b3ull + 0x9e37ull;
    b ^= b >> 29;
  }
  return H128{mix64(a), mix64(b ^ 0x5bd1e9955bd1e995ull)};
}

__device__ __forceinline__ bool h_less(const H128& x, const H128& y) { return x.a != y.a ? x.a < y.a : x.b < y.b; }

// ---------------------------------------------------------------- validator
__device__ __forceinline__ bool ws(uint8_t c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }

// UTF-8 sequence starting at p[0] (>= 0x80); returns its length or 0 if
// invalid for Python's utf-8 codec with 'surrogatepass'
__device__ __forceinline__ int utf8_len(const uint8_t* p, const uint8_t* e) {
  const uint8_t c = p[0];
  int n;
  u32 cp;
  if (c >= 0xc2 && c <= 0xdf) { n = 2; cp = c & 0x1f; }
  else if (c >= 0xe0 && c <= 0xef) { n = 3; cp = c & 0x0f; }
  else if (c >= 0xf0 && c <= 0xf4) { n = 4; cp = c & 0x07; }
  else return 0;
  if (p + n > e) return 0;
  for (int k = 1; k < n; ++k) {
    if ((p[k] & 0xc0) != 0x80) return 0;
    cp = (cp << 6) | (p[k] & 0x3f);
  }
  if ((n == 3 && cp < 0x800) || (n == 4 && (cp < 0x10000 || cp > 0x10ffff))) return 0;
  return n;
}

// scan a JSON string starting after its opening quote; returns the position
// after the closing quote (nullptr if invalid); *esc = it held an escape
__device__ const uint8_t* scan_string(const uint8_t* p, const uint8_t* e, bool* esc) {
  *esc = false;
  while (p < e) {
    const uint8_t c = *p;
    if (c == '"') return p + 1;
    if (c == '\\') {
      *esc = true;
      if (p + 1 >= e) return nullptr;
      const uint8_t d = p[1];
      if (d == 'u') {
        if (p + 6 > e) return nullptr;
        for (int k = 2; k < 6; ++k) {
          const uint8_t h = p[k];
          if (!((h >= '0' && h <= '9') || (h >= 'a' && h <= 'f') || (h >= 'A' && h <= 'F'))) return nullptr;
        }
        p += 6;
      } else if (d == '"' || d == '\\' || d == '/' || d == 'b' || d == 'f' || d == 'n' || d == 'r' || d == 't') {
        p += 2;
      } else {
        return nullptr;
      }
      continue;
    }
    if (c < 0x20) return nullptr;  // strict json.loads: raw control characters are invalid
    if (c >= 0x80) {
      const int n = utf8_len(p, e);
      if (!n) return nullptr;
      p += n;
      continue;
    }
    ++p;
  }
  return nullptr;
}

__device__ const uint8_t* scan_number(const uint8_t* p, const uint8_t* e) {
  if (p < e && *p == '-') ++p;
  if (p >= e) return nullptr;
  if (*p == '0') {
    ++p;
  } else if (*p >= '1' && *p <= '9') {
    const uint8_t* d0 = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p - d0 > 4000) return nullptr;  // CPython's int digit limit: the host decides
  } else {
    return nullptr;
  }
  if (p < e && *p == '.') {
    ++p;
    if (p >= e || !(*p >= '0' && *p <= '9')) return nullptr;
    while (p < e && *p >= '0' && *p <= '9') ++p;
  }
  if (p < e && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    if (p >= e || !(*p >= '0' && *p <= '9')) return nullptr;
    while (p < e && *p >= '0' && *p <= '9') ++p;
  }
  return p;
}

__device__ __forceinline__ bool lit(const uint8_t* p, const uint8_t* e, const char* s, int n) {
  if (p + n > e) return false;
  for (int k = 0; k < n; ++k)
    if (p[k] != (uint8_t)s[k]) return false;
  return true;
}

// Validate one JSON value (any depth) starting at p; returns the end or
// nullptr (invalid / needs the host: NaN, Infinity, nesting beyond 64)
__device__ const uint8_t* skip_value(const uint8_t* p, const uint8_t* e) {
  u64 stack = 0;  // bit per level: 1 = object, 0 = array
  int depth = 0;
  // state: 0 expect value, 1 after value (expect , or close), 2 expect key (or } right after {), 3 expect key
  int st = 0;
  while (true) {
    while (p < e && ws(*p)) ++p;
    if (p >= e) return nullptr;
    const uint8_t c = *p;
    if (st == 0) {
      if (c == '{' || c == '[') {
        if (depth == 64) return nullptr;
        stack = (stack << 1) | (c == '{' ? 1u : 0u);
        ++depth;
        ++p;
        if (c == '{') {
          st = 2;
        } else {
          while (p < e && ws(*p)) ++p;
          if (p < e && *p == ']') {
            ++p;
            stack >>= 1;
            --depth;
            st = 1;
          } else {
            st = 0;
          }
        }
        if (depth == 0 && st == 1) return p;
        continue;
      }
      if (c == '"') {
        bool esc;
        p = scan_string(p + 1, e, &esc);
        if (!p) return nullptr;
      } else if (c == '-' || (c >= '0' && c <= '9')) {
        p = scan_number(p, e);
        if (!p) return nullptr;
      } else if (lit(p, e, "true", 4)) {
        p += 4;
      } else if (lit(p, e, "false", 5)) {
        p += 5;
      } else if (lit(p, e, "null", 4)) {
        p += 4;
      } else {
        return nullptr;  // includes NaN / Infinity / -Infinity (host decides)
      }
      if (depth == 0) return p;
      st = 1;
      continue;
    }
    if (st == 1) {
      const bool obj = stack & 1u;
      if (c == ',') {
        ++p;
        st = obj ? 3 : 0;
        continue;
      }
      if ((obj && c == '}') || (!obj && c == ']')) {
        ++p;
        stack >>= 1;
        --depth;
        if (depth == 0) return p;
        st = 1;
        continue;
      }
      return nullptr;
    }
    // st 2 / 3: a key
    if (st == 2 && c == '}') {
      ++p;
      stack >>= 1;
      --depth;
      if (depth == 0) return p;
      st = 1;
      continue;
    }
    if (c != '"') return nullptr;
    bool esc;
    p = scan_string(p + 1, e, &esc);
    if (!p) return nullptr;
    while (p < e && ws(*p)) ++p;
    if (p >= e || *p != ':') return nullptr;
    ++p;
    st = 0;
  }
}

// value of a requested field: a plain string, null, or a list of plain
// strings. kind: 1 value, 2 host, 3 present without a value (null, []);
// span: the string's content, or the whole list ([...], *is_list)
__device__ const uint8_t* field_value(const uint8_t* p, const uint8_t* e, int* kind, int* nelem, H128* out,
                                      const uint8_t** span, int* span_len, bool* is_list) {
  while (p < e && ws(*p)) ++p;
  if (p >= e) return nullptr;
  if (lit(p, e, "null", 4)) {
    *kind = 3;
    *nelem = 0;
    return p + 4;
  }
  const uint8_t* v0 = p;
  H128 el[LIST_MAX];
  int n = 0;
  if (*p == '"') {
    bool esc;
    const uint8_t* q = scan_string(p + 1, e, &esc);
    if (!q) return nullptr;
    if (esc) {
      *kind = 2;
      return q;
    }
    el[n++] = elem_hash(p + 1, q - 1 - (p + 1));
    *span = p + 1;
    *span_len = (int)(q - 1 - (p + 1));
    *is_list = false;
    p = q;
  } else if (*p == '[') {
    ++p;
    bool first = true;
    while (true) {
      while (p < e && ws(*p)) ++p;
      if (p >= e) return nullptr;
      if (*p == ']' && first) {
        ++p;
        break;
      }
      if (*p != '"') {  // non-string element: str(v) formatting is the host's
        const uint8_t* q = skip_value(p, e);
        if (!q) return nullptr;
        *kind = 2;
        // still validate the rest of the list
        p = q;
      } else {
        bool esc;
        const uint8_t* q = scan_string(p + 1, e, &esc);
        if (!q) return nullptr;
        if (esc || n == LIST_MAX) *kind = 2;
        else el[n++] = elem_hash(p + 1, q - 1 - (p + 1));
        p = q;
      }
      first = false;
      while (p < e && ws(*p)) ++p;
      if (p >= e) return nullptr;
      if (*p == ',') {
        ++p;
        continue;
      }
      if (*p == ']') {
        ++p;
        break;
      }
      return nullptr;
    }
    if (*kind == 2) return p;
    *span = v0;
    *span_len = (int)(p - v0);
    *is_list = true;
  } else {
    const uint8_t* q = skip_value(p, e);  // number / bool / object: host formatting / errors
    if (!q) return nullptr;
    *kind = 2;
    return q;
  }
  // sorted distinct element hashes -> the value hash
  for (int i = 1; i < n; ++i) {
    const H128 x = el[i];
    int j = i - 1;
    while (j >= 0 && h_less(x, el[j])) {
      el[j + 1] = el[j];
      --j;
    }
    el[j + 1] = x;
  }
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (m == 0 || el[i].a != el[m - 1].a || el[i].b != el[m - 1].b) el[m++] = el[i];
  *nelem = m;
  if (m == 0) {
    *kind = 3;
    return p;
  }
  u64 a = 0x243f6a8885a308d3ull ^ (u64)m, b = 0x13198a2e03707344ull;
  for (int i = 0; i < m; ++i) {
    a = mix64(a ^ el[i].a) + 0x9e3779b97f4a7c15ull;
    b = mix64(b ^ el[i].b ^ (a >> 7));
  }
  out->a = a;
  out->b = b;
  *kind = 1;
  return p;
}

// per record: 0 = fast path ok, 1 = the host must evaluate it
__global__ void jsonl_extract_kernel(const uint8_t* __restrict__ buf, const long long* __restrict__ rs,
                                     const long long* __restrict__ re, long long n_rec, JsonlFields f,
                                     uint8_t* kind_out, uint8_t* nelem_out, u64* ha, u64* hb, long long* vstart,
                                     int* vlen, uint8_t* host) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= n_rec) return;
  const uint8_t* p = buf + rs[r];
  const uint8_t* e = buf + re[r];
  int kind[JL_MAX_FIELDS], nel[JL_MAX_FIELDS], sl[JL_MAX_FIELDS];
  long long so[JL_MAX_FIELDS];
  H128 h[JL_MAX_FIELDS];
  for (int k = 0; k < f.n; ++k) {
    kind[k] = 0;
    nel[k] = 0;
    h[k] = H128{0, 0};
    so[k] = -1;
    sl[k] = 0;
  }
  bool bad = false;
  for (const uint8_t* q = p; q < e; ++q)
    if (*q == 0) bad = true;  // NUL: json.loads(bytes) may pick another encoding
  if (e - p >= 3 && p[0] == 0xef && p[1] == 0xbb && p[2] == 0xbf) bad = true;  // BOM
  while (!bad && p < e && ws(*p)) ++p;
  if (!bad && (p >= e || *p != '{')) bad = true;  // not an object: the host applies the parser
  if (!bad) {
    ++p;
    int st = 2;  // 2: key or '}', 3: key, 1: ',' or '}'
    while (true) {
      while (p < e && ws(*p)) ++p;
      if (p >= e) {
        bad = true;
        break;
      }
      if (st == 1) {
        if (*p == ',') {
          ++p;
          st = 3;
          continue;
        }
        if (*p == '}') {
          ++p;
          break;
        }
        bad = true;
        break;
      }
      if (st == 2 && *p == '}') {
        ++p;
        break;
      }
      if (*p != '"') {
        bad = true;
        break;
      }
      bool esc;
      const uint8_t* ks = p + 1;
      const uint8_t* q = scan_string(ks, e, &esc);
      if (!q || esc) {  // an escaped key may spell a field name: the host decodes it
        bad = true;
        break;
      }
      const long long klen = q - 1 - ks;
      p = q;
      while (p < e && ws(*p)) ++p;
      if (p >= e || *p != ':') {
        bad = true;
        break;
      }
      ++p;
      int fk = -1;
      for (int k = 0; k < f.n && fk < 0; ++k) {
        const long long a0 = f.off[k], n = f.off[k + 1] - a0;
        if (n != klen) continue;
        bool eq = true;
        for (long long t = 0; t < n && eq; ++t) eq = f.names[a0 + t] == ks[t];
        if (eq) fk = k;
      }
      if (fk >= 0) {  // the last occurrence wins (json.loads)
        int kd = 0, ne = 0, sn = 0;
        H128 hv{0, 0};
        const uint8_t* sp = nullptr;
        bool lst = false;
        q = field_value(p, e, &kd, &ne, &hv, &sp, &sn, &lst);
        if (!q) {
          bad = true;
          break;
        }
        kind[fk] = kd;
        nel[fk] = ne;
        h[fk] = hv;
        // span: content of a string value (>= 0), or ~start of a list value
        so[fk] = kd == 1 ? (lst ? ~(long long)(sp - buf) : (long long)(sp - buf)) : -1;
        sl[fk] = sn;
      } else {
        q = skip_value(p, e);
        if (!q) {
          bad = true;
          break;
        }
      }
      p = q;
      st = 1;
    }
    if (!bad) {
      while (p < e && ws(*p)) ++p;
      if (p != e) bad = true;  // trailing bytes: "Extra data"
    }
  }
  for (int k = 0; k < f.n; ++k) {
    bad |= kind[k] == 2;
    kind_out[r * f.n + k] = (uint8_t)kind[k];
    nelem_out[r * f.n + k] = (uint8_t)(nel[k] > 255 ? 255 : nel[k]);
    ha[r * f.n + k] = h[k].a;
    hb[r * f.n + k] = h[k].b;
    vstart[r * f.n + k] = so[k];
    vlen[r * f.n + k] = sl[k];
  }
  host[r] = bad ? 1 : 0;
}

}  // namespace mx

using namespace mx;

extern "C" {

int mx_jsonl_records(const uint8_t* buf, int64_t n_bytes, int64_t* rec_start, int64_t* rec_end, int64_t* rec_line,
                     int64_t capacity, int64_t* n_records, int64_t* n_lines, void* stream) {
  if (!buf || !n_records || n_bytes < 0 || (n_bytes % 16) != 0 || (reinterpret_cast<uintptr_t>(buf) % 16) != 0)
    return mx_fail(MX_ERR_INVALID, "jsonl buffer: null, or not a 16-byte aligned multiple of 16 bytes");
  cudaStream_t s = (cudaStream_t)stream;
  const long long nw = n_bytes / 16;
  DevBuf<u64> cnt;
  MX_CUDA_TRY(cnt.alloc(1, s));
  // pass 1: newline count (the total lands in a one-word scan)
  DevBuf<long long> nl;
  long long L = 0;
  {
    MX_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(u64), s));
    if (int rc = gs_run(nw, CountF{reinterpret_cast<const uint4*>(buf), cnt.p}, s)) return rc;
    u64 h = 0;
    MX_CUDA_TRY(cudaMemcpyAsync(&h, cnt.p, sizeof(u64), cudaMemcpyDeviceToHost, s));
    MX_CUDA_TRY(cudaStreamSynchronize(s));
    L = (long long)h;
  }
  if (n_lines) *n_lines = L;
  if (L == 0) {
    *n_records = 0;
    return MX_OK;
  }
  MX_CUDA_TRY(nl.alloc(L, s));
  if (int rc = gs_run(nw, NewlineF{reinterpret_cast<const uint4*>(buf), nl.p}, s)) return rc;
  if (!rec_start) {  // sizing call
    MX_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(u64), s));
    if (int rc = gs_run(L, NonEmptyF{nl.p, cnt.p}, s)) return rc;
    u64 h = 0;
    MX_CUDA_TRY(cudaMemcpyAsync(&h, cnt.p, sizeof(u64), cudaMemcpyDeviceToHost, s));
    MX_CUDA_TRY(cudaStreamSynchronize(s));
    *n_records = (long long)h;
    return MX_OK;
  }
  MX_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(u64), s));
  // the caller sized the outputs with a previous sizing call
  if (int rc = gs_run(L, RecCountF{RecordF{nl.p, reinterpret_cast<long long*>(rec_start), reinterpret_cast<long long*>(rec_end),
                                       reinterpret_cast<long long*>(rec_line)},
                               cnt.p}, s)) return rc;
  u64 h = 0;
  MX_CUDA_TRY(cudaMemcpyAsync(&h, cnt.p, sizeof(u64), cudaMemcpyDeviceToHost, s));
  MX_CUDA_TRY(cudaStreamSynchronize(s));
  if ((long long)h > capacity) return mx_fail(MX_ERR_INVALID, "jsonl records: %llu > capacity %lld", h, (long long)capacity);
  *n_records = (long long)h;
  return MX_OK;
}

int mx_jsonl_extract(const uint8_t* buf, const int64_t* rec_start, const int64_t* rec_end, int64_t n_records,
                     const uint8_t* field_names, const int64_t* field_offsets, int32_t n_fields, uint8_t* kind,
                     uint8_t* nelem, uint64_t* hash_a, uint64_t* hash_b, int64_t* value_start, int32_t* value_len,
                     uint8_t* host, void* stream) {
  if (n_fields < 0 || n_fields > JL_MAX_FIELDS)
    return mx_fail(MX_ERR_UNSUPPORTED, "%d requested fields (at most %d)", n_fields, JL_MAX_FIELDS);
  if (n_records == 0) return MX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  JsonlFields f{n_fields, field_names, reinterpret_cast<const long long*>(field_offsets)};
  jsonl_extract_kernel<<<(unsigned)((n_records + 127) / 128), 128, 0, s>>>(
      buf, reinterpret_cast<const long long*>(rec_start), reinterpret_cast<const long long*>(rec_end), n_records, f,
      kind, nelem, reinterpret_cast<u64*>(hash_a), reinterpret_cast<u64*>(hash_b),
      reinterpret_cast<long long*>(value_start), value_len, host);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

}  // extern "C"
