// musr_io.cpp -- native reader / writer of the muSR data file (SURVEY.md 8(f)
// row 3: fast .musr ingest).  Host code in libmusr_b200.so, C ABI in
// include/musr_b200.h (musr_file_*).
//
// Format and semantics are the reference's (pkg/src/blk/io.py:109-212):
//
//   DETECTOR <int>        starts a block (finishing the previous one)
//   dt <float> | t0 <int> | n0_slot <int> | nbkg_slot <int>
//   map <int>*  | func <float>*  | counts <int>*   (a new `counts` line replaces)
//   any other line continues `counts` once the block has one
//
// Reading follows load_musr_data (io.py:143-212) decision for decision so the
// first error, in file order, is the reference's:
//   * lines split like Python text mode (\n, \r\n, \r), stripped and split on
//     Python's ASCII whitespace; blank and '#' lines skipped;
//   * key dispatch order DETECTOR, (no block -> "data before any DETECTOR
//     header"), dt, t0, n0_slot, nbkg_slot, map, func, counts, continuation,
//     unknown key; int()/float() failures and a missing value are "malformed";
//   * a block is finished (missing keys in the order dt, t0, n0_slot,
//     nbkg_slot, map, counts -> first negative count -> negative map entry
//     (TheoryBinding, theory.py:370-376) -> empty histogram -> dt <= 0
//     (MusrDataset, musr.py:78-88)) when the next DETECTOR line or EOF is
//     reached, i.e. after every line of the block;
//   * int tokens follow Python int(): [+-]digits with single '_' between
//     digits; float tokens follow Python float(): decimal with optional
//     exponent or inf/infinity/nan, '_' between digits, no hex; conversion is
//     strtod (correctly rounded, like CPython).
// Inputs outside this byte-exact subset -- non-ASCII bytes, integers beyond
// int64 -- return MUSR_IO_UNSUPPORTED and the Python wrapper
// (musrio.py) parses that file with its restatement of io.py.
//
// Speed: the file is read once; lines are parsed by n threads over
// contiguous byte ranges (numbers into per-thread buffers, key lines and runs
// of continuation lines as items), then one sequential pass replays the
// reference's state machine over the items and the counts are gathered.
//
// Writing follows store_musr_data (io.py:124-140): the caller passes each
// detector's header text (DETECTOR ... func lines, formatted on the Python
// side with the reference's f-strings) and its counts; the counts are
// truncated to int64 like ndarray.astype(np.int64) and written 16 per line
// ("counts " / "  " prefixes), formatted in parallel.

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/musr_b200.h"

namespace {

enum Key : uint8_t { K_DETECTOR, K_DT, K_T0, K_N0, K_NBKG, K_MAP, K_FUNC, K_COUNTS, K_OTHER };

inline bool py_space(unsigned char c) {  // str.isspace() on ASCII
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}

// Python int() on an ASCII token.  0 ok, 1 invalid, 2 outside int64.
int parse_int(const char* s, const char* e, int64_t* out) {
  bool neg = false;
  if (s < e && (*s == '+' || *s == '-')) neg = (*s++ == '-');
  if (s == e || !(*s >= '0' && *s <= '9')) return 1;
  unsigned long long v = 0;
  bool big = false;
  bool prev_us = false;
  for (; s < e; ++s) {
    const char c = *s;
    if (c == '_') {
      if (prev_us) return 1;
      prev_us = true;
      continue;
    }
    if (!(c >= '0' && c <= '9')) return 1;
    prev_us = false;
    const unsigned d = (unsigned)(c - '0');
    if (v > (ULLONG_MAX - d) / 10) big = true;
    else v = v * 10 + d;
  }
  if (prev_us) return 1;  // trailing underscore
  if (big || v > (neg ? 9223372036854775808ull : 9223372036854775807ull)) return 2;
  *out = neg ? (int64_t)(0 - v) : (int64_t)v;
  return 0;
}

// digits with single underscores between digits: returns end or nullptr
const char* digitpart(const char* s, const char* e, std::string* acc) {
  if (s == e || !(*s >= '0' && *s <= '9')) return nullptr;
  while (s < e) {
    if (*s >= '0' && *s <= '9') {
      acc->push_back(*s++);
    } else if (*s == '_' && s + 1 < e && s[1] >= '0' && s[1] <= '9') {
      ++s;
    } else {
      break;
    }
  }
  return s;
}

bool ieq(const char* s, const char* e, const char* word) {
  const size_t n = std::strlen(word);
  if ((size_t)(e - s) != n) return false;
  for (size_t i = 0; i < n; ++i) {
    char c = s[i];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    if (c != word[i]) return false;
  }
  return true;
}

// Python float() on an ASCII token.  true on success.
bool parse_float(const char* s, const char* e, double* out) {
  std::string buf;
  const char* p = s;
  if (p < e && (*p == '+' || *p == '-')) buf.push_back(*p++);
  if (ieq(p, e, "inf") || ieq(p, e, "infinity") || ieq(p, e, "nan")) {
    buf.append(p, e);
    *out = std::strtod(buf.c_str(), nullptr);
    return true;
  }
  bool mant = false;
  if (p < e && *p >= '0' && *p <= '9') {
    p = digitpart(p, e, &buf);
    if (!p) return false;
    mant = true;
  }
  if (p < e && *p == '.') {
    buf.push_back('.');
    ++p;
    if (p < e && *p >= '0' && *p <= '9') {
      p = digitpart(p, e, &buf);
      if (!p) return false;
      mant = true;
    }
  }
  if (!mant) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    buf.push_back('e');
    ++p;
    if (p < e && (*p == '+' || *p == '-')) buf.push_back(*p++);
    p = digitpart(p, e, &buf);
    if (!p) return false;
  }
  if (p != e) return false;
  *out = std::strtod(buf.c_str(), nullptr);
  return true;
}

Key classify(const char* s, const char* e) {
  const size_t n = (size_t)(e - s);
  auto is = [&](const char* w) { return n == std::strlen(w) && std::memcmp(s, w, n) == 0; };
  if (is("DETECTOR")) return K_DETECTOR;
  if (is("dt")) return K_DT;
  if (is("t0")) return K_T0;
  if (is("n0_slot")) return K_N0;
  if (is("nbkg_slot")) return K_NBKG;
  if (is("map")) return K_MAP;
  if (is("func")) return K_FUNC;
  if (is("counts")) return K_COUNTS;
  return K_OTHER;
}

// One parsed unit in file order: a key line, or a run of consecutive
// non-key lines (their integers appended to the thread's buffer).
struct Item {
  Key key;
  bool bad;              // key line: malformed; run: some line malformed (bad_line)
  int64_t line;          // local line number of the key line / first line of the run
  int64_t bad_line;      // run: local line number of the first malformed line
  int64_t first_off;     // byte offset / length of the (stripped) first line,
  int64_t first_len;     //   for the error messages the Python side formats
  int64_t bad_off, bad_len;
  int64_t ival;          // DETECTOR / t0 / n0_slot / nbkg_slot value
  double fval;           // dt
  size_t off, n;         // values in the thread buffer (ints, or doubles for func)
};

struct Chunk {
  std::vector<Item> items;
  std::vector<int64_t> ints;
  std::vector<double> dbls;
  int64_t lines = 0;     // physical lines in the chunk
  bool unsupported = false;
};

// byte classes: 0 other, 1 Python whitespace (not a line end), 2 digit, 3 line end
struct CharClass {
  unsigned char c[256];
  CharClass() {
    for (int i = 0; i < 256; ++i) c[i] = 0;
    for (int i = 0; i < 256; ++i)
      if (py_space((unsigned char)i)) c[i] = 1;
    for (int i = '0'; i <= '9'; ++i) c[i] = 2;
    c[(unsigned char)'\n'] = c[(unsigned char)'\r'] = 3;
  }
};
const CharClass kClass;

// Integers of one line from p (just after the key token, or its start for a
// continuation line) to the line end, fused tokenize + Python int().  Returns
// the line end; *bad = some token is not an int (the rest of the line is
// skipped), *big = some int is outside int64.
const char* line_ints(const char* p, const char* hi, std::vector<int64_t>* out, bool* bad,
                      bool* big) {
  const unsigned char* cls = kClass.c;
  while (p < hi) {
    unsigned k = cls[(unsigned char)*p];
    if (k == 1) { ++p; continue; }
    if (k == 3) break;
    const char* t = p;  // token
    while (p < hi && cls[(unsigned char)*p] == 2) ++p;  // plain digit run (common case)
    if (p > t && p - t <= 18 && (p == hi || cls[(unsigned char)*p] & 1)) {
      int64_t v = 0;
      for (const char* q = t; q < p; ++q) v = v * 10 + (*q - '0');
      out->push_back(v);
      continue;
    }
    while (p < hi && !(cls[(unsigned char)*p] & 1)) ++p;  // token end (space or line end)
    int64_t v;
    const int r = parse_int(t, p, &v);
    if (r == 0) { out->push_back(v); continue; }
    if (r == 2) *big = true;
    *bad = true;
    while (p < hi && cls[(unsigned char)*p] != 3) ++p;
    break;
  }
  return p;
}

void parse_chunk(const char* base, size_t lo, size_t hi_off, Chunk* ck) {
  const unsigned char* cls = kClass.c;
  // at most one integer per two bytes; reserving (virtual memory, touched
  // only as filled) avoids the reallocation copies of a growing buffer
  ck->ints.reserve((hi_off - lo) / 2 + 16);
  const char* hi = base + hi_off;
  std::vector<std::pair<const char*, const char*>> tok;
  int64_t ln = 0;
  const char* p = base + lo;
  Item* run = nullptr;  // open run of non-key lines
  while (p < hi) {
    ++ln;
    const char* ls = p;  // line start
    while (p < hi && cls[(unsigned char)*p] == 1) ++p;
    const char* s = p;   // stripped start
    const char* t_end = p;
    while (t_end < hi && !(cls[(unsigned char)*t_end] & 1)) ++t_end;  // first token
    Key k = K_OTHER;
    bool skip = (s == hi || cls[(unsigned char)*s] == 3 || *s == '#');
    if (!skip) k = classify(s, t_end);
    const char* e;  // line end (before the terminator)
    if (!skip && (k == K_OTHER || k == K_COUNTS)) {
      // hot path: integers, fused with the scan to the line end
      const size_t before = ck->ints.size();
      bool bad = false, big = false;
      if (k == K_OTHER && run && run->bad) {
        e = t_end;
        while (e < hi && cls[(unsigned char)*e] != 3) ++e;
      } else {
        e = line_ints(k == K_OTHER ? s : t_end, hi, &ck->ints, &bad, &big);
      }
      if (big) ck->unsupported = true;
      const char* se = e;
      while (se > s && cls[(unsigned char)se[-1]] == 1) --se;
      const int64_t soff = (int64_t)(s - base), slen = (int64_t)(se - s);
      if (k == K_OTHER) {
        if (!run) {
          ck->items.push_back(Item{K_OTHER, false, ln, -1, soff, slen, 0, 0, 0, 0.0, before, 0});
          run = &ck->items.back();
        }
        if (!run->bad && bad) {
          ck->ints.resize(before);  // a malformed line contributes nothing after the error
          run->bad = true;
          run->bad_line = ln;
          run->bad_off = soff;
          run->bad_len = slen;
        }
        run->n = ck->ints.size() - run->off;
      } else {
        run = nullptr;
        Item it{K_COUNTS, bad, ln, -1, soff, slen, 0, 0, 0, 0.0, before, 0};
        if (bad) ck->ints.resize(before);
        it.n = ck->ints.size() - before;
        ck->items.push_back(it);
      }
    } else {
      e = t_end;
      while (e < hi && cls[(unsigned char)*e] != 3) ++e;
      if (!skip) {
        const char* se = e;
        while (se > s && cls[(unsigned char)se[-1]] == 1) --se;
        tok.clear();
        for (const char* q = s; q < se;) {
          while (q < se && cls[(unsigned char)*q] == 1) ++q;
          const char* r = q;
          while (r < se && cls[(unsigned char)*r] != 1) ++r;
          if (r > q) tok.emplace_back(q, r);
          q = r;
        }
        run = nullptr;
        Item it{k, false, ln, -1, (int64_t)(s - base), (int64_t)(se - s), 0, 0, 0, 0.0, 0, 0};
        auto one_int = [&]() {
          if (tok.size() < 2) { it.bad = true; return; }
          const int r = parse_int(tok[1].first, tok[1].second, &it.ival);
          if (r == 2) ck->unsupported = true;
          it.bad = r != 0;
        };
        switch (k) {
          case K_DETECTOR: case K_T0: case K_N0: case K_NBKG:
            one_int();
            break;
          case K_DT:
            it.bad = tok.size() < 2 || !parse_float(tok[1].first, tok[1].second, &it.fval);
            break;
          case K_MAP:
            it.off = ck->ints.size();
            for (size_t i = 1; i < tok.size(); ++i) {
              int64_t v;
              const int r = parse_int(tok[i].first, tok[i].second, &v);
              if (r == 2) ck->unsupported = true;
              if (r != 0) { it.bad = true; break; }
              ck->ints.push_back(v);
            }
            it.n = ck->ints.size() - it.off;
            break;
          case K_FUNC:
            it.off = ck->dbls.size();
            for (size_t i = 1; i < tok.size(); ++i) {
              double v;
              if (!parse_float(tok[i].first, tok[i].second, &v)) { it.bad = true; break; }
              ck->dbls.push_back(v);
            }
            it.n = ck->dbls.size() - it.off;
            break;
          default:
            break;
        }
        ck->items.push_back(it);
      }
    }
    (void)ls;
    // consume the line terminator (\n, \r\n or \r)
    p = e;
    if (p < hi) p += (*p == '\r' && p + 1 < hi && p[1] == '\n') ? 2 : 1;
  }
  ck->lines = ln;
}

struct Seg {  // a piece of a block's counts: [off, off+n) of chunk c's ints
  int c;
  size_t off, n;
};

struct Block {
  int64_t index = 0;
  double dt = 0.0;
  int64_t t0 = 0, n0 = 0, nbkg = 0;
  bool has_dt = false, has_t0 = false, has_n0 = false, has_nbkg = false, has_map = false,
       has_counts = false;
  std::vector<int64_t> map;
  std::vector<double> func;
  std::vector<Seg> segs;  // the counts, as pieces of the chunks' integer buffers
  int64_t n_counts = 0;
};

int nthreads_for(int requested, size_t bytes) {
  int n = requested > 0 ? requested : (int)std::thread::hardware_concurrency();
  if (n < 1) n = 1;
  const size_t per = 4u << 20;  // >= 4 MiB per thread
  n = (int)std::min<size_t>((size_t)n, std::max<size_t>(1, bytes / per));
  return std::min(n, 64);
}

}  // namespace

struct musr_file {
  std::vector<Block> blocks;
  std::vector<Chunk> chunks;  // own the parsed integers the blocks' segments point into
};

extern "C" {

int musr_file_load(const char* path, int n_threads, musr_file** out, musr_io_error* err) {
  if (!path || !out || !err) return MUSR_ERR_ARG;
  *out = nullptr;
  std::memset(err, 0, sizeof(*err));
  err->detector = err->bin = err->line = -1;
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) {
    err->code = MUSR_IO_OS;
    err->bin = errno;
    return MUSR_ERR_IO;
  }
  struct stat st;
  std::vector<char> data;
  // +1: a full buffer after st_size bytes means the file grew; read on
  if (fstat(fd, &st) == 0 && st.st_size > 0) data.resize((size_t)st.st_size + 1);
  size_t got = 0;
  while (true) {
    if (got == data.size()) data.resize(std::max<size_t>(4096, data.size() * 2));
    const ssize_t r = ::read(fd, data.data() + got, data.size() - got);
    if (r < 0) {
      if (errno == EINTR) continue;
      err->code = MUSR_IO_OS;
      err->bin = errno;
      ::close(fd);
      return MUSR_ERR_IO;
    }
    if (r == 0) break;
    got += (size_t)r;
  }
  ::close(fd);
  data.resize(got);
  const char* base = data.data();
  {
    unsigned char any = 0;  // OR of all bytes: bit 7 set <=> a non-ASCII byte
    for (size_t i = 0; i < got; ++i) any |= (unsigned char)base[i];
    if (any & 0x80) {
      err->code = MUSR_IO_UNSUPPORTED;
      return MUSR_ERR_IO;
    }
  }

  // chunk boundaries at line starts (a "\r\n" pair is never split)
  const int nt = nthreads_for(n_threads, got);
  std::vector<size_t> cut(nt + 1, got);
  cut[0] = 0;
  for (int t = 1; t < nt; ++t) {
    size_t p = std::max(cut[t - 1], got * (size_t)t / (size_t)nt);
    while (p < got && base[p - 1] != '\n' && base[p - 1] != '\r') ++p;
    if (p < got && base[p - 1] == '\r' && base[p] == '\n') ++p;
    cut[t] = p;
  }
  musr_file* f = new musr_file();
  f->chunks.resize(nt);
  std::vector<Chunk>& chunks = f->chunks;
  {
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t)
      pool.emplace_back(parse_chunk, base, cut[t], cut[t + 1], &chunks[t]);
    parse_chunk(base, cut[0], cut[1], &chunks[0]);
    for (auto& th : pool) th.join();
  }
  for (auto& ck : chunks)
    if (ck.unsupported) {
      err->code = MUSR_IO_UNSUPPORTED;
      delete f;
      return MUSR_ERR_IO;
    }

  // sequential replay of io.py:171-212 over the items
  auto fail_line = [&](int code, int64_t line, int64_t off, int64_t len) {
    err->code = code;
    err->line = line;
    err->text_off = off;
    err->text_len = len;
    return MUSR_ERR_IO;
  };
  std::vector<Block>& blocks = f->blocks;
  bool open_block = false;
  Block cur;
  auto finish = [&](Block& b) -> int {
    static const char* names[] = {"dt", "t0", "n0_slot", "nbkg_slot", "map", "counts"};
    const bool have[] = {b.has_dt, b.has_t0, b.has_n0, b.has_nbkg, b.has_map, b.has_counts};
    std::string miss;
    for (int i = 0; i < 6; ++i)
      if (!have[i]) miss += (miss.empty() ? "" : ", ") + std::string(names[i]);
    err->detector = b.index;
    if (!miss.empty()) {
      err->code = MUSR_IO_MISSING;
      std::snprintf(err->missing, sizeof(err->missing), "%s", miss.c_str());
      return MUSR_ERR_IO;
    }
    int64_t bin = 0;
    for (const Seg& sg : b.segs) {
      const int64_t* v = chunks[sg.c].ints.data() + sg.off;
      for (size_t i = 0; i < sg.n; ++i, ++bin)
        if (v[i] < 0) {
          err->code = MUSR_IO_NEGATIVE;
          err->bin = bin;
          return MUSR_ERR_IO;
        }
    }
    for (int64_t m : b.map)
      if (m < 0) {
        err->code = MUSR_IO_BAD_MAP;
        return MUSR_ERR_IO;
      }
    if (b.n_counts < 1) {
      err->code = MUSR_IO_EMPTY_HIST;
      return MUSR_ERR_IO;
    }
    if (b.dt <= 0.0) {  // NaN passes, as in MusrDataset
      err->code = MUSR_IO_BAD_DT;
      return MUSR_ERR_IO;
    }
    err->detector = -1;
    blocks.push_back(std::move(b));
    return MUSR_OK;
  };
  int rc = MUSR_OK;
  int64_t line0 = 0;
  for (int c = 0; c < nt && rc == MUSR_OK; ++c) {
    Chunk& ck = chunks[c];
    for (const Item& it : ck.items) {
      const int64_t line = line0 + it.line;
      if (it.key == K_DETECTOR) {
        if (open_block && (rc = finish(cur)) != MUSR_OK) {
          // io.py:177-178: finish() runs inside the DETECTOR line's try, where the
          // TheoryBinding ValueError of a negative map entry becomes that line's
          // "malformed line" FormatError (at EOF it stays a TheoryError)
          if (err->code == MUSR_IO_BAD_MAP) {
            err->detector = -1;
            rc = fail_line(MUSR_IO_MALFORMED, line, it.first_off, it.first_len);
          }
          break;
        }
        open_block = false;
        if (it.bad) { rc = fail_line(MUSR_IO_MALFORMED, line, it.first_off, it.first_len); break; }
        cur = Block();
        cur.index = it.ival;
        open_block = true;
        continue;
      }
      if (!open_block) {
        rc = fail_line(MUSR_IO_BEFORE_HEADER, line, it.first_off, it.first_len);
        break;
      }
      if (it.key == K_OTHER) {
        if (!cur.has_counts) {
          rc = fail_line(MUSR_IO_UNKNOWN_KEY, line, it.first_off, it.first_len);
          break;
        }
        if (it.n) {
          cur.segs.push_back(Seg{c, it.off, it.n});
          cur.n_counts += (int64_t)it.n;
        }
        if (it.bad) {
          rc = fail_line(MUSR_IO_MALFORMED, line0 + it.bad_line, it.bad_off, it.bad_len);
          break;
        }
        continue;
      }
      if (it.bad) { rc = fail_line(MUSR_IO_MALFORMED, line, it.first_off, it.first_len); break; }
      switch (it.key) {
        case K_DT: cur.dt = it.fval; cur.has_dt = true; break;
        case K_T0: cur.t0 = it.ival; cur.has_t0 = true; break;
        case K_N0: cur.n0 = it.ival; cur.has_n0 = true; break;
        case K_NBKG: cur.nbkg = it.ival; cur.has_nbkg = true; break;
        case K_MAP:
          cur.map.assign(ck.ints.begin() + it.off, ck.ints.begin() + it.off + it.n);
          cur.has_map = true;
          break;
        case K_FUNC:
          cur.func.assign(ck.dbls.begin() + it.off, ck.dbls.begin() + it.off + it.n);
          break;
        case K_COUNTS:
          cur.segs.clear();
          cur.n_counts = 0;
          if (it.n) {
            cur.segs.push_back(Seg{c, it.off, it.n});
            cur.n_counts = (int64_t)it.n;
          }
          cur.has_counts = true;
          break;
        default:
          break;
      }
    }
    line0 += ck.lines;
  }
  if (rc == MUSR_OK && open_block) rc = finish(cur);
  if (rc == MUSR_OK && blocks.empty()) {
    err->code = MUSR_IO_NO_BLOCKS;
    rc = MUSR_ERR_IO;
  }
  if (rc != MUSR_OK) {
    delete f;
    return rc;
  }
  *out = f;
  return MUSR_OK;
}

int musr_file_n_detectors(const musr_file* f) { return f ? (int)f->blocks.size() : 0; }

int musr_file_detector(const musr_file* f, int i, musr_detector_info* info) {
  if (!f || !info || i < 0 || i >= (int)f->blocks.size()) return MUSR_ERR_ARG;
  const Block& b = f->blocks[(size_t)i];
  info->index = b.index;
  info->dt = b.dt;
  info->t0_bin = b.t0;
  info->n0_slot = b.n0;
  info->nbkg_slot = b.nbkg;
  info->n_map = (int64_t)b.map.size();
  info->n_func = (int64_t)b.func.size();
  info->n_counts = b.n_counts;
  return MUSR_OK;
}

int musr_file_copy(const musr_file* f, int i, int64_t* map, double* func, double* counts_f64,
                   int64_t* counts_i64) {
  if (!f || i < 0 || i >= (int)f->blocks.size()) return MUSR_ERR_ARG;
  const Block& b = f->blocks[(size_t)i];
  if (map && !b.map.empty()) std::memcpy(map, b.map.data(), b.map.size() * 8);
  if (func && !b.func.empty()) std::memcpy(func, b.func.data(), b.func.size() * 8);
  size_t k = 0;
  for (const Seg& sg : b.segs) {
    const int64_t* v = f->chunks[sg.c].ints.data() + sg.off;
    if (counts_i64) std::memcpy(counts_i64 + k, v, sg.n * 8);
    if (counts_f64)
      for (size_t i = 0; i < sg.n; ++i) counts_f64[k + i] = (double)v[i];
    k += sg.n;
  }
  return MUSR_OK;
}

void musr_file_free(musr_file* f) { delete f; }

// ---- writer ------------------------------------------------------------------

}  // extern "C"

namespace {

// ndarray.astype(np.int64) of one double (x86: NaN/inf/out of range -> INT64_MIN)
inline int64_t to_i64(double x) {
  if (!(x > -9223372036854775808.0 && x < 9223372036854775808.0)) return INT64_MIN;
  return (int64_t)x;
}

inline char* put_i64(char* p, int64_t v) {
  char tmp[24];
  int n = 0;
  unsigned long long u = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
  do { tmp[n++] = (char)('0' + u % 10); u /= 10; } while (u);
  if (v < 0) *p++ = '-';
  while (n) *p++ = tmp[--n];
  return p;
}

// counts lines of one detector, [row_lo, row_hi) of its 16-value rows
void format_rows(const double* c, int64_t n, int64_t row_lo, int64_t row_hi, std::string* out) {
  out->resize((size_t)(row_hi - row_lo) * (16 * 21 + 8));
  char* p = &(*out)[0];
  for (int64_t r = row_lo; r < row_hi; ++r) {
    const int64_t lo = r * 16, hi = std::min<int64_t>(lo + 16, n);
    if (r == 0) { std::memcpy(p, "counts ", 7); p += 7; }
    else { *p++ = ' '; *p++ = ' '; }
    for (int64_t k = lo; k < hi; ++k) {
      if (k > lo) *p++ = ' ';
      p = put_i64(p, to_i64(c[k]));
    }
    *p++ = '\n';
  }
  out->resize((size_t)(p - out->data()));
}

}  // namespace

extern "C" {

int musr_file_store(const char* path, int n_det, const char* const* headers,
                    const double* const* counts, const int64_t* n_counts, int n_threads,
                    musr_io_error* err) {
  if (!path || n_det < 0 || (n_det && (!headers || !counts || !n_counts)) || !err)
    return MUSR_ERR_ARG;
  std::memset(err, 0, sizeof(*err));
  // work units: (detector, row range) of ~64K rows
  struct Unit { int d; int64_t lo, hi; };
  std::vector<Unit> units;
  int64_t total_rows = 0;
  for (int d = 0; d < n_det; ++d) {
    const int64_t rows = (n_counts[d] + 15) / 16;
    for (int64_t lo = 0; lo < rows; lo += 65536) units.push_back({d, lo, std::min(rows, lo + 65536)});
    total_rows += rows;
  }
  std::vector<std::string> text(units.size());
  int nt = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
  nt = std::max(1, std::min<int>(nt, (int)std::max<size_t>(1, units.size())));
  {
    auto work = [&](int t) {
      for (size_t u = (size_t)t; u < units.size(); u += (size_t)nt)
        format_rows(counts[units[u].d], n_counts[units[u].d], units[u].lo, units[u].hi, &text[u]);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  }
  (void)total_rows;
  FILE* fp = std::fopen(path, "wb");
  if (!fp) {
    err->code = MUSR_IO_OS;
    err->bin = errno;
    return MUSR_ERR_IO;
  }
  // "\n".join(lines): every detector contributes header lines, counts lines
  // and one empty line; the join puts no newline after the final empty line.
  size_t u = 0;
  bool ok = true;
  for (int d = 0; d < n_det && ok; ++d) {
    const size_t hl = std::strlen(headers[d]);
    ok = std::fwrite(headers[d], 1, hl, fp) == hl;
    for (; ok && u < units.size() && units[u].d == d; ++u)
      ok = std::fwrite(text[u].data(), 1, text[u].size(), fp) == text[u].size();
    if (ok && d + 1 < n_det) ok = std::fputc('\n', fp) != EOF;
  }
  if (std::fclose(fp) != 0) ok = false;
  if (!ok) {
    err->code = MUSR_IO_OS;
    err->bin = errno;
    return MUSR_ERR_IO;
  }
  return MUSR_OK;
}

}  // extern "C"
