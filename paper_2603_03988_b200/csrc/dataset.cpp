// SPDX-License-Identifier: Apache-2.0
// Request ingest (SURVEY.md section 8(f) "next 3"): the reference's JSONL dataset format
// `rankformer.dataset` v1 (dataset_io.cpp:14-56 writer, :58-162 reader) read into the
// structure-of-arrays batches sort_forward takes, in pinned host memory so the per-step
// host -> device copies run at full link speed.
//
// The reference parses with nlohmann::json (vendored, not in this image); this is a small
// recursive-descent JSON reader for the value kinds the schema uses (objects, arrays,
// integers, reals, strings, literals). Validation and error texts follow read_dataset:
// "dataset line N, field 'F': what" (DatasetFormatError, dataset_io.hpp:12-25), status 1.
#include <cuda_runtime.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/sort_b200.h"
#include "plan.hpp"

namespace sortk {

extern thread_local std::string g_last_error;  // runtime.cu (sort_last_error)

namespace {

struct JVal {
  enum Kind { Null, Bool, Int, Real, Str, Arr, Obj } kind = Null;
  int64_t i = 0;
  double r = 0.0;
  bool b = false;
  std::string s;
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;
  const JVal* find(const char* k) const {
    for (const auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const char* p;
  const char* e;
  bool ok = true;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(e - p) < n || std::strncmp(p, w, n) != 0) return false;
    p += n;
    return true;
  }
  JVal value() {
    JVal v;
    ws();
    if (p >= e) {
      ok = false;
      return v;
    }
    const char c = *p;
    if (c == '{') {
      v.kind = JVal::Obj;
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return v;
      }
      while (ok) {
        ws();
        JVal k = value();
        if (!ok || k.kind != JVal::Str) {
          ok = false;
          break;
        }
        ws();
        if (p >= e || *p != ':') {
          ok = false;
          break;
        }
        ++p;
        JVal x = value();
        v.o.emplace_back(std::move(k.s), std::move(x));
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          break;
        }
        ok = false;
      }
      return v;
    }
    if (c == '[') {
      v.kind = JVal::Arr;
      ++p;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return v;
      }
      while (ok) {
        v.a.push_back(value());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          break;
        }
        ok = false;
      }
      return v;
    }
    if (c == '"') {
      v.kind = JVal::Str;
      ++p;
      while (p < e && *p != '"') {
        if (*p == '\\' && p + 1 < e) ++p;
        v.s.push_back(*p++);
      }
      if (p >= e) ok = false;
      ++p;
      return v;
    }
    if (lit("true")) {
      v.kind = JVal::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = JVal::Bool;
      return v;
    }
    if (lit("null")) return v;
    // number
    const char* s = p;
    bool real = false;
    if (p < e && (*p == '-' || *p == '+')) ++p;
    while (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '-' || *p == '+')) {
      if (*p == '.' || *p == 'e' || *p == 'E') real = true;
      ++p;
    }
    if (p == s) {
      ok = false;
      return v;
    }
    const std::string num(s, p);
    errno = 0;
    if (real) {
      v.kind = JVal::Real;
      v.r = std::strtod(num.c_str(), nullptr);
    } else {
      v.kind = JVal::Int;
      v.i = std::strtoll(num.c_str(), nullptr, 10);
      v.r = static_cast<double>(v.i);
      if (errno == ERANGE) ok = false;
    }
    return v;
  }
};

struct FormatError : ConfigError {
  FormatError(size_t line, const std::string& field, const std::string& what)
      : ConfigError("dataset line " + std::to_string(line) + ", field '" + field + "': " + what) {}
};

int64_t as_int(const JVal& v, size_t line, const char* field) {
  if (v.kind != JVal::Int) throw FormatError(line, field, "type must be number (integer)");
  return v.i;
}
int32_t as_i32(const JVal& v, size_t line, const char* field) {
  const int64_t x = as_int(v, line, field);
  if (x < std::numeric_limits<int32_t>::min() || x > std::numeric_limits<int32_t>::max())
    throw FormatError(line, field, "integer out of range");
  return static_cast<int32_t>(x);
}

}  // namespace

struct Dataset {
  // one parsed RequestSample (data.hpp:32-38)
  struct Rec {
    int64_t id = 0, ts = 0;
    std::vector<int32_t> profile, item, action, scene, cand, click, cart, purchase;
    std::vector<int64_t> hts;
    int n_side = 0;
  };
  std::vector<Rec> recs;
  // pinned SoA staging of the last batch
  int32_t *p_item = nullptr, *p_action = nullptr, *p_scene = nullptr, *p_prof = nullptr, *p_cand = nullptr;
  int64_t *p_ts = nullptr, *p_req = nullptr;
  size_t cap_item = 0, cap_action = 0, cap_scene = 0, cap_ts = 0, cap_c = 0, cap_b = 0, cap_p = 0;
  std::map<void*, bool> pinned;  // allocation -> page-locked (false: plain host memory, no driver)
  void release(void* q) {
    if (!q) return;
    if (pinned[q]) cudaFreeHost(q); else std::free(q);
    pinned.erase(q);
  }
  ~Dataset() {
    for (void* q : {static_cast<void*>(p_item), static_cast<void*>(p_action), static_cast<void*>(p_scene),
                    static_cast<void*>(p_prof), static_cast<void*>(p_cand), static_cast<void*>(p_ts),
                    static_cast<void*>(p_req)})
      release(q);
  }
};

// read_dataset (dataset_io.cpp:58-162)
static void parse_dataset(const std::string& path, Dataset& ds) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw RuntimeFailure("read_dataset: cannot open " + path);
  std::string line;
  size_t line_no = 0;
  if (!std::getline(in, line)) throw FormatError(1, "header", "empty file");
  ++line_no;
  JParser hp{line.data(), line.data() + line.size()};
  JVal header = hp.value();
  hp.ws();
  if (!hp.ok || hp.p != hp.e || header.kind != JVal::Obj) throw FormatError(1, "header", "not a JSON object");
  const JVal* sn = header.find("schema");
  if (!sn || sn->kind != JVal::Str || sn->s != "rankformer.dataset") throw FormatError(1, "schema", "unknown schema name");
  const JVal* ver = header.find("version");
  if (!ver || ver->kind != JVal::Int || ver->i != 1) throw FormatError(1, "version", "unsupported schema version");
  if (const JVal* n = header.find("records"); n && n->kind == JVal::Int && n->i > 0)
    ds.recs.reserve(static_cast<size_t>(n->i));
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    JParser rp{line.data(), line.data() + line.size()};
    JVal rec = rp.value();
    rp.ws();
    if (!rp.ok || rp.p != rp.e || rec.kind != JVal::Obj) throw FormatError(line_no, "record", "malformed JSON");
    auto require = [&](const char* f) -> const JVal& {
      const JVal* v = rec.find(f);
      if (!v) throw FormatError(line_no, f, "missing");
      return *v;
    };
    Dataset::Rec s;
    s.id = as_int(require("request_id"), line_no, "record");
    s.ts = as_int(require("ts"), line_no, "record");
    const JVal& prof = require("profile");
    if (prof.kind != JVal::Arr) throw FormatError(line_no, "record", "profile must be an array");
    for (const JVal& x : prof.a) s.profile.push_back(as_i32(x, line_no, "record"));
    const JVal& hist = require("history");
    if (hist.kind != JVal::Arr) throw FormatError(line_no, "history", "not an array");
    int64_t prev_ts = std::numeric_limits<int64_t>::min();
    for (const JVal& h : hist.a) {
      if (h.kind != JVal::Arr || h.a.size() != 4)
        throw FormatError(line_no, "history", "event must be [item,action,ts,scene]");
      const int32_t item = as_i32(h.a[0], line_no, "history");
      const int32_t action = as_i32(h.a[1], line_no, "history");
      if (action < 0 || action > 2) throw FormatError(line_no, "history.action", "out of range");
      const int64_t ts = as_int(h.a[2], line_no, "history");
      const int32_t scene = as_i32(h.a[3], line_no, "history");
      if (ts < prev_ts) throw FormatError(line_no, "history.ts", "timestamps must be non-decreasing");
      if (ts >= s.ts) throw FormatError(line_no, "history.ts", "event not before request");
      prev_ts = ts;
      s.item.push_back(item);
      s.action.push_back(action);
      s.hts.push_back(ts);
      s.scene.push_back(scene);
    }
    const JVal& cands = require("candidates");
    if (cands.kind != JVal::Arr || cands.a.empty())
      throw FormatError(line_no, "candidates", "must be a non-empty array");
    for (const JVal& cj : cands.a) {
      if (cj.kind != JVal::Arr || cj.a.size() != 5)
        throw FormatError(line_no, "candidates", "candidate must be [item,click,cart,purchase,[side...]]");
      const int32_t item = as_i32(cj.a[0], line_no, "candidates");
      const int32_t click = as_i32(cj.a[1], line_no, "candidates");
      const int32_t cart = as_i32(cj.a[2], line_no, "candidates");
      const int32_t purchase = as_i32(cj.a[3], line_no, "candidates");
      if (cj.a[4].kind != JVal::Arr) throw FormatError(line_no, "candidates", "side features must be an array");
      for (const JVal& x : cj.a[4].a)
        if (x.kind != JVal::Int && x.kind != JVal::Real) throw FormatError(line_no, "candidates", "side feature type");
      if ((click | cart | purchase) >> 1 || click < 0 || cart < 0 || purchase < 0)
        throw FormatError(line_no, "candidates.labels", "labels must be 0/1");
      if (purchase > click) throw FormatError(line_no, "candidates.purchase", "purchase=1 requires click=1");
      if (cart > click) throw FormatError(line_no, "candidates.cart", "cart=1 requires click=1");
      s.cand.push_back(item);
      s.click.push_back(click);
      s.cart.push_back(cart);
      s.purchase.push_back(purchase);
      s.n_side = std::max(s.n_side, static_cast<int>(cj.a[4].a.size()));
    }
    ds.recs.push_back(std::move(s));
  }
}

// Pinned staging (page-locked: full-speed, asynchronous host -> device copies); plain host
// memory when no CUDA driver is present (parsing and packing are host-only work).
template <class T>
static void ensure_pinned(Dataset& ds, T*& p, size_t& cap, size_t n) {
  if (n <= cap && p) return;
  ds.release(p);
  p = nullptr;
  void* q = nullptr;
  bool pin = true;
  if (cudaHostAlloc(&q, std::max<size_t>(n, 1) * sizeof(T), cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    pin = false;
    q = std::malloc(std::max<size_t>(n, 1) * sizeof(T));
    if (!q) throw RuntimeFailure("dataset: out of host memory");
  }
  ds.pinned[q] = pin;
  p = static_cast<T*>(q);
  cap = n;
}

}  // namespace sortk

using namespace sortk;

extern "C" {


int sort_dataset_open(const char* path, SortDataset* out) {
  try {
    if (!path || !out) throw ConfigError("null argument");
    auto ds = std::make_unique<Dataset>();
    parse_dataset(path, *ds);
    *out = reinterpret_cast<SortDataset>(ds.release());
    return SORT_OK;
  } catch (const ConfigError& e) {
    g_last_error = e.what();
    return SORT_CONFIG_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SORT_RUNTIME_FAILURE;
  }
}

void sort_dataset_close(SortDataset d) { delete reinterpret_cast<Dataset*>(d); }

int64_t sort_dataset_size(SortDataset d) {
  return d ? static_cast<int64_t>(reinterpret_cast<Dataset*>(d)->recs.size()) : -1;
}

int sort_dataset_batch(SortDataset d, int64_t first, int32_t count, int32_t n_hist, int32_t n_cand,
                       int32_t n_profile_fields, SortBatch* batch, float* labels, int64_t* request_ids) {
  try {
    Dataset* ds = reinterpret_cast<Dataset*>(d);
    if (!ds || !batch) throw ConfigError("null argument");
    if (count < 1 || first < 0 || first + count > static_cast<int64_t>(ds->recs.size()))
      throw ConfigError("dataset batch out of range");
    const size_t B = static_cast<size_t>(count);
    ensure_pinned(*ds, ds->p_item, ds->cap_item, B * n_hist);
    ensure_pinned(*ds, ds->p_action, ds->cap_action, B * n_hist);
    ensure_pinned(*ds, ds->p_scene, ds->cap_scene, B * n_hist);
    ensure_pinned(*ds, ds->p_ts, ds->cap_ts, B * n_hist);
    ensure_pinned(*ds, ds->p_cand, ds->cap_c, B * n_cand);
    ensure_pinned(*ds, ds->p_req, ds->cap_b, B);
    ensure_pinned(*ds, ds->p_prof, ds->cap_p, B * std::max(n_profile_fields, 1));
    for (size_t b = 0; b < B; ++b) {
      const Dataset::Rec& r = ds->recs[static_cast<size_t>(first) + b];
      if (static_cast<int>(r.item.size()) != n_hist || static_cast<int>(r.cand.size()) != n_cand ||
          static_cast<int>(r.profile.size()) != n_profile_fields)
        throw ConfigError("dataset record " + std::to_string(first + static_cast<int64_t>(b)) +
                          " does not match the batch geometry (history " + std::to_string(r.item.size()) +
                          ", candidates " + std::to_string(r.cand.size()) + ", profile " +
                          std::to_string(r.profile.size()) + "): one handle serves one geometry");
      // candidate side groups are not configured on this path (side_width() == 0): the
      // reference tokenizer rejects any other width (tokenizer.cpp:116-120), so do we
      if (r.n_side != 0)
        throw ConfigError("tokenizer: candidate side feature width " + std::to_string(r.n_side) +
                          " != configured 0 (dataset record " + std::to_string(first + static_cast<int64_t>(b)) + ")");
      std::memcpy(ds->p_item + b * n_hist, r.item.data(), n_hist * 4);
      std::memcpy(ds->p_action + b * n_hist, r.action.data(), n_hist * 4);
      std::memcpy(ds->p_scene + b * n_hist, r.scene.data(), n_hist * 4);
      std::memcpy(ds->p_ts + b * n_hist, r.hts.data(), n_hist * 8);
      std::memcpy(ds->p_cand + b * n_cand, r.cand.data(), n_cand * 4);
      std::memcpy(ds->p_prof + b * n_profile_fields, r.profile.data(), n_profile_fields * 4);
      ds->p_req[b] = r.ts;
      if (labels)
        for (int j = 0; j < n_cand; ++j) {
          labels[(b * n_cand + j) * 3 + 0] = static_cast<float>(r.click[j]);
          labels[(b * n_cand + j) * 3 + 1] = static_cast<float>(r.cart[j]);
          labels[(b * n_cand + j) * 3 + 2] = static_cast<float>(r.purchase[j]);
        }
      if (request_ids) request_ids[b] = r.id;
    }
    batch->batch = count;
    batch->hist_item = ds->p_item;
    batch->hist_action = ds->p_action;
    batch->hist_scene = ds->p_scene;
    batch->hist_ts = ds->p_ts;
    batch->req_ts = ds->p_req;
    batch->profile = ds->p_prof;
    batch->cand_item = ds->p_cand;
    return SORT_OK;
  } catch (const ConfigError& e) {
    g_last_error = e.what();
    return SORT_CONFIG_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SORT_RUNTIME_FAILURE;
  }
}

}  // extern "C"
