// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// The UNMODIFIED reference OverlapRegistry / infer_overlap_closure (overlap.hpp) on batches
// described with the product's coh_view / coh_mode records (include/cohere_b200.h), so the
// GPU registry and closure can be compared field by field.  View i is named "v" + its
// zero-padded name_rank (std::string order == rank order), buffer k is "b<k>" with length
// max(hi) + 1, scalar j (a mode without the view flag) is "s<j>".
#include <cstdio>
#include <string>
#include <vector>

#include "cohere/cohere.hpp"
#include "cohere_b200.h"

using namespace cohere;

namespace {

std::string vname(uint32_t rank) {
  char b[16];
  std::snprintf(b, sizeof b, "v%08u", rank);
  return b;
}

Declarations decls_of(const coh_view* v, uint32_t n, uint32_t n_scalars, std::vector<std::string>& names) {
  Declarations d;
  for (uint32_t j = 0; j < n_scalars; ++j) d.add_scalar({"s" + std::to_string(j), {}});
  uint32_t nb = 0;
  for (uint32_t i = 0; i < n; ++i) nb = std::max(nb, v[i].buffer + 1);
  std::vector<int> len(nb, 0);
  for (uint32_t i = 0; i < n; ++i) len[v[i].buffer] = std::max(len[v[i].buffer], v[i].hi + 1);
  for (uint32_t b = 0; b < nb; ++b)
    if (len[b]) d.add_buffer({"b" + std::to_string(b), len[b], {}});
  names.resize(n);
  for (uint32_t i = 0; i < n; ++i) {
    names[i] = vname(v[i].name_rank);
    d.add_view({names[i], "b" + std::to_string(v[i].buffer), v[i].lo, v[i].hi, {}});
  }
  return d;
}

}  // namespace

extern "C" int ref_registry_query(const coh_view* views, uint32_t n, const uint32_t* probes, uint32_t n_probes,
                                  uint32_t* hits, uint32_t stride, uint32_t* count, int segment_tree) {
  std::vector<std::string> names;
  Declarations d = decls_of(views, n, 0, names);
  OverlapRegistry reg = build_registry(d, segment_tree ? OverlapRegistry::Backend::SegmentTree
                                                       : OverlapRegistry::Backend::SortedList);
  std::map<std::string, uint32_t> idx;
  for (uint32_t i = 0; i < n; ++i) idx[names[i]] = i;
  for (uint32_t q = 0; q < n_probes; ++q) {
    auto h = reg.query(names[probes[q]]);
    count[q] = (uint32_t)h.size();
    for (uint32_t k = 0; k < h.size() && k < stride; ++k) hits[(uint64_t)q * stride + k] = idx[h[k]];
  }
  return 0;
}

extern "C" int ref_overlap_closure(const coh_view* views, uint32_t n, uint32_t n_scalars, const coh_mode* modes,
                                   const uint32_t* off, uint32_t n_blocks, coh_mode* out, uint32_t stride,
                                   uint32_t* out_count, int32_t* status) {
  std::vector<std::string> names;
  Declarations d = decls_of(views, n, n_scalars, names);
  OverlapRegistry reg = build_registry(d);
  std::map<std::string, uint32_t> idx;
  for (uint32_t i = 0; i < n; ++i) idx[names[i]] = i;
  for (uint32_t b = 0; b < n_blocks; ++b) {
    std::vector<AccessMode> ms;
    for (uint32_t k = off[b]; k < off[b + 1]; ++k) {
      AccessMode m;
      m.kind = static_cast<AccessMode::Kind>(modes[k].kind);
      m.site = modes[k].site ? Site::Remote : Site::Local;
      m.view = (modes[k].flags & 1u) ? names[modes[k].var] : "s" + std::to_string(modes[k].var);
      m.shadow = (modes[k].flags & 2u) != 0;
      ms.push_back(m);
    }
    try {
      auto r = infer_overlap_closure(ms, reg, d);
      out_count[b] = (uint32_t)r.size();
      status[b] = -1;
      for (uint32_t k = 0; k < r.size() && k < stride; ++k) {
        coh_mode& o = out[(uint64_t)b * stride + k];
        const bool is_view = d.find_view(r[k].view) != nullptr;
        o.var = is_view ? idx[r[k].view] : (uint32_t)std::stoul(r[k].view.substr(1));
        o.kind = (uint8_t)r[k].kind;
        o.site = r[k].site == Site::Remote ? 1 : 0;
        o.flags = (uint8_t)((is_view ? 1u : 0u) | (r[k].shadow ? 2u : 0u));
        o.pad = 0;
      }
    } catch (const OverlapInferenceError& e) {
      status[b] = (int32_t)idx[e.view];
      out_count[b] = 0;
    }
  }
  return 0;
}
