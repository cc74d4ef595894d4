// libstrata_b200: batch grouping (reference: cli.cpp:358-399 build_batch_groups).
#include "strata/batch_groups.hpp"

#include <map>
#include <string>

namespace strata {

std::vector<BatchGroup> build_batch_groups(const RunSet& runs) {
  using Entry = std::pair<const RunSet::GroupKey, std::vector<TraceBundle>>;
  std::map<std::uint32_t, const Entry*> deepest;
  for (const Entry& e : runs.groups) {
    auto it = deepest.find(e.first.batch_size);
    if (it == deepest.end() || e.first.levels.size() > it->second->first.levels.size() ||
        (e.first.levels.size() == it->second->first.levels.size() && it->second->first.levels < e.first.levels))
      deepest[e.first.batch_size] = &e;
  }
  // one GPU pass over every selected run
  std::vector<TraceBundle> all;
  for (const auto& [batch, e] : deepest)
    for (const TraceBundle& b : e->second) all.push_back(b);
  std::vector<std::string> errors;
  std::vector<CorrelationResult> results = correlate_all(all, &errors);
  std::vector<BatchGroup> groups;
  std::size_t i = 0;
  for (const auto& [batch, e] : deepest) {
    BatchGroup g;
    g.batch_size = batch;
    g.levels = e->first.levels;
    g.input.batch_size = batch;
    for (const TraceBundle& bundle : e->second) {
      if (!errors[i].empty()) throw TraceError(errors[i]);
      CorrelationResult& r = results[i++];
      if (demand_serialized_rerun(r.ambiguities))
        throw TraceError("trace " + std::to_string(bundle.meta.trace_id) + " has " +
                         std::to_string(r.ambiguities.size()) +
                         " ambiguous spans; resolve them first (correlate --serialized-rerun) or profile serialized");
      g.input.runs.push_back(std::move(r.tree));
    }
    groups.push_back(std::move(g));
  }
  return groups;
}

}  // namespace strata
