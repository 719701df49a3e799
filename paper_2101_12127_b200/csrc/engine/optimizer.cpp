// optimizer.cpp -- static rewrites to a fixed point (include/dpb200/
// datapipe.hpp).  Rule set, priority order, attribute merging and the
// synthesized-UDF naming follow the reference's contract
// (/root/reference/proj/docs/formats.md:152-186, optimizer.cpp:143-400):
//   map_map_fusion        map(f).map(g) -> map((f)>>(g)); downstream p wins,
//                         AUTOTUNE absorbing; device step chains concatenate
//   filter_filter_fusion  filter(p).filter(q) -> filter((p)&&(q))
//   map_filter_fusion     map(f).filter(p) -> map(f, fused_filter_udf=p)
//   map_vectorization     never fires: device UDFs register no vectorized
//                         variant (it would pre-empt map_and_batch,
//                         SURVEY.md 3.3)
//   map_batch_fusion      map(f).batch(b) -> map_and_batch(f, b) unless the
//                         map carries a fused predicate
//   shuffle_repeat_fusion shuffle.repeat -> shuffle(fused_with_repeat=true)
#include <algorithm>
#include <sstream>

#include "dpb200/datapipe.hpp"

namespace datapipe::b200 {

namespace {

constexpr int kMaxPasses = 100;

int64_t MergeParallelism(int64_t up, int64_t down) { return (up == kAutotune || down == kAutotune) ? kAutotune : down; }

struct Engine {
  const RuleSet& rules;
  UdfRegistry& reg;
  RewriteReport* report;
  bool changed = false;

  NodePtr Apply(const char* rule, const std::string& path, const std::function<NodePtr()>& build) {
    NodePtr r;
    try {
      r = build();
    } catch (const PipelineError& e) {
      throw PipelineError(ErrorCode::kRuleProducedInvalidGraph, std::string(rule) + ": " + e.what());
    }
    report->applied.push_back({rule, path});
    changed = true;
    return r;
  }

  bool IsMap(const std::string& n) { return reg.Contains(n) && !reg.Get(n).map.empty(); }
  bool IsPred(const std::string& n) { return reg.Contains(n) && reg.Get(n).predicate.has_value(); }

  std::string Conjunction(const std::string& p, const std::string& q) {
    std::string name = "(" + p + ")&&(" + q + ")";
    if (!reg.Contains(name)) {
      UdfRegistry::Entry e;
      DevicePredicate c = *reg.Get(p).predicate;
      const auto& tq = reg.Get(q).predicate->terms;
      c.terms.insert(c.terms.end(), tq.begin(), tq.end());
      e.predicate = std::move(c);
      reg.Register(name, std::move(e));
    }
    return name;
  }

  NodePtr TryMapMap(const NodePtr& n, const std::string& path) {
    if (n->kind() != NodeKind::kMap) return nullptr;
    const auto& in = n->inputs()[0];
    if (in->kind() != NodeKind::kMap || in->HasAttr("fused_filter_udf")) return nullptr;
    const std::string &f = in->GetString("udf"), &g = n->GetString("udf");
    if (!IsMap(f) || !IsMap(g)) return nullptr;
    return Apply(kMapMapFusion, path, [&] {
      std::string name = "(" + f + ")>>(" + g + ")";
      if (!reg.Contains(name)) {
        UdfRegistry::Entry e;
        e.map = reg.Get(f).map;
        const auto& gm = reg.Get(g).map;
        e.map.insert(e.map.end(), gm.begin(), gm.end());
        if (reg.Get(f).cost_hint_ns && reg.Get(g).cost_hint_ns)
          e.cost_hint_ns = *reg.Get(f).cost_hint_ns + *reg.Get(g).cost_hint_ns;
        reg.Register(name, std::move(e));
      }
      Attrs a{{"udf", name},
              {"num_parallel_calls", MergeParallelism(in->GetInt("num_parallel_calls"), n->GetInt("num_parallel_calls"))}};
      if (n->HasAttr("fused_filter_udf")) a["fused_filter_udf"] = n->GetString("fused_filter_udf");
      return Build(NodeKind::kMap, {in->inputs()[0]}, std::move(a), reg);
    });
  }

  NodePtr TryFilterFilter(const NodePtr& n, const std::string& path) {
    if (n->kind() != NodeKind::kFilter) return nullptr;
    const auto& in = n->inputs()[0];
    if (in->kind() != NodeKind::kFilter) return nullptr;
    const std::string &p = in->GetString("udf"), &q = n->GetString("udf");
    if (!IsPred(p) || !IsPred(q)) return nullptr;
    // device conjunctions hold at most 8 terms on one quantity
    const auto &pp = *reg.Get(p).predicate, &pq = *reg.Get(q).predicate;
    if (pp.on != pq.on || pp.terms.size() + pq.terms.size() > 8) return nullptr;
    return Apply(kFilterFilterFusion, path, [&] {
      return Build(NodeKind::kFilter, {in->inputs()[0]}, {{"udf", Conjunction(p, q)}}, reg);
    });
  }

  NodePtr TryMapFilter(const NodePtr& n, const std::string& path) {
    if (n->kind() != NodeKind::kFilter) return nullptr;
    const auto& in = n->inputs()[0];
    if (in->kind() != NodeKind::kMap) return nullptr;
    const std::string& p = n->GetString("udf");
    if (!IsPred(p)) return nullptr;
    return Apply(kMapFilterFusion, path, [&] {
      Attrs a = in->attrs();
      a["fused_filter_udf"] = in->HasAttr("fused_filter_udf") ? Conjunction(in->GetString("fused_filter_udf"), p) : p;
      return Build(NodeKind::kMap, {in->inputs()[0]}, std::move(a), reg);
    });
  }

  NodePtr TryMapBatch(const NodePtr& n, const std::string& path) {
    if (n->kind() != NodeKind::kBatch) return nullptr;
    const auto& in = n->inputs()[0];
    if (in->kind() != NodeKind::kMap || in->HasAttr("fused_filter_udf")) return nullptr;
    const std::string& f = in->GetString("udf");
    if (!IsMap(f)) return nullptr;
    return Apply(kMapBatchFusion, path, [&] {
      Attrs a{{"udf", f}, {"batch_size", n->GetInt("batch_size")}, {"num_parallel_calls", in->GetInt("num_parallel_calls")}};
      if (n->GetBoolOr("drop_remainder", false)) a["drop_remainder"] = true;
      return Build(NodeKind::kMapAndBatch, {in->inputs()[0]}, std::move(a), reg);
    });
  }

  NodePtr TryShuffleRepeat(const NodePtr& n, const std::string& path) {
    if (n->kind() != NodeKind::kRepeat) return nullptr;
    const auto& in = n->inputs()[0];
    if (in->kind() != NodeKind::kShuffle || in->GetBoolOr("fused_with_repeat", false)) return nullptr;
    return Apply(kShuffleRepeatFusion, path, [&] {
      Attrs sa = in->attrs();
      sa["fused_with_repeat"] = true;
      NodePtr fused = Build(NodeKind::kShuffle, {in->inputs()[0]}, std::move(sa), reg);
      return Build(NodeKind::kRepeat, {fused}, n->attrs(), reg);
    });
  }

  NodePtr TryRules(const NodePtr& n, const std::string& path) {
    for (const auto& rule : rules.order()) {
      NodePtr r;
      if (rule == kMapMapFusion) r = TryMapMap(n, path);
      else if (rule == kFilterFilterFusion) r = TryFilterFilter(n, path);
      else if (rule == kMapFilterFusion) r = TryMapFilter(n, path);
      else if (rule == kMapBatchFusion) r = TryMapBatch(n, path);
      else if (rule == kShuffleRepeatFusion) r = TryShuffleRepeat(n, path);
      if (r) return r;
    }
    return nullptr;
  }

  NodePtr Rewrite(const NodePtr& n, const std::string& path) {
    std::vector<NodePtr> inputs;
    bool changed_inputs = false;
    for (size_t i = 0; i < n->inputs().size(); ++i) {
      const auto& in = n->inputs()[i];
      NodePtr r = Rewrite(in, path + "/" + NodeKindName(in->kind()) + "@" + std::to_string(i));
      changed_inputs |= (r != in);
      inputs.push_back(std::move(r));
    }
    NodePtr cur = changed_inputs ? Build(n->kind(), std::move(inputs), n->attrs(), reg) : n;
    for (;;) {
      NodePtr r = TryRules(cur, path);
      if (!r) break;
      cur = std::move(r);
    }
    return cur;
  }
};

}  // namespace

const std::vector<std::string>& RuleSet::AllRuleNames() {
  static const std::vector<std::string> all = {kMapMapFusion,     kFilterFilterFusion, kMapFilterFusion,
                                               kMapVectorization, kMapBatchFusion,     kShuffleRepeatFusion};
  return all;
}

RuleSet RuleSet::Default() {
  RuleSet r;
  r.order_ = AllRuleNames();
  return r;
}

void RuleSet::Disable(const std::string& name) {
  const auto& all = AllRuleNames();
  if (std::find(all.begin(), all.end(), name) == all.end())
    throw PipelineError(ErrorCode::kInvalidAttr, "unknown rule: " + name);
  order_.erase(std::remove(order_.begin(), order_.end(), name), order_.end());
}

bool RuleSet::IsEnabled(const std::string& name) const {
  return std::find(order_.begin(), order_.end(), name) != order_.end();
}

std::string RewriteReport::ToString() const {
  std::ostringstream os;
  os << "passes: " << iterations << "\n";
  if (applied.empty()) os << "no rewrites applied\n";
  for (const auto& r : applied) os << r.rule << " at " << r.node_path << "\n";
  return os.str();
}

std::pair<DatasetGraph, RewriteReport> Optimize(const DatasetGraph& graph, const RuleSet& rules,
                                                UdfRegistry& registry) {
  if (!graph.root()) throw PipelineError(ErrorCode::kValidationFailed, "empty graph");
  RewriteReport report;
  NodePtr root = graph.root();
  for (int pass = 1;; ++pass) {
    if (pass > kMaxPasses)
      throw PipelineError(ErrorCode::kRewriteDiverged, "rewrite did not reach a fixed point in 100 passes");
    Engine e{rules, registry, &report};
    NodePtr r = e.Rewrite(root, "/" + std::string(NodeKindName(root->kind())) + "@0");
    report.iterations = pass;
    if (!e.changed) break;
    root = std::move(r);
  }
  return {DatasetGraph(root), report};
}

}  // namespace datapipe::b200
