// Host planner: Alg. 3 (QuesadillaSort) and the strategy -> device-group
// lowering.  Re-implemented from the paper and the reference's behaviour
// (proj/src/planner.cpp, plan.cpp, transpose.cpp); follow sets are 64-bit
// masks exactly as ModeSet (ordering.hpp:16-33).
#include <algorithm>
#include <string>

#include "internal.hpp"

namespace qb200 {

namespace {

uint64_t bit(uint32_t m) { return uint64_t{1} << m; }

// f(ord, p): modes after p in ord (planner.cpp:12-17).
uint64_t follow(const uint32_t* ord, uint32_t rank, uint32_t p) {
  uint32_t pos = 0;
  while (pos < rank && ord[pos] != p) ++pos;
  if (pos == rank) invalid("mode " + std::to_string(p) + " does not appear in the ordering");
  uint64_t s = 0;
  for (uint32_t i = pos + 1; i < rank; ++i) s |= bit(ord[i]);
  return s;
}

uint64_t simple_follow(uint32_t rank, uint32_t p) {
  // follow set of p in (0, 1, ..., rank-1): every mode > p.
  uint64_t all = rank == 64 ? ~uint64_t{0} : bit(rank) - 1;
  return all & ~((bit(p) << 1) - 1);
}

}  // namespace

void check_ordering(const uint32_t* ord, uint32_t rank) {
  if (rank == 0 || rank > QD_MAX_RANK)
    invalid("ordering rank must be in 1.." + std::to_string(QD_MAX_RANK));
  uint64_t seen = 0;
  for (uint32_t i = 0; i < rank; ++i) {
    if (ord[i] >= rank)
      invalid("ordering contains mode " + std::to_string(ord[i]) + " outside 0.." +
              std::to_string(rank - 1));
    if (seen & bit(ord[i])) invalid("ordering repeats mode " + std::to_string(ord[i]));
    seen |= bit(ord[i]);
  }
}

// Scan for the longest run of target positions whose mode still needs a sort
// (its target follow set escapes its simple follow set), emit those sorts
// lowest priority first behind the settled prefix l, grow the prefix, repeat.
// Positions at or beyond `want` never get their own sort.
std::vector<Step> plan_to_prefix(const uint32_t* target, uint32_t rank, uint32_t want) {
  check_ordering(target, rank);
  std::vector<Step> steps;
  uint32_t l = 0;
  while (l < want) {
    uint32_t k = l;
    while (k + 1 < rank) {
      const uint32_t m = target[k];
      if ((follow(target, rank, m) & ~simple_follow(rank, m)) == 0) break;
      ++k;
    }
    for (uint32_t j = std::min(k, want); j > l; --j) steps.push_back({l, target[j - 1]});
    l = k + 1;
  }
  return steps;
}

int required_sort_count(const uint32_t* source, const uint32_t* target, uint32_t rank) {
  check_ordering(source, rank);
  check_ordering(target, rank);
  int count = 0;
  for (uint32_t i = 0; i < rank; ++i) {
    const uint32_t p = target[i];
    if (follow(target, rank, p) & ~follow(source, rank, p)) ++count;
  }
  return count;
}

std::vector<uint32_t> apply_transition(const uint32_t* cur, uint32_t rank, Step s) {
  check_ordering(cur, rank);
  if (s.mode >= rank) invalid("step mode out of range");
  if (s.prefix_len >= rank) invalid("step prefix length out of range");
  uint32_t pos = 0;
  while (cur[pos] != s.mode) ++pos;
  if (pos < s.prefix_len) invalid("sort mode lies inside the bucketing prefix");
  std::vector<uint32_t> out(cur, cur + s.prefix_len);
  out.push_back(s.mode);
  out.insert(out.end(), cur + s.prefix_len, cur + pos);
  out.insert(out.end(), cur + pos + 1, cur + rank);
  return out;
}

namespace {

// Consecutive steps with equal prefix_len compose into one stable sort on the
// combined key (later steps are more significant): one device group.
void lower_steps(const uint32_t* target, const std::vector<Step>& steps,
                 std::vector<Group>& groups) {
  for (uint32_t i = 0; i < steps.size();) {
    uint32_t j = i;
    while (j < steps.size() && steps[j].prefix_len == steps[i].prefix_len) ++j;
    Group g;
    g.prefix.assign(target, target + steps[i].prefix_len);
    for (uint32_t s = j; s > i; --s) g.keys.push_back(steps[s - 1].mode);
    g.first_step = i;
    g.n_steps = j - i;
    groups.push_back(std::move(g));
    i = j;
  }
}

}  // namespace

std::vector<Group> strategy_groups(const uint32_t* target, uint32_t rank,
                                   qd_strategy_kind kind, uint32_t k,
                                   std::vector<Step>* steps_out) {
  check_ordering(target, rank);
  std::vector<Step> steps;
  std::vector<Group> groups;
  switch (kind) {
    case QD_QUESADILLA:  // transpose.cpp:93
      steps = plan_to_prefix(target, rank, rank);
      lower_steps(target, steps, groups);
      break;
    case QD_FULL_RADIX:  // transpose.cpp:95-99
      for (uint32_t j = rank; j > 0; --j) steps.push_back({0, target[j - 1]});
      lower_steps(target, steps, groups);
      break;
    case QD_TOPK: {  // transpose.cpp:100-107
      if (k < 1 || k > rank) invalid("top-K prefix length must be in 1..rank");
      steps = plan_to_prefix(target, rank, k);
      lower_steps(target, steps, groups);
      if (k < rank) {
        // parallel_topk_bucket_sort (parallel.cpp:190-248): each maximal run of
        // the first k target modes is stably sorted by the remaining modes.
        // Not a histogram pass, so not logged (strategy_pass_cost).
        Group g;
        g.prefix.assign(target, target + k);
        g.keys.assign(target + k, target + rank);
        g.first_step = static_cast<uint32_t>(steps.size());
        g.n_steps = 0;
        g.check_range = false;
        groups.push_back(std::move(g));
      }
      break;
    }
    case QD_COMPARISON_SORT: {  // transpose.cpp:108-110 (no histogram passes)
      Group g;
      g.keys.assign(target, target + rank);
      g.check_range = false;
      groups.push_back(std::move(g));
      break;
    }
    default:
      invalid("unknown strategy kind");
  }
  // the rows' ordering before each group, from a simple source (0, 1, ...):
  // a group leaves its prefix, then its keys, then the other modes as they were
  std::vector<uint32_t> cur(rank);
  for (uint32_t m = 0; m < rank; ++m) cur[m] = m;
  for (Group& g : groups) {
    g.first_digit_scattered = rank > 1 && !g.keys.empty() && g.keys.back() == cur[rank - 1];
    std::vector<uint32_t> next(g.prefix);
    next.insert(next.end(), g.keys.begin(), g.keys.end());
    for (uint32_t m : cur)
      if (std::find(next.begin(), next.end(), m) == next.end()) next.push_back(m);
    cur = next;
  }
  if (steps_out) *steps_out = steps;
  return groups;
}

}  // namespace qb200
