// validate_plan, see validate.cpp.
#pragma once

#include <string>
#include <vector>

#include "reshard/plan_core.hpp"

namespace reshard {
namespace core {

/// Violations of the plan invariants + destination coverage; empty on success.
/// drop >= 0 removes transfer `drop` (canonical order) first (fault injection).
std::vector<std::string> validate_plan(const PlanCore& P, const std::vector<FlatXfer>& flat, std::int64_t drop = -1);

}  // namespace core
}  // namespace reshard
