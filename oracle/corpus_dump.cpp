// Test-infrastructure dumper over the reference (femopt) -- NOT product code.
//
// Prints the reference's own verification corpus as IR JSON: every kernel of
// corpus::all_json() (proj/tests/kernels.hpp:321-342, the set test_backend.cpp
// :167-182 runs through emit_c and the interpreter) and the 20 plan-optimality
// kernels corpus::plan_kernel_json(0..19) (kernels.hpp:348-363).  The corpus is
// generated code in the reference (kernels.hpp:17-21), so its IR is taken from
// there rather than restated.  Built by `make -C oracle corpus` from the sources
// where they lie; output goes to oracle/_ref/ only.
#include <iostream>
#include <string>

#include "kernels.hpp"

int main() {
  nlohmann::json out = nlohmann::json::array();
  for (auto& [name, j] : corpus::all_json()) out.push_back({{"name", name}, {"ir", j}});
  for (int v = 0; v < 20; ++v)
    out.push_back({{"name", "plan" + std::to_string(v)}, {"ir", corpus::plan_kernel_json(v)}});
  std::cout << out.dump() << "\n";
  return 0;
}
