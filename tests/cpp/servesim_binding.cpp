// Compiles the C++ binding (include/ssn.hpp) against the UNMODIFIED reference
// headers and checks, host-side, that every record of servesim's
// default_catalog() (profile.hpp:469-507) is a valid TinyCNN control tuple
// for the engine, and that invalid tuples raise the reference's exception type.
#include <cstdio>
#include <stdexcept>

#include "servesim/profile.hpp"
#include "ssn.hpp"

int main() {
  const servesim::Catalog cat = servesim::default_catalog();
  ssn_supernet_desc d{};
  d.family = SSN_FAMILY_TINYCNN;
  d.dtype = SSN_DTYPE_F32;
  d.image_size = 32;
  d.num_classes = 10;
  d.max_batch = 8;
  for (std::size_t i = 0; i < cat.size(); ++i) {
    ssn::CfgView v(cat.at(i).config);
    uint64_t n = 0;
    ssn::check(ssn_plan_stat_count(&d, &v.c, &n));
    std::printf("%s %llu\n", cat.at(i).id.c_str(), static_cast<unsigned long long>(n));
  }
  servesim::SubnetConfig bad = cat.at(0).config;
  bad.width_multipliers.assign(4, 1.5);
  try {
    ssn::CfgView v(bad);
    uint64_t n = 0;
    ssn::check(ssn_plan_stat_count(&d, &v.c, &n));
    return 1;
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what());
  }
  return 0;
}
