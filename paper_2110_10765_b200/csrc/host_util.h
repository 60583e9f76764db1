// Host-side error plumbing shared by the C-ABI translation units.
#pragma once
#include <string>

namespace cim {
int set_error(int code, const std::string &msg);  // returns code
void clear_error();
}  // namespace cim
