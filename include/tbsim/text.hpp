// tbsim/text.hpp -- number formatting shared by every CSV writer
// (twin of proj/include/tbsim/text.hpp).
#pragma once

#include <string>

namespace tbsim {

std::string fmt_ms(double v);     // %.6f with trailing zeros (and '.') trimmed
std::string fmt_ratio(double v);  // %.3f

}  // namespace tbsim
