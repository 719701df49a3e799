// fastdiv.hpp -- per-constant-set proof of normalize_fast (k_prove.cu).
#pragma once

namespace dpk {

// True when normalize_fast(v, mean_c, std_c, RN(1 / std_c)) equals
// __fdiv_rn(v - mean_c, std_c) bit for bit for every fp32 v in [+0, 255] and
// every channel c, checked exhaustively on the current device at first use
// (cached).  False on any failure to run the check.
bool fast_div_proven(const float mean[3], const float stdv[3]);

}  // namespace dpk
