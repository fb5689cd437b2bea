// A/B tuning switches, in ONE place.  Production builds return the measured-best
// defaults (no environment reads); a profiling build (-DVC_TUNING, e.g.
// `python -m paper_2501_08453_b200.build --tuning`) reads VC_<name> from the
// environment once per switch so variants can be interleaved on one box.
// The measured alternatives are listed in DESIGN.md §4 "A/B switches".
#pragma once
#include <stdlib.h>

namespace vc {

inline int tuning_int(const char* env, int def) {
#ifdef VC_TUNING
  const char* v = getenv(env);
  return v ? atoi(v) : def;
#else
  (void)env;
  return def;
#endif
}

inline bool tuning_debug() { return tuning_int("VC_GEMM_DEBUG", 0) != 0; }

}  // namespace vc
