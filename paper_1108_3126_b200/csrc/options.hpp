// Process-wide tuning and test switches (rxg_set_option in include/rxg.h).
// They change which kernel variant or table layout runs, never results.
#pragma once

namespace rxg {

// The value set for `name`, or nullptr when unset.
const char* option(const char* name);

}  // namespace rxg
