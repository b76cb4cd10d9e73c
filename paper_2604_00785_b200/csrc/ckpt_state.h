// Shard files of the sharded-optimizer checkpoint, see ckpt_state.cpp.
#pragma once
#include <string>
#include <vector>

#include "ckpt.h"
#include "optim.h"

namespace b2 {

struct ShardWritten {
    int64_t bytes = 0;  // 0 on ranks that are not their shard's writer
    uint32_t crc = 0;
    int model_shard = 0;
    bool writer = false;
};

// Collective over every owning group. names[p]: the parameter's record name prefix;
// dims[p]: its shape (empty -> {numel}). full = false writes weights only (.w16).
ShardWritten write_state_shard(ShardedOptimizer& opt, const std::string& dir, const std::vector<std::string>& names,
                               const std::vector<std::vector<int64_t>>& dims, bool full);
// Every rank reads its own model shard's file (and shard ep = 0's for non-expert params);
// no collective. full = false restores weights only.
void restore_state_shard(ShardedOptimizer& opt, const std::string& dir, const std::vector<std::string>& names,
                         const std::vector<std::vector<int64_t>>& dims, bool full);

}  // namespace b2
