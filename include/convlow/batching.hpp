// convlow/batching.hpp -- partitioned batch execution (the
// reference's src/batching.cpp is absent, CMakeLists.txt:24).  On B200 a
// partition is a batch shard; execute_partitioned runs the shards through the
// device path (one stream, or one GPU each in the multi-GPU driver).
#pragma once

#include <vector>

#include "convlow/lowering.hpp"

namespace convlow {

struct PartitionPlan {
    std::size_t partitions = 1;
    std::vector<std::size_t> partition_sizes;
    std::vector<std::size_t> threads_per_partition;
};

struct FootprintReport {
    std::uint64_t lowered_bytes_per_partition = 0;
    std::uint64_t peak_bytes = 0;
    LoweringStrategy strategy = LoweringStrategy::Type1;
};

PartitionPlan plan_partitions(std::size_t b, std::size_t total_threads, std::size_t p);
FootprintReport footprint(LoweringStrategy strategy, const LayerConfig& layer, std::size_t partition_size);

struct PartitionedResult {
    OutputBatch output;
    PhaseTimings timing;
    FootprintReport footprint;
};
PartitionedResult execute_partitioned(const DataBatch& batch, const KernelBank& bank, LoweringStrategy strategy,
                                      const PartitionPlan& plan, ConvGeometry geom = {});

}  // namespace convlow
