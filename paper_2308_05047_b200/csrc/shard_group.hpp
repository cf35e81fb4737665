// In-process shard groups (shard.cu) behind the single-engine handle
// (engine.cu): an shs_engine created with options.n_devices >= 2 (or a state
// larger than one device under n_devices < 0) owns G shards, one per listed
// device (a device may repeat: virtual shards), all driven by the calling
// thread. Row N1 of the coverage table: the reference's C++ API reaches the
// multi-GPU engine unchanged (include/shorsim_b200.hpp).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/shorsim_b200.h"
#include "host_model.hpp"

struct ShmBarrier;
using shs::u64;
using shs::u128;
int shards_run(const std::vector<shs_shard*>& L, ShmBarrier* bar, u64 seed, u64 idx, u128* j_out,
               u128* js_out, shs_stage_trace* trace);

struct ShardGroup {
    std::vector<shs_shard*> shards;
    uint64_t N = 0, S = 0;
    uint32_t t = 0;
    bool pending = false;
    double p0 = 0, p1 = 0;
};

int group_create(const shs_problem& problem, const shs_error& error, const shs_options& options,
                 const std::vector<int>& devices, ShardGroup** out);
void group_destroy(ShardGroup* g);
int group_run(ShardGroup* g, u64 seed, u64 idx, u128* j, u128* js, shs_stage_trace* trace);
int group_state_init(ShardGroup* g);
int group_stage_probs(ShardGroup* g, uint32_t s, u128 prefix, double* p0, double* p1);
int group_stage_collapse(ShardGroup* g, int src_group, double p_src);
// x, global [first, first+count) (zero where no shard covers it)
int group_state_read(ShardGroup* g, int x, uint64_t first, uint64_t count, double* host);
int group_stage_read(ShardGroup* g, int x, uint64_t first, uint64_t count, double* host);
int group_state_gather(ShardGroup* g, int x, const uint64_t* idx, uint64_t count, double* host);
uint64_t group_launches(const ShardGroup* g);
int group_set_sparse(ShardGroup* g, bool on);
uint32_t group_sparse_stages(const ShardGroup* g);
int shard_device(const shs_shard* sh);
uint64_t group_device_bytes(const ShardGroup* g);
// the devices a state of N amplitudes needs (SHS_DEVICES overrides); 1 = fits one device
int plan_devices(uint64_t N, int first_device, std::vector<int>* devices);
