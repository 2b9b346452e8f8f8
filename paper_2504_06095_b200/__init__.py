"""B200-native NTP gradient reshard-and-reduce (arXiv 2504.06095 hot path).

Public API mirrors the reference package ``ntpsim``:

* ``shardmap``   -- build_shard_map, build_reshard_plan, apply_plan,
                    naive_contiguous_sync_volumes, attention_head_partition
* ``tpnumerics`` -- MlpLayer, MlpReplica, uniform_grad_sync, nonuniform_grad_sync
* ``reconfig``   -- TP-n1 -> TP-n2 weight / optimizer-state reshard
* ``dist``       -- one process per GPU: peer-memory sync over NVLink/NVSwitch
* ``dist_dp``    -- DP > 2 with one degraded replica (NCCL among the healthy ones)
* ``dist_reconfig`` -- the failure reconfiguration across processes (peer pulls)
* ``linear``     -- tcgen05 uneven-shard MLP linears writing the unit-major arenas
* ``step``       -- the degraded-replica backward with every layer's sync overlapped

All device work runs in libntp_b200.so (csrc/, sm_100a); there is no CPU
fallback.
"""

__version__ = "0.1.0"
