"""B200-native WAGMA-SGD group-model-averaging hot path (arXiv 2005.00124).

Drop-in for the hot path of the reference package `wagma`:

- ``topology``   butterfly / XOR-rotating schedule (C++ generator)
- ``collective`` GroupAllreduce / SyncAllreduce over a DeviceContext
- ``optim``      EtaSchedule, OptimizerConfig, GroupAveragingOptimizer
                 (one fused sm_100a launch per iteration)
- ``straggler``  StragglerPolicy / DelayModel (deterministic victims)
- ``context``    DeviceContext: device arena, CUDA-IPC peer mapping
- ``driver``     replay and straggler-emulation drivers

The compute lives in ``libwagma_b200.so`` (csrc/, C ABI in
include/wagma_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"
