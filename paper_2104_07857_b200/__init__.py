"""B200-native ZeRO-Infinity partitioned data-parallel step (drop-in for the reference `infinisim` hot path).

Modules:
  store     — TierStore / BufferPool / IoTicket: the infinity offload engine (reference store.py)
  partition — PartitionedTensor, partition / allgather / reduce_scatter / broadcast_fetch
  schedule  — trace_schedule / plan_prefetch / Timeline
  tiling    — TiledLinear, tile_linear / forward_tiled / backward_tiled
  harness   — SPEC train-harness: init_partitioned / train_step / chunked_adam_step / run_training
  gpt       — the GPT ZeRO-3 engine used by the BASELINE configs
  kernels   — tensor wrappers over libzinf.so (csrc/, C ABI in include/zinf.h)
"""

__version__ = "0.1.0"
