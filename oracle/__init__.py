"""CPU oracle for the ZeRO-Infinity partitioned data-parallel step.

TEST INFRASTRUCTURE ONLY. Nothing under ``oracle/`` is part of the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the
checker or the timed CPU baseline. The product package
``paper_2104_07857_b200`` never imports it and has no CPU fallback.

What it restates (reference = ``/root/reference``):

* ``numerics``  — binary16 / bfloat16 round-to-nearest-even
  and the counter-based uniform init shared bit-for-bit with the CUDA init kernel.
* ``partition`` — PartitionedTensor / partition / allgather / reduce_scatter /
  broadcast_fetch.
* ``adam``      — chunked mixed-precision Adam and the fused
  reduce-scatter + cast + Adam the engine runs per layer.
* ``tiling``    — tile_linear / forward_tiled / backward_tiled.
* ``schedule``  — trace_schedule / plan_prefetch.
* ``harness``   — the SPEC toy train_step / run_training.
* ``gpt``       — the GPT-block generalisation of train_step used by the
  BASELINE configs (numpy forward/backward).
* ``store_ref`` — the reference ``infinisim.store`` itself, imported from
  ``/root/reference/pkg/src`` when present (fixture generation only).

Parity pinning: the reference ships no tests. The store
semantics are pinned by running the reference ``store.py`` itself
(``tests/golden/make_golden.py``); the hot-path arithmetic (partition,
reduce-scatter, Adam, tiling, train_step) exists in the reference only as the
SPEC contract, so it is pinned by the SPEC's own examples and acceptance
criteria — "parity pinned to SPEC examples; no reference
code exists for these functions".
"""
