"""CPU oracle for the B200 hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the CPU baseline --
never on the product path (paper_2404_02015_b200 never imports it).

  _ref/            the reference C++ sources compiled in place (Makefile)
  numerics_ref.c   C restatement of paged decode attention + a bf16 GEMV
                   baseline (parity unpinned: the reference has no numerics)
  llama_ref.py     numpy LLaMA-1 forward with the GPU path's rounding points
  alloc_ref.py     restatement of the physical head-block id policy
"""
