"""B200-native MuxServe hot path: ADBS scheduling over a unified head-wise KV
pool, with sm_100a kernels for decode attention, KV append and tcgen05 GEMMs.

Everything runs in libmux.so (csrc/); this package is the ctypes mirror of the
reference's C++ API (see host.py and include/mux.h).
"""
from ._lib import LIB_PATH, Infeasible, InvalidArgument, LogicError, MuxError, header_symbols, lib  # noqa: F401
from .host import (CATALOG, AllocResult, BlockPool, EngineParams, Entry, LLMSpec, Placement,  # noqa: F401
                   ParallelCandidate, QuotaInput, TraceRequest, parallel_candidates, Unit, adapt_quota, blocks_for_tokens, blocks_per_token, byte_share_partitions,
                   decode_attention_headwise, gemm_bf16, init_token_block_quota, kv_append,
                   prefill_attention,
                   rope_table, simulate, spec, weight_tile)

__version__ = "0.1.0"
