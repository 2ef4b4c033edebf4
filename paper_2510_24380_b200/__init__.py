"""B200-native drop-in for APEX's exhaustive enumeration-and-retrieval path.

Public API mirrors the reference `apexcsl.engine` hot path (engine.py:80-92,
265-313, 345-398); compute runs in libapexb200.so (sm_100a kernels behind the
C ABI in include/apex_b200.h).  See DESIGN.md.
"""

from .csl import (CslLibrary, LibraryError, MultiIndex, ReactionSpec, RgroupSpec, SynthonRecord, decode_index,
                  deserialize_library, library_fingerprint, product_count, serialize_library)
from .engine import (Constraint, ContributionTable, EngineError, QuerySpec, ScoredCompound, TopKResult, bind,
                     precompute_contributions, search_topk_batched, search_topk_many, search_topk_stream)

__version__ = "0.1.0"
