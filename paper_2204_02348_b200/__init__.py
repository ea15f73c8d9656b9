"""B200-native digHolo batch hot path (arXiv 2204.02348), drop-in for holopipe.

Public surface: ``api`` (handle API mirroring holopipe.api), ``engine.Engine``
(staged engine mirroring holopipe.engine.Engine), and the C ABI in
include/holo_b200.h implemented by lib/libholo_b200.so (sm_100a CUDA).
"""

__version__ = "0.1.0"
