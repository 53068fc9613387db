"""B200-native (sm_100a) SOCKET sparse-decode hot path (arxiv 2602.06283).

    from paper_2602_06283_b200 import ops, Config, SocketDecoder

The compute lives in libsocket_b200.so (C ABI: include/socket_b200.h); this
package only marshals torch tensors to it.  Importing `ops` requires the
library to be built (`python -m paper_2602_06283_b200.build`); there is no
CPU fallback.
"""
from .ops import Config, KV_SHARED, PER_QHEAD  # noqa: F401
from . import ops  # noqa: F401
from .engine import SocketDecoder  # noqa: F401

__all__ = ["Config", "KV_SHARED", "PER_QHEAD", "ops", "SocketDecoder"]
