"""B200-native (sm_100a) hot path of batch speculative decoding (EqSpec / EXSpec,
arXiv 2510.22876): verify -> repad/positions/masks -> KV realign, and EXSpec pool
regrouping, behind the C ABI of libspecdec.so (include/specdec.h).

    _abi      ctypes binding with the C names (argument marshalling only)
    eqspec    EqSpecBatch: device-resident batch state + one round (K1 -> K3 -> K2)
    exspec    SequencePool: EXSpec pool epochs (K4 plan, gather / verify / write-back)
    build     nvcc build of libspecdec.so (sm_100a), in-tree
"""
from . import _abi  # noqa: F401

__all__ = ["_abi"]
