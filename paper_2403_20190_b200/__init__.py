"""hewisard-b200: batched TFHE programmable bootstrapping at q = 2^32 on B200.

B200-native (sm_100a) re-implementation of the hot path of the reference
"Homomorphic WiSARDs" package (`hewisard`, arXiv 2403.20190): the CMUX-ladder
external product, blind rotation, sample extraction, LWE key switching and
PBS, behind a Python API that mirrors `hewisard.tfhe`.
"""

__version__ = "0.1.0"

from . import params  # noqa: F401
from ._lib import EncodingError, TfheError  # noqa: F401
