"""pcmm-b200: plaintext-ciphertext matrix multiplication over EC-ElGamal / P-256
on NVIDIA B200 (sm_100a), by Cussen's compression-reconstruction algorithm
(arXiv 2504.14497, Alg. 3).  The product is the C-ABI library libpcmm.so
(include/pcmm.h); `pcmm` is its thin Python binding."""
from . import pcmm  # noqa: F401
from .pcmm import (CUSSEN, SCHOOLBOOK, PCMMError, decrypt_small, encrypt, keygen, load,  # noqa: F401
                   mul_cussen, mul_schoolbook, normalize, status)
