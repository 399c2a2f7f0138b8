"""Independent references for pinning the oracle (NOT the oracle, NOT the GPU path).

* k*G comes from the `cryptography` package (OpenSSL), a library independent of
  both implementations in this repo.
* curve constants are the SEC 2 / FIPS 186-4 published values; p is also
  checked against the formula printed in the paper.
"""
from cryptography.hazmat.primitives.asymmetric import ec

P = 2**256 - 2**224 + 2**192 + 2**96 - 1
Q = int("ffffffff00000000ffffffffffffffffbce6faada7179e84f3b9cac2fc632551", 16)
B = int("5ac635d8aa3a93e7b3ebbd55769886bc651d06b0cc53b0f63bce3c3e27d2604b", 16)
GX = int("6b17d1f2e12c4247f8bce6e563a440f277037d812deb33a0f4a13945d898c296", 16)
GY = int("4fe342e2fe1a7f9b8ee7eb4a7c0f9e162bce33576b315ececbb6406837bf51f5", 16)
INF = bytes(64)


def mulG(k: int) -> bytes:
    """Canonical bytes of k*G (x||y big-endian; infinity = 64 zero bytes) via OpenSSL."""
    k %= Q
    if k == 0:
        return INF
    pn = ec.derive_private_key(k, ec.SECP256R1()).public_key().public_numbers()
    return pn.x.to_bytes(32, "big") + pn.y.to_bytes(32, "big")


def enc_closed_form(x: int, R: int, c: int) -> bytes:
    """Eq. 5: ciphertext of message c with randomness R = (R G, (x R + c) G)."""
    return mulG(R) + mulG(x * R + c)
