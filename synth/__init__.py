"""Seeded synthetic edge streams (inputs only: no part of the method's arithmetic lives here).

Shared by the oracle tests and the CUDA path's tests / bench, which is the one
thing the two sides are allowed to share.  See DESIGN.md "Input recipe".
"""
from .graphs import CONFIGS, chung_lu, config_stream, er, finalize, rmat, tiny_stream

__all__ = ["CONFIGS", "chung_lu", "config_stream", "er", "finalize", "rmat", "tiny_stream"]
