"""Seeded synthetic input generators (summaries + launch records).

Shared by the oracle side and the CUDA side as *inputs only*: nothing here
computes address ranges, overlaps or verdicts.
"""
