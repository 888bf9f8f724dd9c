"""B200-native Picker runtime validator (arXiv 2410.23661).

Batched instance-level idempotency validation of GPU kernel launch records
against per-kernel access summaries, in hand-written CUDA for sm_100a behind a C
ABI (include/picker.h).  See DESIGN.md.
"""
from .validator import (CODE_NAMES, NUM_COUNTS, Picker, PickerError, compile_summaries,  # noqa: F401
                        records_tensor, summary_text, verify_summaries)
