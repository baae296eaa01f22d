"""paper_2605_24259_b200 -- B200-native batched resident-KV-claim arbitration.

Submodules:
  rkc  -- thin ctypes binding of the C-ABI library librkc.so (include/rkc.h)
  gen  -- seeded synthetic trace generator (inputs only)
"""
