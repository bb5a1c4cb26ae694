"""B200-native MatMul-free LM block forward (arxiv 2406.02528).

The compute path is libtern.so (hand-written sm_100a CUDA behind the C ABI in
include/tern.h).  `_lib` is the argument-marshalling binding, `model` the
stack driver, `synth` the seeded input generators.  Importing the package
does not load the CUDA library; `paper_2406_02528_b200._lib.load()` does and
raises if it is missing -- there is no CPU fallback.
"""
__all__ = ["_lib", "model", "synth", "build"]
