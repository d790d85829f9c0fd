"""B200-native ARCQuant (arxiv 2601.07475) hot path: ARC-NVFP4 quantize + block-scaled
tcgen05 GEMM behind the C-ABI library ``libarc.so`` (see include/arc.h).

``paper_2601_07475_b200.arc`` is the thin ctypes binding (loads libarc.so and fails
loudly if it is missing); ``tp`` holds the tensor-parallel wrappers; ``synth`` the
seeded synthetic inputs.  Nothing here computes on the CPU.
"""
