"""Seeded synthetic inputs shared by the oracle harness and the GPU path.

This package holds NONE of the method's arithmetic (no base64 encode/decode
math, no alphabet map).  It only produces the byte streams, lengths and
corruption positions described in DESIGN.md §"Input recipe":

* ``gen.splitmix_bytes(seed, begin, end)`` -- host (numpy) implementation of
  the counter-based byte generator G(seed, j).
* ``gpu_gen.fill(tensor, seed, begin)`` -- the same generator as a CUDA kernel
  (``inputs/libb64gen.so``), tested equal to the numpy twin.
* ``workloads`` -- per-config recipes (C1..C5) built from numpy's
  ``default_rng(seed)``.
"""
