"""Seeded synthetic inputs shared by the tests, the bench and the oracle legs.

This package holds NO arithmetic of the method (no pre-scaling, Bjorck,
composition or convolution).  It only describes workload shapes
(``synth.configs``) and draws seeded random numbers (``synth.gen``).  Both the
CUDA path and the oracle consume what it produces; neither is imported here.
"""
