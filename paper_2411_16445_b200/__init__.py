"""B200-native cable-cell integration loop (arXiv 2411.16445 reference `mcsim`).

The hot path — Engine::advance_to / step_cell / fast_forward_to of the
reference (proj/src/engine.cpp) — runs as hand-written sm_100a kernels behind
the C ABI in include/mcg.h.  This package is the host-side mirror of the
reference's Recipe / Engine API plus its network builders.
"""
from .engine import CellView, Checkpoint, Engine, EngineOptions, GroupView, SpikeRecord  # noqa: F401
from .recipe import (CellKindSpec, ConnectionSpec, ConnectionTable, EngineError,  # noqa: F401
                     HhMembrane, HomeostasisParams, LifMembrane, MorphologyError, NoMembrane,
                     NumericError, PlacementSpec, PoissonSource, PoissonWindow, ProbeSpec,
                     ProbeWhat, PrpUnitSpec, Recipe, Region, RegularSource, ScriptedSource,
                     Segment, SelectionPolicy, SpeciesSpec, StcParams, StdpParams, SynKind,
                     SynSpec, TargetingError)
