"""B200-native executor for FusionStitching's hot path (stitched fusion groups).

The product is libsfx.so (C ABI in include/sfx.h): each fusion group the
reference planner emits runs as ONE generated sm_100a kernel.  `host` is the
Python mirror of the reference's run_program / run_compiled interface.
"""

from .host import (  # noqa: F401
    CompiledGraph, CompileReport, Context, ExecError, GraphDesc, Kernel, KernelProgram, ParseError,
    TensorGraph, codegen, default_context, graph_from_json, lib, load_bundle, parse_graph, run_compiled,
    run_program,
)
