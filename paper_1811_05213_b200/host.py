"""Host-side mirror of the reference executor interface over the C ABI.

The reference's hot path is C++ (`run_program`, exec.hpp:60-61;
`run_compiled`, pipeline.hpp:50-51).  The product boundary is libsfx.so
(include/sfx.h); this module is the thin ctypes mirror used by the tests, the
benchmark and Python callers, with the reference's names and argument meaning:

    graph  = parse_graph(text)                       # ir.cpp:340-443 (mean lowering included)
    report = CompileReport.from_bundle(bundle)        # compile_graph output, exported by the
                                                      # reference itself (oracle/_ref/ref_tool)
    outs   = run_program(report.kernels[i].program, graph, externals)   # list, comp.roots order
    values = run_compiled(report, graph, inputs)                        # dict of graph outputs

Arrays are numpy float32/int32, row-major.  Errors raise ExecError (the
reference's exception type name, exec.hpp:21-23) carrying sfx_last_error().
There is no CPU fallback: without libsfx.so or a GPU every call raises.
"""

from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsfx.so")

MAX_RANK = 8
OPCODES = {
    "parameter": 0, "constant": 1, "elementwise": 2, "reshape": 3, "bitcast": 4,
    "transpose": 5, "broadcast": 6, "reduce": 7, "batch_matmul": 8, "library_call": 9,
}
EW_KINDS = ["add", "sub", "mul", "max", "min", "neg", "compare", "select", "scale",
            "exp", "log", "div", "pow", "tanh", "sqrt", "rsqrt"]
REDUCERS = {"sum": 0, "max": 1, "min": 2}
STRATEGIES = {"auto": 0, "literal": 1, "map": 2, "row": 3, "col": 4, "colbc": 5}
EXPENSIVE = {"exp", "log", "div", "pow", "tanh", "sqrt", "rsqrt"}


class ExecError(RuntimeError):
    """Mirror of stitchfuse::ExecError; `status` is the sfx_status code."""

    def __init__(self, msg, status=5):
        super().__init__(msg)
        self.status = status


class ParseError(ExecError):
    pass


# --------------------------------------------------------------------------- ABI

class SfxInstr(C.Structure):
    _fields_ = [
        ("id", C.c_char_p), ("opcode", C.c_int32), ("kind", C.c_int32), ("dtype", C.c_int32),
        ("rank", C.c_int32), ("dims", C.c_int64 * MAX_RANK), ("n_operands", C.c_int32),
        ("operands", C.c_int32 * 3), ("permutation", C.c_int64 * MAX_RANK), ("n_dim_map", C.c_int32),
        ("broadcast_dim_map", C.c_int64 * MAX_RANK), ("n_reduce_dims", C.c_int32),
        ("reduce_dims", C.c_int64 * MAX_RANK), ("reducer", C.c_int32), ("scalar", C.c_double),
        ("n_literal", C.c_int64), ("literal", C.POINTER(C.c_double)),
    ]


class SfxStmt(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("instr", C.c_int32), ("split_dim", C.c_int64), ("sword", C.c_int64),
        ("sched_type", C.c_int32), ("dest", C.c_int32), ("offset", C.c_int64), ("bytes", C.c_int64),
        ("root_index", C.c_int32),
    ]


class SfxMemberPlan(C.Structure):
    _fields_ = [("arena_offset", C.c_int64), ("split_dim", C.c_int64), ("sword", C.c_int64), ("sched_type", C.c_int32)]


class SfxProgram(C.Structure):
    _fields_ = [
        ("n_members", C.c_int32), ("members", C.POINTER(C.c_int32)), ("n_roots", C.c_int32),
        ("roots", C.POINTER(C.c_int32)), ("fusion_root", C.c_int32), ("blocks", C.c_int64),
        ("block_threads", C.c_int32), ("arena_bytes", C.c_int64), ("n_stmts", C.c_int32),
        ("stmts", C.POINTER(SfxStmt)), ("member_plans", C.POINTER(SfxMemberPlan)),
    ]


class SfxGraphDesc(C.Structure):
    _fields_ = [
        ("n_instrs", C.c_int32), ("instrs", C.POINTER(SfxInstr)), ("n_outputs", C.c_int32),
        ("outputs", C.POINTER(C.c_int32)), ("n_programs", C.c_int32), ("programs", C.POINTER(SfxProgram)),
    ]


class SfxCompileOpts(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("debug_checks", C.c_int32), ("rows_per_cta", C.c_int32),
                ("threads_per_row", C.c_int32), ("items_per_thread", C.c_int32), ("row_pipeline", C.c_int32),
                ("pipe_warps", C.c_int32), ("pipe_stages", C.c_int32), ("pipe_ctas_per_sm", C.c_int32),
                ("cross_rank", C.c_int32), ("host_stream", C.c_int32)]


class SfxKernelInfo(C.Structure):
    _fields_ = [
        ("strategy", C.c_char_p), ("entry", C.c_char_p), ("n_inputs", C.c_int32), ("n_outputs", C.c_int32),
        ("grid", C.c_int64), ("block", C.c_int32), ("smem_bytes", C.c_int32), ("workspace_bytes", C.c_int64),
        ("algorithmic_bytes", C.c_int64), ("registers", C.c_int32), ("vector_width", C.c_int32),
    ]


EXPORTS = [
    "sfx_abi_version", "sfx_last_error", "sfx_ctx_create", "sfx_ctx_destroy", "sfx_alloc", "sfx_free",
    "sfx_host_alloc", "sfx_host_free", "sfx_memcpy_h2d", "sfx_memcpy_d2h", "sfx_memset_d32",
    "sfx_stream_sync", "sfx_launch_count", "sfx_program_compile", "sfx_program_codegen",
    "sfx_kernel_get_info", "sfx_kernel_input_instrs", "sfx_program_launch", "sfx_kernel_destroy",
    "sfx_graph_compile", "sfx_graph_param_instrs", "sfx_graph_kernel", "sfx_graph_kernel_count", "sfx_graph_run",
    "sfx_graph_run_host", "sfx_graph_destroy", "sfx_nccl_unique_id", "sfx_nccl_init",
    "sfx_allreduce_sum_f32", "sfx_peer_create", "sfx_peer_open", "sfx_program_time", "sfx_program_signature",
    "sfx_template_param_has", "sfx_template_param_put", "sfx_template_params_text", "sfx_graph_fetch",
    "sfx_graph_run_host_async",
]
ABI_VERSION = 3
PEER_HANDLE_BYTES = 64
PEER_MAX_RANKS = 8

_lib = None


def lib():
    """Loads libsfx.so (fails loudly: there is no fallback executor)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExecError(f"libsfx.so not built ({LIB_PATH}); run __graft_entry__.build()", 3)
    L = C.CDLL(LIB_PATH)
    vp, u64, i32, i64 = C.c_void_p, C.c_uint64, C.c_int32, C.c_int64
    sig = {
        "sfx_abi_version": (i32, []),
        "sfx_last_error": (C.c_char_p, []),
        "sfx_ctx_create": (i32, [i32, C.POINTER(vp)]),
        "sfx_ctx_destroy": (i32, [vp]),
        "sfx_alloc": (i32, [vp, u64, C.POINTER(u64)]),
        "sfx_free": (i32, [vp, u64]),
        "sfx_host_alloc": (i32, [vp, u64, C.POINTER(vp)]),
        "sfx_host_free": (i32, [vp, vp]),
        "sfx_memcpy_h2d": (i32, [vp, u64, vp, u64, vp]),
        "sfx_memcpy_d2h": (i32, [vp, vp, u64, u64, vp]),
        "sfx_memset_d32": (i32, [vp, u64, C.c_uint32, u64, vp]),
        "sfx_stream_sync": (i32, [vp, vp]),
        "sfx_launch_count": (i64, [vp]),
        "sfx_program_compile": (i32, [vp, C.POINTER(SfxGraphDesc), i32, C.POINTER(SfxCompileOpts), C.POINTER(vp)]),
        "sfx_program_codegen": (i32, [C.POINTER(SfxGraphDesc), i32, C.POINTER(SfxCompileOpts), C.c_char_p, u64,
                                      C.c_char_p, u64, C.c_char_p, u64]),
        "sfx_kernel_get_info": (i32, [vp, C.POINTER(SfxKernelInfo)]),
        "sfx_kernel_input_instrs": (i32, [vp, C.POINTER(i32), i32]),
        "sfx_program_launch": (i32, [vp, C.POINTER(u64), i32, C.POINTER(u64), i32, vp]),
        "sfx_kernel_destroy": (i32, [vp]),
        "sfx_graph_compile": (i32, [vp, C.POINTER(SfxGraphDesc), C.POINTER(SfxCompileOpts), C.POINTER(vp)]),
        "sfx_graph_param_instrs": (i32, [vp, C.POINTER(i32), i32, C.POINTER(i32)]),
        "sfx_graph_kernel": (i32, [vp, i32, C.POINTER(vp)]),
        "sfx_graph_kernel_count": (i32, [vp, C.POINTER(i32), C.POINTER(i32)]),
        "sfx_graph_run": (i32, [vp, C.POINTER(u64), i32, C.POINTER(u64), i32, vp, i32]),
        "sfx_graph_run_host": (i32, [vp, C.POINTER(vp), i32, C.POINTER(vp), i32, vp]),
        "sfx_graph_destroy": (i32, [vp]),
        "sfx_nccl_unique_id": (i32, [vp]),
        "sfx_nccl_init": (i32, [vp, vp, i32, i32]),
        "sfx_allreduce_sum_f32": (i32, [vp, u64, u64, vp]),
        "sfx_peer_create": (i32, [vp, u64, vp]),
        "sfx_peer_open": (i32, [vp, vp, i32, i32]),
        "sfx_program_time": (i32, [vp, C.POINTER(SfxGraphDesc), i32, C.POINTER(SfxCompileOpts), i32,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "sfx_program_signature": (i32, [C.POINTER(SfxGraphDesc), i32, C.POINTER(SfxCompileOpts), C.c_char_p, u64]),
        "sfx_template_param_has": (i32, [C.c_char_p]),
        "sfx_template_param_put": (i32, [C.c_char_p, i32, i32, i32, i32, C.c_double, C.c_double, C.c_char_p]),
        "sfx_template_params_text": (i32, [C.c_char_p, u64, C.POINTER(u64)]),
        "sfx_graph_fetch": (i32, [vp, i32, vp, u64, vp]),
        "sfx_graph_run_host_async": (i32, [vp, C.POINTER(vp), i32, C.POINTER(vp), i32, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.sfx_abi_version() != ABI_VERSION:
        raise ExecError(f"libsfx.so ABI {L.sfx_abi_version()} != {ABI_VERSION}; rebuild it", 3)
    _lib = L
    return L


def _check(status):
    if status != 0:
        msg = lib().sfx_last_error().decode(errors="replace")
        raise ExecError(msg, status)


# --------------------------------------------------------------------------- IR

@dataclass
class Instruction:
    """Mirror of stitchfuse::Instruction (ir.hpp:82-99)."""
    id: str
    op: str                      # "parameter", "constant", "add", ..., "reduce", ...
    operands: list = field(default_factory=list)
    shape: list = field(default_factory=list)
    dtype: str = "f32"
    permutation: list = field(default_factory=list)
    broadcast_dim_map: list = field(default_factory=list)
    reduce_dims: list = field(default_factory=list)
    reducer: str = "sum"
    scalar: float = 0.0
    value: list | None = None    # constant literal (len 1 = splat)
    callee: str = ""

    @property
    def opcode(self) -> str:
        return "elementwise" if self.op in EW_KINDS else self.op

    def numel(self) -> int:
        n = 1
        for d in self.shape:
            n *= int(d)
        return n

    def np_dtype(self):
        return np.float32 if self.dtype == "f32" else np.int32


class TensorGraph:
    """Mirror of stitchfuse::TensorGraph (ir.hpp:103-125)."""

    def __init__(self, instructions, outputs):
        self.instructions = list(instructions)
        self.outputs = list(outputs)
        self.index = {ins.id: i for i, ins in enumerate(self.instructions)}
        self.users = {ins.id: set() for ins in self.instructions}
        for ins in self.instructions:
            for op in ins.operands:
                self.users[op].add(ins.id)

    def at(self, id) -> Instruction:
        return self.instructions[self.index[id]]

    def parameters(self):
        return [i for i in self.instructions if i.op == "parameter"]

    def topological_order(self):
        """ir.cpp:137-155: Kahn with a sorted ready list."""
        pending = {i.id: len(set(i.operands)) for i in self.instructions}
        ready = sorted(i for i, n in pending.items() if n == 0)
        order = []
        while ready:
            v = ready.pop(0)
            order.append(v)
            for u in sorted(self.users[v]):
                pending[u] -= 1
                if pending[u] == 0:
                    ready.append(u)
                    ready.sort()
        if len(order) != len(self.instructions):
            raise ParseError("graph contains a cycle", 1)
        return order


def graph_from_json(doc) -> TensorGraph:
    instrs = []
    for j in doc["instructions"]:
        v = j.get("value")
        instrs.append(Instruction(
            id=j["id"], op=j["op"], operands=list(j.get("operands", [])), shape=list(j["shape"]),
            dtype=j.get("dtype", "f32"), permutation=list(j.get("permutation", [])),
            broadcast_dim_map=list(j.get("broadcast_dim_map", [])), reduce_dims=list(j.get("reduce_dims", [])),
            reducer=j.get("reducer", "sum"), scalar=float(j.get("scalar", 0.0)),
            value=None if v is None else (list(v) if isinstance(v, list) else [v]), callee=j.get("callee", "")))
    return TensorGraph(instrs, doc["outputs"])


def parse_graph(text: str) -> TensorGraph:
    """Parses the reference graph format and applies its mean lowering
    (reduce mean -> `<id>.sum` + scale(1/n), ir.cpp:396-428)."""
    doc = json.loads(text) if isinstance(text, str) else text
    out = []
    by_id = {}
    for j in doc["instructions"]:
        j = dict(j)
        if j["op"] == "reduce" and j.get("reducer", "sum") == "mean":
            s = dict(j, id=j["id"] + ".sum", reducer="sum")
            out.append(s)
            by_id[s["id"]] = s
            j = {"id": j["id"], "op": "scale", "operands": [s["id"]], "shape": j["shape"],
                 "dtype": j.get("dtype", "f32"), "scalar": 0.0, "_mean": True}
        out.append(j)
        by_id[j["id"]] = j
    for j in out:
        if j.get("op") == "scale" and float(j.get("scalar", 0.0)) == 0.0 and j.get("operands") and \
                by_id.get(j["operands"][0], {}).get("op") == "reduce":
            s = by_id[j["operands"][0]]
            src = by_id[s["operands"][0]]
            n_in = int(np.prod(src["shape"], dtype=np.int64))
            n_out = int(np.prod(s["shape"], dtype=np.int64))
            j["scalar"] = 1.0 / float(n_in // n_out)
        j.pop("_mean", None)
    return graph_from_json({"instructions": out, "outputs": doc["outputs"]})


@dataclass
class KernelProgram:
    """Mirror of stitchfuse::KernelProgram + FusedComputation (kernelgen.hpp:48-54, fusion.hpp:20-25)."""
    fusion_root: str
    members: list
    roots: list
    blocks: int
    block_threads: int
    arena_bytes: int
    statements: list   # dicts as exported by ref_tool
    dump: str = ""
    # the geometry the executor reads members with (KernelProgram.arena_offsets,
    # SchedulePlan.per_instruction: id -> [split_dim, sword, "row"|"col"]); None =
    # the statements' own
    arena_offsets: dict | None = None
    per_instruction: dict | None = None


@dataclass
class CompiledKernel:
    program: KernelProgram


@dataclass
class CompileReport:
    """Mirror of stitchfuse::CompileReport (pipeline.hpp:33-40)."""
    kernels: list
    baseline_kernels: int
    fused_kernels: int
    fusion_ratio: float
    unfused: list

    @staticmethod
    def from_bundle(bundle) -> "CompileReport":
        ks = []
        for k in bundle["kernels"]:
            ks.append(CompiledKernel(KernelProgram(
                fusion_root=k["fusion_root"], members=list(k["members"]), roots=list(k["roots"]),
                blocks=int(k["blocks"]), block_threads=int(k["block_threads"]),
                arena_bytes=int(k["arena_bytes"]), statements=list(k["statements"]), dump=k.get("dump", ""),
                arena_offsets=k.get("arena_offsets"), per_instruction=k.get("per_instruction"))))
        return CompileReport(ks, bundle["baseline_kernels"], bundle["fused_kernels"], bundle["fusion_ratio"],
                             list(bundle.get("unfused", [])))


def load_bundle(path):
    with open(path) as f:
        b = json.load(f)
    return graph_from_json(b["graph"]), CompileReport.from_bundle(b), b


# --------------------------------------------------------------------------- descriptors

class GraphDesc:
    """Flattens (TensorGraph, [KernelProgram]) into sfx_graph_desc, keeping the
    ctypes buffers alive for the lifetime of this object."""

    def __init__(self, graph: TensorGraph, programs):
        self.graph = graph
        self.programs = list(programs)
        n = len(graph.instructions)
        self._instrs = (SfxInstr * max(n, 1))()
        self._keep = []
        idx = graph.index
        for i, ins in enumerate(graph.instructions):
            s = self._instrs[i]
            bid = ins.id.encode()
            self._keep.append(bid)
            s.id = bid
            s.opcode = OPCODES[ins.opcode]
            if ins.op == "library_call":  # SFX_CALLEE_*
                s.kind = {"matmul": 0, "opaque": 1}.get(ins.callee, -1)
            else:
                s.kind = EW_KINDS.index(ins.op) if ins.op in EW_KINDS else 0
            s.dtype = 0 if ins.dtype == "f32" else 1
            if len(ins.shape) > MAX_RANK:
                raise ExecError(f"rank of {ins.id} exceeds {MAX_RANK}", 1)
            s.rank = len(ins.shape)
            for k, d in enumerate(ins.shape):
                s.dims[k] = int(d)
            s.n_operands = len(ins.operands)
            for k, o in enumerate(ins.operands):
                s.operands[k] = idx[o]
            for k, p in enumerate(ins.permutation):
                s.permutation[k] = int(p)
            s.n_dim_map = len(ins.broadcast_dim_map)
            for k, d in enumerate(ins.broadcast_dim_map):
                s.broadcast_dim_map[k] = int(d)
            s.n_reduce_dims = len(ins.reduce_dims)
            for k, d in enumerate(ins.reduce_dims):
                s.reduce_dims[k] = int(d)
            s.reducer = REDUCERS.get(ins.reducer, 0)
            s.scalar = float(ins.scalar)
            if ins.value is not None:
                lit = (C.c_double * len(ins.value))(*[float(v) for v in ins.value])
                self._keep.append(lit)
                s.n_literal = len(ins.value)
                s.literal = C.cast(lit, C.POINTER(C.c_double))
        outs = (C.c_int32 * max(len(graph.outputs), 1))(*[idx[o] for o in graph.outputs])
        self._keep.append(outs)
        progs = (SfxProgram * max(len(self.programs), 1))()
        for pi, prog in enumerate(self.programs):
            sp = progs[pi]
            mem = (C.c_int32 * len(prog.members))(*[idx[m] for m in prog.members])
            roots = (C.c_int32 * len(prog.roots))(*[idx[r] for r in prog.roots])
            stmts = (SfxStmt * max(len(prog.statements), 1))()
            for si, st in enumerate(prog.statements):
                t = stmts[si]
                kind = st["kind"]
                t.kind = {"materialize": 0, "barrier": 1, "inline": 2}[kind]
                if kind != "barrier":
                    t.instr = idx[st["instr"]]
                if kind == "materialize":
                    sd, sw, ty = st["schedule"]
                    t.split_dim, t.sword, t.sched_type = int(sd), int(sw), (0 if ty == "row" else 1)
                    if st["dest"] == "shared":
                        t.dest, t.offset, t.bytes = 0, int(st["offset"]), int(st["bytes"])
                    else:
                        t.dest, t.root_index = 1, int(st["root_index"])
            self._keep += [mem, roots, stmts]
            if prog.arena_offsets is not None and prog.per_instruction is not None:
                plans = (SfxMemberPlan * len(prog.members))()
                for mi, m in enumerate(prog.members):
                    sd, sw, ty = prog.per_instruction.get(m, [0, 1, "row"])
                    plans[mi].arena_offset = int(prog.arena_offsets.get(m, -1))
                    plans[mi].split_dim, plans[mi].sword = int(sd), int(sw)
                    plans[mi].sched_type = 0 if ty == "row" else 1
                self._keep.append(plans)
                sp.member_plans = C.cast(plans, C.POINTER(SfxMemberPlan))
            sp.n_members, sp.members = len(prog.members), C.cast(mem, C.POINTER(C.c_int32))
            sp.n_roots, sp.roots = len(prog.roots), C.cast(roots, C.POINTER(C.c_int32))
            sp.fusion_root = idx[prog.fusion_root] if prog.fusion_root in idx else -1
            sp.blocks, sp.block_threads, sp.arena_bytes = prog.blocks, prog.block_threads, prog.arena_bytes
            sp.n_stmts, sp.stmts = len(prog.statements), C.cast(stmts, C.POINTER(SfxStmt))
        self._keep.append(progs)
        self.desc = SfxGraphDesc(n, C.cast(self._instrs, C.POINTER(SfxInstr)), len(graph.outputs),
                                 C.cast(outs, C.POINTER(C.c_int32)), len(self.programs),
                                 C.cast(progs, C.POINTER(SfxProgram)))

    def ref(self):
        return C.byref(self.desc)


def compile_opts(strategy="auto", rows_per_cta=0, threads_per_row=0, items_per_thread=0, row_pipeline=0,
                 pipe_warps=0, pipe_stages=0, pipe_ctas_per_sm=0, cross_rank=0, host_stream=0, debug_checks=0):
    return SfxCompileOpts(STRATEGIES[strategy], int(debug_checks), rows_per_cta, threads_per_row, items_per_thread, row_pipeline,
                          pipe_warps, pipe_stages, pipe_ctas_per_sm, int(bool(cross_rank)), int(bool(host_stream)))


def codegen(graph: TensorGraph, program: KernelProgram, strategy="auto", **kw):
    """Lowers one group and NVRTC-compiles it for sm_100a without touching a GPU.
    Returns (cuda_source, cubin_path, strategy_note)."""
    gd = GraphDesc(graph, [program])
    src = C.create_string_buffer(1 << 22)
    path = C.create_string_buffer(4096)
    strat = C.create_string_buffer(1024)
    opts = compile_opts(strategy, **kw)
    _check(lib().sfx_program_codegen(gd.ref(), 0, C.byref(opts), src, len(src), path, len(path), strat, len(strat)))
    return src.value.decode(), path.value.decode(), strat.value.decode()


def codegen_barrier(graph: TensorGraph, report: "CompileReport", k: int, **kw):
    """Like codegen() for the k-th unfused matmul barrier of a compiled module
    (instruction order), which runs as its own kernel."""
    programs = [kk.program for kk in report.kernels]
    gd = GraphDesc(graph, programs)
    src = C.create_string_buffer(1 << 22)
    path = C.create_string_buffer(4096)
    strat = C.create_string_buffer(1024)
    opts = compile_opts(**kw)
    _check(lib().sfx_program_codegen(gd.ref(), len(programs) + k, C.byref(opts), src, len(src), path, len(path),
                                     strat, len(strat)))
    return src.value.decode(), path.value.decode(), strat.value.decode()


# --------------------------------------------------------------------------- runtime

class Context:
    """sfx_ctx: device + pooled device buffer manager."""

    def __init__(self, device=0):
        h = C.c_void_p()
        _check(lib().sfx_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            lib().sfx_ctx_destroy(self.h)
            self.h = None

    def alloc(self, nbytes) -> int:
        p = C.c_uint64()
        _check(lib().sfx_alloc(self.h, int(nbytes), C.byref(p)))
        return p.value

    def free(self, ptr):
        _check(lib().sfx_free(self.h, int(ptr)))

    def h2d(self, dptr, arr: np.ndarray, stream=0):
        arr = np.ascontiguousarray(arr)
        _check(lib().sfx_memcpy_h2d(self.h, int(dptr), arr.ctypes.data, arr.nbytes, C.c_void_p(stream)))
        self.sync(stream)

    def d2h(self, arr: np.ndarray, dptr, stream=0):
        _check(lib().sfx_memcpy_d2h(self.h, arr.ctypes.data, int(dptr), arr.nbytes, C.c_void_p(stream)))
        self.sync(stream)

    def sync(self, stream=0):
        _check(lib().sfx_stream_sync(self.h, C.c_void_p(stream)))

    def launch_count(self) -> int:
        return int(lib().sfx_launch_count(self.h))

    # ---- batch-crossing column reductions across GPUs (NCCL) ----
    def nccl_init(self, unique_id: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(lib().sfx_nccl_init(self.h, buf, nranks, rank))

    def allreduce_sum_f32(self, dptr: int, count: int, stream=0):
        _check(lib().sfx_allreduce_sum_f32(self.h, int(dptr), int(count), C.c_void_p(stream)))


    # ---- peer-memory group: column sums combined across ranks inside the kernel ----
    def peer_create(self, nbytes=1 << 24) -> bytes:
        """Allocates this rank's symmetric peer arena; returns its IPC handle."""
        buf = C.create_string_buffer(PEER_HANDLE_BYTES)
        _check(lib().sfx_peer_create(self.h, int(nbytes), buf))
        return buf.raw

    def peer_open(self, handles, rank: int):
        """Opens every rank's arena (handles in rank order, as exchanged out of band)."""
        blob = b"".join(bytes(h) for h in handles)
        if len(blob) != PEER_HANDLE_BYTES * len(handles):
            raise ExecError("peer handles must be 64 bytes each", 1)
        buf = C.create_string_buffer(blob, len(blob))
        _check(lib().sfx_peer_open(self.h, buf, len(handles), rank))

    def peer_init(self, rank: int, world: int, all_gather, nbytes=1 << 24):
        """peer_create + exchange + peer_open; `all_gather(obj) -> list` is the
        out-of-band exchange (e.g. torch.distributed.all_gather_object)."""
        if world > PEER_MAX_RANKS:
            raise ExecError(f"peer group of {world} ranks exceeds {PEER_MAX_RANKS}", 1)
        mine = self.peer_create(nbytes)
        handles = all_gather(mine)
        if len(handles) != world or bytes(handles[rank]) != mine:
            raise ExecError("peer handle exchange returned an inconsistent list", 1)
        self.peer_open(handles, rank)


def torch_all_gather(obj):
    """all_gather for Context.peer_init over the default torch.distributed group."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().sfx_nccl_unique_id(buf))
    return buf.raw


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class Kernel:
    """One fused group lowered to one stitched sm_100a kernel (run_program twin)."""

    def __init__(self, ctx: Context, graph: TensorGraph, program: KernelProgram, strategy="auto", **kw):
        self.ctx, self.graph, self.program = ctx, graph, program
        self._gd = GraphDesc(graph, [program])
        h = C.c_void_p()
        opts = compile_opts(strategy, **kw)
        _check(lib().sfx_program_compile(ctx.h, self._gd.ref(), 0, C.byref(opts), C.byref(h)))
        self.h = h
        self._owned = True
        self.roots = list(program.roots)
        self._load_info()

    @classmethod
    def _borrow(cls, ctx, graph, program, handle):
        k = cls.__new__(cls)
        k.ctx, k.graph, k.program, k.h, k._owned, k._gd = ctx, graph, program, handle, False, None
        k.roots = list(program.roots) if program is not None else []
        k._load_info()
        return k

    def _load_info(self):
        info = SfxKernelInfo()
        _check(lib().sfx_kernel_get_info(self.h, C.byref(info)))
        self.info = {
            "strategy": info.strategy.decode(), "entry": info.entry.decode(), "n_inputs": info.n_inputs,
            "n_outputs": info.n_outputs, "grid": info.grid, "block": info.block, "smem_bytes": info.smem_bytes,
            "workspace_bytes": info.workspace_bytes, "algorithmic_bytes": info.algorithmic_bytes,
            "registers": info.registers, "vector_width": info.vector_width,
        }
        buf = (C.c_int32 * max(info.n_inputs, 1))()
        _check(lib().sfx_kernel_input_instrs(self.h, buf, info.n_inputs))
        self.input_ids = [self.graph.instructions[buf[i]].id for i in range(info.n_inputs)]

    def launch(self, in_ptrs, out_ptrs, stream=0):
        ins = (C.c_uint64 * max(len(in_ptrs), 1))(*[int(p) for p in in_ptrs])
        outs = (C.c_uint64 * max(len(out_ptrs), 1))(*[int(p) for p in out_ptrs])
        _check(lib().sfx_program_launch(self.h, ins, len(in_ptrs), outs, len(out_ptrs), C.c_void_p(stream)))

    def close(self):
        if self.h and self._owned:
            lib().sfx_kernel_destroy(self.h)
        self.h = None


class CompiledGraph:
    """The whole compiled module on device (run_compiled twin)."""

    def __init__(self, ctx: Context, graph: TensorGraph, report: CompileReport, strategy="auto", **kw):
        self.ctx, self.graph, self.report = ctx, graph, report
        self._gd = GraphDesc(graph, [k.program for k in report.kernels])
        h = C.c_void_p()
        opts = compile_opts(strategy, **kw)
        _check(lib().sfx_graph_compile(ctx.h, self._gd.ref(), C.byref(opts), C.byref(h)))
        self.h = h
        n = C.c_int32()
        buf = (C.c_int32 * (len(graph.instructions) + 1))()
        _check(lib().sfx_graph_param_instrs(h, buf, len(graph.instructions), C.byref(n)))
        self.param_ids = [graph.instructions[buf[i]].id for i in range(n.value)]
        self.kernels = []
        for i, k in enumerate(report.kernels):
            kh = C.c_void_p()
            _check(lib().sfx_graph_kernel(h, i, C.byref(kh)))
            self.kernels.append(Kernel._borrow(ctx, graph, k.program, kh))
        # unfused matmul barriers (one kernel each, after the planned groups)
        nk, npl = C.c_int32(), C.c_int32()
        _check(lib().sfx_graph_kernel_count(h, C.byref(nk), C.byref(npl)))
        unfused = set(report.unfused)
        self.unfused_ids = [i.id for i in graph.instructions if i.id in unfused]  # C-side order
        assert len(self.unfused_ids) == nk.value - npl.value
        self.barrier_kernels = []
        for i, u in zip(range(npl.value, nk.value), self.unfused_ids):
            kh = C.c_void_p()
            _check(lib().sfx_graph_kernel(h, i, C.byref(kh)))
            k = Kernel._borrow(ctx, graph, None, kh)
            k.roots = [u]
            self.barrier_kernels.append(k)

    @property
    def launches_per_run(self) -> int:
        return len(self.kernels) + len(self.barrier_kernels)

    def run(self, param_ptrs, out_ptrs, stream=0, cuda_graph=False):
        ps = (C.c_uint64 * max(len(param_ptrs), 1))(*[int(p) for p in param_ptrs])
        os_ = (C.c_uint64 * max(len(out_ptrs), 1))(*[int(p) for p in out_ptrs])
        _check(lib().sfx_graph_run(self.h, ps, len(param_ptrs), os_, len(out_ptrs), C.c_void_p(stream),
                                   1 if cuda_graph else 0))

    def run_host(self, params: dict, outputs: dict | None = None, stream=0):
        """Host arrays in, host arrays out (copies inside)."""
        arrs = [np.ascontiguousarray(params[i], dtype=self.graph.at(i).np_dtype()) for i in self.param_ids]
        if outputs is None:
            outputs = {o: np.empty(self.graph.at(o).shape, self.graph.at(o).np_dtype()) for o in self.graph.outputs}
        pin = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
        pout = (C.c_void_p * max(len(outputs), 1))(*[outputs[o].ctypes.data for o in self.graph.outputs])
        _check(lib().sfx_graph_run_host(self.h, pin, len(arrs), pout, len(self.graph.outputs), C.c_void_p(stream)))
        return outputs

    def run_host_async(self, param_ptrs, out_ptrs, stream):
        """sfx_graph_run_host_async: pinned host pointers (param slot order /
        graph output order), complete when `stream` is."""
        pin = (C.c_void_p * max(len(param_ptrs), 1))(*[int(p) for p in param_ptrs])
        pout = (C.c_void_p * max(len(out_ptrs), 1))(*[int(p) for p in out_ptrs])
        _check(lib().sfx_graph_run_host_async(self.h, pin, len(param_ptrs), pout, len(out_ptrs), C.c_void_p(stream)))

    def fetch(self, instr_id: str, stream=0) -> np.ndarray:
        """A value the latest run on `stream` left in HBM (an intermediate group
        root, or a dense constant): sfx_graph_fetch."""
        ins = self.graph.at(instr_id)
        a = np.empty(ins.shape, ins.np_dtype())
        _check(lib().sfx_graph_fetch(self.h, self.graph.index[instr_id], C.c_void_p(a.ctypes.data), a.nbytes,
                                     C.c_void_p(stream)))
        return a

    def close(self):
        if self.h:
            lib().sfx_graph_destroy(self.h)
        self.h = None


def constant_value(ins: Instruction) -> np.ndarray:
    """stitchfuse::constant_value (exec.cpp:215-229): splat or dense literal,
    each double narrowed to the element type."""
    n = ins.numel()
    lit = list(ins.value or [])
    if len(lit) != 1 and len(lit) != n:
        raise ExecError("constant literal size mismatch for " + ins.id)
    raw = np.array(lit if len(lit) == n else lit * n, dtype=np.float64)
    v = raw.astype(np.float32) if ins.dtype == "f32" else raw.astype(np.int64).astype(np.int32)
    return v.reshape(ins.shape)


def _to_device(ctx, arr):
    p = ctx.alloc(max(arr.nbytes, 4))
    ctx.h2d(p, arr)
    return p


def run_program(program: KernelProgram, graph: TensorGraph, externals: dict, strategy="auto", ctx=None, **kw):
    """Device twin of stitchfuse::run_program (exec.cpp:296-412): one stitched
    launch; returns one array per root in comp.roots order."""
    ctx = ctx or default_context()
    k = Kernel(ctx, graph, program, strategy, **kw)
    ptrs = []
    try:
        ins = []
        for i in k.input_ids:
            if i not in externals:
                raise ExecError("missing external value " + i)
            ins.append(_to_device(ctx, np.ascontiguousarray(externals[i], dtype=graph.at(i).np_dtype())))
        ptrs += ins
        outs = [ctx.alloc(max(graph.at(r).numel() * 4, 4)) for r in program.roots]
        ptrs += outs
        k.launch(ins, outs)
        ctx.sync()
        res = []
        for r, p in zip(program.roots, outs):
            a = np.empty(graph.at(r).shape, graph.at(r).np_dtype())
            ctx.d2h(a, p)
            res.append(a)
        return res
    finally:
        for p in ptrs:
            ctx.free(p)
        k.close()


def run_compiled(report: CompileReport, graph: TensorGraph, inputs: dict, strategy="auto", ctx=None,
                 values="outputs"):
    """Device twin of stitchfuse::run_compiled (pipeline.cpp:65-133).

    values="outputs": the graph outputs (what callers of the reference read,
    stitchfuse.cpp:236-237).  values="all": the reference's whole map
    (pipeline.cpp:104-118) — every parameter, constant, unfused instruction and
    group root; intermediates are read back from HBM after the run
    (sfx_graph_fetch)."""
    if values not in ("outputs", "all"):
        raise ValueError("values must be 'outputs' or 'all'")
    ctx = ctx or default_context()
    cg = CompiledGraph(ctx, graph, report, strategy)
    try:
        for p in cg.param_ids:
            if p not in inputs:
                raise ExecError("missing input for parameter " + p)
        out = cg.run_host(inputs)
        if values == "outputs":
            return out
        full = {}
        roots = set(cg.unfused_ids)
        for k in report.kernels:
            roots.update(k.program.roots)
        for ins in graph.instructions:
            if ins.op == "parameter":
                full[ins.id] = np.asarray(inputs[ins.id], dtype=ins.np_dtype()).reshape(ins.shape)
            elif ins.op == "constant":
                full[ins.id] = constant_value(ins)
            elif ins.id in out:
                full[ins.id] = out[ins.id]
            elif ins.id in roots:
                full[ins.id] = cg.fetch(ins.id)
        return full
    finally:
        cg.close()
