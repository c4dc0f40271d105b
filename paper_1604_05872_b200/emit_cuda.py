"""emit_cuda -- femopt kernel IR -> sm_100a CUDA kernel.

The reference's only backend is ``emit_c`` (/root/reference/proj/src/emit_c.cpp:
108-174): a C function ``fn(double* outputs..., const double* input tables...,
double constants...)`` (each group in name order, :137-140) whose element
loop runs every cell, with pre-evaluated tables baked in as ``static const``
(:143-159) and outputs accumulated with ``+=`` into caller-zeroed arrays
(:91-92,129).  This module is the GPU counterpart for ANY femopt IR -- the
raw kernels of ir.py as well as femopt's optimized output (``to_json``):

  * the order-free element loop becomes the grid: one thread per cell;
  * everything inside it is emitted as the same loop nest, in the same
    statement and operand order as emit_c, compiled with ``--fmad=false``
    (the oracle's ``-ffp-contract=off``), so results match femopt's own
    emitted C bit for bit on the same inputs;
  * input tables are kernel arguments (device pointers), pre-evaluated tables
    are ``__device__ const`` arrays in the module, constants are by value;
  * the element count is a runtime argument (femopt bakes it as a literal).

It handles arity-1 (element vectors) and arity-2 (element matrices) nests
alike -- whatever femopt's validator accepts (kernel.cpp:246-392).  The
hand-written kernels in csrc/ remain the fast path for the BASELINE forms;
this is the generic one: correct for every femopt kernel, thread-per-cell
fast.

IR forms accepted (proj/README.md:68-100): flat ``statements`` with ``level``
(loops open lazily in declaration order) or a nested ``body`` with
``{"loop": {...}}`` nodes, as femopt writes it.
"""
from __future__ import annotations

import json
import re

import numpy as np

_CALLS = {"fabs": "fabs", "sqrt": "sqrt", "exp": "exp", "log": "log", "pow": "pow",
          "sin": "sin", "cos": "cos", "tan": "tan", "atan": "atan", "atan2": "atan2",
          "cbrt": "cbrt", "fmin": "fmin", "fmax": "fmax", "abs": "fabs"}


class IRError(ValueError):
    pass


# ----------------------------------------------------------------------------
# IR -> nested tree
# ----------------------------------------------------------------------------
def _lhs(st):
    lhs = st["lhs"]
    if isinstance(lhs, str):
        return lhs, []
    return lhs[0], list(lhs[1:])


def _tree(ir: dict) -> list:
    """Normalize to [("loop", index, begin, end, body, class) | ("stmt", name, idx, op, rhs)]."""
    ext = ir["indices"]

    def from_nested(nodes):
        out = []
        for n in nodes:
            if "loop" in n:
                L = n["loop"]
                out.append(("loop", L["index"], int(L.get("begin", 0)),
                            int(L.get("end", ext[L["index"]])), from_nested(L["body"]),
                            L.get("class")))
            elif "body" in n and "index" in n:  # nested form of the input schema
                out.append(("loop", n["index"], int(n.get("begin", 0)),
                            int(n.get("end", ext[n["index"]])), from_nested(n["body"]),
                            n.get("class")))
            else:
                name, idx = _lhs(n)
                out.append(("stmt", name, idx, n.get("op", "="), n["rhs"]))
        return out

    if "body" in ir:
        return from_nested(ir["body"])
    loops = [L["index"] for L in ir["loops"]]
    classes = {L["index"]: L.get("class") for L in ir["loops"]}
    root: list = []
    stack = [root]  # stack[d] = body list at depth d
    for st in ir["statements"]:
        if "body" in st and "index" in st:
            stack[-1].append(from_nested([st])[0])
            continue
        level = int(st["level"])
        if level > len(loops):
            raise IRError(f"statement level {level} exceeds the loop nest")
        while len(stack) - 1 > level:  # close deeper loops
            stack.pop()
        while len(stack) - 1 < level:  # open loops lazily, in declaration order
            idx = loops[len(stack) - 1]
            node = ("loop", idx, 0, int(ext[idx]), [], classes.get(idx))
            stack[-1].append(node)
            stack.append(node[4])
        name, idx = _lhs(st)
        stack[-1].append(("stmt", name, idx, st.get("op", "="), st["rhs"]))
    return root


# ----------------------------------------------------------------------------
# code generation
# ----------------------------------------------------------------------------
def _lit(x: float) -> str:
    x = float(x)
    if x == 0.0:
        return "0.0"
    if np.isfinite(x) and x == int(x) and abs(x) < 2 ** 52:
        return f"{int(x)}.0"
    return x.hex()


_IDENT = re.compile(r"^[A-Za-z_][A-Za-z0-9_]*$")


def _ident(name: str) -> str:
    if not _IDENT.match(name):
        raise IRError(f"bad name {name!r}")
    return name


class Emitted:
    """Generated CUDA source and the calling convention of its kernel."""

    def __init__(self, source, fn, outputs, inputs, constants, preevaluated, e_index, extents,
                 dims):
        self.source = source
        self.fn = fn
        self.outputs = outputs          # names, emit_c order
        self.inputs = inputs            # input-table names, emit_c order
        self.constants = constants      # names, emit_c order
        self.preevaluated = preevaluated
        self.e_index = e_index          # the order-free element index (or None)
        self.extents = extents          # index -> extent (the IR's; e is runtime)
        self.dims = dims                # array name -> dims

    def shape(self, name: str, ncells: int) -> tuple:
        return tuple(ncells if d == self.e_index else int(self.extents[d])
                     for d in self.dims[name])

    def size(self, name: str, ncells: int) -> int:
        return int(np.prod(self.shape(name, ncells), dtype=np.int64))


def _op_counts(tree, J, ext):
    """Arithmetic nodes executed per cell outside / inside the row loops (J)."""
    def ops(x):
        if isinstance(x, list) and x and x[0] in ("+", "*", "/", "call"):
            return max(1, len(x) - 2) + sum(ops(a) for a in x[1:])
        if isinstance(x, list) and x and x[0] == "sym":
            return 0
        return 0

    tot = [0, 0]

    def walk(nodes, mult, inJ):
        for n in nodes:
            if n[0] == "loop":
                _, idx, b, e, body, cls = n
                if cls == "orderfree":
                    walk(body, mult, inJ)
                else:
                    walk(body, mult * max(0, e - b), inJ or idx == J)
            else:
                tot[1 if inJ else 0] += mult * (1 + ops(n[4]))

    walk(tree, 1, False)
    return tot


def _warp_plan(tree, outputs, dims, temps, e_index, ext):
    """The warp-per-cell mapping, if the nest allows it: the output rows (first
    linear index J) are spread over the lanes, every other loop runs in full on
    each lane.  Returns J or None."""
    if e_index is None:
        return None
    rows = {tuple(dims[o][:2]) for o in outputs}
    if len(rows) != 1:
        return None
    (e0, J), = rows
    if e0 != e_index or J is None:
        return None
    ok = True
    written_in_J, read_outside_J = set(), set()

    def names_in(x, acc):
        if isinstance(x, str):
            acc.add(x)
        elif isinstance(x, list) and x:
            if x[0] == "sym":
                acc.add(x[1])
            for a in x[1:]:
                names_in(a, acc)

    def walk(nodes, inJ):
        nonlocal ok
        for n in nodes:
            if n[0] == "loop":
                _, idx, b, e, body, _ = n
                if idx == J:
                    if inJ or b != 0 or e != ext[J]:
                        ok = False
                    walk(body, True)
                else:
                    walk(body, inJ)
            else:
                _, name, idx, op, rhs = n
                used = set()
                names_in(rhs, used)
                if any(o in used for o in outputs):
                    ok = False  # outputs are write-only in femopt nests
                if name in outputs:
                    if not inJ or op != "+=" or idx[:2] != [e_index, J]:
                        ok = False
                elif inJ:
                    written_in_J.add(name)
                if not inJ:
                    read_outside_J.update(used)

    walk(tree, False)
    if not ok or (written_in_J & read_outside_J):
        return None
    return J


def emit(ir: dict | str, fn: str = "femopt_kernel", strategy: str = "auto") -> Emitted:
    """Generate the kernel.  ``strategy``: "thread" (one thread per cell), "warp"
    (one warp per cell, output rows over the lanes, accumulators in registers),
    or "auto" (warp when the nest allows it and the output has >= 8 rows)."""
    if isinstance(ir, str):
        ir = json.loads(ir)
    ext = {k: int(v) for k, v in ir["indices"].items()}
    tables = ir.get("tables", {})
    consts = ir.get("constants", {}) or {}
    outputs = sorted(ir["outputs"])
    tree = _tree(ir)

    # the element loop: a single top-level loop that is order-free (femopt's
    # class; an unclassified top-level loop over "e" counts as one)
    e_index = None
    top_loops = [n for n in tree if n[0] == "loop"]
    if len(top_loops) == 1:
        _, idx, _, _, _, cls = top_loops[0]
        if cls == "orderfree" or (cls is None and idx == "e"):
            e_index = idx

    dims = {}
    for name, t in tables.items():
        dims[name] = list(t["dims"])
    # outputs / temporaries from the statements
    temps: dict[str, list] = {}

    def scan(nodes):
        for n in nodes:
            if n[0] == "loop":
                scan(n[4])
            else:
                _, name, idx, op, rhs = n
                if name in outputs:
                    prev = dims.get(name)
                    if prev is not None and prev != idx:
                        raise IRError(f"output {name} written with different subscripts")
                    dims[name] = list(idx)
                elif name in tables:
                    raise IRError(f"statement writes table {name}")
                else:
                    prev = temps.get(name)
                    if prev is not None and prev != idx:
                        raise IRError(f"temporary {name} used with different subscripts")
                    temps[name] = list(idx)

    scan(tree)
    for o in outputs:
        if o not in dims:
            raise IRError(f"output {o} is never written")

    J = _warp_plan(tree, outputs, dims, temps, e_index, ext)
    if strategy == "auto":
        strategy = "thread"
        if J is not None and ext[J] >= 8:
            o_out, o_in = _op_counts(tree, J, ext)
            # the warp mapping repeats the out-of-row work on every lane
            if 31 * o_out < 0.25 * o_in:
                strategy = "warp"
    if strategy == "warp" and J is None:
        raise IRError("the warp mapping does not apply to this nest")
    if strategy not in ("thread", "warp"):
        raise IRError(f"unknown strategy {strategy!r}")
    warp = strategy == "warp"
    acc_dims = {d for o in outputs for d in dims[o][2:]}
    R = (ext[J] + 31) // 32 if warp else 0
    rest = {o: int(np.prod([ext[d] for d in dims[o][2:]], dtype=np.int64)) for o in outputs}

    inputs = sorted(n for n, t in tables.items() if t.get("provenance", "input") != "preevaluated")
    preev = sorted(n for n, t in tables.items() if t.get("provenance", "input") == "preevaluated")
    cnames = sorted(consts)

    def ext_of(d):
        return "E" if d == e_index else str(ext[d])

    def offset(name, idx):
        dd = dims[name]
        if len(idx) != len(dd):
            raise IRError(f"{name} subscripted with {idx}, declared {dd}")
        if not idx:
            return "0"
        expr = f"(long)i_{idx[0]}"
        for d, i in zip(dd[1:], idx[1:]):
            expr = f"({expr} * {ext_of(d)} + i_{i})"
        return expr

    # Printed exactly as emit_c prints it (emit_c.cpp:47-80: precedence-driven,
    # nested sums/products flattened, C's left-to-right evaluation), so the
    # generated arithmetic is femopt's emitted arithmetic, operation for operation.
    def expr(x, prec=0) -> str:
        if isinstance(x, (int, float)) and not isinstance(x, bool):
            s_ = _lit(x)
            return f"({s_})" if float(x) < 0 and prec >= 1 else s_
        if isinstance(x, str):
            if x in temps:
                if temps[x]:
                    raise IRError(f"array temporary {x} read without subscripts")
                return f"v_{_ident(x)}"
            if x in consts:
                return f"c_{_ident(x)}"
            raise IRError(f"unknown scalar {x!r}")
        op = x[0]
        if op == "sym":
            name, idx = x[1], list(x[2:])
            if name in tables:
                return f"t_{_ident(name)}[{offset(name, idx)}]"
            if name in temps:
                t_idx = temps[name]
                if len(idx) != len(t_idx):
                    raise IRError(f"temporary {name} subscript count")
                flat = "0"
                for d, i in zip(t_idx, idx):
                    flat = f"({flat} * {ext[d]} + i_{i})"
                return f"v_{_ident(name)}[{flat}]"
            if name in outputs:
                return f"o_{_ident(name)}[{offset(name, idx)}]"
            raise IRError(f"unknown array {name!r}")
        if op == "+":
            s_ = " + ".join(expr(a, 0) for a in x[1:])
            return f"({s_})" if prec >= 1 else s_
        if op == "*":
            s_ = " * ".join(expr(a, 1) for a in x[1:])
            return f"({s_})" if prec >= 2 else s_
        if op == "/":
            if len(x) != 3:
                raise IRError("'/' takes two operands")
            s_ = f"{expr(x[1], 1)} / {expr(x[2], 2)}"
            return f"({s_})" if prec >= 2 else s_
        if op == "call":
            fnm = x[1]
            if fnm not in _CALLS:
                raise IRError(f"unsupported call {fnm!r}")
            return f"{_CALLS[fnm]}(" + ", ".join(expr(a, 0) for a in x[2:]) + ")"
        raise IRError(f"unknown operator {op!r}")

    lines = []

    def emit_nodes(nodes, ind):
        pad = "  " * ind
        for n in nodes:
            if n[0] == "loop":
                _, idx, b, e, body, _ = n
                if idx == e_index:
                    raise IRError("nested element loop")
                if warp and idx == J:  # this lane's rows: J = lane + 32 r
                    lines.append(f"{pad}#pragma unroll")
                    lines.append(f"{pad}for (int r_ = 0; r_ < {R}; ++r_) {{")
                    lines.append(f"{pad}  const int i_{_ident(J)} = lane_ + 32 * r_;")
                    lines.append(f"{pad}  if (i_{J} < {e}) {{")
                    emit_nodes(body, ind + 2)
                    lines.append(f"{pad}  }}")
                    lines.append(f"{pad}}}")
                    continue
                if warp and e - b <= 64 and idx in acc_dims and \
                        (e - b) * _op_counts(body, None, ext)[0] <= 4096:
                    lines.append(f"{pad}#pragma unroll")  # accumulators stay in registers
                lines.append(f"{pad}for (int i_{_ident(idx)} = {b}; i_{idx} < {e}; ++i_{idx}) {{")
                emit_nodes(body, ind + 1)
                lines.append(f"{pad}}}")
            else:
                _, name, idx, op, rhs = n
                if name in outputs and warp:
                    flat = "0"
                    for d, i in zip(dims[name][2:], idx[2:]):
                        flat = f"({flat} * {ext[d]} + i_{i})"
                    target = f"a_{name}[r_ * {rest[name]} + {flat}]"
                elif name in outputs:
                    target = f"o_{name}[{offset(name, idx)}]"
                elif temps[name]:
                    flat = "0"
                    for d, i in zip(temps[name], idx):
                        flat = f"({flat} * {ext[d]} + i_{i})"
                    target = f"v_{name}[{flat}]"
                else:
                    target = f"v_{name}"
                if op == "+=":
                    lines.append(f"{pad}{target} += {expr(rhs)};")
                elif op == "=":
                    lines.append(f"{pad}{target} = {expr(rhs)};")
                else:
                    raise IRError(f"unknown assignment {op!r}")

    # kernel body
    if e_index is not None:
        body = top_loops[0][4]
        pre = [n for n in tree if n is not top_loops[0]]
    else:
        body, pre = tree, []
    if any(n[0] == "stmt" and n[1] in outputs for n in pre):
        raise IRError("output written outside the element loop")
    emit_nodes(pre, 1)
    if warp:
        lines.append(f"  const long i_{e_index} = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;")
        lines.append("  const int lane_ = threadIdx.x & 31;")
        lines.append(f"  if (i_{e_index} >= E) return;")
        for o in outputs:
            lines.append(f"  double a_{o}[{R * rest[o]}];")
            lines.append("  #pragma unroll")
            lines.append(f"  for (int x_ = 0; x_ < {R * rest[o]}; ++x_) a_{o}[x_] = 0.0;")
    elif e_index is not None:
        lines.append(f"  const long i_{e_index} = (long)blockIdx.x * blockDim.x + threadIdx.x;")
        lines.append(f"  if (i_{e_index} >= E) return;")
    else:
        lines.append("  if (blockIdx.x != 0 || threadIdx.x != 0) return;")
    emit_nodes(body, 1)
    if warp:  # the output += contract: one add per entry, rows contiguous
        for o in outputs:
            lines.append("  #pragma unroll")
            lines.append(f"  for (int r_ = 0; r_ < {R}; ++r_) {{")
            lines.append(f"    const long row_ = lane_ + 32 * r_;")
            lines.append(f"    if (row_ < {ext[J]}) {{")
            lines.append(f"      double* dst_ = o_{o} + (i_{e_index} * {ext[J]} + row_) * {rest[o]};")
            lines.append(f"      for (int x_ = 0; x_ < {rest[o]}; ++x_) dst_[x_] += a_{o}[r_ * {rest[o]} + x_];")
            lines.append("    }")
            lines.append("  }")

    decl = []
    for name in sorted(temps):
        idx = temps[name]
        if idx:
            if e_index in idx:
                raise IRError(f"temporary {name} indexed by the element loop")
            n = int(np.prod([ext[d] for d in idx]))
            decl.append(f"  double v_{_ident(name)}[{n}];")
        else:
            decl.append(f"  double v_{_ident(name)};")

    params = [f"double* __restrict__ o_{_ident(o)}" for o in outputs]
    params += [f"const double* __restrict__ t_{_ident(t)}" for t in inputs]
    params += [f"const double c_{_ident(c)}" for c in cnames]
    params.append("const long E")

    src = ["// generated by paper_1604_05872_b200.emit_cuda from a femopt kernel IR"]
    for name in preev:
        vals = np.asarray(tables[name]["values"], dtype=np.float64).reshape(-1)
        body_vals = ",".join(_lit(v) for v in vals)
        src.append(f"__device__ const double t_{_ident(name)}[{max(len(vals), 1)}] = {{{body_vals}}};")
    src.append(f'extern "C" __global__ void __launch_bounds__(128) {_ident(fn)}(' + ", ".join(params)
               + ") {")
    src += decl
    src += lines
    src.append("}")
    em = Emitted("\n".join(src) + "\n", fn, outputs, inputs, cnames, preev, e_index, ext, dims)
    em.strategy = strategy
    return em


# ----------------------------------------------------------------------------
# runtime: NVRTC -> cubin -> driver module (the context torch has made current)
# ----------------------------------------------------------------------------
def compile_cubin(source: str, name: str = "femopt_kernel.cu", arch: str = "sm_100a") -> bytes:
    """NVRTC: generated source -> sm_100a cubin (no FMA contraction, IEEE div/sqrt)."""
    from cuda.bindings import nvrtc

    err, prog = nvrtc.nvrtcCreateProgram(source.encode(), name.encode(), 0, [], [])
    if int(err) != 0:
        raise RuntimeError(f"nvrtcCreateProgram: {err}")
    opts = [f"--gpu-architecture={arch}".encode(), b"--fmad=false", b"--prec-div=true",
            b"--prec-sqrt=true", b"-std=c++17", b"-default-device"]
    (err,) = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
    if int(err) != 0:
        _, n = nvrtc.nvrtcGetProgramLogSize(prog)
        log = b" " * n
        nvrtc.nvrtcGetProgramLog(prog, log)
        raise RuntimeError("NVRTC compile failed:\n" + log.decode(errors="replace"))
    err, n = nvrtc.nvrtcGetCUBINSize(prog)
    if int(err) != 0:
        raise RuntimeError(f"nvrtcGetCUBINSize: {err}")
    cubin = b" " * n
    (err,) = nvrtc.nvrtcGetCUBIN(prog, cubin)
    if int(err) != 0:
        raise RuntimeError(f"nvrtcGetCUBIN: {err}")
    nvrtc.nvrtcDestroyProgram(prog)
    return cubin


class IRKernel:
    """A femopt IR compiled for the B200: ``run`` on device arrays, ``argv`` with
    emit_c's host calling convention (outputs accumulated with +=)."""

    BLOCK = 128

    def __init__(self, ir: dict | str, fn: str = "femopt_kernel", strategy: str = "auto"):
        self.em = emit(ir, fn, strategy)
        self.cubin = compile_cubin(self.em.source, fn + ".cu")
        self._func = None

    def _function(self):
        if self._func is None:
            import torch
            from cuda.bindings import driver as cu

            torch.cuda.init()
            torch.zeros(1, device="cuda")  # primary context current on this thread
            (err,) = cu.cuInit(0)
            if int(err) != 0:
                raise RuntimeError(f"cuInit: {err}")
            err, mod = cu.cuModuleLoadData(self.cubin)
            if int(err) != 0:
                raise RuntimeError(f"cuModuleLoadData: {err}")
            err, fn = cu.cuModuleGetFunction(mod, self.em.fn.encode())
            if int(err) != 0:
                raise RuntimeError(f"cuModuleGetFunction: {err}")
            self._mod, self._func = mod, fn
        return self._func

    def run(self, outputs: dict, inputs: dict, constants: dict | None, ncells: int,
            stream=None) -> None:
        """Device-resident run: ``outputs``/``inputs`` map names to CUDA tensors
        (float64, contiguous, sized for ``ncells``); outputs accumulate (+=)."""
        import ctypes

        import torch
        from cuda.bindings import driver as cu

        f = self._function()
        em = self.em
        constants = constants or {}
        vals, types = [], []
        for name in em.outputs:
            t = outputs[name]
            assert t.dtype == torch.float64 and t.is_cuda and t.is_contiguous()
            if t.numel() != em.size(name, ncells):
                raise ValueError(f"output {name}: {t.numel()} values, need {em.size(name, ncells)}")
            vals.append(t.data_ptr())
            types.append(ctypes.c_void_p)
        for name in em.inputs:
            t = inputs[name]
            assert t.dtype == torch.float64 and t.is_cuda and t.is_contiguous()
            if t.numel() != em.size(name, ncells):
                raise ValueError(f"input {name}: {t.numel()} values, need {em.size(name, ncells)}")
            vals.append(t.data_ptr())
            types.append(ctypes.c_void_p)
        for name in em.constants:
            vals.append(float(constants[name]))
            types.append(ctypes.c_double)
        vals.append(int(ncells))
        types.append(ctypes.c_long)
        n_threads = (ncells * (32 if em.strategy == "warp" else 1)) if em.e_index is not None else 1
        grid = max(1, (n_threads + self.BLOCK - 1) // self.BLOCK)
        s = torch.cuda.current_stream().cuda_stream if stream is None else (
            stream if isinstance(stream, int) else stream.cuda_stream)
        (err,) = cu.cuLaunchKernel(f, grid, 1, 1, self.BLOCK, 1, 1, 0, s,
                                   (tuple(vals), tuple(types)), 0)
        if int(err) != 0:
            raise RuntimeError(f"cuLaunchKernel: {err}")

    def argv(self, outputs: list, inputs: list, constants: list | None, ncells: int) -> None:
        """emit_c's calling convention on host numpy arrays: outputs (emit_c order)
        are accumulated into with +=, inputs/constants in emit_c order."""
        import torch

        dev = torch.device("cuda")
        o = {n: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).to(dev)
             for n, a in zip(self.em.outputs, outputs)}
        t = {n: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).to(dev)
             for n, a in zip(self.em.inputs, inputs)}
        c = dict(zip(self.em.constants, constants or []))
        self.run(o, t, c, ncells)
        torch.cuda.synchronize()
        for n, a in zip(self.em.outputs, outputs):
            a.reshape(-1)[:] = o[n].cpu().numpy()

    def run_ir_tables(self, ir: dict, outputs: dict | None = None) -> dict:
        """Run on the tables embedded in ``ir`` (femopt IRs carry their data);
        returns numpy outputs starting from zero (the reference's contract)."""
        import torch

        dev = torch.device("cuda")
        E = int(ir["indices"][self.em.e_index]) if self.em.e_index else 1
        tabs = ir.get("tables", {})
        t = {n: torch.tensor(np.asarray(tabs[n]["values"], dtype=np.float64), device=dev)
             for n in self.em.inputs}
        o = {n: torch.zeros(self.em.size(n, E), dtype=torch.float64, device=dev)
             for n in self.em.outputs}
        self.run(o, t, ir.get("constants", {}), E)
        torch.cuda.synchronize()
        return {n: v.cpu().numpy().reshape(self.em.shape(n, E)) for n, v in o.items()}
