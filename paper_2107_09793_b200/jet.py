"""Thin ctypes binding of libjetb200 (include/jetb200.h): argument marshalling only.

Every step of the hot path runs inside the library's CUDA kernels; PyTorch provides
device memory (the workspace) and the stream.  There is no CPU fallback: importing this
module fails loudly if the in-tree ``libjetb200.so`` is missing.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libjetb200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the CUDA extension is required; there is no fallback path)")

_lib = ctypes.CDLL(LIB_PATH)

JT_C64, JT_C128 = 0, 1
_DT = {"c64": JT_C64, "complex64": JT_C64, "c128": JT_C128, "complex128": JT_C128}

c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_i32 = ctypes.POINTER(c_i32)
P_i64 = ctypes.POINTER(c_i64)
P_dbl = ctypes.POINTER(c_dbl)


class PlannerOpts(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("trials", c_i32), ("threads", c_i32), ("n_sliced", c_i32),
                ("width_cap", c_i32), ("reconf_sweeps", c_i32), ("reconf_leaves", c_i32),
                ("time_budget_s", c_dbl), ("bytes_weight", c_dbl), ("candidates", c_i32),
                ("model_hbm_gbs", c_dbl), ("model_cuda_tflops", c_dbl), ("model_tc_tflops", c_dbl),
                ("model_launch_us", c_dbl), ("model_esize", c_dbl), ("slice_objective", c_i32),
                ("partition", c_i32)]


class Cost(ctypes.Structure):
    _fields_ = [("n_sl", c_i64), ("flop_sl", c_dbl), ("flop_shared", c_dbl), ("e_flsl", c_dbl),
                ("e_fltask", c_dbl), ("exact_reuse", c_dbl), ("prefix", c_dbl), ("max_width", c_dbl),
                ("bytes_sl", c_dbl), ("n_steps", c_i64), ("n_sliced", c_i32), ("n_batch", c_i64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ExecStats(ctypes.Structure):
    _fields_ = [("slices_done", c_i64), ("node_launches", c_i64), ("kernel_launches", c_i64),
                ("flop_executed", c_dbl), ("bytes_executed", c_dbl), ("k2_time_ms", c_dbl),
                ("k2_timed_launches", c_i64), ("k2_timed_bytes", c_dbl), ("k2_timed_flop", c_dbl),
                ("k3_time_ms", c_dbl), ("k3_timed_launches", c_i64), ("k3_timed_bytes", c_dbl),
                ("k3_timed_flop", c_dbl), ("h2d_bytes", c_i64),
                ("k4_time_ms", c_dbl), ("k4_timed_launches", c_i64), ("k4_timed_bytes", c_dbl),
                ("k4_timed_flop", c_dbl), ("k3g_time_ms", c_dbl), ("k3g_timed_launches", c_i64),
                ("k3g_timed_bytes", c_dbl), ("k3g_timed_flop", c_dbl), ("k2s_time_ms", c_dbl),
                ("k2s_timed_launches", c_i64), ("k2s_timed_bytes", c_dbl), ("k2s_timed_flop", c_dbl)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("jt_last_error", ctypes.c_char_p, [])
_sig("jt_version", ctypes.c_char_p, [])
_sig("jt_network_create", c_i32, [c_i32, c_i32, ctypes.POINTER(c_vp)])
_sig("jt_network_add_gate", c_i32, [c_vp, c_i32, P_i32, P_dbl])
_sig("jt_network_close", c_i32, [c_vp, P_i32])
_sig("jt_network_close_batch", c_i32, [c_vp, P_i32, P_i32, c_i32])
_sig("jt_network_info", c_i32, [c_vp, P_i64, P_i64])
_sig("jt_network_export", c_i32, [c_vp, ctypes.c_char_p])
_sig("jt_network_destroy", None, [c_vp])
_sig("jt_plan_create", c_i32, [c_vp, P_i64, c_i64, P_i64, c_i32, ctypes.POINTER(c_vp)])
_sig("jt_plan_greedy", c_i32, [c_vp, ctypes.POINTER(PlannerOpts), ctypes.POINTER(c_vp)])
_sig("jt_plan_sizes", c_i32, [c_vp, P_i64, P_i32])
class Memory(ctypes.Structure):
    _fields_ = [("total_bytes", c_i64), ("leaf_bytes", c_i64), ("arena_bytes", c_i64), ("peak_live_bytes", c_i64),
                ("no_deletion_bytes", c_i64), ("cache_bytes", c_i64), ("peak_live_noshare_bytes", c_i64),
                ("scratch_bytes", c_i64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_sig("jt_plan_slice", c_i32, [c_vp, P_i64, c_i64, ctypes.POINTER(PlannerOpts), ctypes.POINTER(c_vp)])
_sig("jt_plan_get", c_i32, [c_vp, P_i64, P_i64])
_sig("jt_plan_cost", c_i32, [c_vp, ctypes.POINTER(Cost)])
_sig("jt_plan_prefix_flop", c_i32, [c_vp, c_i64, c_i64, P_dbl])
_sig("jt_plan_export", c_i32, [c_vp, ctypes.c_char_p])
_sig("jt_plan_destroy", None, [c_vp])
_sig("jt_exec_workspace_bytes", c_i32, [c_vp, c_i32, P_i64])
_sig("jt_exec_describe", c_i32, [c_vp, c_i32, ctypes.c_char_p])
_sig("jt_exec_memory", c_i32, [c_vp, c_i32, ctypes.POINTER(Memory)])
_sig("jt_exec_create", c_i32, [c_vp, c_i32, c_i32, c_vp, c_i64, c_vp, ctypes.POINTER(c_vp)])
_sig("jt_exec_contract", c_i32, [c_vp, c_i64, c_i64, c_vp, P_dbl])
_sig("jt_exec_contract_noreuse", c_i32, [c_vp, c_i64, c_i64, c_vp, P_dbl])
_sig("jt_exec_contract_host", c_i32, [c_vp, c_i64, c_i64, P_dbl])
_sig("jt_exec_stats_get", c_i32, [c_vp, ctypes.POINTER(ExecStats)])
_sig("jt_exec_upload_leaves", c_i32, [c_vp])
_sig("jt_exec_set_profiling", c_i32, [c_vp, c_i32])
_sig("jt_exec_stats_reset", c_i32, [c_vp])
_sig("jt_exec_invalidate", c_i32, [c_vp])
_sig("jt_exec_destroy", None, [c_vp])
_sig("jt_debug_emulate_host", c_i32, [c_vp, c_i32, c_i64, c_i64, P_dbl, c_i32])
_sig("jt_debug_time_node", c_i32, [c_vp, c_i64, c_i32, P_dbl, P_dbl, P_dbl, P_i32])
_sig("jt_amplitude", c_i32, [c_vp, c_i32, c_i32, P_dbl])
_sig("jt_permute", c_i32, [c_i32, c_vp, c_vp, c_i32, P_i32, c_vp])

EXPORTED = ["jt_last_error", "jt_version", "jt_network_create", "jt_network_add_gate", "jt_network_close",
            "jt_network_close_batch", "jt_network_info", "jt_network_export", "jt_network_destroy", "jt_plan_create", "jt_plan_greedy", "jt_plan_slice",
            "jt_plan_sizes", "jt_plan_get", "jt_plan_cost", "jt_plan_prefix_flop", "jt_plan_export",
            "jt_plan_destroy", "jt_exec_workspace_bytes", "jt_exec_describe", "jt_exec_memory", "jt_exec_create", "jt_exec_contract",
            "jt_exec_contract_noreuse", "jt_exec_contract_host", "jt_exec_stats_get",
            "jt_exec_upload_leaves", "jt_exec_set_profiling", "jt_exec_stats_reset",
            "jt_exec_invalidate", "jt_exec_destroy", "jt_amplitude", "jt_permute", "jt_debug_emulate_host",
            "jt_debug_time_node"]


class JetError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[jt status {code}] {msg}")
        self.code = code


def _check(st):
    if st != 0:
        raise JetError(st, _lib.jt_last_error().decode())


def version():
    return _lib.jt_version().decode()


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(P_i32)


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(P_i64)


class Network:
    """jt_network: circuit -> closed tensor network."""

    def __init__(self, n_wires, d):
        h = c_vp()
        _check(_lib.jt_network_create(n_wires, d, ctypes.byref(h)))
        self._h = h
        self.n_wires, self.d = n_wires, d
        self.open_wires = ()

    @classmethod
    def from_circuit(cls, circuit, bitstring, open_wires=None):
        """open_wires: batch of amplitudes over these wires (jt_network_close_batch)."""
        net = cls(circuit.n_wires, circuit.d)
        for g in circuit.gates:
            net.add_gate(g.wires, g.u)
        if open_wires is None:
            net.close(bitstring)
        else:
            net.close_batch(bitstring, open_wires)
        return net

    def add_gate(self, wires, u):
        w, wp = _i32(list(wires))
        u = np.ascontiguousarray(np.asarray(u, dtype=np.complex128))
        ud = u.view(np.float64)
        _check(_lib.jt_network_add_gate(self._h, len(w), wp, ud.ctypes.data_as(P_dbl)))

    def close(self, bits):
        b, bp = _i32(list(bits))
        _check(_lib.jt_network_close(self._h, bp))
        self.open_wires = ()

    def close_batch(self, bits, open_wires):
        b, bp = _i32(list(bits))
        o, op = _i32(list(open_wires))
        _check(_lib.jt_network_close_batch(self._h, bp, op, len(o)))
        self.open_wires = tuple(int(w) for w in open_wires)

    def info(self):
        nt, nl = c_i64(), c_i64()
        _check(_lib.jt_network_info(self._h, ctypes.byref(nt), ctypes.byref(nl)))
        return nt.value, nl.value

    def export(self, path):
        _check(_lib.jt_network_export(self._h, path.encode()))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.jt_network_destroy(self._h)
            self._h = None


class Plan:
    """jt_plan: SSA contraction path + sliced labels."""

    def __init__(self, handle, net):
        self._h = handle
        self.net = net

    @classmethod
    def create(cls, net, ssa_path, sliced_labels=()):
        p = np.asarray(ssa_path, dtype=np.int64).reshape(-1)
        pa, pp = _i64(p)
        s, sp = _i64(list(sliced_labels))
        h = c_vp()
        _check(_lib.jt_plan_create(net._h, pp, len(pa) // 2, sp, len(s), ctypes.byref(h)))
        return cls(h, net)

    @classmethod
    def greedy(cls, net, seed=1, trials=64, threads=0, n_sliced=0, width_cap=0, reconf_sweeps=-1,
               reconf_leaves=0, time_budget_s=0.0, bytes_weight=0.0, candidates=0, model=None,
               slice_objective=0, partition=0):
        """jt_plan_greedy.  slice_objective: 0 = sliced cost, 1 = shared-work aware (executed
        prefix-cache cost)."""
        m = model or {}
        o = PlannerOpts(seed, trials, threads, n_sliced, width_cap, reconf_sweeps, reconf_leaves, time_budget_s,
                        bytes_weight, candidates, m.get("hbm_gbs", 0.0), m.get("cuda_tflops", 0.0),
                        m.get("tc_tflops", 0.0), m.get("launch_us", 0.0), m.get("esize", 0.0), slice_objective,
                        partition)
        h = c_vp()
        _check(_lib.jt_plan_greedy(net._h, ctypes.byref(o), ctypes.byref(h)))
        return cls(h, net)

    @classmethod
    def slice_path(cls, net, ssa_path, n_sliced=0, width_cap=0, bytes_weight=0.0, slice_objective=1):
        """jt_plan_slice: greedy slicing along a FIXED path, by default choosing
        the labels that maximise shared work (the executed prefix-cache cost)."""
        p = np.asarray(ssa_path, dtype=np.int64).reshape(-1)
        o = PlannerOpts(0, 0, 0, n_sliced, width_cap, -1, 0, 0.0, bytes_weight, 0, 0.0, 0.0, 0.0, 0.0, 0.0,
                        slice_objective, 0)
        h = c_vp()
        _check(_lib.jt_plan_slice(net._h, p.ctypes.data_as(P_i64), len(p) // 2, ctypes.byref(o), ctypes.byref(h)))
        return cls(h, net)

    def sizes(self):
        ns, nk = c_i64(), c_i32()
        _check(_lib.jt_plan_sizes(self._h, ctypes.byref(ns), ctypes.byref(nk)))
        return ns.value, nk.value

    @property
    def ssa_path(self):
        ns, nk = self.sizes()
        p = np.zeros(2 * ns, dtype=np.int64)
        s = np.zeros(max(nk, 1), dtype=np.int64)
        _check(_lib.jt_plan_get(self._h, p.ctypes.data_as(P_i64), s.ctypes.data_as(P_i64)))
        return [(int(p[2 * i]), int(p[2 * i + 1])) for i in range(ns)]

    @property
    def sliced_labels(self):
        ns, nk = self.sizes()
        p = np.zeros(max(2 * ns, 1), dtype=np.int64)
        s = np.zeros(max(nk, 1), dtype=np.int64)
        _check(_lib.jt_plan_get(self._h, p.ctypes.data_as(P_i64), s.ctypes.data_as(P_i64)))
        return [int(x) for x in s[:nk]]

    def cost(self):
        c = Cost()
        _check(_lib.jt_plan_cost(self._h, ctypes.byref(c)))
        return c.as_dict()

    def prefix_flop(self, begin, end):
        f = c_dbl()
        _check(_lib.jt_plan_prefix_flop(self._h, begin, end, ctypes.byref(f)))
        return f.value

    def export(self, path):
        _check(_lib.jt_plan_export(self._h, path.encode()))

    def workspace_bytes(self, dtype="c64"):
        b = c_i64()
        _check(_lib.jt_exec_workspace_bytes(self._h, _DT[dtype], ctypes.byref(b)))
        return b.value

    def memory(self, dtype="c64"):
        """jt_exec_memory: workspace, peak live, no-deletion and prefix-cache bytes (fig. m10_memory)."""
        m = Memory()
        _check(_lib.jt_exec_memory(self._h, _DT[dtype], ctypes.byref(m)))
        return m.as_dict()

    def concurrent_slices(self, budget_bytes, dtype="c64"):
        """How many slice subsets (executors sharing the read-only leaves) fit in budget_bytes of
        device memory, decided a priori from the memory report."""
        m = self.memory(dtype)
        per = m["total_bytes"] - m["leaf_bytes"]
        return max(0, (budget_bytes - m["leaf_bytes"]) // per) if per > 0 else 0

    def describe_exec(self, dtype="c64"):
        import json
        import tempfile

        with tempfile.NamedTemporaryFile(suffix=".json") as f:
            _check(_lib.jt_exec_describe(self._h, _DT[dtype], f.name.encode()))
            return json.load(open(f.name))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.jt_plan_destroy(self._h)
            self._h = None


class Exec:
    """jt_exec on one GPU; the workspace is a torch uint8 tensor owned by this object."""

    def __init__(self, plan, dtype="c64", device=None, stream=None, workspace=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("Exec needs a CUDA device (no CPU fallback)")
        self.plan = plan
        self.dtype = dtype
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        nbytes = plan.workspace_bytes(dtype)
        if workspace is None:
            workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        assert workspace.numel() >= nbytes
        self.ws = workspace
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        h = c_vp()
        _check(_lib.jt_exec_create(plan._h, _DT[dtype], dev.index, c_vp(workspace.data_ptr()), workspace.numel(),
                                   c_vp(self.stream.cuda_stream), ctypes.byref(h)))
        self._h = h

    def contract(self, begin, end, acc, slice_values=False, reuse=True):
        """acc: torch float64 CUDA tensor with 2 entries (complex128), += sum s_sigma."""
        vals = np.zeros(2 * max(end - begin, 1), dtype=np.float64) if slice_values else None
        vp = vals.ctypes.data_as(P_dbl) if slice_values else None
        fn = _lib.jt_exec_contract if reuse else _lib.jt_exec_contract_noreuse
        _check(fn(self._h, begin, end, c_vp(acc.data_ptr()), vp))
        if slice_values:
            return vals[: 2 * (end - begin)].view(np.complex128)
        return None

    def contract_host(self, begin, end):
        """Sum of runs [begin, end) on the host: a complex, or n_batch complex for batch plans."""
        nb = self.plan.cost()["n_batch"]
        out = np.zeros(2 * nb, dtype=np.float64)
        _check(_lib.jt_exec_contract_host(self._h, begin, end, out.ctypes.data_as(P_dbl)))
        return complex(out[0], out[1]) if nb == 1 and not self.plan.net.open_wires else out.view(np.complex128)

    def stats(self):
        s = ExecStats()
        _check(_lib.jt_exec_stats_get(self._h, ctypes.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        _check(_lib.jt_exec_stats_reset(self._h))

    def upload_leaves(self):
        _check(_lib.jt_exec_upload_leaves(self._h))

    def set_profiling(self, on=True):
        _check(_lib.jt_exec_set_profiling(self._h, 1 if on else 0))

    def time_node(self, order_index, reps=5):
        """DEBUG: mean ms per launch of one node (see jetb200.h)."""
        ms, by, fl, kd = c_dbl(), c_dbl(), c_dbl(), c_i32()
        _check(_lib.jt_debug_time_node(self._h, order_index, reps, ctypes.byref(ms), ctypes.byref(by),
                                       ctypes.byref(fl), ctypes.byref(kd)))
        return {"ms": ms.value, "bytes": by.value, "flop": fl.value, "kind": kd.value}

    def invalidate(self):
        _check(_lib.jt_exec_invalidate(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.jt_exec_destroy(self._h)
            self._h = None


def debug_emulate_host(plan, begin, end, dtype="c128", reuse=True):
    """TEST ONLY: the compiled launch descriptors executed on the host (see jetb200.h)."""
    vals = np.zeros(2 * max(end - begin, 1), dtype=np.float64)
    _check(_lib.jt_debug_emulate_host(plan._h, _DT[dtype], begin, end, vals.ctypes.data_as(P_dbl), 1 if reuse else 0))
    return vals[: 2 * (end - begin)].view(np.complex128)


def amplitude(plan, dtype="c64", device=0):
    """<x|U|0> (complex), or the batch of n_batch amplitudes (complex128 array, y-indexed)."""
    nb = plan.cost()["n_batch"]
    out = np.zeros(2 * nb, dtype=np.float64)
    _check(_lib.jt_amplitude(plan._h, _DT[dtype], device, out.ctypes.data_as(P_dbl)))
    return complex(out[0], out[1]) if nb == 1 and not plan.net.open_wires else out.view(np.complex128)


def permute(src, perm, out=None):
    """K1: dst[pi(i)] = src[i] for a 2^n complex CUDA tensor; address bit b -> bit perm[b]."""
    import torch

    n = len(perm)
    assert src.numel() == 1 << n and src.is_cuda and src.is_contiguous()
    dt = {torch.complex64: JT_C64, torch.complex128: JT_C128}[src.dtype]
    if out is None:
        out = torch.empty_like(src)
    p, pp = _i32(list(perm))
    _check(_lib.jt_permute(dt, c_vp(src.data_ptr()), c_vp(out.data_ptr()), n, pp,
                           c_vp(torch.cuda.current_stream(src.device).cuda_stream)))
    return out
