"""Python mirror of the reference's coexec interface, bound to the native
B200 engine through include/ecl_engine.h.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/coexec/{core,schedulers,engine,metrics}.hpp so
the parity tests read like the reference's own Catch2 tests.  Everything
here is marshalling: validation, scheduling, the engine and the kernels run
in libcoexec.so / libecl_cuda.so.
"""
from __future__ import annotations

import ctypes
import enum
import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple, Union

import numpy as np

from . import _native as N

# ---------------------------------------------------------------------------
# errors (error.hpp:11-97)

ErrorCode = enum.Enum("ErrorCode", [(n, i) for i, n in enumerate(N.ERROR_NAMES)])


class Error(RuntimeError):
    """coexec::Error: carries an ErrorCode."""

    def __init__(self, code: ErrorCode, message: str):
        super().__init__(message)
        self.code = code


class EngineFailure(RuntimeError):
    """coexec::EngineFailure: every error of one run (has_errors/get_errors)."""

    def __init__(self, errors: List[Error]):
        super().__init__("engine failed: " + (str(errors[0]) if errors else ""))
        self.errors = errors

    def has(self, code: ErrorCode) -> bool:
        return any(e.code == code for e in self.errors)


def _raise(status: int, message: Optional[str] = None):
    raise Error(ErrorCode[N.code_name(status)], message if message is not None else N.last_error())


def _check(status: int):
    if status != 0:
        _raise(status)


# ---------------------------------------------------------------------------
# core types (core.hpp:14-237)

class BackendKind(enum.Enum):
    Simulated = "simulated"
    Cuda = "cuda"


@dataclass
class Backend:
    kind: BackendKind = BackendKind.Simulated
    ordinal: int = 0
    queue_depth: int = 2
    copy_split_items: int = 1 << 23
    widen_per_8: int = 8

    def to_json(self):
        if self.kind == BackendKind.Simulated:
            return {"kind": "simulated"}
        return {"kind": "cuda", "ordinal": self.ordinal, "queue_depth": self.queue_depth,
                "copy_split_items": self.copy_split_items, "widen_per_8": self.widen_per_8}


@dataclass
class DeviceProfile:
    id: str
    name: str = ""
    computing_power: float = 1.0
    launch_overhead_ms: float = 0.0
    bandwidth_bytes_per_ms: float = 1.0
    backend: Backend = field(default_factory=Backend)
    min_package_work_groups: int = 1
    kernel: str = ""  # per-device specialization "<kernel>@<variant>"; "" = the program's kernel

    def to_json(self):
        j = {"id": self.id, "name": self.name or self.id, "computing_power": self.computing_power,
             "launch_overhead_ms": self.launch_overhead_ms, "bandwidth_bytes_per_ms": self.bandwidth_bytes_per_ms,
             "backend": self.backend.to_json(), "min_package_work_groups": self.min_package_work_groups}
        if self.kernel:
            j["kernel"] = self.kernel
        return j

    @staticmethod
    def from_json(j) -> "DeviceProfile":
        b = j.get("backend", {"kind": "simulated"})
        backend = Backend(BackendKind(b["kind"]), b.get("ordinal", 0), b.get("queue_depth", 2),
                          b.get("copy_split_items", 1 << 23), b.get("widen_per_8", 8))
        return DeviceProfile(j["id"], j.get("name", j["id"]), j.get("computing_power", 1.0),
                             j.get("launch_overhead_ms", 0.0), j.get("bandwidth_bytes_per_ms", 1.0), backend,
                             j.get("min_package_work_groups", 0), j.get("kernel", ""))


def cuda_device(id: str, ordinal: int = 0, power: float = 1.0, queue_depth: int = 2,
                min_package_work_groups: int = 1, widen_per_8: int = 8,
                copy_split_items: int = 1 << 23, kernel: str = "") -> DeviceProfile:
    return DeviceProfile(id, id, power, 0.0, 1.0,
                         Backend(BackendKind.Cuda, ordinal, queue_depth, copy_split_items, widen_per_8),
                         min_package_work_groups, kernel)


def simulated_device(id: str, power: float, overhead_ms: float = 0.0, bandwidth: float = float(1 << 20),
                     min_wg: int = 1) -> DeviceProfile:
    return DeviceProfile(id, id, power, overhead_ms, bandwidth, Backend(), min_wg)


@dataclass
class BufferDesc:
    name: str
    element_size_bytes: int = 1
    element_count: int = 1

    def size_bytes(self) -> int:
        return self.element_size_bytes * self.element_count

    def to_json(self):
        return {"name": self.name, "element_size_bytes": self.element_size_bytes, "element_count": self.element_count}


@dataclass
class OutPattern:
    out_indices: int = 1
    work_items: int = 1


ArgValue = Union[int, float]


@dataclass
class ProgramSpec:
    global_work_size: int = 0
    local_work_size: int = 1
    in_buffers: List[BufferDesc] = field(default_factory=list)
    out_buffers: List[BufferDesc] = field(default_factory=list)
    out_pattern: OutPattern = field(default_factory=OutPattern)
    kernel: str = ""
    args: List[ArgValue] = field(default_factory=list)

    def to_json(self):
        return {"kernel": self.kernel, "global_work_size": self.global_work_size,
                "local_work_size": self.local_work_size,
                "out_pattern": {"out_indices": self.out_pattern.out_indices,
                                "work_items": self.out_pattern.work_items},
                "in_buffers": [b.to_json() for b in self.in_buffers],
                "out_buffers": [b.to_json() for b in self.out_buffers],
                "args": [a if isinstance(a, (int, np.integer)) and not isinstance(a, bool) else float(a)
                         for a in self.args]}


class ValidatedProgram:
    """A ProgramSpec that passed validate_program (core.hpp:91-143)."""

    def __init__(self, spec: ProgramSpec, total_wg: int):
        self._spec = spec
        self._total_wg = total_wg

    def spec(self) -> ProgramSpec:
        return self._spec

    def total_work_groups(self) -> int:
        return self._total_wg

    def global_work_size(self) -> int:
        return self._spec.global_work_size

    def local_work_size(self) -> int:
        return self._spec.local_work_size


def validate_program(spec: ProgramSpec) -> ValidatedProgram:
    total = ctypes.c_uint64(0)
    _check(N.lib.ecl_validate_program(json.dumps(spec.to_json()).encode(), ctypes.byref(total)))
    return ValidatedProgram(spec, total.value)


@dataclass
class Package:
    seq: int = 0
    device_index: int = 0
    device_id: str = ""
    offset_wg: int = 0
    size_wg: int = 0
    t_enqueue_ms: float = 0.0
    t_start_ms: float = 0.0
    t_end_ms: float = 0.0

    def end_wg(self) -> int:
        return self.offset_wg + self.size_wg


@dataclass
class OutRange:
    offset: int = 0
    count: int = 0


def out_range_for(pkg: Package, prog: ValidatedProgram) -> OutRange:
    off, cnt = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _check(N.lib.ecl_out_range_for(json.dumps(prog.spec().to_json()).encode(), pkg.offset_wg, pkg.size_wg,
                                   ctypes.byref(off), ctypes.byref(cnt)))
    return OutRange(off.value, cnt.value)


def tiles_exactly(packages: Sequence[Package], total_wg: int) -> bool:
    n = len(packages)
    offs = (ctypes.c_uint64 * max(1, n))(*[p.offset_wg for p in packages])
    sizes = (ctypes.c_uint64 * max(1, n))(*[p.size_wg for p in packages])
    return N.lib.ecl_tiles_exactly(offs, sizes, n, total_wg) == 1


class ClockMode(enum.Enum):
    Virtual = "virtual"
    Wall = "wall"


@dataclass
class ExecutionTrace:
    raw: dict

    @property
    def packages(self) -> List[Package]:
        return [Package(p["seq"], p["device_index"], p["device_id"], p["offset_wg"], p["size_wg"],
                        p["t_enqueue_ms"], p["t_start_ms"], p["t_end_ms"]) for p in self.raw["packages"]]

    @property
    def t_total_ms(self) -> float:
        return self.raw["t_total_ms"]

    @property
    def per_device_time_ms(self) -> Dict[str, float]:
        return self.raw["per_device_time_ms"]

    @property
    def scheduler(self) -> str:
        return self.raw["scheduler"]

    @property
    def init_ms(self) -> float:
        return self.raw["init_ms"]

    def to_json_string(self) -> str:
        return json.dumps(self.raw, indent=2)

    def to_csv(self) -> str:
        return _checked_string(N.lib.ecl_trace_csv, json.dumps(self.raw).encode())

    def to_svg(self) -> str:
        """The Introspector package chart (reference chart.hpp:52-154)."""
        return _checked_string(N.lib.ecl_chart_svg, json.dumps(self.raw).encode())


def _checked_string(fn, *args) -> str:
    s = N.read_string(fn, *args)
    if isinstance(s, int):
        _raise(s)
    return s


# ---------------------------------------------------------------------------
# experiment harness (experiment.hpp:67-181, config.hpp:159-195)

def run_experiment(config_path: str, scheduler: Optional[dict] = None, out_dir: Optional[str] = None,
                   exclude_init: Optional[bool] = None, write_traces: bool = True, write_csv: bool = False,
                   write_charts: bool = True, dump_pgm: bool = False) -> dict:
    """Runs an experiment file (solo baselines + scheduler matrix, warm-up
    discard, medians); writes traces / charts / summary.json under the
    output directory and returns the parsed summary (plus "summary_file")."""
    o: dict = {"write_traces": write_traces, "write_csv": write_csv, "write_charts": write_charts,
               "dump_pgm": dump_pgm}
    if scheduler is not None:
        o["scheduler"] = scheduler
    if out_dir is not None:
        o["out_dir"] = str(out_dir)
    if exclude_init is not None:
        o["exclude_init"] = bool(exclude_init)
    buf = ctypes.create_string_buffer(4096)
    rc = N.lib.ecl_experiment_run(str(config_path).encode(), json.dumps(o).encode(), buf, len(buf))
    if rc != 0:
        _raise(rc)
    path = buf.value.decode()
    with open(path) as f:
        summary = json.load(f)
    summary["summary_file"] = path
    return summary


def validate_experiment(config_path: str) -> str:
    """What `coexec validate` prints; raises Error on a bad file."""
    return _checked_string(N.lib.ecl_experiment_validate, str(config_path).encode())


# ---------------------------------------------------------------------------
# schedulers (schedulers.hpp:18-315)

@dataclass
class StaticConfig:
    proportions: List[float] = field(default_factory=list)
    device_order: List[str] = field(default_factory=list)

    def to_json(self):
        j = {"type": "static"}
        if self.proportions:
            j["proportions"] = [float(p) for p in self.proportions]
        if self.device_order:
            j["device_order"] = list(self.device_order)
        return j


@dataclass
class DynamicConfig:
    num_packages: int = 1

    def to_json(self):
        return {"type": "dynamic", "num_packages": self.num_packages}


@dataclass
class HGuidedConfig:
    k: float = 2.0
    powers: List[float] = field(default_factory=list)
    include_device_count: bool = True
    adaptive: bool = False
    ema_alpha: float = 0.5

    def to_json(self):
        j = {"type": "hguided", "k": float(self.k), "include_device_count": self.include_device_count}
        if self.powers:
            j["powers"] = [float(p) for p in self.powers]
        if self.adaptive:
            j["adaptive"] = True
            j["ema_alpha"] = float(self.ema_alpha)
        return j


SchedulerConfig = Union[StaticConfig, DynamicConfig, HGuidedConfig]


def describe(cfg: SchedulerConfig) -> str:
    return N.read_string(N.lib.ecl_describe_scheduler, json.dumps(cfg.to_json()).encode())


def resolve_static(cfg: StaticConfig, devices: Sequence[DeviceProfile]) -> StaticConfig:
    out = N.read_string(N.lib.ecl_resolve_static, json.dumps(cfg.to_json()).encode(),
                        json.dumps([d.to_json() for d in devices]).encode())
    if isinstance(out, int):
        _raise(out)
    j = json.loads(out)
    return StaticConfig(j["proportions"], j["device_order"])


def apply_default_min_package(devices: List[DeviceProfile]) -> None:
    out = N.read_string(N.lib.ecl_apply_default_min_package, json.dumps([d.to_json() for d in devices]).encode())
    if isinstance(out, int):
        _raise(out)
    for d, j in zip(devices, json.loads(out)):
        d.min_package_work_groups = j["min_package_work_groups"]


@dataclass
class PackageRange:
    offset_wg: int
    size_wg: int


class Scheduler:
    """The native scheduler behind the strategy seam (schedulers.hpp:178-183)."""

    def __init__(self, cfg: SchedulerConfig, total_wg: int, devices: Sequence[DeviceProfile]):
        h = ctypes.c_void_p()
        doc = {"scheduler": cfg.to_json(), "devices": [d.to_json() for d in devices], "total_work_groups": total_wg}
        _check(N.lib.ecl_scheduler_create(json.dumps(doc).encode(), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            N.lib.ecl_scheduler_destroy(self._h)
            self._h = None

    def next(self, device_index: int) -> Optional[PackageRange]:
        off, size = ctypes.c_uint64(0), ctypes.c_uint64(0)
        rc = N.lib.ecl_scheduler_next(self._h, device_index, ctypes.byref(off), ctypes.byref(size))
        if rc < 0:
            _raise(rc)
        return PackageRange(off.value, size.value) if rc == 1 else None

    def remaining_work_groups(self) -> int:
        return N.lib.ecl_scheduler_remaining(self._h)

    def observe(self, device: int, work_items: int, busy_ms: float) -> None:
        _check(N.lib.ecl_scheduler_observe(self._h, device, work_items, busy_ms))

    def unclamped_size(self, pending_wg: int, device: int) -> int:
        return N.lib.ecl_scheduler_unclamped(self._h, pending_wg, device)


def make_scheduler(cfg: SchedulerConfig, total_wg: int, devices: Sequence[DeviceProfile]) -> Scheduler:
    return Scheduler(cfg, total_wg, devices)


def static_partition(total_wg: int, resolved: StaticConfig, devices: Sequence[DeviceProfile]) -> List[Package]:
    """One package per device in delivery order (schedulers.hpp:131-168)."""
    s = Scheduler(resolved, total_wg, devices)
    ids = [d.id for d in devices]
    order = resolved.device_order or ids
    out = []
    for seq, dev_id in enumerate(order):
        i = ids.index(dev_id)
        r = s.next(i)
        out.append(Package(seq, i, dev_id, r.offset_wg, r.size_wg))
    out.sort(key=lambda p: p.offset_wg)
    for seq, p in enumerate(out):
        p.seq = seq
    return out


# ---------------------------------------------------------------------------
# metrics (metrics.hpp:19-164)

@dataclass
class MetricsReport:
    balance: float
    speedup: float
    s_max: float
    efficiency: float
    overhead_pct: Optional[float]
    work_share: Dict[str, float]
    notes: List[str]


def make_report(trace: ExecutionTrace, solo_times_ms: Sequence[float],
                reference_ms: Optional[float] = None) -> MetricsReport:
    solo = (ctypes.c_double * max(1, len(solo_times_ms)))(*solo_times_ms)
    out = N.read_string(N.lib.ecl_metrics_report, json.dumps(trace.raw).encode(), solo, len(solo_times_ms),
                        -1.0 if reference_ms is None else float(reference_ms))
    if isinstance(out, int):
        _raise(out)
    j = json.loads(out)
    return MetricsReport(j["balance"], j["speedup"], j["s_max"], j["efficiency"], j.get("overhead_pct"),
                         j["work_share"], j["notes"])


def balance(trace: ExecutionTrace) -> float:
    return make_report(trace, [max(trace.t_total_ms, 1e-300)]).balance


def overhead_pct(t_ms: float, t_reference_ms: float) -> float:
    if not t_reference_ms > 0.0:
        raise Error(ErrorCode.NonPositiveReference, "reference time must be > 0")
    return (t_ms - t_reference_ms) / t_reference_ms * 100.0


# ---------------------------------------------------------------------------
# engine (engine.hpp:21-446)

@dataclass
class EngineConfig:
    devices: List[DeviceProfile] = field(default_factory=list)
    scheduler: SchedulerConfig = field(default_factory=StaticConfig)
    clock_mode: ClockMode = ClockMode.Wall
    seed: int = 0
    exclude_init_from_total: bool = False
    tally: bool = False
    # One process per GPU: {"name": "/shm-name", "rank": r, "world": w, "local_devices": [r]}
    shared: Optional[dict] = None

    def to_json(self, program: ProgramSpec):
        j = {"schema": 1, "program": program.to_json(), "devices": [d.to_json() for d in self.devices],
             "scheduler": self.scheduler.to_json(), "clock_mode": self.clock_mode.value, "seed": self.seed,
             "exclude_init": self.exclude_init_from_total, "tally": self.tally}
        if self.shared:
            j["shared"] = dict(self.shared)
        return j


@dataclass
class RunResult:
    outputs: List[np.ndarray]
    trace: ExecutionTrace


def _as_buffer(a) -> Tuple[int, int]:
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("buffers must be C-contiguous")
        return a.ctypes.data, a.nbytes
    if isinstance(a, (bytes, bytearray)):
        arr = np.frombuffer(a, dtype=np.uint8)
        return arr.ctypes.data, arr.nbytes
    raise TypeError(f"unsupported buffer type {type(a)}")


class Engine:
    """coexec::Engine on B200s.  Construction opens the devices, allocates
    each device's buffer partition and starts one host thread per device."""

    def __init__(self, cfg: EngineConfig, prog: ValidatedProgram):
        self._cfg = cfg
        self._prog = prog
        h = ctypes.c_void_p()
        rc = N.lib.ecl_engine_create(json.dumps(cfg.to_json(prog.spec())).encode(), ctypes.byref(h))
        if rc != 0:
            _raise(rc)
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            N.lib.ecl_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def program(self) -> ValidatedProgram:
        return self._prog

    def init_ms(self) -> float:
        return N.lib.ecl_engine_init_ms(self._h)

    def _fail(self, rc: int):
        n = N.lib.ecl_engine_error_count(self._h)
        if n == 0:
            _raise(rc)
        errors = []
        for i in range(n):
            st = ctypes.c_int(0)
            msg = N.read_string(N.lib.ecl_engine_error, self._h, i, ctypes.byref(st))
            errors.append(Error(ErrorCode[N.code_name(st.value)], msg if isinstance(msg, str) else ""))
        raise EngineFailure(errors)

    def _check_inputs(self, inputs):
        """inputs=None reuses the replicas already resident on the devices."""
        if inputs is None:
            return []
        bufs = self._prog.spec().in_buffers
        if len(inputs) != len(bufs):
            raise Error(ErrorCode.InputSizeMismatch, f"expected {len(bufs)} input buffers, got {len(inputs)}")
        ptrs = []
        for b, a in zip(bufs, inputs):
            p, n = _as_buffer(a)
            if n != b.size_bytes():
                raise Error(ErrorCode.InputSizeMismatch,
                            f"input '{b.name}' is {n} bytes, descriptor says {b.size_bytes()}")
            ptrs.append(p)
        return ptrs

    def _check_outputs(self, outputs: Sequence) -> List[int]:
        """Every output must be a writable, C-contiguous buffer of exactly the
        descriptor's size: the native side writes spec-sized slices."""
        outs = self._prog.spec().out_buffers
        if len(outputs) != len(outs):
            raise Error(ErrorCode.ConfigError, f"expected {len(outs)} output buffers, got {len(outputs)}")
        ptrs = []
        for b, a in zip(outs, outputs):
            if a is None:
                ptrs.append(None)
                continue
            if isinstance(a, bytes) or (isinstance(a, np.ndarray) and not a.flags["WRITEABLE"]):
                raise Error(ErrorCode.ConfigError, f"output '{b.name}' must be a writable buffer")
            p, n = _as_buffer(a)
            if n != b.size_bytes():
                raise Error(ErrorCode.ConfigError, f"output '{b.name}' must be {b.size_bytes()} bytes, got {n}")
            ptrs.append(p)
        return ptrs

    def allocate_outputs(self) -> List[np.ndarray]:
        return [np.zeros(b.size_bytes(), dtype=np.uint8) for b in self._prog.spec().out_buffers]

    def run_into(self, inputs: Sequence, outputs: Optional[Sequence[np.ndarray]],
                 want_trace: bool = True, kernel: Optional[str] = None) -> Optional[ExecutionTrace]:
        """Caller-owned buffers; outputs=None keeps the results device-resident.
        want_trace=False skips serializing the trace (last_trace() has it).
        kernel: run this device kernel id (built-in or register_kernel'ed)
        instead of the program's, for this run only."""
        in_ptrs = self._check_inputs(inputs)
        in_arr = N.pointer_array(in_ptrs)
        out_ptrs = self._check_outputs(outputs) if outputs is not None else []
        out_arr = N.pointer_array(out_ptrs) if outputs is not None else None
        if kernel is None:
            rc = N.lib.ecl_engine_run(self._h, in_arr, len(in_ptrs), out_arr, len(out_ptrs))
        else:
            rc = N.lib.ecl_engine_run_kernel(self._h, kernel.encode(), in_arr, len(in_ptrs), out_arr,
                                             len(out_ptrs))
        if rc != 0:
            self._fail(rc)
        return self.last_trace() if want_trace else None

    def run_steps(self, inputs: Sequence, outputs: Optional[Sequence[np.ndarray]], steps: int,
                  swaps: Sequence[Tuple[int, int]], want_trace: bool = True) -> Optional[ExecutionTrace]:
        """Iterative program: `steps` passes; between passes each (input i,
        output o) pair is exchanged across devices and swapped in place."""
        in_ptrs = self._check_inputs(inputs)
        out_ptrs = self._check_outputs(outputs) if outputs is not None else []
        si = (ctypes.c_uint32 * max(1, len(swaps)))(*[a for a, _ in swaps])
        so = (ctypes.c_uint32 * max(1, len(swaps)))(*[b for _, b in swaps])
        rc = N.lib.ecl_engine_run_steps(self._h, N.pointer_array(in_ptrs), len(in_ptrs),
                                        N.pointer_array(out_ptrs) if out_ptrs else None, len(out_ptrs), steps, si, so,
                                        len(swaps))
        if rc != 0:
            self._fail(rc)
        return self.last_trace() if want_trace else None

    def run(self, inputs: Sequence = (), kernel: Optional[str] = None, cost=None) -> RunResult:
        """Reference semantics: engine-allocated outputs (engine.hpp:219-256).
        run(inputs, kernel, cost) is the reference's plugin overload
        (engine.hpp:223): `kernel` is a device kernel id (built-in or
        register_kernel'ed) run instead of the program's; `cost` (a per-item
        function) is the virtual clock's model and unused by a wall run.
        A virtual-clock engine has no outputs to return (kernels never run on
        the CPU here): it raises ConfigError and run_virtual() gives the trace."""
        if self._cfg.clock_mode == ClockMode.Virtual:
            raise Error(ErrorCode.ConfigError,
                        "virtual clock mode produces a trace only: call run_virtual(); outputs need a wall-clock "
                        "engine on cuda devices")
        outputs = self.allocate_outputs()
        trace = self.run_into(inputs, outputs, kernel=kernel)
        return RunResult(outputs, trace)

    def run_virtual(self, item_costs) -> ExecutionTrace:
        """item_costs: one cost per work-item, a per-item cost function (the
        reference's CostFn), or None for vecscale/synthetic's analytic costs."""
        if callable(item_costs):
            gws = self._prog.global_work_size()
            item_costs = np.array([item_costs(i) for i in range(gws)], dtype=np.float64)
        if item_costs is None:
            rc = N.lib.ecl_engine_run_virtual(self._h, None, 0)
        else:
            c = np.ascontiguousarray(item_costs, dtype=np.float64)
            rc = N.lib.ecl_engine_run_virtual(self._h, c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), c.size)
        if rc != 0:
            self._fail(rc)
        return self.last_trace()

    def gather(self, outputs: Sequence[np.ndarray]) -> None:
        ptrs = self._check_outputs(outputs)
        rc = N.lib.ecl_engine_gather(self._h, N.pointer_array(ptrs), len(ptrs))
        if rc != 0:
            self._fail(rc)

    def native_run(self, inputs: Sequence = (), outputs: Optional[Sequence[np.ndarray]] = None):
        """One launch over the whole grid: returns (kernel_ms, total_ms)."""
        in_ptrs = self._check_inputs(inputs)
        out_ptrs = self._check_outputs(outputs) if outputs is not None else []
        k, t = ctypes.c_double(0), ctypes.c_double(0)
        rc = N.lib.ecl_engine_native_run(self._h, N.pointer_array(in_ptrs), len(in_ptrs),
                                         N.pointer_array(out_ptrs) if out_ptrs else None, len(out_ptrs),
                                         ctypes.byref(k), ctypes.byref(t))
        if rc != 0:
            self._fail(rc)
        return k.value, t.value

    def native_run_split(self, items_per_launch: int) -> float:
        """The same grid as plain sub-launches of `items_per_launch`
        work-items over the first device's two compute streams (resident
        outputs): kernel span in ms."""
        k = ctypes.c_double(0)
        rc = N.lib.ecl_engine_native_run_split(self._h, int(items_per_launch), ctypes.byref(k))
        if rc != 0:
            self._fail(rc)
        return k.value

    def kernel_timing(self, reset: bool = False) -> Tuple[float, int]:
        ms, n = ctypes.c_double(0), ctypes.c_uint64(0)
        _check(N.lib.ecl_engine_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(n), 1 if reset else 0))
        return ms.value, n.value

    def learned_powers(self) -> List[float]:
        """Adaptive HGuided: work-items/ms per device measured by the last run
        (the next run's seeds); [] before a run measured every device."""
        cap = len(self._cfg.devices)
        buf = (ctypes.c_double * max(1, cap))()
        n = ctypes.c_uint32(0)
        _check(N.lib.ecl_engine_learned_powers(self._h, buf, cap, ctypes.byref(n)))
        return [buf[i] for i in range(min(n.value, cap))]

    def last_trace(self) -> ExecutionTrace:
        s = N.read_string(N.lib.ecl_engine_trace_json, self._h)
        if isinstance(s, int):
            _raise(s)
        return ExecutionTrace(json.loads(s))


def run(cfg: EngineConfig, prog: ValidatedProgram, inputs: Sequence = ()) -> RunResult:
    with Engine(cfg, prog) as e:
        return e.run(inputs)


def host_register(a: np.ndarray) -> None:
    """Page-locks a host buffer so per-package D2H copies run async."""
    p, n = _as_buffer(a)
    rc = N.lib.ecl_host_register(p, n)
    if rc != 0:
        raise Error(ErrorCode[N.code_name(rc)], N.device_last_error())


def host_unregister(a: np.ndarray) -> None:
    p, _ = _as_buffer(a)
    N.lib.ecl_host_unregister(p)


class PinnedBuffer:
    """Page-locked host memory (cudaHostAlloc) viewed as a numpy array."""

    def __init__(self, nbytes: int, dtype=np.uint8):
        p = ctypes.c_void_p()
        rc = N.lib.ecl_host_alloc(nbytes, ctypes.byref(p))
        if rc != 0:
            raise Error(ErrorCode[N.code_name(rc)], N.device_last_error())
        self._ptr = p
        raw = (ctypes.c_uint8 * nbytes).from_address(p.value)
        self.array = np.frombuffer(raw, dtype=np.uint8).view(dtype)

    def free(self):
        if getattr(self, "_ptr", None):
            self.array = None
            lib = getattr(N, "lib", None)
            if lib is not None:  # at interpreter exit the module may already be torn down
                lib.ecl_host_free(self._ptr)
            self._ptr = None

    def __del__(self):
        self.free()


def register_kernel(kernel_id: str, image, entry: str) -> str:
    """Registers a device kernel compiled for sm_100a (include/ecl_plugin.h
    ABI) under `kernel_id`: `image` is the cubin / fatbin / PTX bytes or a
    path to such a file.  Returns the id (usable as a program's kernel, a
    per-device kernel, or Engine.run(kernel=...))."""
    if isinstance(image, str) or hasattr(image, "__fspath__"):
        with open(image, "rb") as f:
            image = f.read()
    data = bytes(image) + b"\0"  # PTX is read up to its NUL
    buf = ctypes.create_string_buffer(data, len(data))
    rc = N.lib.ecl_kernel_register(kernel_id.encode(), buf, len(data) - 1, entry.encode())
    if rc != 0:
        raise Error(ErrorCode[N.code_name(rc)], N.device_last_error())
    return kernel_id


def unregister_kernel(kernel_id: str) -> None:
    rc = N.lib.ecl_kernel_unregister(kernel_id.encode())
    if rc != 0:
        raise Error(ErrorCode[N.code_name(rc)], N.device_last_error())


def is_registered_kernel(kernel_id: str) -> bool:
    return N.lib.ecl_kernel_is_plugin(kernel_id.encode()) == 1


def gpu_count() -> int:
    return N.gpu_count()
