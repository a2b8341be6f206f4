"""ctypes binding of include/cel.h (argument marshalling only).

Every step of the coherence path runs inside libcel.so (C++ scheduler +
sm_100a kernels).  There is no fallback: if the library is missing this
module raises at import, and creating an executing runtime without a GPU
fails with CEL_E_CUDA.
"""

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcel.so")
if not os.path.exists(LIB_PATH):
    raise ImportError("libcel.so not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
lib = C.CDLL(LIB_PATH)

OK, W_UNINIT_READ = 0, 1
E_INVALID, E_OUT_OF_BOUNDS, E_OVERLAPPING_WRITE, E_OOM, E_CUDA, E_NCCL, E_STATE = -1, -2, -3, -4, -5, -6, -7

MAPPERS = {"one_to_one": 0, "neighborhood": 1, "all": 2, "fixed": 3, "remap": 4, "neighborhood_axes": 5}
MODES = {"read": 1, "write": 2, "read_write": 3}
SPLITS = {"1d": 0, "2d": 1}
KERNELS = {"fill_hash": 0, "fill_const": 1, "stencil3": 2, "wave5": 3, "jacobi7": 4, "nbody_step": 5,
           "nbody_update": 6, "rsim_row": 7, "probe": 8, "callback": 9}
KERNEL_NAMES = {v: k for k, v in KERNELS.items()}
PROFILE_SLOTS = 14       # kernel kinds 0..9, copy within a GPU (10), peer push (11), stencil shell launches (12),
                         # NCCL all-gather groups (13)
COPY_SLOT = 10
PEER_SLOT = 11
SHELL_SLOT = 12
COLL_SLOT = 13


class cel_box(C.Structure):
    _fields_ = [("min", C.c_uint64 * 3), ("max", C.c_uint64 * 3)]


class cel_range_mapper(C.Structure):
    _fields_ = [("kind", C.c_int32), ("border", C.c_uint32 * 3), ("fixed", cel_box),
                ("from_kernel_dim", C.c_int32 * 3)]


class cel_access(C.Structure):
    _fields_ = [("buf", C.c_uint32), ("mode", C.c_int32), ("map", cel_range_mapper)]


class cel_kernel_params(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("value", C.c_float), ("t", C.c_uint32), ("salt", C.c_uint32)]


class cel_accessor(C.Structure):
    _fields_ = [("base", C.c_void_p), ("alloc_box", cel_box), ("elem_size", C.c_uint32), ("range", cel_box),
                ("oob", C.c_void_p)]


cel_kernel_fn = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(cel_box), C.POINTER(cel_accessor), C.c_int,
                            C.c_void_p)


class cel_task_desc(C.Structure):
    _fields_ = [("dims", C.c_int32), ("range", cel_box), ("split", C.c_int32), ("kernel", C.c_int32),
                ("params", cel_kernel_params), ("fn", cel_kernel_fn), ("fn_user", C.c_void_p),
                ("acc", C.POINTER(cel_access)), ("n_acc", C.c_int32)]


class cel_config(C.Structure):
    _fields_ = [("cuda_devices", C.POINTER(C.c_int)), ("n_devices", C.c_int32), ("execute", C.c_int32),
                ("lookahead", C.c_int32), ("horizon_step", C.c_int32), ("checks", C.c_int32),
                ("instr_log_path", C.c_char_p), ("arena_bytes", C.c_uint64), ("rank", C.c_int32),
                ("world", C.c_int32), ("fast_math", C.c_int32), ("collective", C.c_int32),
                ("bounds_check", C.c_int32), ("n_nodes", C.c_int32)]


class cel_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "n_alloc", "n_free", "n_copy", "n_kernel", "n_horizon", "n_epoch",
        "copies_resize", "copies_coherence", "copies_readback",
        "bytes_resize", "bytes_coherence", "bytes_readback", "bytes_d2d_peer",
        "alloc_bytes_peak", "flushes", "kernel_launches", "copy_launches", "memcpy_calls",
        "event_waits", "remote_waits", "signals", "host_syncs", "gen_ns",
        "exec_ns_alloc", "exec_ns_free", "exec_ns_copy", "exec_ns_kernel", "exec_ns_horizon", "exec_ns_epoch",
        "signal_ns", "remote_wait_ns", "copies_elided", "bytes_elided", "coll_groups", "coll_copies",
        "gather_sets", "n_send", "n_receive", "n_split_receive", "n_await_receive", "pulls", "pull_bytes",
        "coll_allgathers", "tma_copy_launches", "vmm_maps", "vmm_mapped_bytes", "coll_multicast", "staging_elided",
        "staging_materialized", "coll_p2p", "coll_fused", "halo_fused", "halo_in_waits", "halo_chained", "memo_hits", "memo_misses")]


_P = C.c_void_p
lib.cel_runtime_create.argtypes = [C.POINTER(cel_config), C.POINTER(_P)]
lib.cel_ipc_blob_size.restype = C.c_size_t
lib.cel_ipc_export.argtypes = [_P, C.c_void_p]
lib.cel_ipc_import.argtypes = [_P, C.c_int32, C.c_void_p]
lib.cel_buffer_create.argtypes = [_P, C.c_int32, C.POINTER(C.c_uint64), C.c_uint32, C.c_void_p, C.POINTER(C.c_uint32)]
lib.cel_buffer_create_ex.argtypes = [_P, C.c_int32, C.POINTER(C.c_uint64), C.c_uint32, C.c_void_p, C.c_uint32,
                                     C.POINTER(C.c_uint32)]
lib.cel_task_submit.argtypes = [_P, C.POINTER(cel_task_desc), C.POINTER(C.c_uint64)]
lib.cel_wait.argtypes = [_P]
lib.cel_buffer_read.argtypes = [_P, C.c_uint32, C.POINTER(cel_box), C.c_void_p]
lib.cel_buffer_destroy.argtypes = [_P, C.c_uint32]
lib.cel_stats.argtypes = [_P, C.POINTER(cel_stats)]
lib.cel_stats_get.argtypes = [_P, C.POINTER(cel_stats)]
lib.cel_profile_enable.argtypes = [_P, C.c_int32]
lib.cel_profile_read.argtypes = [_P, C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_int32]
lib.cel_runtime_destroy.argtypes = [_P]
lib.cel_trace_dump.argtypes = [_P, C.c_char_p]
lib.cel_last_error.restype = C.c_char_p

BORROW_HOST = 1
SYMBOLS = ["cel_runtime_create", "cel_ipc_blob_size", "cel_ipc_export", "cel_ipc_import", "cel_buffer_create",
           "cel_buffer_create_ex",
           "cel_task_submit", "cel_wait", "cel_buffer_read", "cel_buffer_destroy", "cel_stats", "cel_stats_get",
           "cel_profile_enable", "cel_profile_read", "cel_trace_dump", "cel_runtime_destroy", "cel_last_error"]


class CelError(Exception):
    def __init__(self, code, msg):
        super().__init__("%d: %s" % (code, msg))
        self.code = code


def _check(rc):
    if rc < 0:
        raise CelError(rc, lib.cel_last_error().decode())
    return rc


def _box(mn, mx):
    b = cel_box()
    mn = list(mn) + [0] * (3 - len(mn))
    mx = list(mx) + [1] * (3 - len(mx))
    for d in range(3):
        b.min[d] = int(mn[d])
        b.max[d] = int(mx[d])
    return b


def _mapper(mp):
    m = cel_range_mapper()
    m.kind = MAPPERS[mp[0]]
    m.from_kernel_dim[:] = [-1, -1, -1]
    if mp[0] in ("neighborhood", "neighborhood_axes"):
        bd = list(mp[1]) + [0] * (3 - len(mp[1]))
        m.border[:] = [int(x) for x in bd]
    elif mp[0] in ("fixed", "remap"):
        m.fixed = _box(mp[1][0], mp[1][1])
        if mp[0] == "remap":
            kd = list(mp[2]) + [-1] * (3 - len(mp[2]))
            m.from_kernel_dim[:] = [int(x) for x in kd]
    return m


def task_desc(spec):
    """Marshal a workloads task spec into a cel_task_desc (kept alive by the caller)."""
    d = cel_task_desc()
    d.dims = spec["dims"]
    d.range = _box(*spec["range"])
    d.split = SPLITS[spec.get("split", "1d")]
    d.kernel = KERNELS[spec["kernel"]]
    p = spec.get("params", {})
    d.params.seed = int(p.get("seed", 0))
    d.params.value = float(p.get("value", 0.0))
    d.params.t = int(p.get("t", 0))
    d.params.salt = int(p.get("salt", 0)) & 0xFFFFFFFF
    accs = (cel_access * max(1, len(spec["accesses"])))()
    for i, (bid, mode, mp) in enumerate(spec["accesses"]):
        accs[i].buf = bid
        accs[i].mode = MODES[mode]
        accs[i].map = _mapper(mp)
    d.acc = accs
    d.n_acc = len(spec["accesses"])
    return d, accs


class Runtime:
    """The C-ABI runtime.  Method names follow include/cel.h (cel_ prefix dropped)."""

    def __init__(self, n_devices, cuda_devices=None, execute=True, lookahead="auto", horizon_step=4, checks=True,
                 instr_log_path=None, arena_bytes=0, rank=0, world=1, fast_math=False, collective=True, n_nodes=1,
                 bounds_check=False):
        """n_nodes > 1: virtual-node mode, n_nodes nodes of n_devices devices each
        (cuda_devices lists n_nodes * n_devices entries, node-major); node k's
        instruction log is written to instr_log_path + ".k"."""
        cfg = cel_config()
        devs = list(cuda_devices) if cuda_devices is not None else list(range(n_devices * max(1, n_nodes)))
        self._devs = (C.c_int * len(devs))(*devs)
        cfg.cuda_devices = self._devs
        cfg.n_devices = n_devices
        cfg.execute = 1 if execute else 0
        cfg.lookahead = {"none": 0, "auto": 1, "infinite": 2}[lookahead]
        cfg.horizon_step = horizon_step
        cfg.checks = 1 if checks else 0
        cfg.instr_log_path = instr_log_path.encode() if instr_log_path else None
        cfg.arena_bytes = int(arena_bytes)
        cfg.rank = rank
        cfg.world = world
        cfg.fast_math = 1 if fast_math else 0
        cfg.collective = 1 if collective else 0
        cfg.n_nodes = int(n_nodes)
        cfg.bounds_check = 1 if bounds_check else 0
        h = _P()
        _check(lib.cel_runtime_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.G = n_devices
        self.meta = {}
        self._keep = []

    # -- multi-process plumbing
    def ipc_export(self):
        buf = C.create_string_buffer(lib.cel_ipc_blob_size())
        _check(lib.cel_ipc_export(self.h, buf))
        return buf.raw

    def ipc_import(self, rank, blob):
        _check(lib.cel_ipc_import(self.h, rank, C.c_char_p(blob)))

    # -- the paper's model
    def buffer_create(self, dims, extent, elem_size, host_init=None, borrow=False):
        ext = (C.c_uint64 * 3)(*(list(extent) + [1] * (3 - len(extent))))
        out = C.c_uint32()
        ptr = None
        if host_init is not None:
            host_init = np.ascontiguousarray(host_init)
            assert host_init.nbytes == int(np.prod(extent)) * elem_size
            ptr = host_init.ctypes.data_as(C.c_void_p)
        if borrow:
            self._keep.append(host_init)
            _check(lib.cel_buffer_create_ex(self.h, dims, ext, elem_size, ptr, BORROW_HOST, C.byref(out)))
        else:
            _check(lib.cel_buffer_create(self.h, dims, ext, elem_size, ptr, C.byref(out)))
        self.meta[out.value] = (dims, list(extent), elem_size)
        return out.value

    def task_submit(self, spec):
        d, accs = task_desc(spec)
        tid = C.c_uint64()
        st = _check(lib.cel_task_submit(self.h, C.byref(d), C.byref(tid)))
        return tid.value, st

    def submit_desc(self, d):
        """Submit a pre-marshalled cel_task_desc (hot loops)."""
        tid = C.c_uint64()
        return _check(lib.cel_task_submit(self.h, C.byref(d), C.byref(tid)))

    def wait(self):
        _check(lib.cel_wait(self.h))

    def buffer_read(self, bid, box, out=None):
        """Read `box` back; returns a uint32 array (n0, n1, n2, words) over the box."""
        b = _box(*box)
        es = self.meta[bid][2]
        shape = tuple(int(b.max[d] - b.min[d]) for d in range(3)) + (es // 4,)
        if out is None:
            out = np.zeros(shape, dtype=np.uint32)
        _check(lib.cel_buffer_read(self.h, bid, C.byref(b), out.ctypes.data_as(C.c_void_p)))
        return out

    def buffer_read_into(self, bid, box, ptr):
        b = _box(*box)
        _check(lib.cel_buffer_read(self.h, bid, C.byref(b), C.c_void_p(ptr)))

    def buffer_destroy(self, bid):
        _check(lib.cel_buffer_destroy(self.h, bid))

    def stats(self):
        s = cel_stats()
        _check(lib.cel_stats(self.h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in cel_stats._fields_}

    def profile_enable(self, on=True, stride=1):
        """stride k: time every k-th launch of each kind (average unchanged, less overhead)."""
        _check(lib.cel_profile_enable(self.h, max(1, int(stride)) if on else 0))

    def profile_read(self):
        ms = (C.c_double * PROFILE_SLOTS)()
        cnt = (C.c_uint64 * PROFILE_SLOTS)()
        _check(lib.cel_profile_read(self.h, ms, cnt, PROFILE_SLOTS))
        out = {}
        for k in range(PROFILE_SLOTS):
            if cnt[k]:
                name = {COPY_SLOT: "copy", PEER_SLOT: "copy_peer", SHELL_SLOT: "shell", COLL_SLOT: "coll"}.get(k) or KERNEL_NAMES[k]
                out[name] = (ms[k], cnt[k])
        return out

    def trace_dump(self, path):
        _check(lib.cel_trace_dump(self.h, path.encode()))

    def shutdown(self):
        if self.h is not None:
            h, self.h = self.h, None
            _check(lib.cel_runtime_destroy(h))

    def __del__(self):
        try:
            self.shutdown()
        except Exception:
            pass
