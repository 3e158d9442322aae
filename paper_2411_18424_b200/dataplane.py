"""Real bytes under SwapManager.dispatch: device KV planes, the pinned host
pool, and the libkvswap handle that moves SwapPlans between them.

Reference seam: kvswitch models a swap as timestamps only
(swap.py:181-232); the CPU copy is bookkeeping over host block groups
(cpu_store.py:123-141).  This module owns the memory those blocks name:

* `PagedKVCache` — the rank's GPU KV cache, one plane per layer (or two with
  split K/V), allocated once in HBM by torch (it outlives every swap).
* `HostKVPool` — the CpuStore's swap space: block-major, pinned, device-mapped
  host memory from kvs_host_alloc (cudaHostAlloc Mapped|Portable or
  mmap+mbind+cudaHostRegister).
* `SwapDataPlane` — one kvs handle per rank; `swap()` queues one plan as one
  kernel launch on a caller-chosen stream, `baseline()` queues the
  copy-engine comparators.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _lib
from .geometry import KVGeometry

OpsLike = Union[np.ndarray, Sequence]


def ops_array(ops: OpsLike) -> np.ndarray:
    """TransferOp list / (blocks, gpu_start, cpu_start) tuples -> int32 [n, 3]."""
    if isinstance(ops, np.ndarray):
        arr = np.ascontiguousarray(ops, dtype=np.int32).reshape(-1, 3)
        return arr
    flat = []
    for op in ops:
        if hasattr(op, "blocks"):
            flat.extend((op.blocks, op.gpu_start, op.cpu_start))
        else:
            b, g, c = op
            flat.extend((b, g, c))
    return np.asarray(flat, dtype=np.int32).reshape(-1, 3)


def _stream_handle(stream: Optional[torch.cuda.Stream]) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def numa_nodes() -> int:
    """Number of online NUMA nodes of this host (1 when unknown)."""
    try:
        with open("/sys/devices/system/node/online") as f:
            spec = f.read().strip()
    except OSError:
        return 1
    n = 0
    for part in spec.split(","):
        lo, _, hi = part.partition("-")
        n += int(hi or lo) - int(lo) + 1
    return max(1, n)


def _gpu_bdf(device) -> Optional[str]:
    try:
        idx = torch.device(device if device is not None else "cuda").index
        props = torch.cuda.get_device_properties(idx if idx is not None else 0)
        return f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
    except (RuntimeError, AssertionError, ValueError):
        return None


def _smi_link(device) -> dict:
    import subprocess

    try:
        idx = torch.device(device if device is not None else "cuda").index or 0
        out = subprocess.run(
            ["nvidia-smi", "-i", str(idx), "--format=csv,noheader,nounits",
             "--query-gpu=pcie.link.gen.max,pcie.link.gen.gpumax,pcie.link.width.max"],
            capture_output=True, text=True, timeout=10).stdout.strip()
        gen, gpumax, width = [x.strip() for x in out.split(",")]
        return {"link_speed": f"gen{gen} (device max gen{gpumax})", "link_width": width,
                "source": "nvidia-smi"}
    except (OSError, ValueError, subprocess.SubprocessError):
        return {}


def host_link_info(device=None) -> dict:
    """The GPU's PCIe link as sysfs reports it (speed, width), its NUMA node,
    and the root port it hangs off: GPUs behind one root port share that
    port's host link, which caps their aggregate swap bandwidth."""
    import os

    bdf = _gpu_bdf(device)
    info = {"bdf": bdf, "link_speed": None, "link_width": None, "max_link_speed": None,
            "root_port": None, "numa_node": -1}
    if bdf is None:
        return info
    base = f"/sys/bus/pci/devices/{bdf}"

    def read(name):
        try:
            with open(f"{base}/{name}") as f:
                return f.read().strip()
        except OSError:
            return None

    info["link_speed"] = read("current_link_speed")
    info["max_link_speed"] = read("max_link_speed")
    info["link_width"] = read("current_link_width")
    if info["link_speed"] is None:  # no PCI sysfs in this container: ask the driver
        info.update(_smi_link(device))
    node = read("numa_node")
    info["numa_node"] = int(node) if node not in (None, "") else -1
    try:
        parts = os.path.realpath(base).split("/")
        # /sys/devices/pci0000:00/<root port>/.../<gpu>: the first device below the host bridge
        i = next(k for k, p in enumerate(parts) if p.startswith("pci"))
        info["root_port"] = parts[i + 1] if len(parts) > i + 2 else None
    except (StopIteration, OSError):
        pass
    return info


def pcie_switch_groups(n: int, text: Optional[str] = None) -> dict:
    """GPUs 0..n-1 grouped by shared PCIe switch, from `nvidia-smi topo -mp`
    (the PCIe-only matrix: NVLink would hide the host-link topology).  GPUs
    whose path is PIX / PXB (through PCIe switches only) share a switch's
    uplink to the host, so their swaps share one host link.  Returns
    {"groups": [[gpu, ...], ...], "matrix": {"i-j": relation}} or {} when
    the matrix is unavailable."""
    if text is None:
        import subprocess
        try:
            text = subprocess.run(["nvidia-smi", "topo", "-mp"], capture_output=True, text=True,
                                  timeout=20).stdout
        except (OSError, subprocess.SubprocessError):
            return {}
    rows = [ln.split() for ln in text.splitlines() if ln.strip()]
    head = next((r for r in rows if r and r[0].startswith("GPU") and len(r) > 1
                 and r[1].startswith("GPU")), None)
    if head is None:  # the header row starts with the first column name
        head = next((r for r in rows if "GPU0" in r and not r[0].startswith("GPU0")), None)
    if head is None:
        return {}
    cols = [c for c in head if c.startswith("GPU") and c[3:].isdigit()]
    rel = {}
    for r in rows:
        if r and r[0] in cols:
            i = int(r[0][3:])
            for c, v in zip(cols, r[1:1 + len(cols)]):
                j = int(c[3:])
                if i < n and j < n and i != j:
                    rel[(min(i, j), max(i, j))] = v
    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for (i, j), v in rel.items():
        if v in ("PIX", "PXB"):
            parent[find(i)] = find(j)
    groups: dict = {}
    for g in range(n):
        groups.setdefault(find(g), []).append(g)
    return {"groups": sorted(groups.values()),
            "matrix": {f"{i}-{j}": v for (i, j), v in sorted(rel.items())}}


def gpu_numa_node(device: Union[int, str, torch.device, None]) -> int:
    """NUMA node of the GPU's PCIe root (sysfs), or -1 when unknown.  Each
    rank's swap space belongs on its own GPU's socket: host-link traffic then
    never crosses the inter-socket fabric."""
    bdf = _gpu_bdf(device)
    if bdf is None:
        return -1
    try:
        with open(f"/sys/bus/pci/devices/{bdf}/numa_node") as f:
            return int(f.read().strip())
    except (OSError, ValueError):
        return -1


def sm_partition(device=None, swap_sms: int = 8, swap_streams: int = 2,
                 swap_priority: int = 0, compute_priority: int = -1):
    """Green-context SM partition (kvs_sm_partition): returns
    (swap streams, compute stream, (swap SMs, compute SMs)); the streams are
    torch.cuda.ExternalStream views of the driver streams."""
    lib = _lib.load()
    idx = torch.device(device if device is not None else "cuda").index
    idx = idx if idx is not None else torch.cuda.current_device()
    swaps = (ctypes.c_uint64 * swap_streams)()
    rest = ctypes.c_uint64()
    sms = (ctypes.c_int * 2)()
    _lib.check(lib.kvs_sm_partition(idx, swap_sms, swap_streams, swap_priority, compute_priority,
                                    swaps, ctypes.byref(rest), sms), "kvs_sm_partition")
    dev = torch.device("cuda", idx)
    return ([torch.cuda.ExternalStream(int(h), device=dev) for h in swaps],
            torch.cuda.ExternalStream(int(rest.value), device=dev), (sms[0], sms[1]))


class HostKVPool:
    """Pinned, device-mapped host swap space: [num_blocks, block_bytes] bytes.

    numa_node=None with a `device` places the pool on that GPU's NUMA node
    (mmap + mbind + cudaHostRegister) on multi-socket hosts; single-node hosts
    use cudaHostAlloc."""

    def __init__(self, num_blocks: int, block_bytes: int, numa_node: Optional[int] = -1,
                 register: bool = False, device=None, write_combined: bool = False) -> None:
        if num_blocks < 1 or block_bytes < 16 or block_bytes % 16:
            raise ValueError("host pool needs >= 1 block of a 16-byte multiple")
        lib = _lib.load()
        if numa_node is None:
            numa_node = gpu_numa_node(device) if numa_nodes() > 1 else -1
            register = register or numa_node >= 0
        self.numa_node = numa_node
        self.num_blocks = num_blocks
        self.block_bytes = block_bytes
        self.nbytes = num_blocks * block_bytes
        host = ctypes.c_void_p()
        dev = ctypes.c_void_p()
        if write_combined and register:
            raise ValueError("write-combined pools come from cudaHostAlloc, not registration")
        flags = (_lib.KVS_HOST_REGISTER if register else
                 _lib.KVS_HOST_WRITE_COMBINED if write_combined else _lib.KVS_HOST_DEFAULT)
        _lib.check(lib.kvs_host_alloc(self.nbytes, numa_node, flags,
                                      ctypes.byref(host), ctypes.byref(dev)),
                   "kvs_host_alloc")
        self.host_ptr = int(host.value)
        self.dev_ptr = int(dev.value)
        buf = (ctypes.c_uint8 * self.nbytes).from_address(self.host_ptr)
        self._buf = buf
        self.array = np.frombuffer(buf, dtype=np.uint8).reshape(num_blocks, block_bytes)
        self.tensor = torch.from_numpy(self.array)

    def close(self) -> None:
        if getattr(self, "host_ptr", 0):
            self.tensor = None
            self.array = None
            self._buf = None
            _lib.check(_lib.load().kvs_host_free(ctypes.c_void_p(self.host_ptr)), "kvs_host_free")
            self.host_ptr = 0

    def __del__(self) -> None:  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class PagedKVCache:
    """The rank's KV cache in HBM: planes [P, num_blocks, chunk] of raw bytes.

    `layer(l)` views plane l as the model's [num_blocks, 2, T, H, d] tensor.
    """

    def __init__(self, geometry: KVGeometry, num_blocks: int,
                 device: Union[int, str, torch.device] = "cuda",
                 dtype: torch.dtype = torch.float16) -> None:
        if num_blocks < 1:
            raise ValueError("num_blocks must be >= 1")
        self.geometry = geometry
        self.num_blocks = num_blocks
        self.device = torch.device(device)
        self.dtype = dtype
        self.planes = torch.empty(
            (geometry.num_planes, num_blocks, geometry.plane_chunk_bytes),
            dtype=torch.uint8, device=self.device,
        )

    @property
    def plane_stride(self) -> int:
        return self.geometry.plane_chunk_bytes

    def plane_ptrs(self) -> list[int]:
        base = self.planes.data_ptr()
        step = self.num_blocks * self.geometry.plane_chunk_bytes
        return [base + p * step for p in range(self.geometry.num_planes)]

    def layer(self, l: int) -> torch.Tensor:
        g = self.geometry
        if g.split_kv:
            raise ValueError("split_kv caches expose planes, not fused layers")
        return self.planes[l].view(self.dtype).view(
            self.num_blocks, 2, g.block_tokens, g.heads_per_rank, g.head_dim)


class SwapDataPlane:
    """One libkvswap handle: moves SwapPlans between a PagedKVCache and a HostKVPool."""

    def __init__(self, cache: PagedKVCache, host: HostKVPool,
                 ctas: Optional[dict] = None, threads: Optional[dict] = None) -> None:
        g = cache.geometry
        if host.block_bytes != g.block_bytes:
            raise ValueError(
                f"host pool block {host.block_bytes} B != geometry block {g.block_bytes} B"
            )
        self.lib = _lib.load()
        self.cache = cache
        self.host = host
        self.geometry = g
        geo = _lib.KvsGeometry(g.num_planes, 0, g.plane_chunk_bytes, cache.plane_stride)
        ptrs = (ctypes.c_uint64 * g.num_planes)(*cache.plane_ptrs())
        handle = ctypes.c_void_p()
        dev_index = cache.device.index if cache.device.index is not None else torch.cuda.current_device()
        _lib.check(self.lib.kvs_create(dev_index, ctypes.byref(geo), ptrs,
                                       ctypes.c_void_p(host.dev_ptr), cache.num_blocks,
                                       host.num_blocks, ctypes.byref(handle)), "kvs_create")
        self.handle = handle
        self.device_index = dev_index
        for direction, d in _lib.DIRECTIONS.items():
            c = (ctas or {}).get(direction, 0)
            t = (threads or {}).get(direction, 0)
            self.set_launch(direction, c, t)

    def set_launch(self, direction: str, ctas: int = 0, threads: int = 0) -> None:
        _lib.check(self.lib.kvs_set_launch(self.handle, _lib.DIRECTIONS[direction], ctas, threads),
                   "kvs_set_launch")

    def set_path(self, direction: str, path: str = "lsu", piece_bytes: int = 0,
                 stages: int = 0) -> None:
        """Kernel path per direction: "lsu" (16-B vector LDG/STG) or "bulk" (TMA)."""
        _lib.check(self.lib.kvs_set_path(self.handle, _lib.DIRECTIONS[direction],
                                         _lib.PATHS[path], piece_bytes, stages), "kvs_set_path")

    def set_staging(self, slot_bytes: int = 0, slots: int = 0) -> None:
        """Staging ring of the staged copy-engine path (0 = default 4 x 128 MiB)."""
        _lib.check(self.lib.kvs_set_staging(self.handle, int(slot_bytes), int(slots)),
                   "kvs_set_staging")

    def set_pace(self, direction: str, gbps: float = 0.0) -> None:
        """Hold one direction's LSU kernel to `gbps` GB/s (0 = unpaced)."""
        _lib.check(self.lib.kvs_set_pace(self.handle, _lib.DIRECTIONS[direction], float(gbps)),
                   "kvs_set_pace")

    def set_pace_burst(self, direction: str, burst_bytes: int = 0) -> None:
        """Release paced pieces in bursts of `burst_bytes` (0 = steady)."""
        _lib.check(self.lib.kvs_set_pace_burst(self.handle, _lib.DIRECTIONS[direction],
                                               int(burst_bytes)), "kvs_set_pace_burst")

    def set_budget(self, gbps: float = 0.0) -> None:
        """One GB/s budget shared by swap-out and swap-in (0 = none)."""
        _lib.check(self.lib.kvs_set_budget(self.handle, float(gbps)), "kvs_set_budget")

    def set_layer_group(self, planes: int = 0) -> None:
        """Planes per group in plane-major (layered) order; 0 = auto."""
        _lib.check(self.lib.kvs_set_layer_group(self.handle, planes), "kvs_set_layer_group")

    def set_budget_priority(self, direction: Optional[str]) -> None:
        """Direction that charges the shared budget without waiting (None = neither)."""
        d = -1 if direction is None else _lib.DIRECTIONS[direction]
        _lib.check(self.lib.kvs_set_budget_priority(self.handle, d), "kvs_set_budget_priority")

    def set_budget_share(self, direction: str, gbps: float = 0.0) -> None:
        """Reserve `gbps` of the shared budget for `direction` (0 = none)."""
        _lib.check(self.lib.kvs_set_budget_share(self.handle, _lib.DIRECTIONS[direction],
                                                 float(gbps)), "kvs_set_budget_share")

    @property
    def launches(self) -> int:
        return int(self.lib.kvs_launch_count(self.handle))

    def swap(self, direction: str, ops: OpsLike, stream: Optional[torch.cuda.Stream] = None,
             done_flag: Optional[int] = None, seq: int = 0) -> np.ndarray:
        """Queue one plan (all its TransferOps, all planes) as one kernel launch."""
        arr = ops_array(ops)
        rc = self.lib.kvs_swap(self.handle, _lib.DIRECTIONS[direction],
                               arr.ctypes.data_as(ctypes.c_void_p), arr.shape[0],
                               _stream_handle(stream),
                               ctypes.c_void_p(done_flag) if done_flag else None,
                               seq & 0xFFFFFFFF)
        _lib.check(rc, f"kvs_swap({direction})")
        return arr

    def swap_layered(self, direction: str, ops: OpsLike, plane_flags: int, seq: int,
                     stream: Optional[torch.cuda.Stream] = None) -> np.ndarray:
        """Plane-major swap; plane_flags[p] <- seq once plane (layer) p has landed."""
        arr = ops_array(ops)
        rc = self.lib.kvs_swap_layered(self.handle, _lib.DIRECTIONS[direction],
                                       arr.ctypes.data_as(ctypes.c_void_p), arr.shape[0],
                                       _stream_handle(stream), ctypes.c_void_p(plane_flags),
                                       seq & 0xFFFFFFFF)
        _lib.check(rc, f"kvs_swap_layered({direction})")
        return arr

    def swap_ops(self, direction: str, ops: OpsLike, op_flags: int, seq: int,
                 stream: Optional[torch.cuda.Stream] = None,
                 done_flag: Optional[int] = None) -> np.ndarray:
        """One launch; op_flags[i] <- seq once TransferOp i has landed."""
        arr = ops_array(ops)
        rc = self.lib.kvs_swap_ops(self.handle, _lib.DIRECTIONS[direction],
                                   arr.ctypes.data_as(ctypes.c_void_p), arr.shape[0],
                                   _stream_handle(stream), ctypes.c_void_p(op_flags),
                                   ctypes.c_void_p(done_flag) if done_flag else None,
                                   seq & 0xFFFFFFFF)
        _lib.check(rc, f"kvs_swap_ops({direction})")
        return arr

    def swap_signaled(self, direction: str, ops: OpsLike, seq: int,
                      op_flags: Optional[int] = None, plane_flags: Optional[int] = None,
                      done_flag: Optional[int] = None,
                      stream: Optional[torch.cuda.Stream] = None) -> np.ndarray:
        """One launch with any of: per-op flags, per-plane flags (plane-major
        order), a whole-plan flag; each receives `seq` once its bytes landed."""
        arr = ops_array(ops)
        sig = _lib.KvsSignals(op_flags or None, plane_flags or None, done_flag or None,
                              seq & 0xFFFFFFFF, 0)
        rc = self.lib.kvs_swap_signaled(self.handle, _lib.DIRECTIONS[direction],
                                        arr.ctypes.data_as(ctypes.c_void_p), arr.shape[0],
                                        _stream_handle(stream), ctypes.byref(sig))
        _lib.check(rc, f"kvs_swap_signaled({direction})")
        return arr

    def baseline(self, direction: str, mode: int, ops: OpsLike,
                 stream: Optional[torch.cuda.Stream] = None) -> None:
        """Copy-engine path for the plan (include/kvswap.h): 0 per block
        (vLLM swap_blocks), 1 per run (2D), 2 staged (whole host runs through
        an HBM staging ring + a gather / scatter kernel)."""
        arr = ops_array(ops)
        rc = self.lib.kvs_memcpy_baseline(self.handle, _lib.DIRECTIONS[direction], mode,
                                          arr.ctypes.data_as(ctypes.c_void_p), arr.shape[0],
                                          _stream_handle(stream))
        _lib.check(rc, f"kvs_memcpy_baseline({direction}, mode={mode})")

    def kv_tokens(self, mode: int, segs: np.ndarray, stream: Optional[torch.cuda.Stream] = None,
                  mismatch_ptr: int = 0, planes: Optional[tuple[int, int]] = None) -> None:
        """Write (mode 0) or check (mode 1) the synthetic KV of token segments
        int64 [n, 4] = (request, lo, hi, physical block of token lo), in
        planes [lo, hi) (default: all)."""
        arr = np.ascontiguousarray(segs, dtype=np.int64).reshape(-1, 4)
        p_lo, p_hi = planes if planes is not None else (0, -1)
        rc = self.lib.kvs_kv_tokens(self.handle, mode, arr.ctypes.data_as(ctypes.c_void_p),
                                    arr.shape[0], self.geometry.block_tokens, p_lo, p_hi,
                                    _stream_handle(stream),
                                    ctypes.c_void_p(mismatch_ptr) if mismatch_ptr else None)
        _lib.check(rc, "kvs_kv_tokens")

    def wait_flag(self, stream: Optional[torch.cuda.Stream], flag_ptr: int, value: int) -> None:
        _lib.check(self.lib.kvs_wait_flag(_stream_handle(stream), ctypes.c_void_p(flag_ptr),
                                          value & 0xFFFFFFFF), "kvs_wait_flag")

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.kvs_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self) -> None:  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
