#!/usr/bin/env python
"""Benchmark of the Marrow hot path on B200 (driver contract: one JSON line).

Default workload (BASELINE.json configs[1], the metric's headline config):
the fused Filter Pipeline (Gaussian noise -> solarize -> mirror) on
one 8192x8192 RGBA8 image, rows partitioned across the ranks (strong
scaling).  A step is one run of the whole tree over the image.  Other §8
rows: --workload saxpy|segmentation|mapreduce_sum|mapreduce_dot|mapreduce_max|hysteresis|
nbody|all.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

For N > 1 launch with torchrun (one process per GPU), or plain
`python bench.py --gpus N`, which starts the N local ranks itself; timing is
CUDA events on the launching stream, max over ranks.  `--impl reference` times the CPU
oracle (test infrastructure) as the reference arm on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "elements/s (pixels, particles) at 1/2/4/8 B200; % of HBM roofline"


def peaks():
    p = {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p = {"hbm_gbs": float(m["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)",
             "sm_max_mhz": m.get("sm_max_mhz")}
    return p


def alu_peaks(pk):
    """Peaks of the ALU-bound rows: measured by scripts/microbench_peaks.cu on
    a B200 of this pool (profiles/r02_alu_peaks.jsonl: packed FFMA2 for the
    FP32 pipe, LOP3 for the integer ALU pipe), else the guide's unit counts."""
    sm_mhz = pk.get("sm_max_mhz") or 1965.0
    out = {"nbody": (148 * 128 * 2 * sm_mhz * 1e6 / 1e12, "TFLOP/s",
                     "148 SM x 128 FP32 lanes x 2 flop x max SM clock (guide unit counts)"),
           "hysteresis": (148 * 64 * sm_mhz * 1e6 / 1e12, "Tops/s",
                          "148 SM x 64 integer-ALU lanes x max SM clock (guide unit counts)")}
    path = os.path.join(ROOT, "profiles", "r02_alu_peaks.jsonl")
    try:
        with open(path) as f:
            m = {d["kernel"]: d for d in map(json.loads, f) if d}
        out["nbody"] = (m["ffma2"]["value"], "TFLOP/s",
                        "measured: packed FFMA2 throughput (scripts/microbench_peaks.cu, "
                        "profiles/r02_alu_peaks.jsonl)")
        out["hysteresis"] = (m["lop3"]["value"], "Tops/s",
                             "measured: LOP3 integer-ALU throughput (scripts/microbench_peaks.cu, "
                             "profiles/r02_alu_peaks.jsonl)")
    except (OSError, KeyError, ValueError):
        pass
    return out


# ------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples),
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b and b != 0x1]}


# ------------------------------------------------------------------ distributed
class Dist:
    def __init__(self, gpus):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if gpus != self.world:
            raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={self.world}")
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=self.device_obj())
            self.pg = dist

    def device_obj(self):
        import torch
        return torch.device(f"cuda:{self.local}")

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, v):
        if not self.pg:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device=self.device_obj())
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def bcast_bytes(self, b):
        if not self.pg:
            return b
        obj = [b]
        self.pg.broadcast_object_list(obj, src=0)
        return obj[0]


# ------------------------------------------------------------------ workloads
class Workload:
    """One §8 row: builds the tree, allocates this rank's slice (inputs
    generated on the device, keyed by global index), enqueues one step."""
    name = ""
    unit = ""
    dtype = ""
    kclass = 0
    bound = "hbm"

    def arglist(self, k):
        """The prebuilt argument array of buffer set k (marshalled once)."""
        if not hasattr(self, "_al"):
            self._al = {}
        al = self._al.get(k)
        if al is None:
            al = self._al[k] = self.M.ArgList(list(self.sets[k]))
        return al

    def __init__(self, M, trees, synth, torch, ctx, dev, rank):
        self.M, self.trees, self.synth, self.torch = M, trees, synth, torch
        self.ctx, self.dev, self.rank = ctx, dev, rank
        self.l2 = torch.cuda.get_device_properties(dev).L2_cache_size

    def bound_of(self, cls, launches, steps):
        return self.bound

    def sets_for(self, ws_bytes):
        return max(1, math.ceil(2 * self.l2 / max(1, ws_bytes)))

    # ---- end-to-end leg (the public API with host data every step)
    e2e_mode = None          # "staged": mw_run on pinned HOST args (library overlap);
    e2e_in, e2e_out = (), ()  # "explicit": H2D of sets[0][e2e_in], mw_run, D2H of e2e_out

    def _host_arg(self, a):
        t = a._owner
        h = self.torch.empty(tuple(t.shape), dtype=t.dtype).pin_memory()
        h.copy_(t)
        return self.M.arg(h, a.mode, local_offset=a.local_offset,
                          global_shape=tuple(a.shape[i] for i in range(a.ndim)))

    def e2e_setup(self):
        st = self.sets[0]
        nbytes = lambda t: t.numel() * t.element_size()   # noqa: E731
        h2d = sum(nbytes(st[i]._owner) for i in self.e2e_in)
        d2h = sum(nbytes(st[i]._owner) for i in self.e2e_out) if self.e2e_out else 8   # or one fp64
        if self.e2e_mode == "staged":
            self.e2e_args = [self._host_arg(a) for a in st]
            # the pinned inputs are complete before the timed region: a run's
            # uploads may overlap the previous run's downloads (marrow.h)
            self.M.mw_ctx_set_staging_overlap(self.ctx, True)
            return h2d, d2h
        # Two device buffer sets on two streams: step i+1's uploads overlap
        # step i's downloads (PCIe duplex); the runs themselves stay in FIFO
        # order (each waits for the previous run: the ctx scratch is shared).
        torch, M = self.torch, self.M

        def clone(a):
            t2 = torch.empty_like(a._owner)
            return M.arg(t2, mode=a.mode, local_offset=a.local_offset,
                         global_shape=tuple(a.shape[k] for k in range(a.ndim)))
        dsets = [list(st), [clone(a) for a in st]]
        host_in = [self._host_arg(st[i])._owner for i in self.e2e_in]
        self.e2e_slots = []
        for ds in dsets:
            outs = [(ds[i]._owner, torch.empty(tuple(ds[i]._owner.shape),
                                               dtype=ds[i]._owner.dtype).pin_memory())
                    for i in self.e2e_out]
            ins = [(h, ds[i]._owner) for h, i in zip(host_in, self.e2e_in)]
            self.e2e_slots.append((torch.cuda.Stream(device=self.dev), ds, ins, outs))
        self.e2e_streams = [sl[0] for sl in self.e2e_slots]
        self.e2e_i = 0
        self.e2e_prev = None
        return h2d, d2h

    def e2e_step(self):
        if self.e2e_mode == "staged":
            return self.M.mw_run(self.ctx, self.tree, self.e2e_args)
        torch = self.torch
        s, ds, ins, outs = self.e2e_slots[self.e2e_i % 2]
        self.e2e_i += 1
        with torch.cuda.stream(s):
            for h, d in ins:
                d.copy_(h, non_blocking=True)
            if self.e2e_prev is not None:
                s.wait_event(self.e2e_prev)
            f = self.M.mw_run(self.ctx, self.tree, ds, stream=s)
            ev = torch.cuda.Event()
            ev.record(s)
            self.e2e_prev = ev
            for d, h in outs:
                h.copy_(d, non_blocking=True)
        return f

    def slice(self, L):
        off, ln = self.M.mw_partition(self.ctx, self.tree, L)
        k = len(off) // int(os.environ.get("WORLD_SIZE", "1"))   # this rank's partitions: contiguous
        return off[self.rank * k], sum(ln[self.rank * k:(self.rank + 1) * k])


class Filter(Workload):
    name, unit, dtype = "filter_pipeline_8192x8192_rgba8", "pixels/s", "u8"
    e2e_mode, e2e_in, e2e_out = "staged", (0,), (1,)

    def setup(self, H=8192, W=8192):
        M, t = self.M, self.torch
        self.tree = self.trees.filter_pipeline()
        self.H, self.W = H, W
        self.kclass = M.MW_KC_RGBA
        self.o, self.n = self.slice(H)
        ws = 2 * self.n * W * 4
        self.B = self.sets_for(ws)
        self.sets = []
        for _ in range(self.B):
            src = t.empty((self.n, W, 4), dtype=t.uint8, device=self.dev)
            self.synth.dev_fill_rgba(src, self.synth.SEED_IMAGE, self.o * W)
            dst = t.empty_like(src)
            self.sets.append((M.arg(src, local_offset=self.o, global_shape=(H, W, 4)),
                              M.arg(dst, local_offset=self.o, global_shape=(H, W, 4))))
        self.units = H * W                       # whole-job pixels per step
        self.launch_bytes = 8 * self.n * W       # algorithmic: read 4 B + write 4 B per pixel
        # steps run over rotating buffer sets: a run reads nothing the previous
        # one wrote, so its first loads may overlap the previous run's drain
        M.mw_ctx_set_run_pipelining(self.ctx, True)
        self.l2_note = (f"inputs larger than L2 ({ws >> 20} MiB/rank working set)" if self.B == 1 else
                        f"{self.B} rotating buffer sets ({self.B * ws >> 20} MiB >= 2x L2)")

    def step(self, i):
        return self.M.mw_run(self.ctx, self.tree, self.arglist(i % self.B))

    def roof_bytes(self, cls, launches, steps, res):
        return 8.0 * self.n * self.W * steps if cls == self.M.MW_KC_RGBA else 0.0   # this rank's rows

    def config(self):
        return {"workload": self.name, "image": [self.H, self.W, 4],
                "tree": "pipeline(gauss_noise(seed=4,S=8), solarize(T=128), mirror)",
                "rows_per_rank": self.n, "l2": self.l2_note,
                "runs": "pipelined (mw_ctx_set_run_pipelining): each run's first loads may precede the "
                        "wait for the previous run, whose outputs it does not read; stores stay ordered"}


class Saxpy(Workload):
    name, unit, dtype = "saxpy_map_2^20_fp32", "elements/s", "f32"
    e2e_mode, e2e_in, e2e_out = "staged", (0, 1), (1,)

    def setup(self, n=1 << 20):
        M, t = self.M, self.torch
        self.tree = self.trees.saxpy()
        self.kclass = M.MW_KC_SAXPY
        self.L = n
        self.o, self.n = self.slice(n)
        ws = 8 * self.n
        self.B = self.sets_for(ws)
        self.sets = []
        for _ in range(self.B):
            x = t.empty(self.n, dtype=t.float32, device=self.dev)
            y = t.empty(self.n, dtype=t.float32, device=self.dev)
            self.synth.dev_fill_f32_um11(x, self.synth.SEED_SAXPY_X, self.o)
            self.synth.dev_fill_f32_um11(y, self.synth.SEED_SAXPY_Y, self.o)
            self.sets.append((M.arg(x, local_offset=self.o, global_shape=(n,)),
                              M.arg(y, local_offset=self.o, global_shape=(n,))))
        self.units, self.launch_bytes = n, 12 * self.n
        self.l2_note = f"{self.B} rotating buffer sets ({self.B * ws >> 20} MiB >= 2x L2)"

    def capture(self, stream):
        """2^20 elements are ~2 us of HBM time, below launch latency: the B
        rotating-buffer runs are captured back to back in ONE CUDA graph
        (mw_graph_capture_many); step i is run i of the replayed sequence."""
        self.graph = self.M.mw_graph_capture_many(self.ctx, self.tree, [list(st) for st in self.sets],
                                                  stream)
        self.graphs = [self.graph]
        self.graph_kernels = self.graph.kernels // self.B

    def warm_capture(self, stream):
        """Warm-L2 auxiliary: the same graph shape on buffer set 0 only."""
        self.warm_graph = self.M.mw_graph_capture_many(self.ctx, self.tree,
                                                       [list(self.sets[0])] * self.B, stream)

    def warm_timed(self, timed, k):
        g0, self.graph = self.graph, self.warm_graph
        timed(self.B)
        t = timed(k)[0]
        self.graph = g0
        return t / k

    def extra_aux(self, timed, start, stop, stream):
        """n = 2^28 (3 GiB of traffic per run) shows the
        kernel's own HBM efficiency; and the same rotating-buffer graph with
        its runs strictly serialized (one lane) next to the default
        dependency-aware graph (independent runs on parallel lanes)."""
        torch, M = self.torch, self.M
        out = {}
        n = 1 << 28
        x = torch.empty(n, dtype=torch.float32, device=self.dev)
        y = torch.empty(n, dtype=torch.float32, device=self.dev)
        self.synth.dev_fill_f32_um11(x, self.synth.SEED_SAXPY_X, 0)
        self.synth.dev_fill_f32_um11(y, self.synth.SEED_SAXPY_Y, 0)
        al = M.ArgList([M.arg(x), M.arg(y)])
        ts = []
        for r in range(6):
            start.record(stream)
            M.mw_run(self.ctx, self.tree, al, stream=stream)
            stop.record(stream)
            torch.cuda.synchronize()
            if r:
                ts.append(start.elapsed_time(stop))
        ms = statistics.median(ts)
        gbs = 12.0 * n / (ms / 1e3) / 1e9
        out["n_2p28"] = {"ms_per_run": ms, "achieved_gbs": gbs, "frac": gbs / peaks()["hbm_gbs"]}
        del x, y, al
        lanes0 = M.mw_ctx_get_tuning(self.ctx, M.MW_TUNE_GRAPH_LANES)
        M.mw_ctx_set_tuning(self.ctx, M.MW_TUNE_GRAPH_LANES, 1)
        g1 = M.mw_graph_capture_many(self.ctx, self.tree, [list(st) for st in self.sets], stream)
        M.mw_ctx_set_tuning(self.ctx, M.MW_TUNE_GRAPH_LANES, lanes0)
        g0, self.graph = self.graph, g1
        timed(self.B)
        k = max(self.B, 2000 // self.B * self.B)
        out["serialized_graph_ms_per_step"] = timed(k)[0] / k
        self.graph = g0
        return out

    def run_steps(self, k):
        assert k % self.B == 0, "steps must be a multiple of the buffer-set count"
        for _ in range(k // self.B):
            self.graph.launch(self.stream)
        return []

    def config(self):
        return {"workload": self.name, "n": self.L, "a": 2.5, "l2": self.l2_note,
                "launch": "one CUDA graph replaying the rotating-buffer runs back to back "
                          "(mw_graph_capture_many); a step is one run"}

    def roof_bytes(self, cls, launches, steps, res):
        return 12.0 * self.n * steps


class Segmentation(Workload):
    name, unit, dtype = "segmentation_1024x1024x512_u8", "voxels/s", "u8"
    e2e_mode, e2e_in, e2e_out = "staged", (0,), (1,)

    def setup(self, shape=(512, 1024, 1024)):
        M, t = self.M, self.torch
        self.tree = self.trees.segmentation()
        self.kclass = M.MW_KC_U8
        self.shape = shape
        slab = shape[1] * shape[2]
        self.o, self.n = self.slice(shape[0])
        ws = 2 * self.n * slab
        self.B = self.sets_for(ws)
        self.sets = []
        for _ in range(self.B):
            src = t.empty((self.n,) + shape[1:], dtype=t.uint8, device=self.dev)
            self.synth.dev_fill_u8_stream(src, self.synth.SEED_SEGMENT, self.o * slab)
            dst = t.empty_like(src)
            self.sets.append((M.arg(src, local_offset=self.o, global_shape=shape),
                              M.arg(dst, local_offset=self.o, global_shape=shape)))
        self.units, self.launch_bytes = shape[0] * slab, 2 * self.n * slab
        self.l2_note = (f"inputs larger than L2 ({ws >> 20} MiB/rank)" if self.B == 1 else
                        f"{self.B} rotating buffer sets")
        M.mw_ctx_set_run_pipelining(self.ctx, True)   # a run never reads what the previous wrote

    def step(self, i):
        return self.M.mw_run(self.ctx, self.tree, self.arglist(i % self.B))

    def roof_bytes(self, cls, launches, steps, res):
        return 2.0 * self.n * self.shape[1] * self.shape[2] * steps if cls == self.M.MW_KC_U8 else 0.0

    def config(self):
        return {"workload": self.name, "shape_zyx": list(self.shape), "lo": 85, "hi": 170,
                "slabs_per_rank": self.n, "l2": self.l2_note,
                "runs": "pipelined (mw_ctx_set_run_pipelining), as the filter"}


class MapReduce(Workload):
    unit, dtype = "elements/s", "f32"
    e2e_mode, e2e_out = "explicit", ()

    def __init__(self, *a, dot=True, reduce_op=None):
        super().__init__(*a)
        self.dot = dot
        self.reduce_op = reduce_op   # None: map_reduce(+); else a device reduction stage (NEXT-4)
        self.e2e_in = (0, 1) if dot else (0,)
        self.name = (f"mapreduce_{'dot' if dot else 'sum'}_2^30_fp32" if reduce_op is None
                     else "mapreduce_max_product_2^30_fp32")

    def setup(self, n=1 << 30):
        M, t = self.M, self.torch
        self.tree = (self.trees.mapreduce(self.dot) if self.reduce_op is None
                     else self.trees.mapreduce_sct(self.reduce_op, self.dot))
        self.kclass = M.MW_KC_REDUCE
        self.L = n
        self.o, self.n = self.slice(n)
        nin = 2 if self.dot else 1
        ws = 4 * nin * self.n
        self.B = self.sets_for(ws)
        self.sets = []
        for _ in range(self.B):
            args = []
            for k, seed in enumerate((self.synth.SEED_MR_X, self.synth.SEED_MR_Y)[:nin]):
                v = t.empty(self.n, dtype=t.float32, device=self.dev)
                self.synth.dev_fill_f32_um11(v, seed, self.o)
                args.append(M.arg(v, local_offset=self.o, global_shape=(n,)))
            self.sets.append(tuple(args))
        self.units, self.launch_bytes = n, 4 * nin * self.n
        self.l2_note = f"inputs larger than L2 ({ws >> 20} MiB/rank)"

    def step(self, i):
        return self.M.mw_run(self.ctx, self.tree, self.arglist(i % self.B))

    def roof_bytes(self, cls, launches, steps, res):
        return (8.0 if self.dot else 4.0) * self.n * steps if cls == self.M.MW_KC_REDUCE else 0.0

    def config(self):
        merge = ("+ (canonical 2^16 chunks, fp64)" if self.reduce_op is None
                 else "device reduction stage reduce(max) over x*y (fp64-exact products)")
        return {"workload": self.name, "n": self.L, "merge": merge, "l2": self.l2_note}


class Hysteresis(Workload):
    name, unit, dtype = "hysteresis_16384x16384_u8", "pixels/s", "u8"
    e2e_mode, e2e_in, e2e_out = "explicit", (0,), (1,)

    def __init__(self, *a, check_every=1):
        super().__init__(*a)
        self.ce = check_every

    def setup(self, H=16384, W=16384):
        M, t = self.M, self.torch
        self.tree = self.trees.hysteresis(check_every=self.ce)
        self.kclass = M.MW_KC_STENCIL
        self.H, self.W = H, W
        self.o, self.n = self.slice(H)
        # a rank's share below 2x L2 (N >= 4) rotates over buffer sets (the
        # bit planes themselves are ctx scratch, L2-resident by design)
        ws = 2 * self.n * W
        self.B = self.sets_for(ws)
        self.sets = []
        for _ in range(self.B):
            src = t.empty((self.n, W), dtype=t.uint8, device=self.dev)
            self.synth.dev_fill_u8_stream(src, self.synth.SEED_HYST, self.o * W)
            dst = t.empty_like(src)
            self.sets.append((M.arg(src, local_offset=self.o, global_shape=(H, W)),
                              M.arg(dst, local_offset=self.o, global_shape=(H, W))))
        self.units, self.launch_bytes = H * W, 2 * self.n * W   # per stencil execution
        self.l2_note = (f"inputs larger than L2 ({ws >> 20} MiB/rank)" if self.B == 1 else
                        f"{self.B} rotating buffer sets ({self.B * ws >> 20} MiB >= 2x L2)")

    def step(self, i):
        return self.M.mw_run(self.ctx, self.tree, self.arglist(i % self.B))

    def plane(self, launches, steps):
        # bit planes unless disabled (one partition: one cooperative launch per
        # step; several: one pass kernel per partition per T executions)
        return self.M.mw_ctx_get_tuning(self.ctx, self.M.MW_TUNE_HYST_PLANES) != 0

    def bound_of(self, cls, launches, steps):
        # the bit-plane loop works on L2-resident planes and is bound by the
        # integer ALU / shuffle pipes, not by HBM
        return "alu" if cls == self.M.MW_KC_STENCIL and self.plane(launches, steps) else "hbm"

    def roof_bytes(self, cls, launches, steps, res):
        """Algorithmic work.  Bit-plane path (one cooperative launch per step, or
        per-partition pass kernels):
        pack 1 B + 1/4 B and unpack 1/4 B + 1 B per pixel (U8 class, HBM);
        each Jacobi execution of the dense plane algorithm costs 5 integer ALU
        lane-operations per 32 pixels (2 funnel shifts + 3 LOP3; the 2 shuffles
        run elsewhere) -> 0.15625 ops per pixel-execution (STENCIL class, ALU).
        Byte path: 2 B per pixel per chain and per execution (HBM)."""
        px, E = float(self.n * self.W), float(res.get("executions", 0))
        plane = self.plane(launches, steps)
        if cls == self.M.MW_KC_U8:
            return (2.5 if plane else 4.0) * px * steps
        if cls == self.M.MW_KC_STENCIL:
            return (0.15625 if plane else 2.0) * px * E * steps
        return 0.0

    def config(self):
        return {"workload": self.name, "tree": "pipeline(threshold(173,250), "
                f"loop_while_changed(step, check_every={self.ce}), finalize)",
                "rows_per_rank": self.n, "l2": self.l2_note}


class NBody(Workload):
    name, unit, dtype, bound = "nbody_2^20", "bodies/s", "f32", "alu"
    e2e_mode, e2e_in, e2e_out = "explicit", (0, 1), (0, 1)

    def setup(self, N=1 << 20):
        M, t = self.M, self.torch
        self.tree = self.trees.nbody(1)
        self.kclass = M.MW_KC_NBODY
        self.N = N
        self.o, self.n = self.slice(N)
        pos = t.empty((N, 4), dtype=t.float32, device=self.dev)
        vel = t.empty((N, 4), dtype=t.float32, device=self.dev)
        self.synth.dev_fill_nbody(pos, vel, self.synth.SEED_NBODY, 0, 2.0 ** -20)
        self.sets = [(M.arg(pos, M.MW_COPY), M.arg(vel, M.MW_COPY))]
        self.B = 1
        self.units = N
        self.launch_flops = 20.0 * self.n * N    # GPU Gems convention: 20 flop / interaction
        self.l2_note = "state 32 MiB (compute bound)"

    def step(self, i):
        return self.M.mw_run(self.ctx, self.tree, self.arglist(0))

    def roof_bytes(self, cls, launches, steps, res):   # flops for the ALU-bound row
        return self.launch_flops * steps if cls == self.M.MW_KC_NBODY else 0.0

    def config(self):
        return {"workload": self.name, "bodies": self.N, "eps2": 1e-4, "dt": 1e-3,
                "bodies_per_rank": self.n, "interactions_per_step": self.N * self.N}


# workload-describing config keys shared by both arms
REF_CONFIG = {
    "filter": {"image": [8192, 8192, 4],
               "tree": "pipeline(gauss_noise(seed=4,S=8), solarize(T=128), mirror)"},
    "saxpy": {"n": 1 << 20, "a": 2.5},
    "segmentation": {"shape_zyx": [512, 1024, 1024], "lo": 85, "hi": 170},
    "mapreduce_sum": {"n": 1 << 30}, "mapreduce_dot": {"n": 1 << 30}, "mapreduce_max": {"n": 1 << 30},
    "hysteresis": {"tree": "pipeline(threshold(173,250), loop_while_changed(step, "
                           "check_every=1), finalize)"},
    "nbody": {"bodies": 1 << 20, "eps2": 1e-4, "dt": 1e-3},
    "fft": {"batch": 512, "points": 1 << 16, "tree": "pipeline(fft(2^16), ifft(2^16))"},
}

KCLASS = {0: "saxpy_chain", 1: "rgba_chain (k_rgba_ns)", 2: "u8_chain / plane pack+unpack",
          3: "hysteresis stencil loop", 4: "k_nbody", 5: "k_reduce_chunks", 6: "traits",
          7: "k_fft16 cols / rows (16 x 4096 four-step FFT)"}

class Fft(Workload):
    """NEXT-3: the paper's FFT benchmark: a batch of 512 KiB
    (65536-point complex64) FFTs, each pipelined with its inversion; one unit
    = one FFT -> IFFT of one epu.  256 MiB batch (512 transforms)."""
    name, unit, dtype = "fft_ifft_512x65536_c64", "ffts/s", "f32"
    e2e_mode, e2e_in, e2e_out = "staged", (0,), (1,)

    def setup(self, B=512, log2n=16):
        M, t = self.M, self.torch
        self.tree = self.trees.fft_pipeline(log2n)
        self.kclass = M.MW_KC_FFT
        self.Bt, self.N = B, 1 << log2n
        self.o, self.n = self.slice(B)
        g = (B, self.N, 2)
        ws = 2 * self.n * self.N * 8
        # a rank's share below 2x L2 (N >= 4) rotates over buffer sets, as the filter
        self.B = self.sets_for(ws)
        self.sets = []
        for _ in range(self.B):
            src = t.empty((self.n, self.N, 2), dtype=t.float32, device=self.dev)
            self.synth.dev_fill_f32_um11(src, 11, self.o * self.N * 2)
            dst = t.empty_like(src)
            self.sets.append((M.arg(src, local_offset=self.o, global_shape=g),
                              M.arg(dst, local_offset=self.o, global_shape=g)))
        self.units = B
        self.l2_note = (f"inputs larger than L2 ({ws >> 20} MiB/rank)" if self.B == 1 else
                        f"{self.B} rotating buffer sets ({self.B * ws >> 20} MiB >= 2x L2)")

    def step(self, i):
        return self.M.mw_run(self.ctx, self.tree, self.arglist(i % self.B))

    def roof_bytes(self, cls, launches, steps, res):
        # the fused FFT -> IFFT reads and writes each transform once: 2 x 512 KiB
        return 16.0 * self.n * self.N * steps if cls == self.M.MW_KC_FFT else 0.0

    def config(self):
        return {"workload": self.name, "batch": self.Bt, "points": self.N,
                "tree": "pipeline(fft(2^16), ifft(2^16)) (1/N in the inverse)",
                "ffts_per_rank": self.n, "l2": self.l2_note,
                "flop_convention": "5 N log2 N per transform, 2 transforms per unit"}


WORKLOADS = {"filter": Filter, "saxpy": Saxpy, "segmentation": Segmentation,
             "mapreduce_sum": lambda *a: MapReduce(*a, dot=False),
             "mapreduce_dot": lambda *a: MapReduce(*a, dot=True),
             "mapreduce_max": lambda *a: MapReduce(*a, dot=True, reduce_op=1),
             "hysteresis": Hysteresis, "nbody": NBody, "fft": Fft}


# ------------------------------------------------------------------ oracle legs
def oracle_filter_rate(budget_s, rows_cap=8192, W=8192):
    """Oracle (test infrastructure) on bounded row blocks of the config image."""
    import numpy as np  # noqa: F401

    import synth
    from oracle import kernels as K
    rows, px, spent, blocks = 64, 0, 0.0, 0
    r0 = 0
    while spent < budget_s:
        img = synth.host_rgba(synth.SEED_IMAGE, r0 * W, rows * W).reshape(rows, W, 4)
        t0 = time.perf_counter()
        K.mirror(K.solarize(K.gauss_noise(img, 4, 8, y0=r0), 128))
        spent += time.perf_counter() - t0
        px += rows * W
        blocks += 1
        r0 = (r0 + rows) % rows_cap
    return px / spent, f"{blocks} blocks of {rows}x{W} px rows of the config image", spent


def oracle_generic_rate(name, budget_s):
    """Oracle rate for the other workloads on bounded samples."""
    import numpy as np

    import synth
    from oracle import kernels as K
    spent, units, reps = 0.0, 0, 0
    while spent < budget_s:
        if name == "saxpy":
            n = 1 << 20
            x, y = synth.host_f32_um11(1, 0, n), synth.host_f32_um11(2, 0, n)
            t0 = time.perf_counter(); K.saxpy(2.5, x, y); dt = time.perf_counter() - t0
            what = "whole 2^20 vector"
        elif name == "segmentation":
            n = 1 << 24
            a = synth.host_u8_stream(7, reps * n, n)
            t0 = time.perf_counter(); K.segment(a, 85, 170); dt = time.perf_counter() - t0
            what = "16 slabs of 1024x1024"
        elif name.startswith("mapreduce"):
            n = 1 << 24
            x = synth.host_f32_um11(5, reps * n, n)
            y = synth.host_f32_um11(6, reps * n, n)
            t0 = time.perf_counter()
            if name.endswith("max"):
                K.fold_extreme(x, y)
            else:
                K.dot(x, y) if name.endswith("dot") else K.sum_(x)
            dt = time.perf_counter() - t0
            what = "2^24-element chunks"
        elif name == "hysteresis":
            n = 2048
            g = synth.host_u8_stream(8, 0, n * n).reshape(n, n)
            t0 = time.perf_counter()
            L = K.segment(g, 173, 250); f, _ = K.hyst_bfs(L); K.hyst_finalize(f)
            dt = time.perf_counter() - t0
            what = "2048x2048 tile (threshold + BFS closed form + finalize)"
            n = n * n
        elif name == "fft":
            from oracle import fft as FF
            N = 1 << 16
            x = synth.host_f32_um11(11, reps * 2 * N, 2 * N).reshape(N, 2)
            t0 = time.perf_counter(); FF.fft_chain(FF.as_complex(x), "FI"); dt = time.perf_counter() - t0
            what = "one 65536-point FFT -> IFFT (fp64, numpy pocketfft)"
            n = 1
        elif name == "nbody":
            N = 1 << 20
            pos, _ = synth.host_nbody(9, 0, N, 2.0 ** -20)
            tg = synth.nbody_sample_indices(N, 64)
            t0 = time.perf_counter(); K.nbody_accel(pos, 1e-4, targets=tg); dt = time.perf_counter() - t0
            what = "64 sampled bodies x 2^20 sources (fp64)"
            n = 64
        spent += dt
        units += n if name != "saxpy" else 1 << 20
        reps += 1
    return units / spent, f"{reps} x {what}", spent


def cpu_rate(name, budget_s):
    if name.startswith("filter"):
        return oracle_filter_rate(budget_s)
    key = {"saxpy_map_2^20_fp32": "saxpy", "segmentation_1024x1024x512_u8": "segmentation",
           "mapreduce_sum_2^30_fp32": "mapreduce_sum", "mapreduce_dot_2^30_fp32": "mapreduce_dot",
           "mapreduce_max_product_2^30_fp32": "mapreduce_max",
           "hysteresis_16384x16384_u8": "hysteresis", "nbody_2^20": "nbody",
           "fft_ifft_512x65536_c64": "fft"}[name]
    return oracle_generic_rate(key, budget_s)


# ------------------------------------------------------------------ arms
def host_info():
    """nproc and the CPU model of the box the oracle ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "threads_used": 1}


def run_reference(args, dist):
    """Reference arm: the CPU oracle as it stands, on host cores (rank 0 only)."""
    if dist.rank != 0:
        return
    names = {"filter": ("filter_pipeline_8192x8192_rgba8", "pixels/s", "u8"),
             "saxpy": ("saxpy_map_2^20_fp32", "elements/s", "f32"),
             "segmentation": ("segmentation_1024x1024x512_u8", "voxels/s", "u8"),
             "mapreduce_sum": ("mapreduce_sum_2^30_fp32", "elements/s", "f64"),
             "mapreduce_dot": ("mapreduce_dot_2^30_fp32", "elements/s", "f64"),
             "mapreduce_max": ("mapreduce_max_product_2^30_fp32", "elements/s", "f64"),
             "hysteresis": ("hysteresis_16384x16384_u8", "pixels/s", "u8"),
             "nbody": ("nbody_2^20", "bodies/s", "f64"),
             "fft": ("fft_ifft_512x65536_c64", "ffts/s", "f64")}
    wl = args.workload if args.workload != "all" else "filter"
    name, unit, dtype = names[wl]
    total_budget = float(os.environ.get("MW_REF_BUDGET_S", "90"))   # the whole arm, seconds
    per_step = total_budget / max(1, args.steps + args.warmup)
    for _ in range(args.warmup):
        cpu_rate(name, per_step)
    rates, spent, sample = [], 0.0, ""
    for _ in range(args.steps):
        r, sample, s = cpu_rate(name, per_step)
        rates.append(r)
        spent += s
    value = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * spent / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype,
            "data": "synthetic (SplitMix64, seeded; DESIGN.md input recipe)",
            "config": dict(REF_CONFIG.get(wl, {}), workload=name,
                           arm=("CPU oracle (oracle/fft.py, numpy pocketfft fp64, 1 thread)"
                                if wl == "fft" else "CPU oracle (oracle/, plain C, 1 thread)")),
            "cpu_baseline": {"value": value, "unit": unit, "cores": 1, "kind": "oracle",
                             "sample": f"per step: {sample}", **host_info()},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def comm_check(M, trees, torch, ctx, dist, parts):
    """The library's own communicator spans every rank: a MapReduce sum of
    ones over world x parts x 2^16 elements (each rank holding its rows) must
    all-reduce to exactly that count on every rank."""
    node = trees.mapreduce(False)
    L = dist.world * parts * (1 << 16)
    off, ln = M.mw_partition(ctx, node, L)
    f = dist.rank * parts
    s0, s1 = off[f], off[f + parts - 1] + ln[f + parts - 1]
    x = torch.ones(s1 - s0, dtype=torch.float32, device=dist.device_obj())
    r = M.mw_run(ctx, node, [M.arg(x, local_offset=s0, global_shape=(L,))]).wait().result()
    ok = dist.max(0.0 if r["reduced"] == L else 1.0) == 0.0
    return {"transport": "nccl", "nranks": dist.world, "allreduce_sum_of_ones_ok": ok}


def run_marrow(args, dist, wl_name):
    import torch

    import synth
    from paper_1510_06585_b200 import marrow as M
    from paper_1510_06585_b200 import trees

    dev = dist.device_obj()
    torch.cuda.set_device(dev)
    nccl_id = None
    if dist.world > 1:
        nccl_id = dist.bcast_bytes(M.mw_nccl_unique_id() if dist.rank == 0 else None)
    ctx = M.mw_ctx_create(dist.local, dist.rank, dist.world, args.parts, nccl_id)
    comm = comm_check(M, trees, torch, ctx, dist, args.parts) if dist.world > 1 else None
    w = WORKLOADS[wl_name](M, trees, synth, torch, ctx, dev, dist.rank)
    stream = torch.cuda.Stream(device=dev)   # a real stream (graph capture needs one)
    torch.cuda.set_stream(stream)
    w.setup()
    w.stream = stream
    if hasattr(w, "capture"):
        w.capture(stream)
    torch.cuda.synchronize()
    # warm-up
    if hasattr(w, "run_steps"):
        args.steps = max(w.B, args.steps // w.B * w.B)
        w.run_steps(max(w.B, args.warmup // w.B * w.B))
    else:
        futs = [w.step(i) for i in range(args.warmup)]
        del futs
    torch.cuda.synchronize()
    # Timed region without the per-partition monitoring events: a timing event
    # pair around every launch serialises back-to-back runs (measured: +11 us
    # per 8192^2 filter run, 102 vs 91 us); they are only needed by the
    # rebalancer, which is not part of a step.  Per-kernel times come from a
    # separate monitored pass below.
    M.mw_ctx_set_monitoring(ctx, False)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(k):
        """K steps between a barrier + synchronize on both sides: CUDA events
        on the launch stream, max over ranks (ms for the K steps)."""
        dist.barrier()
        torch.cuda.synchronize()
        start.record(stream)
        fs = w.run_steps(k) if hasattr(w, "run_steps") else [w.step(i) for i in range(k)]
        stop.record(stream)
        torch.cuda.synchronize()
        return dist.max(start.elapsed_time(stop)), fs

    # the median of `trials` timed trials of K steps (min and
    # max reported); clocks sampled over all of them
    trials = []
    with ClockSampler(dist.local) as clocks:
        for tr in range(args.trials):
            l0 = M.mw_ctx_launch_count(ctx)
            t_ms, futs = timed(args.steps)
            launches = M.mw_ctx_launch_count(ctx) - l0
            trials.append(t_ms)
            if tr + 1 < args.trials:
                del futs
    ms_local = statistics.median(trials)
    if hasattr(w, "graphs"):
        launches = w.graph_kernels * args.steps
        res = w.graphs[0].result()
    else:
        res = futs[-1].wait().result()
    del futs
    # monitored pass: CUDA events around every launch (mw_kernel_stats)
    M.mw_ctx_set_monitoring(ctx, True)
    mk = args.steps if hasattr(w, "graphs") else max(3, min(args.steps, 200))
    M.mw_stats_enable(ctx, True)
    if not hasattr(w, "graphs"):
        futs = [w.step(i) for i in range(mk)]
        torch.cuda.synchronize()
        del futs
    kstats = {cls: M.mw_kernel_stats(ctx, cls) for cls in range(M.MW_KC_COUNT)}
    M.mw_stats_enable(ctx, False)
    ms = ms_local   # already the max over ranks, per trial
    value = w.units * args.steps / (ms / 1e3)
    # auxiliaries: warm L2 (one buffer set, B = 1) and per-launch latency (one
    # step, R = 1, then a synchronize; device events and host wall clock)
    aux = {"trials_ms_per_step": [round(t / args.steps, 6) for t in trials],
           "min_ms_per_step": min(trials) / args.steps, "max_ms_per_step": max(trials) / args.steps}
    M.mw_ctx_set_monitoring(ctx, False)
    if w.B > 1 and not hasattr(w, "graphs"):
        b0, w.B = w.B, 1
        kw = max(3, min(args.steps, 500))
        timed(3)
        aux["warm_l2_ms_per_step"] = timed(kw)[0] / kw
        w.B = b0
    elif w.B > 1 and hasattr(w, "warm_capture"):
        w.warm_capture(stream)
        aux["warm_l2_ms_per_step"] = w.warm_timed(timed, args.steps)
    else:
        aux["warm_l2_ms_per_step"] = None   # one set already exceeds L2: cold == warm
    lat_dev, lat_wall = [], []
    a0 = w.arglist(0)
    for _ in range(3 if wl_name == "nbody" else 10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        start.record(stream)
        f1 = M.mw_run(ctx, w.tree, a0, stream=stream)
        stop.record(stream)
        torch.cuda.synchronize()
        lat_wall.append(1e3 * (time.perf_counter() - t0))
        lat_dev.append(start.elapsed_time(stop))
        del f1
    aux["single_step_ms"] = statistics.median(lat_dev)
    aux["single_step_wall_ms"] = statistics.median(lat_wall)
    if hasattr(w, "extra_aux"):
        aux.update(w.extra_aux(timed, start, stop, stream))
    pk = peaks()
    # roofline of the dominant kernel class: algorithmic bytes (flops) of its
    # launches in the timed region / their CUDA-event-measured duration
    nlaunch = {cls: n for cls, (_, n) in kstats.items()}
    alu_peak = alu_peaks(pk)
    breakdown = []
    for cls, (kms, kn) in kstats.items():
        if kn == 0:
            continue
        b = w.roof_bytes(cls, nlaunch, mk, res)
        bd = w.bound_of(cls, nlaunch, mk)
        scale = 1e12 if bd == "alu" else 1e9
        breakdown.append({"class": KCLASS[cls], "bound": bd, "launches": kn, "ms": round(kms, 4),
                          "share": None,
                          "achieved": (b / (kms / 1e3) / scale) if kms > 0 and b else None})
    tot = sum(x["ms"] for x in breakdown) or 1.0
    for x in breakdown:
        x["share"] = round(x["ms"] / tot, 4)
    ksrc = "monitored pass: CUDA events around each launch of the dominant kernel class"
    if breakdown:
        dom = max(breakdown, key=lambda x: x["ms"])
        kms, kn, bound = dom["ms"], dom["launches"], dom["bound"]
        achieved = dom["achieved"] or 0.0
        kname = dom["class"]
        if len(breakdown) == 1 and launches == args.steps and bound != "alu":
            # one launch per step: the timed region itself gives the launch duration
            kms, kn = ms, launches
            achieved = w.roof_bytes(w.kclass, nlaunch, args.steps, res) / (ms / 1e3) / 1e9
            ksrc = "timed region (one launch per step): CUDA events on the launch stream / K"
    else:   # graph replay: no per-launch events; use the step time
        kms, kn, kname, bound = ms, launches, KCLASS[w.kclass], w.bound
        achieved = w.roof_bytes(w.kclass, {}, args.steps, res) / (ms / 1e3) / 1e9
        ksrc = "timed region (graph replay, one kernel per step): CUDA events / K"
    if bound == "alu":
        peak, unit, src = alu_peak["nbody" if wl_name == "nbody" else "hysteresis"]
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": unit,
                "frac": achieved / peak, "traffic": traffic_from_profile(wl_name),
                "peak_src": src, "kernel": kname,
                "kernel_launches": kn, "kernel_avg_us": 1e3 * kms / max(1, kn),
                "kernel_time_source": ksrc}
        if wl_name == "nbody":
            roof["flop_per_interaction"] = 20
    else:
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": traffic_from_profile(wl_name),
                "peak_src": pk["src"], "kernel": kname, "kernel_launches": kn,
                "kernel_avg_us": 1e3 * kms / max(1, kn), "kernel_time_source": ksrc}
    line = {"metric": METRIC, "value": value, "unit": w.unit, "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": w.dtype, "data": "synthetic (SplitMix64 seeded, generated on device per rank)",
            "config": dict(w.config(), parallelism=f"rows/slabs/bodies over {dist.world} GPU(s)",
                           partitions=dist.world * args.parts),
            "roofline": roof, "kernels": breakdown, "gpu_launches": launches,
            "clocks": clocks.summary(), "trials": args.trials, "aux": aux}
    if comm is not None:
        line["comm"] = comm
    if wl_name == "hysteresis":
        line["config"]["executions_E"] = res["executions"]
        line["pixel_executions_per_s"] = value * res["executions"]
    if wl_name == "nbody":
        line["interactions_per_s"] = value * w.N
    if wl_name == "fft":
        import math
        line["gflops_5nlogn"] = value * 2 * 5 * w.N * math.log2(w.N) / 1e9
    # end to end through the C-ABI with HOST buffers (H2D + run + D2H per step)
    if w.e2e_mode:
        h2d, d2h = w.e2e_setup()
        ek = max(3, min(args.steps, 20))
        f = w.e2e_step()
        f.wait()
        torch.cuda.synchronize()
        dist.barrier()
        start.record(stream)
        for es in getattr(w, "e2e_streams", []):
            es.wait_stream(stream)
        futs = [w.e2e_step() for _ in range(ek)]
        for es in getattr(w, "e2e_streams", []):
            stream.wait_stream(es)
        stop.record(stream)
        torch.cuda.synchronize()
        del futs
        ems = dist.max(start.elapsed_time(stop))
        line["e2e"] = {"value": w.units * ek / (ems / 1e3), "unit": w.unit,
                       "h2d_bytes_per_step": h2d * dist.world, "d2h_bytes_per_step": d2h * dist.world,
                       "steps": ek,
                       "path": ("mw_run with MW_LOC_HOST pinned buffers (library-staged chunked "
                                "H2D/compute/D2H overlap on 3 streams)" if w.e2e_mode == "staged" else
                                "pinned H2D of the inputs + mw_run + D2H of the result, two device "
                                "buffer sets on two streams (uploads of step i+1 overlap downloads of "
                                "step i; runs in FIFO order) (tree not host-stageable)")}
    else:
        line["e2e"] = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
        rate, sample, spent = cpu_rate(w.name, args.cpu_budget)
        line["cpu_baseline"] = {"value": rate, "unit": w.unit, "cores": 1, "kind": "oracle",
                                "sample": sample, "seconds": round(spent, 2), **host_info()}
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    ctx.destroy()


def run_rebalance_scenario(args, dist):
    """§8 a9 on one GPU (the E5 analogue): the fused Filter
    Pipeline on a 16384^2 image split into P = 8 virtual partitions; from run
    10 to 29 partition 3 computes 4x slower (slowdown injector, the analogue of
    the paper's CPU-load generator P:1110-1113); after every run the monitor /
    rebalancer runs (mw_rebalance: lbt trigger + proportional re-derivation).
    Reports when it triggered, the distributions and per-partition times, and
    that the output is bitwise identical to the one-partition run."""
    import torch

    import synth
    from paper_1510_06585_b200 import marrow as M
    from paper_1510_06585_b200 import trees
    if dist.world != 1:
        if dist.rank == 0:
            print(json.dumps({"workload": "rebalance", "skipped": "runs on one GPU (virtual partitions)"}))
        return
    H = W = 16384   # big enough that every partition's launch is well above launch latency
    P, runs = 8, 40
    ctx = M.mw_ctx_create(0, 0, 1, P)
    src = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
    synth.dev_fill_rgba(src, synth.SEED_IMAGE, 0)
    dst = torch.empty_like(src)
    node = trees.filter_pipeline()
    for _ in range(5):   # warm-up runs, not monitored
        M.mw_run(ctx, node, [M.arg(src), M.arg(dst)]).wait()
    trace = []
    for k in range(runs):
        M.mw_ctx_set_slowdown(ctx, 3, 4.0 if 10 <= k < 30 else 1.0)
        M.mw_run(ctx, node, [M.arg(src), M.arg(dst)]).wait()
        ms, wall = M.mw_last_timings(ctx)
        rows = M.mw_last_lengths(ctx)
        trig = M.mw_rebalance(ctx)
        st = M.mw_get_balance_state(ctx)
        trace.append({"run": k, "wall_ms": round(wall, 4), "part_ms": [round(x, 4) for x in ms],
                      "rows": rows, "lbt": round(st.lbt, 4), "triggered": trig,
                      "next_dist": [round(x, 4) for x in M.mw_get_distribution(ctx)]})
    ref = torch.empty_like(src)
    c1 = M.mw_ctx_create(0, 0, 1, 1)
    M.mw_run(c1, node, [M.arg(src), M.arg(ref)]).wait()
    same = bool(torch.equal(dst, ref))
    line = {"workload": "filter_rebalance_16384x16384_8parts",
            "metric": "online rebalancing (lbt trigger, proportional re-derivation) under an "
                      "injected 4x slowdown of partition 3 during runs 10-29",
            "trigger_runs": [t["run"] for t in trace if t["triggered"]],
            "bitwise_identical_to_one_partition_run": same,
            "wall_ms": {"balanced": trace[9]["wall_ms"], "slowed_before_rebalance": trace[11]["wall_ms"],
                        "slowed_after_rebalance": trace[25]["wall_ms"],
                        "recovered": trace[39]["wall_ms"]},
            "rows_while_slowed": trace[25]["rows"], "rows_after_recovery": trace[39]["rows"],
            "trace": trace}
    print(json.dumps(line), flush=True)
    ctx.destroy()
    c1.destroy()


def run_rebalance_nbody(args, dist):
    """SURVEY §8(d) C5b rebalance scenario (the analogue of P:1101-1119): the
    2^20-body N-body loop on P = 8 partitions (virtual devices on one GPU),
    40 steps; partition 3 computes 2x slower (slowdown injector: its step is
    repeated) during steps 10-29; after every step the monitor / rebalancer
    runs (mw_rebalance: lbt trigger after three unbalanced runs, proportional
    re-derivation).  A second context without rebalancing runs the same
    trajectory in lockstep: positions and velocities must be bitwise equal at
    every step (COPY state: the distribution never changes the result)."""
    import torch

    import synth
    from paper_1510_06585_b200 import marrow as M
    from paper_1510_06585_b200 import trees
    if dist.world != 1:
        if dist.rank == 0:
            print(json.dumps({"workload": "rebalance_nbody", "skipped": "runs on one GPU (virtual partitions)"}))
        return
    N, P, steps = 1 << 20, 8, 40
    ctx = M.mw_ctx_create(0, 0, 1, P)
    ref = M.mw_ctx_create(0, 0, 1, 1)
    M.mw_ctx_set_monitoring(ref, False)
    pos = torch.empty((N, 4), dtype=torch.float32, device="cuda")
    vel = torch.empty((N, 4), dtype=torch.float32, device="cuda")
    synth.dev_fill_nbody(pos, vel, synth.SEED_NBODY, 0, 2.0 ** -20)
    pr, vr = pos.clone(), vel.clone()
    node = trees.nbody(1)
    a = M.ArgList([M.arg(pos, M.MW_COPY), M.arg(vel, M.MW_COPY)])
    ar = M.ArgList([M.arg(pr, M.MW_COPY), M.arg(vr, M.MW_COPY)])
    trace, identical = [], True
    for k in range(steps):
        M.mw_ctx_set_slowdown(ctx, 3, 2.0 if 10 <= k < 30 else 1.0)
        M.mw_run(ctx, node, a).wait()
        M.mw_run(ref, node, ar).wait()
        same = bool(torch.equal(pos, pr)) and bool(torch.equal(vel, vr))
        identical &= same
        ms, wall = M.mw_last_timings(ctx)
        lens = M.mw_last_lengths(ctx)
        act = [x for x, n in zip(ms, lens) if n > 0]
        dev = min(act) / max(act)
        trig = M.mw_rebalance(ctx)
        st = M.mw_get_balance_state(ctx)
        trace.append({"step": k, "slowed": 10 <= k < 30, "wall_ms": round(wall, 3),
                      "part_ms": [round(x, 3) for x in ms], "bodies": lens, "dev": round(dev, 4),
                      "lbt": round(st.lbt, 4), "triggered": trig, "bitwise_equal": same,
                      "next_dist": [round(x, 5) for x in M.mw_get_distribution(ctx)]})
    trig_steps = [t["step"] for t in trace if t["triggered"]]
    line = {"workload": "nbody_rebalance_2^20_8parts",
            "metric": "online rebalancing (lbt trigger, proportional re-derivation) under a 2x "
                      "slowdown of partition 3 during steps 10-29 (SURVEY 8(d) C5b)",
            "trigger_steps": trig_steps,
            "positions_bitwise_identical_every_step": identical,
            "dev_after_first_trigger_min": min((t["dev"] for t in trace
                                                if trig_steps and trig_steps[0] < t["step"] < 30), default=None),
            "share_of_partition_3_while_slowed": trace[25]["next_dist"][3],
            "share_of_others_while_slowed": trace[25]["next_dist"][0],
            "wall_ms": {"balanced": trace[9]["wall_ms"], "slowed_before_rebalance": trace[11]["wall_ms"],
                        "slowed_after_rebalance": trace[25]["wall_ms"], "recovered": trace[39]["wall_ms"]},
            "trace": trace}
    print(json.dumps(line), flush=True)


def traffic_from_profile(wl_name):
    """dram bytes (read + write) per launch of the dominant kernel, from the
    committed `ncu --set full` summary under profiles/ (null if absent)."""
    path = os.path.join(ROOT, "profiles", "dram_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(wl_name)
    except Exception:
        return None


def self_launch(n):
    """`python bench.py --gpus N` outside torchrun: start N local ranks (one
    process per GPU, the torchrun environment on 127.0.0.1), forward rank 0's
    JSON line, exit with the worst return code.  NCCL's INFO log (init: rank
    and nranks of every communicator) goes to stderr so stdout keeps one line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    rcs = [p.wait() for p in procs]
    sys.exit(max(rcs, key=abs))


def main():
    if "WORLD_SIZE" not in os.environ:
        for i, a in enumerate(sys.argv):
            g = a.split("=", 1)[1] if a.startswith("--gpus=") else (
                sys.argv[i + 1] if a == "--gpus" and i + 1 < len(sys.argv) else None)
            if g is not None and int(g) > 1:
                self_launch(int(g))
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="marrow", choices=["marrow", "reference"])
    ap.add_argument("--workload", default="filter",
                    choices=list(WORKLOADS) + ["all", "rebalance", "rebalance_nbody"])
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--trials", type=int, default=5,
                    help="timed trials of K steps; the line reports the median (min/max in aux)")
    ap.add_argument("--parts", type=int, default=1,
                    help="virtual partitions per GPU (uniform distribution vector)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        if int(os.environ.get("RANK", "0")) != 0:
            return   # the reference arm runs on rank 0 alone; the other ranks exit 0
        dist = Dist.__new__(Dist)
        dist.world, dist.rank, dist.local, dist.pg = args.gpus, 0, 0, None
    else:
        dist = Dist(args.gpus)
    if args.impl == "reference":
        if args.steps is None:
            args.steps = 10
        run_reference(args, dist)
        return
    if args.workload == "rebalance_nbody":
        run_rebalance_nbody(args, dist)
        return
    if args.workload == "rebalance":
        run_rebalance_scenario(args, dist)
        return
    names = list(WORKLOADS) if args.workload == "all" else [args.workload]
    # K per trial (x `--trials`): short enough that the default run stays
    # below the ~0.2 s of continuous load after which the power cap lowers
    # the SM clock (scripts/probe_power.py)
    default_steps = {"filter": 200, "saxpy": 4992, "segmentation": 200, "mapreduce_sum": 60,
                     "mapreduce_dot": 40, "mapreduce_max": 40, "hysteresis": 20, "nbody": 3, "fft": 100}
    user_steps = args.steps
    for n in names:
        args.steps = user_steps or default_steps[n]
        run_marrow(args, dist, n)
    if dist.pg:
        dist.pg.destroy_process_group()


if __name__ == "__main__":
    main()
