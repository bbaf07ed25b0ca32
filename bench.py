"""Benchmark: D8 flow accumulation Gcells/s on B200 (BASELINE.json metric).

Workload (N=1): config 3 of BASELINE.json -- 32768 x 32768 float32 fractal DEM
(seed 4), 10% NoData coast, depression-filled, f32 weights U(0.5,1.5) on a
2^-23 grid, fp64 accumulation, 4096 x 4096 tiles.  One step = one call of the
whole hot path (H1 D8 -> H2-H4 pass 1 -> H5 graph -> H6 pass 2) through the
C ABI on device-resident inputs.  Inputs (8 GiB) and the output (8 GiB) are far
larger than the 126 MB L2, so no explicit flush is needed between steps.

`--impl reference` times the CPU oracle (the paper's method as the oracle
implements it, single-threaded) on a bounded sample of the same workload.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
       (N > 1: launched under torchrun, one rank per GPU, row strips.)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "D8 flow-accum Gcells/s at 1/2/4/8 B200; achieved % of HBM roofline"
CFG = "cfg3"
# algorithmic bytes per cell (DESIGN.md §6 "Roofline"): each kernel's own
# input + output, once per cell.  cfg3: f32 w -> f64; cfg4: w = 1 -> u64.
SPECS = {
    "cfg3": {"atype": "f64", "weighted": True, "bytes_min": 16, "bytes_d8": 5, "bytes_block": 13,
             "desc": "32768x32768 f32 DEM seed 4, 10% NoData, filled, f32 w -> f64"},
    "cfg4": {"atype": "u64", "weighted": False, "bytes_min": 12, "bytes_d8": 5, "bytes_block": 9,
             "desc": "131072x131072 f32 DEM seed 5, 30% NoData, filled, w = 1 -> u64"},
}
BYTES_MIN = 16        # z 4 + w 4 + A 8                    (whole path: method input + output)
BYTES_D8 = 5          # z 4 -> dirs 1                      (k_d8, H1)
BYTES_BLOCK = 13      # dirs 1 + w 4 -> A_blk 8 (in place) (k_pass1: H2-H4, RETAIN accumulation + records)


def select_config(name):
    global CFG, BYTES_MIN, BYTES_D8, BYTES_BLOCK
    CFG = name
    s = SPECS[name]
    BYTES_MIN, BYTES_D8, BYTES_BLOCK = s["bytes_min"], s["bytes_d8"], s["bytes_block"]
HBM_FALLBACK = 6650.0


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


class Clocks:
    """Sample SM clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            p = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_inputs(rows=None):
    import inputs

    t0 = time.time()
    cfg = inputs.make_config(CFG, rows, rows)
    return cfg, time.time() - t0


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample(cfg, max_rows=4096, characterise=False):
    """The oracle (as it stands) on a bounded sample: the first `max_rows` rows
    of the workload, full width, D8 + fp64 accumulation (single thread).
    With `characterise`, the oracle's workload statistics of the same sample
    (longest flow path, outlets, NoFlow, max A, height
    histogram) are added."""
    import oracle

    r = min(max_rows, cfg.rows)
    z = np.ascontiguousarray(cfg.dem[:r])
    w = np.ascontiguousarray(cfg.w[:r]) if cfg.w is not None else None
    t0 = time.perf_counter()
    d = oracle.d8(z)
    t1 = time.perf_counter()
    if w is not None:
        oracle.accumulate(d, w, kind="f64")
    else:
        oracle.accumulate(d)
    t2 = time.perf_counter()
    cells = r * cfg.cols
    out = {"value": cells / (t2 - t0) / 1e9, "unit": "Gcells/s", "cores": 1, "kind": "oracle",
           "sample": f"rows [0,{r}) x {cfg.cols} cols of {CFG} (O-D8 + O-ACC "
                     f"{'fp64' if w is not None else 'u64'} Kahn, one thread), "
                     f"{t2 - t0:.1f} s",
           "d8_gcells_s": cells / (t1 - t0) / 1e9, "acc_gcells_s": cells / (t2 - t1) / 1e9,
           "nproc": os.cpu_count(), "cpu_model": cpu_model()}
    if characterise:
        st = oracle.stats(d, nbins=16)
        hist = [int(x) for x in st["height_hist"]]
        data = int((d != 255).sum())
        out["workload"] = {
            "sample_cells": cells, "data_cells": data, "nodata_frac": round(1 - data / cells, 4),
            "longest_flow_path": int(st["max_height"]), "outlets": int(st["outlets"]),
            "noflow": int(st["noflow"]), "max_acc_unit_w": int(st["max_acc"]),
            "height_hist_0_to_14_and_15plus": hist,
            "sources_frac": round(hist[0] / data, 4)}
    return out


def arm_config(cfg, world):
    """The `config` object both arms print (the workload, no model keys)."""
    return {"workload": f"{CFG}: {SPECS[CFG]['desc'].split(' ', 1)[1]}"
                        + (f" (run at {cfg.rows}x{cfg.cols})" if cfg.rows != int(SPECS[CFG]['desc'].split('x')[0]) else "")
                        + f", {cfg.tile[0]}x{cfg.tile[1]} tiles",
            "parallelism": f"row strips x{world} (NCCL)" if world > 1 else "single GPU",
            "tiling": ("one GPU: every tile is resident, so the tiles and the perimeter graph are solved as "
                       "one uncut graph over the 32x32 block exits (identical results, linearity); the "
                       f"{cfg.tile[0]}x{cfg.tile[1]} tiles set the records and the strip / multi-GPU exchange")
            if world == 1 else f"{cfg.tile[0]}x{cfg.tile[1]} tiles, tile records all-gathered (C2)",
            "l2": "inputs and output (GiBs) >> 126 MB L2 (no flush needed)",
            "nodata_frac": round(float(cfg.meta.get("nodata_frac", 0.0)), 4)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, _ = make_inputs(args.rows)
    sample_rows = min(1024, cfg.rows)
    for _ in range(args.warmup):
        cpu_sample(cfg, sample_rows)
    vals = [cpu_sample(cfg, sample_rows) for _ in range(args.steps)]
    v = float(np.median([x["value"] for x in vals]))
    cb = dict(vals[0])
    cb["value"] = v
    ms = sample_rows * cfg.cols / (v * 1e9) * 1e3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {"metric": METRIC, "value": v, "unit": "Gcells/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": SPECS[CFG]["atype"],
            "data": "synthetic", "impl": "reference",
            "config": arm_config(cfg, world),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "Gcells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def shared_inputs(args, world, rank):
    """World 1: generate in-process.  World > 1: rank 0 generates once into
    shared memory, the other ranks map it (each then uploads only its strip)."""
    import torch.distributed as dist

    if world == 1:
        cfg, gen_s = make_inputs(args.rows)
        return cfg, gen_s
    shm = os.environ.get("FA_BENCH_SHM", "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp")
    base = os.path.join(shm, f"fa_bench_{os.environ.get('MASTER_PORT', '0')}")
    gen_s = 0.0
    if rank == 0:
        cfg, gen_s = make_inputs(args.rows)
        np.save(base + "_z.npy", cfg.dem)
        if cfg.w is not None:
            np.save(base + "_w.npy", cfg.w)
        meta = [cfg.rows, cfg.cols, cfg.tile[0], cfg.tile[1], cfg.meta.get("nodata_frac", 0.0)]
    else:
        meta = None
    obj = [meta]
    dist.broadcast_object_list(obj, src=0)
    dist.barrier()
    import inputs

    rows, cols, tr, tc, ndf = obj[0]
    spec = SPECS[CFG]
    cfg = inputs.Config(name=CFG, rows=rows, cols=cols, tile=(tr, tc), atype=spec["atype"],
                        dem=np.load(base + "_z.npy", mmap_mode="r"),
                        w=np.load(base + "_w.npy", mmap_mode="r") if spec["weighted"] else None,
                        meta={"nodata_frac": ndf})
    return cfg, gen_s


def gpu_numa_affinity(index: int):
    """Bind this process to the CPUs of the GPU's NUMA node, so pinned host
    buffers are first touched (allocated) on that node; returns the node."""
    try:
        import torch

        bus = torch.cuda.get_device_properties(index).pci_bus_id if hasattr(
            torch.cuda.get_device_properties(index), "pci_bus_id") else None
        if bus is None:
            import pynvml

            pynvml.nvmlInit()
            bus = pynvml.nvmlDeviceGetPciInfo(pynvml.nvmlDeviceGetHandleByIndex(index)).busId
            bus = bus.decode() if isinstance(bus, bytes) else bus
        bus = bus.lower()
        if len(bus.split(":")[0]) == 8:  # nvml: 00000000:1B:00.0 -> sysfs 0000:1b:00.0
            bus = bus[4:]
        node = int(open(f"/sys/bus/pci/devices/{bus}/numa_node").read())
        if node < 0:
            return None
        cpus = set()
        for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
            a, _, e = part.partition("-")
            cpus.update(range(int(a), int(e or a) + 1))
        os.sched_setaffinity(0, cpus)
        return node
    except Exception:
        return None


def pcie_rates(torch, stream, h_in, d_in, h_out, d_out):
    """Copy bandwidth per direction on the bench's own pinned buffers (GB/s)."""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(stream):
        for t, s in zip(d_in, h_in):
            t.copy_(s, non_blocking=True)  # warm-up
        ev[0].record(stream)
        for t, s in zip(d_in, h_in):
            t.copy_(s, non_blocking=True)
        ev[1].record(stream)
        ev[2].record(stream)
        h_out.copy_(d_out, non_blocking=True)
        ev[3].record(stream)
    stream.synchronize()
    nin = sum(t.numel() * t.element_size() for t in h_in)
    nout = h_out.numel() * h_out.element_size()
    # both directions at once (two streams): the bound of a pipelined queue of rasters
    s2 = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    done2 = torch.cuda.Event()
    torch.cuda.synchronize()
    e0.record(stream)
    s2.wait_event(e0)
    with torch.cuda.stream(stream):
        for t, s in zip(d_in, h_in):
            t.copy_(s, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
        done2.record(s2)
    stream.wait_event(done2)
    e1.record(stream)
    stream.synchronize()
    return {"h2d_gbs": nin / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9,
            "d2h_gbs": nout / (ev[2].elapsed_time(ev[3]) * 1e-3) / 1e9,
            "both_ms": e0.elapsed_time(e1), "both_gbs": (nin + nout) / (e0.elapsed_time(e1) * 1e-3) / 1e9}


SMALL = (("cfg0", 8, "512^2 DEM seed 1, filled, w=1 -> u32, 1 tile (launch-bound; no roofline claim)"),
         ("cfg1", 8, "8192^2 DEM seed 2, 5% NoData, filled, w=1 -> u32, 2048^2 tiles"),
         ("cfg2", 5, "4096^2 D8 serpentine (depth 16.7M), w=1 -> u32, 1 tile"))


def small_configs(torch, fa, local, stream, peak, steps=10):
    """BASELINE.json configs 0-2 on this GPU (the parity configs, timed the
    same way as the headline: device-resident inputs, CUDA events around
    `steps` calls of fa_accumulate, each call returning after completion)."""
    import inputs

    out = {}
    for name, bpc, desc in SMALL:
        cfg = inputs.make_config(name)
        with torch.cuda.stream(stream):
            src = torch.from_numpy(cfg.dem if cfg.dem is not None else cfg.dirs).cuda()
            acc = torch.empty((cfg.rows, cfg.cols), dtype=torch.uint32, device="cuda")
        stream.synchronize()
        kw = {"dem": src} if cfg.dem is not None else {"dirs": src}
        with fa.Context(local, stream=stream, tile=cfg.tile) as c:
            for _ in range(3):
                c.accumulate(atype="u32", out=acc, **kw)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                c.accumulate(atype="u32", out=acc, **kw)
            e1.record(stream)
            e1.synchronize()
            st = c.stats()
        ms = e0.elapsed_time(e1) / steps
        cells = cfg.rows * cfg.cols
        gbs = cells * bpc / (ms * 1e-3) / 1e9
        out[name] = {"workload": desc, "value": cells / (ms * 1e-3) / 1e9, "unit": "Gcells/s", "ms_per_step": ms,
                     "bytes_per_cell": bpc, "roofline_frac": gbs / peak,
                     "phases_ms": {"pass1": st["ms_pass1"], "graph": st["ms_graph"], "pass2": st["ms_pass2"]},
                     "graph_nodes": int(st["graph_nodes"]), "launches": int(st["launches"])}
        del src, acc
    return out


def run_gpu(args):
    import torch

    from paper_1608_04431_b200 import fa

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    cfg, gen_s = shared_inputs(args, world, rank)
    H, W = cfg.rows, cfg.cols
    if world > 1:
        from paper_1608_04431_b200 import dist as fdist

        r0, nr = fdist.strip_bounds(H, cfg.tile[0], rank, world)
        nid = fdist.broadcast_nccl_id()
    else:
        r0, nr = 0, H
    atype = SPECS[CFG]["atype"]
    adt = torch.float64 if atype == "f64" else torch.uint64
    # memory: z 4 + A 8 + dirs 1 B per cell, plus ~10 B of pass-1 / graph state
    need = nr * W * 23
    free = torch.cuda.mem_get_info(local)[0]
    if need > free:
        sys.stderr.write(f"bench.py: {CFG} needs ~{need / 1e9:.0f} GB per GPU at {world} GPU(s); "
                         f"{free / 1e9:.0f} GB free (cfg4 runs on 8 GPUs)\n")
        sys.exit(2)
    z_np = np.ascontiguousarray(cfg.dem[r0:r0 + nr])
    w_np = np.ascontiguousarray(cfg.w[r0:r0 + nr]) if cfg.w is not None else None
    stream = torch.cuda.Stream()
    ctx = fa.Context(local, stream=stream, tile=cfg.tile)
    with torch.cuda.stream(stream):
        dz = torch.from_numpy(z_np).cuda()
        dw = torch.from_numpy(w_np).cuda() if w_np is not None else None
        acc = torch.empty((nr, W), dtype=adt, device="cuda")
    stream.synchronize()

    def call(dem, w, out):
        if world > 1:
            ctx.accumulate_dist(nid, rank, world, H, r0, dem=dem, w=w, atype=atype, out=out)
        else:
            ctx.accumulate(dem=dem, w=w, atype=atype, out=out)

    for _ in range(max(args.warmup, 3)):
        call(dz, dw, acc)
    torch.cuda.synchronize()
    p1, gr, p2, launches, kd8, kblk = [], [], [], [], [], []
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            call(dz, dw, acc)
            s = ctx.stats()
            p1.append(s["ms_pass1"])
            gr.append(s["ms_graph"])
            p2.append(s["ms_pass2"])
            kd8.append(s.get("ms_d8", 0.0))
            kblk.append(s.get("ms_block", 0.0))
            launches.append(s.get("launches", 0))
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = H * W / (ms * 1e-3) / 1e9

    # ---- e2e: the same public call with pinned HOST inputs/outputs: H2D of
    # z and w and D2H of A inside the timed region (the library stages host
    # buffers itself on one GPU; the multi-GPU call takes device buffers, so
    # the copies are issued here on the same stream)
    numa = gpu_numa_affinity(local)  # pinned buffers on the GPU's NUMA node
    hz = torch.from_numpy(z_np).pin_memory()
    hw = torch.from_numpy(w_np).pin_memory() if w_np is not None else None
    ha = torch.empty((nr, W), dtype=adt).pin_memory()
    pcie = pcie_rates(torch, stream, [x for x in (hz, hw) if x is not None], [x for x in (dz, dw) if x is not None],
                      ha, acc)

    def e2e_call():
        if world > 1:
            with torch.cuda.stream(stream):
                dz.copy_(hz, non_blocking=True)
                if dw is not None:
                    dw.copy_(hw, non_blocking=True)
            call(dz, dw, acc)
            with torch.cuda.stream(stream):
                ha.copy_(acc, non_blocking=True)
            stream.synchronize()
        else:
            call(hz, hw, ha)

    e2e_call()  # warm-up
    e2e_steps = max(1, min(args.steps, 3))
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": H * W / (e2e_ms * 1e-3) / 1e9, "unit": "Gcells/s",
           "h2d_bytes_per_step": int(hz.numel() * 4 + (hw.numel() * 4 if hw is not None else 0)) * world,
           "d2h_bytes_per_step": int(ha.numel() * adt.itemsize) * world, "ms_per_step": e2e_ms,
           "pcie_h2d_gbs": round(pcie["h2d_gbs"], 1), "pcie_d2h_gbs": round(pcie["d2h_gbs"], 1),
           "pcie_both_directions_gbs": round(pcie["both_gbs"], 1),
           "pcie_both_directions_ms": round(pcie["both_ms"], 1),
           "pinned_numa_node": numa,
           "call": "fa_accumulate with pinned host buffers (the library stages them through the device)"}
    if world == 1 and not args.no_batch:
        # a queue of K rasters through fa_accumulate_batch: every step still
        # uploads its z and w and downloads its A (same pinned buffers), but
        # the upload of raster i+1 and the download of raster i-1 overlap the
        # device work of raster i (PCIe is full duplex).  Pipeline fill and
        # drain are inside the timed region.
        nb = max(args.steps, 3)
        ctx.accumulate_batch(dems=[hz] * 2, ws=[hw] * 2 if hw is not None else None, atype=atype,
                             outs=[ha] * 2)  # warm-up (device buffer sets into the pool)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.accumulate_batch(dems=[hz] * nb, ws=[hw] * nb if hw is not None else None, atype=atype, outs=[ha] * nb)
        b_ms = (time.perf_counter() - t0) * 1e3 / nb
        sb = ctx.stats()
        single = {k: e2e[k] for k in ("value", "ms_per_step", "call")}
        e2e.update({"value": H * W / (b_ms * 1e-3) / 1e9, "ms_per_step": b_ms, "rasters": nb,
                    "device_ms_per_raster": sb["ms_compute"] / nb,
                    "call": f"fa_accumulate_batch over {nb} rasters (pinned host buffers; each step uploads its z, w "
                            "and downloads its A; raster i+1's upload and raster i-1's download overlap raster i)",
                    "single_call": single})

    # ---- out-of-core path (N2): the same workload streamed from the pinned
    # host buffers one tile row (4096 rows) at a time, z and w uploaded twice
    ooc = None
    extras = world == 1 and not args.no_ooc and CFG == "cfg3"
    if extras:
        sr = cfg.tile[0]
        ctx.accumulate_streamed(dem=hz, w=hw, atype="f64", strip_rows=sr, out=ha)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ctx.accumulate_streamed(dem=hz, w=hw, atype="f64", strip_rows=sr, out=ha)
        ooc_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
        so = ctx.stats()
        ooc = {"value": H * W / (ooc_ms * 1e-3) / 1e9, "unit": "Gcells/s", "ms_per_step": ooc_ms,
               "strip_rows": sr, "strips": -(-H // sr), "pcie_bytes_per_step": so["bytes_exchanged"],
               "pcie_gbs_both_directions": so["bytes_exchanged"] / (ooc_ms * 1e-3) / 1e9,
               "call": "fa_accumulate_streamed (host buffers, pinned)"}

    # ---- absorption (N3): the same workload with a per-cell alpha ~ U[0.9, 1)
    # (seeded, generated on the device), device-resident, library CUDA events
    absorb = None
    if extras:
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        with torch.cuda.stream(stream):
            al = 0.9 + 0.1 * torch.rand((nr, W), generator=g, device="cuda", dtype=torch.float32)
        stream.synchronize()
        ctx.accumulate_absorb(al, dem=dz, w=dw, out=acc)  # warm-up
        ts = []
        for _ in range(3):
            ctx.accumulate_absorb(al, dem=dz, w=dw, out=acc)
            ts.append(ctx.stats()["ms_total"])
        ams = float(np.median(ts))
        absorb = {"value": H * W / (ams * 1e-3) / 1e9, "unit": "Gcells/s", "ms_per_step": ams,
                  "alpha": "U[0.9,1) seed 5", "call": "fa_accumulate_absorb (device buffers)"}
        del al

    # ---- depression filling (N4): fa_fill on cfg3's unfilled terrain (G2 + G3)
    fillm = None
    if extras and args.rows is None:
        import inputs

        zr = inputs.terrain(4, H, W)
        inputs.coast(zr, 4, 0.10)
        with torch.cuda.stream(stream):
            dzr = torch.from_numpy(zr).cuda()
            zf = torch.empty_like(dzr)
        stream.synchronize()
        ctx.fill(dzr, out=zf)  # warm-up
        fts = []
        for _ in range(2):
            ctx.fill(dzr, out=zf)
            fts.append(ctx.stats())
        fms = float(np.median([t["ms_total"] for t in fts]))
        ok = bool(torch.equal(zf, dz))  # the bench DEM is this terrain filled on the CPU (G4)
        fillm = {"value": H * W / (fms * 1e-3) / 1e9, "unit": "Gcells/s", "ms_per_step": fms,
                 "launches": int(fts[-1]["launches"]), "equals_cpu_fill": ok,
                 "call": "fa_fill (device buffers, unfilled cfg3 terrain)"}
        del dzr, zf

    peak, peak_src = hbm_peak()
    mp1, mgr, mp2 = float(np.mean(p1)), float(np.mean(gr)), float(np.mean(p2))
    md8, mblk = float(np.mean(kd8)), float(np.mean(kblk))
    # dominant kernel: the pass-1 block kernel, timed alone by the library with
    # CUDA events recorded on its launch stream around the launch
    dom, dom_ms, dom_bytes = "k_pass1", (mblk if mblk > 0 else mp1), BYTES_BLOCK
    achieved = nr * W * dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom)
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "Gcells/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": atype,
        "data": "synthetic",
        "config": arm_config(cfg, world),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_cell": dom_bytes,
                     "whole_path": {"bytes_per_cell": BYTES_MIN,
                                    "achieved": H * W * BYTES_MIN / (ms * 1e-3) / 1e9 / world,
                                    "frac": H * W * BYTES_MIN / (ms * 1e-3) / 1e9 / world / peak}},
        "phases_ms": {"pass1": mp1, "graph": mgr, "pass2": mp2},
        "kernels": {"k_d8": {"ms": md8, "bytes_per_cell": BYTES_D8,
                             "achieved_gbs": nr * W * BYTES_D8 / (md8 * 1e-3) / 1e9 if md8 > 0 else None},
                    "k_pass1": {"ms": mblk, "bytes_per_cell": BYTES_BLOCK,
                                "achieved_gbs": nr * W * BYTES_BLOCK / (mblk * 1e-3) / 1e9 if mblk > 0 else None}},
        "clocks": clk.summary(),
        "e2e": e2e,
        "out_of_core": ooc,
        "absorption": absorb,
        "fill": fillm,
        "gpu_launches": int(np.sum(launches)) if launches and launches[0] else None,
        "input_gen_s": round(gen_s, 1),
    }
    if extras:
        line["configs"] = small_configs(torch, fa, local, stream, peak)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_sample(cfg, 4096 if args.rows is None else min(4096, args.rows),
                                          characterise=True)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=None, help="smaller square variant (debug only)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ooc", action="store_true", help="skip the out-of-core and absorption measurements")
    ap.add_argument("--no-batch", action="store_true",
                    help="e2e from single fa_accumulate calls only (no fa_accumulate_batch queue)")
    ap.add_argument("--config", default="cfg3", choices=sorted(SPECS),
                    help="cfg3 (default; 1/2/4/8 GPUs) or cfg4 (17.2G cells, ~50 GB per GPU at 8 GPUs)")
    ap.add_argument("--gen-only", action="store_true", help="time the input generation on the host and exit")
    args = ap.parse_args()
    select_config(args.config)
    if args.gen_only:
        cfg, gen_s = make_inputs(args.rows)
        print(json.dumps({"config": CFG, "rows": cfg.rows, "cols": cfg.cols, "input_gen_s": round(gen_s, 1),
                          "cells": cfg.rows * cfg.cols, "nproc": os.cpu_count(),
                          "nodata_frac": round(float(cfg.meta.get("nodata_frac", 0.0)), 4)}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # not under torchrun: launch one rank per GPU ourselves (never time
        # N ranks on fewer GPUs -- fail loudly instead)
        import socket

        import torch

        ndev = torch.cuda.device_count()
        if ndev < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but this box has {ndev} CUDA device(s)\n")
            sys.exit(2)
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if world is not None and int(world) != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}\n")
        sys.exit(2)
    run_gpu(args)


if __name__ == "__main__":
    main()
