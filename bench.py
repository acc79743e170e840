"""Benchmark: SLICER IF codec encode+decode throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c2|c3|c4|c4sweep|c5]

One step = encode of the whole per-GPU batch of synthetic IFs (ATKF -> MS -> ABQ -> CSR
bit-pack -> .sif with CRC) followed by decode of those payloads back to dense fp32, inputs
resident in HBM.  N>1: one process per GPU (bench.py re-launches itself under
torch.distributed.run when WORLD_SIZE is unset), independent IF streams per rank
(sid = rank * B + i), no data-path collectives ("scaling": "weak"); the timing is the max
over ranks.  Every timed payload and decode is checked against digests of the
REFERENCE's own output for the same IF (tests/golden/workloads.npz) -> "parity".
`--impl reference` times the reference's CPU implementation of the path (slicer from
baseline/_ref when installed, else the oracle/ port) on the host cores on a bounded sample
of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import hashlib
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IF encode+decode GB/s per GPU (and 8-GPU aggregate) vs HBM roofline; bits/element"

CONFIGS = {
    # configs[0]: one ResNet IF round trip through the drop-in encode()/decode() (latency)
    "c1": dict(kind=0, rows=1024, cols=196, batch=1, dtype="fp32", latency=True,
               workload="C1: one ResNet-50 split-point IF 1x1024x14x14 fp32 round trip through the drop-in "
                        "encode()/decode() API (latency)"),
    # BASELINE.json configs[1]: ResNet-50 IF batch 256 (headline, N=1 workload)
    "c2": dict(kind=0, rows=1024, cols=196, batch=256, dtype="fp32", depth=4,
               workload="C2: ResNet-50 split-point IF 1x1024x14x14 fp32 (rows=1024 channels, cols=196), "
                        "batch 256 clients per GPU, synthetic ReLU-sparse"),
    # configs[2]: Llama decode-step hidden states, 1 token x 4096, 1024 clients
    "c3": dict(kind=1, rows=1, cols=4096, batch=1024, dtype="bf16", depth=8,
               workload="C3: Llama-class decode-step hidden state 1x4096 bf16, 1024 concurrent clients"),
    # configs[3]: Llama prefill IF 2048 x 4096 bf16, batch 32
    "c4": dict(kind=1, rows=2048, cols=4096, batch=32, dtype="bf16", depth=4,
               workload="C4: Llama-class prefill IF 2048x4096 bf16, batch 32"),
    # configs[3] sweep: BASELINE.md §4.2 grid on the C4 batch
    "c4sweep": dict(kind=1, rows=2048, cols=4096, batch=32, dtype="bf16", depth=2, sweep=True,
                    workload="C4 sweep: Llama-class prefill IF 2048x4096 bf16, batch 32, s x delta x lambda grid "
                             "(BASELINE.md §4.2) plus fixed Q=[8,4,2]"),
    # configs[4]: 8192 independent client streams (mixed vision/LLM shapes) sharded over the
    # GPUs of the job (strong scaling: the 8192 are split, not replicated)
    "c5": dict(mixed=8192, dtype="mixed bf16/fp32", depth=2,
               workload="C5: 8192 independent client IF streams, mixed shapes by sid mod 8 (0-3 decode token "
                        "1x4096 bf16, 4-6 ResNet IF 1024x196 fp32, 7 prefill chunk 256x4096 bf16), sharded over "
                        "the job's GPUs by longest-processing-time on bytes"),
}
CODEC = dict(s=0.9, lam=0.0, m_plus=3, m_minus=3, q_bit=8, delta=0.01)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6552.0)), "measured"
    return 6650.0, "fallback"


def _ncu_traffic(config: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get(config)
    return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled with NVML every ~1 ms while the
    timed region runs (a background thread; nvidia-smi's 50 ms period is too coarse for a
    sub-second region)."""

    NAMES = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
             0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.max_mhz = None
        self._stop = None
        self._thr = None

    def _run(self):
        import pynvml

        h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
        get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), int(get_reasons(h))))
            except Exception:  # noqa: BLE001
                break
            time.sleep(0.001)

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._stop = threading.Event()
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        except Exception:  # noqa: BLE001
            self._thr = None
        return self

    def __exit__(self, *exc):
        if self._thr is not None:
            self._stop.set()
            self._thr.join(timeout=2)

    def summary(self):
        if not self.samples:
            return None
        mhz = [m for m, _ in self.samples]
        bits = 0
        for _, r in self.samples:
            bits |= r
        reasons = sorted(n for b, n in self.NAMES.items() if bits & b)
        return dict(sm_mhz=statistics.median(mhz), sm_max_mhz=self.max_mhz, reasons=reasons, samples=len(mhz),
                    source="nvml, 1 ms period")


# ------------------------------------------------------------------------- parity digests
def _golden():
    """Digests of the REFERENCE's payload / decoded bits for every benchmarked IF
    (tests/golden/make_workload_golden.py ran slicer itself), or None."""
    import numpy as np

    p = os.path.join(ROOT, "tests", "golden", "workloads.npz")
    return dict(np.load(p)) if os.path.exists(p) else None


def _sha16(b) -> bytes:
    return hashlib.sha256(b).digest()[:16]


class Parity:
    """Counts payloads / decodes compared with the reference digests."""

    def __init__(self, gold, name):
        self.g = gold
        self.name = name
        self.checked = 0
        self.mismatches = 0
        self.missing = 0

    def payload(self, sid, nbytes, digest):
        if self.g is None or f"{self.name}_len" not in self.g or sid >= len(self.g[f"{self.name}_len"]):
            self.missing += 1
            return
        self.checked += 1
        if int(self.g[f"{self.name}_len"][sid]) != int(nbytes) or \
                self.g[f"{self.name}_payload_sha"][sid].tobytes() != digest:
            self.mismatches += 1

    def decode(self, sid, digest):
        if self.g is None or f"{self.name}_dec_sha" not in self.g or sid >= len(self.g[f"{self.name}_dec_sha"]):
            self.missing += 1
            return
        self.checked += 1
        if self.g[f"{self.name}_dec_sha"][sid].tobytes() != digest:
            self.mismatches += 1

    def merged(self, pg):
        if pg is None:
            return self.checked, self.mismatches, self.missing
        import torch

        t = torch.tensor([self.checked, self.mismatches, self.missing], dtype=torch.int64)
        pg.all_reduce(t)
        return [int(v) for v in t]

    def summary(self, pg=None, what="every timed payload and decode"):
        c, m, x = self.merged(pg)
        return dict(checked=c, mismatches=m, unchecked=x, against="reference digests (tests/golden/workloads.npz, "
                    "generated by running slicer.encode/serialize/deserialize/decode on the same IFs)", what=what)


def _check_encoder(par, enc, sids, offs=None):
    """Payload digests of every IF of a BatchEncoder / ListEncoder (one D2H copy)."""
    lens = enc.out_len.cpu().numpy()
    host = enc.out.reshape(-1).cpu().numpy()
    if offs is None:
        offs = [i * enc.cap for i in range(len(sids))]
    for i, sid in enumerate(sids):
        par.payload(sid, lens[i], _sha16(host[offs[i]:offs[i] + int(lens[i])].tobytes()))
    return int(lens[: len(sids)].sum())


def _check_decoded(par, ys, sids):
    for y, sid in zip(ys, sids):
        par.decode(sid, _sha16(y.contiguous().cpu().numpy().reshape(-1).view("uint32").tobytes()))


# ------------------------------------------------------------------------- CPU arms
def _ref_path():
    p = os.path.join(ROOT, "baseline", "_ref")
    return p if os.path.exists(os.path.join(p, "slicer", "codec.py")) else None


def _cpu_worker(args):
    """One IF through the CPU implementation: 'reference' = the unmodified slicer package
    (baseline/_ref) via its public API, 'port' = the oracle/ NumPy restatement."""
    kind, rows, cols, sid, cfgd, impl = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np

    from oracle.synth import synth

    x = synth(kind, rows, cols, sid)
    if impl == "reference":
        rp = _ref_path()
        if rp not in sys.path:
            sys.path.insert(0, rp)
        import slicer

        cfg = slicer.CodecConfig(**cfgd)
        t0 = time.perf_counter()
        blob = slicer.serialize(slicer.encode(slicer.DenseTensor(rows, cols, x), cfg, sid))
        y = slicer.decode(slicer.deserialize(blob))
        dt = time.perf_counter() - t0
        ybits = np.ascontiguousarray(y.values, dtype=np.float32).reshape(-1).view(np.uint32).tobytes()
    else:
        from oracle import sif_oracle as O

        t0 = time.perf_counter()
        blob = O.encode_bytes(x, O.Cfg(**cfgd), sid)
        y = O.decode_bytes(blob)
        dt = time.perf_counter() - t0
        ybits = y.reshape(-1).view(np.uint32).tobytes()
    return dt, len(blob), _sha16(blob), _sha16(ybits), sid


def cpu_measure_jobs(jobs, raw_per_step: int, steps: int, warmup: int, cores: int, impl: str, par=None):
    """Times the CPU implementation on host cores: each step encodes+decodes the IFs of
    `jobs` (kind, rows, cols, sid, codec) in a process pool (one process per core)."""
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    jobs = [j + (impl,) for j in jobs]
    with ctx.Pool(cores) as pool:
        for _ in range(warmup):
            pool.map(_cpu_worker, jobs[: max(1, cores)])
        t0 = time.perf_counter()
        plen = 0
        for k in range(steps):
            res = pool.map(_cpu_worker, jobs, chunksize=1)
            plen = sum(r[1] for r in res)
            if par is not None and k == 0:
                for _dt, n, ps, ds, sid in res:
                    par.payload(sid, n, ps)
                    par.decode(sid, ds)
        wall = time.perf_counter() - t0
    raw = steps * raw_per_step
    return dict(value=raw / wall / 1e9, seconds=wall, payload_bytes=plen, raw_bytes=raw)


def _mixed_sample(n_if: int):
    """Deterministic subsample of the C5 mix keeping its 4:3:1 proportions (every k-th sid)."""
    from paper_2511_11608_b200.shard import mixed_workload

    mix = mixed_workload(8192)
    groups = max(1, n_if // 8)
    gstride = max(1, 1024 // groups)  # 1024 groups of 8 sids in the mix
    sids = [(g * gstride) * 8 + k for g in range(groups) for k in range(8)]
    return [(sid,) + tuple(mix[sid]) for sid in sids]


# Seconds of one core per IF round trip (measured on the GPU boxes' host CPUs, round 1/2).
_PER_IF = {"port": {"c1": 0.1, "c2": 0.1, "c3": 0.004, "c4": 5.0, "c4sweep": 5.0, "c5": 0.03},
           "reference": {"c1": 0.4, "c2": 0.4, "c3": 0.02, "c4": 14.0, "c4sweep": 14.0, "c5": 0.15}}


def cpu_measure(conf, name, impl, steps, warmup, cores, step_seconds=1.5, par=None):
    """The CPU implementation on a bounded sample of the workload: the first n IFs of the
    GPU arm's rank-0 batch (same sids, so the sample is also a parity set), n sized so
    one step takes about `step_seconds` on `cores` processes."""
    per_if = _PER_IF[impl][name]
    batch = conf.get("batch", conf.get("mixed"))
    n_if = int(min(batch, max(cores, step_seconds * cores / per_if)))
    if conf.get("mixed"):
        n_if = max(8, n_if // 8 * 8)
        sample = _mixed_sample(n_if)
        jobs = [(kind, r, c, sid, CODEC) for sid, kind, r, c, _b in sample]
        raw = sum(r * c * b for _sid, _k, r, c, b in sample)
        elems = sum(r * c for _sid, _k, r, c, _b in sample)
        desc = f"{n_if} streams of the C5 mix (every k-th group of 8 sids)"
    else:
        b_in = 4 if conf["dtype"] == "fp32" else 2
        jobs = [(conf["kind"], conf["rows"], conf["cols"], i, CODEC) for i in range(n_if)]
        raw = n_if * conf["rows"] * conf["cols"] * b_in
        elems = n_if * conf["rows"] * conf["cols"]
        desc = f"sids 0..{n_if - 1} of the workload (the GPU arm's first {n_if} IFs)"
    r = cpu_measure_jobs(jobs, raw, steps, warmup, cores, impl, par)
    r["sample"] = f"{desc} per step, {cores} processes, " + (
        "reference slicer package (baseline/_ref, unmodified, public API)" if impl == "reference"
        else "oracle/ NumPy port of the reference")
    r["bits_per_element"] = 8.0 * r["payload_bytes"] / elems
    r["n_if"] = n_if
    return r


def run_reference(args, conf, rank):
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    name = args.config if args.config in _PER_IF["port"] else "c2"
    impl = "reference" if _ref_path() else "port"
    gold = _golden()
    par = Parity(gold, {"c4sweep": "c4", "c1": "c2"}.get(name, name))
    steps = args.steps if name not in ("c4", "c4sweep") else max(1, min(args.steps, 3))
    r = cpu_measure(conf, name, impl, steps, args.warmup, cores, par=par)  # W warm-up steps (each a bounded sample)
    port = None
    if impl == "reference":  # the NumPy port beside it, same sample rule
        p2 = cpu_measure(conf, name, "port", max(1, min(steps, 3)), 1, cores)
        port = dict(value=round(p2["value"], 6), unit="GB/s", cores=cores, kind="port", sample=p2["sample"])
    line = dict(metric=METRIC, value=round(r["value"], 6), unit="GB/s", n_gpus=args.gpus, steps=steps,
                warmup=args.warmup, ms_per_step=r["seconds"] * 1e3 / max(1, steps), higher_is_better=True,
                scaling="strong" if conf.get("mixed") else "weak", vs_baseline=None, dtype=conf["dtype"],
                data="synthetic", config=dict(workload=conf["workload"], codec=CODEC, sample=r["sample"]),
                impl="reference",
                cpu_baseline=dict(value=round(r["value"], 6), unit="GB/s", cores=cores, kind=impl, sample=r["sample"]),
                port_baseline=port,
                e2e=dict(value=round(r["value"], 6), unit="GB/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                bits_per_element=round(r["bits_per_element"], 6),
                parity=par.summary(what="the CPU sample's payloads and decodes"))
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------- GPU arm helpers
# Algorithmic bytes per launch of the kernels that carry the path's compulsory traffic
# (B_alg = T*b_in + P + P + T*b_out per IF); the other kernels of the
# pipeline move only intermediate data and count 0.
def _alg_bytes(name, raw, payload, dense_out):
    return {"enc_stream": raw, "enc_pack": payload, "enc_crc": payload, "sif_dcrc_kernel": payload,
            "sif_scatter_kernel": dense_out + payload, "enc_token": raw + payload,
            "sif_dec_small": payload + dense_out}.get(name, 0)


def _kernel_profile(sif, step, steps):
    """Per-kernel average launch durations: the same steps again with every library kernel
    bracketed by CUDA events on its stream (sif_profile_enable)."""
    import ctypes

    import torch

    L = sif._lib.load()
    L.sif_profile_enable(1)
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    L.sif_profile_enable(0)
    ms = (ctypes.c_double * 64)()
    cnt = (ctypes.c_int32 * 64)()
    nk = L.sif_profile_read(ms, cnt, 64)
    out = {}
    for k in range(max(0, nk)):
        if cnt[k]:
            out[L.sif_profile_kernel_name(k).decode()] = dict(ms_total=ms[k], launches=int(cnt[k]))
    return out


def _kernel_table(kprof, steps, raw_bytes, payload_total, dense_out):
    kernels = {}
    prof_ms = sum(v["ms_total"] for v in kprof.values()) or 1.0
    for name, v in kprof.items():
        per = v["ms_total"] / v["launches"]
        alg = _alg_bytes(name, raw_bytes, payload_total, dense_out)
        kernels[name] = dict(us_per_launch=round(per * 1e3, 2), launches_per_step=v["launches"] // steps,
                             share=round(v["ms_total"] / prof_ms, 4), alg_bytes_per_launch=alg,
                             alg_gbs=round(alg / (per * 1e-3) / 1e9, 1) if alg else 0.0)
    return kernels


def _roofline(kernels, config, hbm, peak_kind):
    # dominant kernel: the one that moves the most compulsory (algorithmic) bytes (ties:
    # the longer one)
    cand = [k for k, v in kernels.items() if v["alg_bytes_per_launch"]]
    if not cand:
        return None
    dom = max(cand, key=lambda k: (kernels[k]["alg_bytes_per_launch"], kernels[k]["us_per_launch"]))
    kd = kernels[dom]
    return dict(bound="hbm", kernel=dom, achieved=kd["alg_gbs"], peak=hbm, unit="GB/s",
                frac=round(kd["alg_gbs"] / hbm, 4), traffic=(_ncu_traffic(config) or {}).get(dom),
                peak_source=peak_kind, algorithmic_bytes_per_launch=kd["alg_bytes_per_launch"],
                us_per_launch=kd["us_per_launch"], share_of_step=kd["share"],
                note="per-launch duration from CUDA events around each library kernel in an instrumented "
                     "repeat of the timed steps")


class Dist:
    """One process per GPU.  NCCL when every rank has its own device; ranks that share a
    device (a dry run with fewer GPUs than --gpus) use gloo for the timing reductions."""

    def __init__(self, rank, world, local_rank):
        import torch

        self.rank, self.world = rank, world
        ndev = max(1, torch.cuda.device_count())
        self.device_index = local_rank % ndev
        self.oversubscribed = world > ndev
        torch.cuda.set_device(self.device_index)
        self.dev = torch.device("cuda", self.device_index)
        self.pg = None
        if world > 1:
            import torch.distributed as dist

            if self.oversubscribed:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, vals):
        if not self.pg:
            return list(vals)
        import torch

        t = torch.tensor(list(vals), dtype=torch.float64, device="cpu" if self.oversubscribed else self.dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return [float(v) for v in t.cpu()]

    @property
    def cpu_pg(self):
        """For integer reductions of host counters (gloo needs CPU tensors; NCCL CUDA)."""
        return self

    def all_reduce(self, t):
        if not self.pg:
            return
        if self.oversubscribed:
            self.pg.all_reduce(t)
        else:
            tt = t.to(self.dev)
            self.pg.all_reduce(tt)
            t.copy_(tt.cpu())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()

    def parallelism(self, what):
        s = f"dp{self.world} ({what})"
        if self.oversubscribed:
            s += f"; DRY RUN: {self.world} ranks share the visible GPU(s), timings are not a scaling result"
        return s


def _time_pipe(pipe, steps, d, local_rank):
    import torch

    stream = torch.cuda.current_stream()
    d.barrier()
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        pipe.begin()
        for _ in range(steps):
            pipe.step()
        pipe.end()
        t_end.record(stream)
        torch.cuda.synchronize()
    d.barrier()
    return t_start.elapsed_time(t_end) / steps, clk


def _seq_split(enc, dec, steps):
    """encode / decode split of one step, sequential on one stream (not overlapped)."""
    import torch

    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        ev[i][0].record(stream)
        enc.run()
        ev[i][1].record(stream)
        dec.run()
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    return (sum(e[0].elapsed_time(e[1]) for e in ev) / steps, sum(e[1].elapsed_time(e[2]) for e in ev) / steps)


def _time_e2e(rt, steps, d):
    import torch

    stream = torch.cuda.current_stream()
    for _ in range(2):
        rt.run()
    torch.cuda.synchronize()
    d.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        rt.run()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def _cpu_line(args, conf, name, d):
    if d.rank != 0 or not args.cpu_baseline or d.world > 1:
        return None, None
    cores = len(os.sched_getaffinity(0))
    par = Parity(_golden(), {"c4sweep": "c4", "c1": "c2"}.get(name, name))
    r = cpu_measure(conf, name, "port", 2, 1, cores, par=par)
    return dict(value=round(r["value"], 6), unit="GB/s", cores=cores, kind="port",
                sample=r["sample"] + f" x 2 steps ({r['seconds']:.1f} s)"), par


# ------------------------------------------------------------------------- GPU arm: batches
def run_ours(args, conf, d, local_rank):
    import math

    import torch

    import paper_2511_11608_b200 as sif

    rank, world = d.rank, d.world
    B, N, K = conf["batch"], conf["rows"], conf["cols"]
    tdt = torch.float32 if conf["dtype"] == "fp32" else torch.bfloat16
    b_in = 4 if conf["dtype"] == "fp32" else 2
    raw_bytes = B * N * K * b_in
    dense_out = B * N * K * 4
    cfg = sif.CodecConfig(**CODEC)
    # one input batch per pipeline slot (distinct buffers); enough of them that the set of
    # batches a run cycles through exceeds the 126 MB L2 (C3: 16 batches of 8.4 MB)
    nin = max(args.depth, min(32, math.ceil(126e6 / raw_bytes) + 1)) if raw_bytes < 126e6 else args.depth
    shift = max(1, B // nin)
    slot_inputs = []
    for j in range(nin):
        sids = [rank * B + (i + j * shift) % B for i in range(B)]
        xs = torch.empty((B, N, K), dtype=tdt, device=d.dev)
        for i, sid in enumerate(sids):
            sif.synthetic(conf["kind"], N, K, sid, out=xs[i])
        slot_inputs.append((xs, sids))
    pipe = sif.BatchPipeline(slot_inputs[0][0], cfg, slot_inputs[0][1], graphs=args.graph, slot_inputs=slot_inputs)
    pipe.begin()
    for _ in range(args.warmup):
        pipe.step()
    pipe.end()
    torch.cuda.synchronize()
    st_ms, clk = _time_pipe(pipe, args.steps, d, local_rank)
    pipe.check()  # status after timing (must all be OK)
    # parity: every slot's payloads and decodes vs the reference digests
    par = Parity(_golden(), args.config)
    payload_total = 0
    for sl in pipe.slots:
        payload_total = _check_encoder(par, sl["enc"], sl["seeds"])
        _check_decoded(par, [sl["dec"].out[i] for i in range(B)], sl["seeds"])
    sl0 = pipe.slots[0]
    payload_total = int(sl0["enc"].out_len.cpu().numpy().sum())
    alg_enc = raw_bytes + payload_total
    alg_dec = payload_total + dense_out
    enc_ms, dec_ms = _seq_split(sl0["enc"], sl0["dec"], args.steps)
    st_ms, enc_ms, dec_ms = d.max([st_ms, enc_ms, dec_ms])
    kprof = _kernel_profile(sif, lambda: (sl0["enc"].run(), sl0["dec"].run()), args.steps)

    # ---- e2e through the public API with host buffers (pinned), copies inside the timing:
    # HostRoundTrip pipelines H2D of x, encode, decode and D2H of y over sub-batches
    x_host = sl0["xs"].cpu().pin_memory()
    # sub-batches: one per 16 MB (at most 8); small batches (C3) still split in 4 so the H2D
    # and D2H copies overlap the kernels (measured: C3 e2e 14.3 -> 17.9 GB/s)
    parts = args.parts or (max(1, min(8, raw_bytes // (16 << 20))) if raw_bytes >= (16 << 20) else min(4, B))
    rt = sif.HostRoundTrip(x_host, cfg, sl0["seeds"], parts=parts)
    e2e_ms = _time_e2e(rt, max(2, min(args.steps, 10)), d)
    rt.check()
    assert torch.equal(rt.y_host, sl0["dec"].out.cpu()), "e2e decode differs"
    (e2e_ms,) = d.max([e2e_ms])
    cpu, cpar = _cpu_line(args, conf, args.config, d)
    parity = par.summary(d if world > 1 else None)
    if rank == 0:
        hbm, peak_kind = _peaks()
        value = world * raw_bytes / (st_ms * 1e-3) / 1e9
        step_gbs = (alg_enc + alg_dec) / (st_ms * 1e-3) / 1e9
        kernels = _kernel_table(kprof, args.steps, raw_bytes, payload_total, dense_out)
        in_set = nin * raw_bytes
        line = dict(
            metric=METRIC, value=round(value, 3), unit="GB/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
            ms_per_step=round(st_ms, 5), higher_is_better=True, scaling="weak", vs_baseline=None,
            dtype=conf["dtype"], data="synthetic (integer-exact device generator, SURVEY.md §8(d))",
            config=dict(workload=conf["workload"], codec=CODEC, if_shape=[N, K], batch_per_gpu=B,
                        parallelism=d.parallelism("independent IF streams per GPU, no collectives"),
                        launch=("CUDA graph per step" if args.graph else "direct launches") +
                               f", {nin} pipeline slots on separate streams, each with its own input batch "
                               "(step i decode overlaps step i+1 encode)",
                        l2=("per-step inputs %.0f MB/GPU exceed the 126 MB L2; %d distinct input batches rotate; "
                            "no flush" % (raw_bytes / 1e6, nin)) if raw_bytes > 126e6 else
                           ("per-step inputs %.1f MB/GPU; %d distinct input batches (%.0f MB in total, above the "
                            "126 MB L2) rotate so no step re-reads L2-resident inputs; no flush" %
                            (raw_bytes / 1e6, nin, in_set / 1e6))),
            roofline=_roofline(kernels, args.config, hbm, peak_kind),
            roofline_step=dict(achieved=round(step_gbs, 2), frac=round(step_gbs / hbm, 4), unit="GB/s",
                               algorithmic_bytes_per_step=alg_enc + alg_dec,
                               note="encode_ms/decode_ms from a sequential (non-overlapped) repeat",
                               encode_ms=round(enc_ms, 5), decode_ms=round(dec_ms, 5),
                               encode_gbs=round(alg_enc / (enc_ms * 1e-3) / 1e9, 2),
                               decode_gbs=round(alg_dec / (dec_ms * 1e-3) / 1e9, 2)),
            kernels=kernels,
            bits_per_element=round(8.0 * payload_total / (B * N * K), 6),
            raw_gbs_per_gpu=round(raw_bytes / (st_ms * 1e-3) / 1e9, 3),
            e2e=dict(value=round(world * raw_bytes / (e2e_ms * 1e-3) / 1e9, 3), unit="GB/s",
                     h2d_bytes_per_step=rt.h2d_bytes, d2h_bytes_per_step=rt.d2h_bytes,
                     ms_per_step=round(e2e_ms, 4),
                     api="HostRoundTrip: pinned host IFs -> H2D -> encode -> .sif (device) -> decode -> D2H, "
                         f"{parts} sub-batch(es) pipelined over 3 streams"),
            gpu_launches=sum(v["launches"] for v in kprof.values()),
            clocks=clk.summary(),
            parity=parity,
            cpu_baseline=cpu,
        )
        if cpar is not None:
            line["cpu_baseline"]["parity"] = dict(checked=cpar.checked, mismatches=cpar.mismatches)
        print(json.dumps(line), flush=True)
    d.close()


# ------------------------------------------------------------------------- GPU arm: C1 latency
def run_latency(args, conf, d, local_rank):
    """configs[0]: one ResNet IF round trip through the drop-in API.  Three numbers:
    `value` -- encode(x) -> decode(p) on a device-resident IF, the reference-shaped call
    (plan + launches + status read per call); `planned` -- the same IF through a reused
    plan captured in a CUDA graph (a serving loop); `e2e` -- host numpy-like CPU tensor in,
    host fp32 tensor out."""
    import torch

    import paper_2511_11608_b200 as sif

    N, K = conf["rows"], conf["cols"]
    raw = N * K * 4
    cfg = sif.CodecConfig(**CODEC)
    x = sif.synthetic(conf["kind"], N, K, d.rank)
    par = Parity(_golden(), "c2")
    stream = torch.cuda.current_stream()

    def api_round_trip(xx):
        p = sif.encode(xx, cfg, seed=d.rank)
        return p, sif.decode(p)

    for _ in range(args.warmup):
        api_round_trip(x)
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            p, y = api_round_trip(x)
        e1.record(stream)
        torch.cuda.synchronize()
    api_ms = e0.elapsed_time(e1) / args.steps
    par.payload(d.rank, p.nbytes, _sha16(p.to_bytes()))
    par.decode(d.rank, _sha16(y.cpu().numpy().reshape(-1).view("uint32").tobytes()))
    # reused plan + CUDA graph
    pipe = sif.BatchPipeline(x.unsqueeze(0), cfg, [d.rank], depth=1, graphs=True)
    for _ in range(args.warmup):
        pipe.step()
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(args.steps):
        pipe.step()
        pipe.end()
    g1.record(stream)
    torch.cuda.synchronize()
    planned_ms = g0.elapsed_time(g1) / args.steps
    pipe.check()
    kprof = _kernel_profile(sif, pipe.slots[0]["fn"], args.steps)
    # host in / host out through the drop-in API
    xh = x.cpu()
    for _ in range(args.warmup):
        sif.decode(sif.encode(xh, cfg, seed=d.rank)).cpu()
    torch.cuda.synchronize()
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for _ in range(args.steps):
        ph = sif.encode(xh, cfg, seed=d.rank)
        yh = sif.decode(ph).cpu()
    h1.record(stream)
    torch.cuda.synchronize()
    host_ms = h0.elapsed_time(h1) / args.steps
    assert torch.equal(yh, y.cpu())
    api_ms, planned_ms, host_ms = d.max([api_ms, planned_ms, host_ms])
    if d.rank == 0:
        hbm, peak_kind = _peaks()
        kernels = _kernel_table(kprof, args.steps, raw, p.nbytes, N * K * 4)
        alg = raw + 2 * p.nbytes + N * K * 4
        line = dict(
            metric=METRIC, value=round(d.world * raw / (api_ms * 1e-3) / 1e9, 4), unit="GB/s", n_gpus=d.world,
            steps=args.steps, warmup=args.warmup, ms_per_step=round(api_ms, 5), higher_is_better=True,
            scaling="weak", vs_baseline=None, dtype="fp32", data="synthetic (integer-exact device generator)",
            config=dict(workload=conf["workload"], codec=CODEC, if_shape=[N, K],
                        parallelism=d.parallelism("one IF per GPU"),
                        l2="single 0.8 MB IF: L2-resident by design (a latency measurement)"),
            latency_us=dict(api_round_trip=round(api_ms * 1e3, 1), planned_graph_round_trip=round(planned_ms * 1e3, 1),
                            host_in_host_out=round(host_ms * 1e3, 1),
                            note="api = encode(x) + decode(p) with a device-resident x (plan, upload, launches, "
                                 "status read per call, as the reference API is synchronous); planned = reused "
                                 "plan replayed as one CUDA graph"),
            roofline=_roofline(kernels, "c1", hbm, peak_kind),
            roofline_step=dict(achieved=round(alg / (planned_ms * 1e-3) / 1e9, 2),
                               frac=round(alg / (planned_ms * 1e-3) / 1e9 / hbm, 4), unit="GB/s",
                               algorithmic_bytes_per_step=alg, note="planned graph round trip"),
            kernels=kernels,
            bits_per_element=round(8.0 * p.nbytes / (N * K), 6),
            e2e=dict(value=round(d.world * raw / (host_ms * 1e-3) / 1e9, 4), unit="GB/s", h2d_bytes_per_step=raw,
                     d2h_bytes_per_step=N * K * 4, ms_per_step=round(host_ms, 4),
                     api="encode(host tensor) -> decode -> .cpu(): the drop-in API with host buffers"),
            gpu_launches=sum(v["launches"] for v in kprof.values()),
            clocks=clk.summary(),
            parity=par.summary(what="the IF's payload and decode"),
        )
        print(json.dumps(line), flush=True)
    d.close()


# ------------------------------------------------------------------------- GPU arm: C4 sweep
def sweep_points():
    pts = []
    for s in (0.5, 0.7, 0.8, 0.9, 0.95):
        for dl in (0.01, 0.05, 0.1, 0.2):
            for lam in (0.0, 0.1):
                pts.append(dict(CODEC, s=s, delta=dl, lam=lam))
    pts.append(dict(CODEC, mode="fixed_q", fixed_q=(8, 4, 2, 8, 4, 2)))
    return pts


def run_sweep(args, conf, d, local_rank):
    """the C4 batch at every (s, delta, lambda) point plus fixed Q; each
    point timed like the C4 line (pipelined graphs, 2 input batches), IF sid 0 of every
    point checked against the reference's payload/decode digests."""
    import torch

    import paper_2511_11608_b200 as sif

    B, N, K = conf["batch"], conf["rows"], conf["cols"]
    raw_bytes = B * N * K * 2
    gold = _golden()
    slot_inputs = []
    for j in range(2):
        sids = [d.rank * B + (i + j * (B // 2)) % B for i in range(B)]
        xs = torch.empty((B, N, K), dtype=torch.bfloat16, device=d.dev)
        for i, sid in enumerate(sids):
            sif.synthetic(conf["kind"], N, K, sid, out=xs[i])
        slot_inputs.append((xs, sids))
    steps = max(2, min(args.steps, 5))
    pts, total_ms, total_raw = [], 0.0, 0
    par = Parity(gold, "c4sweep")
    clk_all = None
    for pi, kw in enumerate(sweep_points()):
        cfg = sif.CodecConfig(**kw)
        pipe = sif.BatchPipeline(slot_inputs[0][0], cfg, slot_inputs[0][1], graphs=args.graph,
                                 slot_inputs=slot_inputs)
        pipe.begin()
        for _ in range(3):
            pipe.step()
        pipe.end()
        torch.cuda.synchronize()
        st_ms, clk = _time_pipe(pipe, steps, d, local_rank)
        if clk_all is None:
            clk_all = clk
        pipe.check()
        (st_ms,) = d.max([st_ms])
        sl = pipe.slots[0]
        lens = sl["enc"].out_len.cpu().numpy()
        ok = None
        if d.rank == 0:  # sid 0 sits at batch position 0 of slot 0
            n0 = par.mismatches
            p0 = sl["enc"].payloads()[0]
            par.payload(pi, p0.nbytes, _sha16(p0.to_bytes()))
            par.decode(pi, _sha16(sl["dec"].out[0].cpu().numpy().reshape(-1).view("uint32").tobytes()))
            ok = par.mismatches == n0
        pts.append(dict(s=kw["s"], delta=kw["delta"], lam=kw["lam"], mode=kw.get("mode", "abq"),
                        fixed_q=list(kw.get("fixed_q", ())), gbs=round(raw_bytes / (st_ms * 1e-3) / 1e9, 2),
                        ms_per_step=round(st_ms, 4), bits_per_element=round(8.0 * float(lens.sum()) / (B * N * K), 5),
                        ref_bits_per_element_sid0=(round(8.0 * float(gold["c4sweep_len"][pi]) / (N * K), 5)
                                                   if gold is not None and "c4sweep_len" in gold else None),
                        parity_sid0=ok))
        total_ms += st_ms * steps
        total_raw += raw_bytes * steps
        del pipe
        torch.cuda.empty_cache()
    if d.rank == 0:
        hbm, _ = _peaks()
        line = dict(metric=METRIC, value=round(d.world * total_raw / (total_ms * 1e-3) / 1e9, 3), unit="GB/s",
                    n_gpus=d.world, steps=steps, warmup=3, ms_per_step=round(total_ms / len(pts) / steps, 5),
                    higher_is_better=True, scaling="weak", vs_baseline=None, dtype="bf16",
                    data="synthetic (integer-exact device generator)",
                    config=dict(workload=conf["workload"], if_shape=[N, K], batch_per_gpu=B,
                                parallelism=d.parallelism("independent IF streams per GPU"),
                                l2="per-step inputs 537 MB/GPU exceed the 126 MB L2; 2 input batches; no flush",
                                value_note="aggregate over the 41 points (total raw bytes / total time)"),
                    sweep=pts, peak_gbs=hbm, clocks=clk_all.summary() if clk_all else None,
                    parity=par.summary(what="IF sid 0 of every sweep point"))
        print(json.dumps(line), flush=True)
    d.close()


# ------------------------------------------------------------------------- GPU arm: C5 mixed
def run_ours_mixed(args, conf, d, local_rank):
    """C5: this rank's share of the 8192 mixed streams (LPT by bytes), one ListEncoder launch
    sequence per step, pipelined over `depth` slots like the homogeneous configs."""
    import torch

    import paper_2511_11608_b200 as sif
    from paper_2511_11608_b200.shard import mixed_workload, shard_streams

    rank, world = d.rank, d.world
    mix = mixed_workload(conf["mixed"])
    mine = shard_streams([(r, c, b) for _k, r, c, b in mix], world, rank)
    xs, seeds = [], []
    for sid in mine:
        kind, r, c, b = mix[sid]
        t = torch.empty((r, c), dtype=torch.float32 if b == 4 else torch.bfloat16, device=d.dev)
        sif.synthetic(kind, r, c, sid, out=t)
        xs.append(t)
        seeds.append(sid)
    cfg = sif.CodecConfig(**CODEC)
    raw_bytes = sum(mix[sid][1] * mix[sid][2] * mix[sid][3] for sid in mine)
    job_raw = sum(r * c * b for _k, r, c, b in mix)
    elems = sum(mix[sid][1] * mix[sid][2] for sid in mine)
    dense_out = 4 * elems
    pipe = sif.BatchPipeline(xs, cfg, seeds, depth=args.depth, graphs=args.graph)
    pipe.begin()
    for _ in range(args.warmup):
        pipe.step()
    pipe.end()
    torch.cuda.synchronize()
    st_ms, clk = _time_pipe(pipe, args.steps, d, local_rank)
    pipe.check()
    par = Parity(_golden(), "c5")
    for sl in pipe.slots:
        _check_encoder(par, sl["enc"], seeds, offs=sl["enc"].offs)
        _check_decoded(par, sl["dec"].outs, seeds)
    slot0 = pipe.slots[0]
    enc, dec = slot0["enc"], slot0["dec"]
    payload_total = int(enc.out_len.cpu().numpy()[: len(mine)].sum())
    alg_enc, alg_dec = raw_bytes + payload_total, payload_total + dense_out
    enc_ms, dec_ms = _seq_split(enc, dec, args.steps)
    st_ms, enc_ms, dec_ms = d.max([st_ms, enc_ms, dec_ms])
    kprof = _kernel_profile(sif, lambda: (enc.run(), dec.run()), args.steps)
    # e2e: pinned host streams -> H2D -> encode -> decode -> D2H (ListRoundTrip)
    rt = sif.ListRoundTrip([x.cpu() for x in xs], cfg, seeds, parts=4)
    e2e_ms = _time_e2e(rt, max(2, min(args.steps, 10)), d)
    rt.check()
    for k in (0, len(xs) // 2, len(xs) - 1):
        assert torch.equal(rt.y(k), dec.outs[k].cpu()), "e2e decode differs"
    (e2e_ms,) = d.max([e2e_ms])
    cpu, cpar = _cpu_line(args, conf, "c5", d)
    parity = par.summary(d if world > 1 else None)
    if rank == 0:
        hbm, peak_kind = _peaks()
        step_gbs = (alg_enc + alg_dec) / (st_ms * 1e-3) / 1e9
        kernels = _kernel_table(kprof, args.steps, raw_bytes, payload_total, dense_out)
        counts = {}
        for sid in mine:
            counts[mix[sid][1:3]] = counts.get(mix[sid][1:3], 0) + 1
        line = dict(
            metric=METRIC, value=round(job_raw / (st_ms * 1e-3) / 1e9, 3), unit="GB/s", n_gpus=world,
            steps=args.steps, warmup=args.warmup, ms_per_step=round(st_ms, 5), higher_is_better=True,
            scaling="strong", vs_baseline=None, dtype=conf["dtype"],
            data="synthetic (integer-exact device generator, SURVEY.md §8(d))",
            config=dict(workload=conf["workload"], codec=CODEC, streams_total=conf["mixed"],
                        streams_rank0=len(mine), shapes_rank0={f"{r}x{c}": n for (r, c), n in counts.items()},
                        parallelism=d.parallelism("streams sharded by LPT on bytes, no collectives"),
                        launch=("CUDA graph per step" if args.graph else "direct launches") +
                               f", {args.depth} pipeline slot(s) on separate streams",
                        l2="per-step inputs %.0f MB/GPU exceed the 126 MB L2; no flush" % (raw_bytes / 1e6)),
            roofline=_roofline(kernels, "c5", hbm, peak_kind),
            roofline_step=dict(achieved=round(step_gbs, 2), frac=round(step_gbs / hbm, 4), unit="GB/s",
                               algorithmic_bytes_per_step=alg_enc + alg_dec, encode_ms=round(enc_ms, 5),
                               decode_ms=round(dec_ms, 5)),
            kernels=kernels,
            bits_per_element=round(8.0 * payload_total / elems, 6),
            raw_gbs_per_gpu=round(raw_bytes / (st_ms * 1e-3) / 1e9, 3),
            e2e=dict(value=round(job_raw / (e2e_ms * 1e-3) / 1e9, 3), unit="GB/s", h2d_bytes_per_step=rt.h2d_bytes,
                     d2h_bytes_per_step=rt.d2h_bytes, ms_per_step=round(e2e_ms, 4),
                     api="ListRoundTrip: pinned host streams -> H2D -> encode -> .sif (device) -> decode -> D2H, "
                         "4 groups pipelined over 3 streams"),
            gpu_launches=sum(v["launches"] for v in kprof.values()),
            clocks=clk.summary(),
            parity=parity,
            cpu_baseline=cpu,
        )
        if cpar is not None:
            line["cpu_baseline"]["parity"] = dict(checked=cpar.checked, mismatches=cpar.mismatches)
        print(json.dumps(line), flush=True)
    d.close()


def _relaunch(args) -> int:
    """--gpus N > 1 without a launcher: re-run this script under torch.distributed.run with
    one process per GPU (rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the kernels directly instead of replaying CUDA graphs")
    ap.add_argument("--parts", type=int, default=None,
                    help="e2e: host round-trip sub-batches (default: one per 16 MB of input, at most 8)")
    ap.add_argument("--depth", type=int, default=None,
                    help="pipeline slots: consecutive steps overlap on this many streams (1 = sequential); "
                         "default per config (measured, tools/sweep_depth*.sh)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    conf = CONFIGS[args.config]
    if args.depth is None:
        args.depth = conf.get("depth", 3)
    if args.impl == "reference":
        run_reference(args, conf, rank)
        return
    d = Dist(rank, world, local_rank)
    if conf.get("latency"):
        run_latency(args, conf, d, local_rank)
    elif conf.get("sweep"):
        run_sweep(args, conf, d, local_rank)
    elif conf.get("mixed"):
        run_ours_mixed(args, conf, d, local_rank)
    else:
        run_ours(args, conf, d, local_rank)


if __name__ == "__main__":
    main()
