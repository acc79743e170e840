"""Benchmark: SLICER IF codec encode+decode throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c3|c4]

One step = encode of the whole per-GPU batch of synthetic IFs (ATKF -> MS -> ABQ -> CSR
bit-pack -> .sif with CRC) followed by decode of those payloads back to dense fp32, inputs
resident in HBM.  N>1: one process per GPU (torchrun), independent IF streams per rank
(sid = rank * B + i), no data-path collectives ("scaling": "weak"); the timing is the max
over ranks.  `--impl reference` times the CPU reference restatement (oracle/) on the
host cores on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IF encode+decode GB/s per GPU (and 8-GPU aggregate) vs HBM roofline; bits/element"

CONFIGS = {
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


# ------------------------------------------------------------------------- CPU arm
def _cpu_worker(args):
    kind, rows, cols, sid, cfgd = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import sif_oracle as O
    from oracle.synth import synth

    x = synth(kind, rows, cols, sid)
    t0 = time.perf_counter()
    blob = O.encode_bytes(x, O.Cfg(**cfgd), sid)
    y = O.decode_bytes(blob)
    dt = time.perf_counter() - t0
    return dt, len(blob), int(y.size)


def cpu_measure_jobs(jobs, raw_per_step: int, steps: int, warmup: int, cores: int):
    """Times the oracle (CPU restatement of the reference) on host cores: each step
    encodes+decodes the IFs of `jobs` (kind, rows, cols, sid, codec) in a process pool."""
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for _ in range(warmup):
            pool.map(_cpu_worker, jobs[: max(1, cores)])
        t0 = time.perf_counter()
        plen = 0
        for _ in range(steps):
            res = pool.map(_cpu_worker, jobs)
            plen = sum(r[1] for r in res)
        wall = time.perf_counter() - t0
    raw = steps * raw_per_step
    return dict(value=raw / wall / 1e9, seconds=wall, payload_bytes=plen, raw_bytes=raw)


def cpu_measure(conf, n_if: int, steps: int, warmup: int, cores: int):
    """The oracle on a bounded sample of `n_if` IFs of the workload shape."""
    if conf.get("mixed"):
        return cpu_measure_mixed(conf, n_if, steps, warmup, cores)
    b_in = 4 if conf["dtype"] == "fp32" else 2
    jobs = [(conf["kind"], conf["rows"], conf["cols"], 100000 + i, CODEC) for i in range(n_if)]
    return cpu_measure_jobs(jobs, n_if * conf["rows"] * conf["cols"] * b_in, steps, warmup, cores)


def _mixed_sample(n_if: int):
    """Deterministic subsample of the C5 mix keeping its 4:3:1 proportions (every k-th sid)."""
    from paper_2511_11608_b200.shard import mixed_workload

    mix = mixed_workload(8192)
    groups = max(1, n_if // 8)
    gstride = max(1, 1024 // groups)  # 1024 groups of 8 sids in the mix
    sids = [(g * gstride) * 8 + k for g in range(groups) for k in range(8)]
    return [(sid,) + tuple(mix[sid]) for sid in sids]


def cpu_measure_mixed(conf, n_if: int, steps: int, warmup: int, cores: int):
    sample = _mixed_sample(n_if)
    jobs = [(kind, r, c, sid, CODEC) for sid, kind, r, c, _b in sample]
    raw = sum(r * c * b for _sid, _k, r, c, b in sample)
    return cpu_measure_jobs(jobs, raw, steps, warmup, cores)


def run_reference(args, conf, rank):
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    per_if = {"c2": 0.15, "c3": 0.004, "c4": 8.0, "c5": 0.03}[args.config]
    batch = conf.get("batch", conf.get("mixed"))
    n_if = max(cores, int(min(batch, max(cores, 2.0 * cores / per_if))))
    n_if = min(n_if, batch)
    if conf.get("mixed"):
        n_if = max(8, n_if // 8 * 8)
    r = cpu_measure(conf, n_if, args.steps, args.warmup, cores)
    sample = f"{n_if} IFs of the workload shape per step (of {batch}), {cores} processes, oracle/ NumPy port"
    line = dict(metric=METRIC, value=round(r["value"], 6), unit="GB/s", n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=r["seconds"] * 1e3 / max(1, args.steps), higher_is_better=True,
                scaling="weak", vs_baseline=None, dtype=conf["dtype"], data="synthetic",
                config=dict(workload=conf["workload"], codec=CODEC, sample=sample),
                impl="reference",
                cpu_baseline=dict(value=round(r["value"], 6), unit="GB/s", cores=cores, kind="port", sample=sample),
                e2e=dict(value=round(r["value"], 6), unit="GB/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                bits_per_element=8.0 * r["payload_bytes"] / (
                    sum(rr * cc for _s, _k, rr, cc, _b in _mixed_sample(n_if)) if conf.get("mixed")
                    else n_if * conf["rows"] * conf["cols"]))
    if conf.get("mixed"):
        line["scaling"] = "strong"
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------- GPU arm
# Algorithmic bytes per launch of the kernels that carry the path's compulsory traffic
# (B_alg = T*b_in + P + P + T*b_out per IF); the other kernels of the
# pipeline move only intermediate data and count 0.
def _alg_bytes(name, raw, payload, dense_out):
    return {"enc_stream": raw, "enc_pack": payload, "enc_crc": payload, "sif_dcrc_kernel": payload,
            "sif_scatter_kernel": dense_out + payload}.get(name, 0)


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
    ms = (ctypes.c_double * 32)()
    cnt = (ctypes.c_int32 * 32)()
    nk = L.sif_profile_read(ms, cnt, 32)
    out = {}
    for k in range(max(0, nk)):
        if cnt[k]:
            out[L.sif_profile_kernel_name(k).decode()] = dict(ms_total=ms[k], launches=int(cnt[k]))
    return out


def run_ours(args, conf, rank, world, local_rank):
    import torch

    import paper_2511_11608_b200 as sif

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    B, N, K = conf["batch"], conf["rows"], conf["cols"]
    tdt = torch.float32 if conf["dtype"] == "fp32" else torch.bfloat16
    b_in = 4 if conf["dtype"] == "fp32" else 2
    xs = torch.empty((B, N, K), dtype=tdt, device=dev)
    for i in range(B):
        sif.synthetic(conf["kind"], N, K, rank * B + i, out=xs[i])
    cfg = sif.CodecConfig(**CODEC)
    enc = sif.BatchEncoder(xs, cfg, [rank * B + i for i in range(B)])
    enc.run().check()
    lens = enc.out_len.cpu().numpy()
    cap = enc.cap
    ys = torch.empty((B, N, K), dtype=torch.float32, device=dev)
    dec = sif.BatchDecoder([enc.out.data_ptr() + i * cap for i in range(B)], lens, N, K, out=ys)
    dec.run().check()
    torch.cuda.synchronize()
    payload_total = int(lens.sum())
    raw_bytes = B * N * K * b_in
    dense_out = B * N * K * 4
    alg_enc = raw_bytes + payload_total
    alg_dec = payload_total + dense_out
    stream = torch.cuda.current_stream()

    def step():
        enc.run()
        dec.run()

    # Timed region: BatchPipeline -- two slots (payload buffers) on two streams, each step a
    # CUDA-graph replay of encode+decode; step i's decode overlaps step i+1's encode.
    pipe = sif.BatchPipeline(xs, cfg, [rank * B + i for i in range(B)], depth=args.depth, graphs=args.graph)
    pipe.begin()
    for _ in range(args.warmup):
        pipe.step()
    pipe.end()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        pipe.begin()
        for i in range(args.steps):
            pipe.step()
        pipe.end()
        t_end.record(stream)
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    total_ms = t_start.elapsed_time(t_end)
    st_ms = total_ms / args.steps
    pipe.check()  # status after timing (must all be OK)
    assert torch.equal(pipe.ys(0), pipe.ys(len(pipe.slots) - 1)), "slots disagree"

    # encode / decode split of one step, sequential on one stream (not overlapped)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        ev[i][0].record(stream)
        enc.run()
        ev[i][1].record(stream)
        dec.run()
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    enc_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / args.steps
    dec_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / args.steps
    if pg:
        t = torch.tensor([st_ms, enc_ms, dec_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        st_ms, enc_ms, dec_ms = [float(v) for v in t.cpu().numpy()]

    # per-kernel durations (instrumented repeat of the same steps, after the timed region)
    kprof = _kernel_profile(sif, step, args.steps)

    # ---- e2e through the public API with host buffers (pinned), copies inside the timing:
    # HostRoundTrip pipelines H2D of x, encode, decode and D2H of y over sub-batches on
    # separate streams
    x_host = xs.cpu().pin_memory()
    parts = max(1, min(8, raw_bytes // (16 << 20)))  # pipelining pays off only for large transfers
    rt = sif.HostRoundTrip(x_host, cfg, [rank * B + i for i in range(B)], parts=parts)
    e2e_steps = max(2, min(args.steps, 10))
    for _ in range(2):
        rt.run()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        rt.run()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    rt.check()
    assert torch.equal(rt.y_host, ys.cpu()), "e2e decode differs"
    if pg:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_ms = float(t.item())

    cpu = None
    if rank == 0 and args.cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        per_if = {"c2": 0.15, "c3": 0.004, "c4": 8.0}[args.config]
        n_if = min(conf["batch"], max(cores, int(2.0 * cores / per_if)))
        r = cpu_measure(conf, n_if, 2, 1, cores)
        cpu = dict(value=round(r["value"], 6), unit="GB/s", cores=cores, kind="port",
                   sample=f"{n_if} IFs of the workload shape x 2 steps, {cores} processes, oracle/ NumPy port "
                          f"({r['seconds']:.1f} s)")

    if rank == 0:
        hbm, peak_kind = _peaks()
        value = world * raw_bytes / (st_ms * 1e-3) / 1e9
        step_gbs = (alg_enc + alg_dec) / (st_ms * 1e-3) / 1e9
        kernels = {}
        prof_ms = sum(v["ms_total"] for v in kprof.values()) or 1.0
        for name, v in kprof.items():
            per = v["ms_total"] / v["launches"]
            alg = _alg_bytes(name, raw_bytes, payload_total, dense_out)
            kernels[name] = dict(us_per_launch=round(per * 1e3, 2), launches_per_step=v["launches"] // args.steps,
                                 share=round(v["ms_total"] / prof_ms, 4), alg_bytes_per_launch=alg,
                                 alg_gbs=round(alg / (per * 1e-3) / 1e9, 1) if alg else 0.0)
        # dominant kernel: the one that moves the most compulsory (algorithmic) bytes (ties:
        # the longer one) -- the decode scatter writing the dense IF in every config
        cand = [k for k, v in kernels.items() if v["alg_bytes_per_launch"]]
        dom = max(cand, key=lambda k: (kernels[k]["alg_bytes_per_launch"], kernels[k]["us_per_launch"])) \
            if cand else None
        traffic = (_ncu_traffic(args.config) or {}).get(dom) if dom else None
        roof = None
        if dom:
            kd = kernels[dom]
            roof = dict(bound="hbm", kernel=dom, achieved=kd["alg_gbs"], peak=hbm, unit="GB/s",
                        frac=round(kd["alg_gbs"] / hbm, 4), traffic=traffic, peak_source=peak_kind,
                        algorithmic_bytes_per_launch=kd["alg_bytes_per_launch"], us_per_launch=kd["us_per_launch"],
                        share_of_step=kd["share"],
                        note="per-launch duration from CUDA events around each library kernel in an instrumented "
                             "repeat of the timed steps")
        line = dict(
            metric=METRIC, value=round(value, 3), unit="GB/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
            ms_per_step=round(st_ms, 5), higher_is_better=True, scaling="weak", vs_baseline=None,
            dtype=conf["dtype"], data="synthetic (integer-exact device generator, SURVEY.md §8(d))",
            config=dict(workload=conf["workload"], codec=CODEC, if_shape=[N, K], batch_per_gpu=B,
                        parallelism=f"dp{world} (independent IF streams per GPU, no collectives)",
                        launch=("CUDA graph per step" if args.graph else "direct launches") +
                               f", {args.depth} pipeline slot(s) on separate streams (step i decode overlaps "
                               f"step i+1 encode)",
                        l2="per-step inputs %.0f MB/GPU %s the 126 MB L2; no flush" %
                           (raw_bytes / 1e6, "exceed" if raw_bytes > 126e6 else "fit in")),
            roofline=roof,
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
            cpu_baseline=cpu,
        )
        print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


def run_ours_mixed(args, conf, rank, world, local_rank):
    """C5: this rank's share of the 8192 mixed streams (LPT by bytes), one ListEncoder launch
    sequence per step, pipelined over `depth` slots like the homogeneous configs."""
    import torch

    import paper_2511_11608_b200 as sif
    from paper_2511_11608_b200.shard import mixed_workload, shard_streams

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    mix = mixed_workload(conf["mixed"])
    mine = shard_streams([(r, c, b) for _k, r, c, b in mix], world, rank)
    xs, seeds = [], []
    for sid in mine:
        kind, r, c, b = mix[sid]
        t = torch.empty((r, c), dtype=torch.float32 if b == 4 else torch.bfloat16, device=dev)
        sif.synthetic(kind, r, c, sid, out=t)
        xs.append(t)
        seeds.append(sid)
    cfg = sif.CodecConfig(**CODEC)
    raw_bytes = sum(mix[sid][1] * mix[sid][2] * mix[sid][3] for sid in mine)
    job_raw = sum(r * c * b for _k, r, c, b in mix)
    elems = sum(mix[sid][1] * mix[sid][2] for sid in mine)
    dense_out = 4 * elems
    pipe = sif.BatchPipeline(xs, cfg, seeds, depth=args.depth, graphs=args.graph)
    slot0 = pipe.slots[0]
    payload_total = int(slot0["enc"].out_len.cpu().numpy().sum())
    alg_enc, alg_dec = raw_bytes + payload_total, payload_total + dense_out
    stream = torch.cuda.current_stream()
    pipe.begin()
    for _ in range(args.warmup):
        pipe.step()
    pipe.end()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        pipe.begin()
        for _ in range(args.steps):
            pipe.step()
        pipe.end()
        t_end.record(stream)
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    st_ms = t_start.elapsed_time(t_end) / args.steps
    pipe.check()
    assert torch.equal(pipe.ys(0), pipe.ys(len(pipe.slots) - 1)), "slots disagree"
    enc, dec = slot0["enc"], slot0["dec"]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        ev[i][0].record(stream)
        enc.run()
        ev[i][1].record(stream)
        dec.run()
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    enc_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / args.steps
    dec_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / args.steps
    if pg:
        t = torch.tensor([st_ms, enc_ms, dec_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        st_ms, enc_ms, dec_ms = [float(v) for v in t.cpu().numpy()]
    kprof = _kernel_profile(sif, lambda: (enc.run(), dec.run()), args.steps)
    # e2e: pinned host streams -> H2D -> encode -> decode -> D2H (ListRoundTrip)
    rt = sif.ListRoundTrip([x.cpu() for x in xs], cfg, seeds, parts=4)
    for _ in range(2):
        rt.run()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    e2e_steps = max(2, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        rt.run()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    rt.check()
    for k in (0, len(xs) // 2, len(xs) - 1):
        assert torch.equal(rt.y(k), dec.outs[k].cpu()), "e2e decode differs"
    if pg:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_ms = float(t.item())
    cpu = None
    if rank == 0 and args.cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        n_if = max(8, min(2048, int(2.0 * cores / 0.03)) // 8 * 8)
        r = cpu_measure_mixed(conf, n_if, 2, 1, cores)
        cpu = dict(value=round(r["value"], 6), unit="GB/s", cores=cores, kind="port",
                   sample=f"{n_if} streams of the mix (every k-th group of 8 sids) x 2 steps, {cores} processes, "
                          f"oracle/ NumPy port ({r['seconds']:.1f} s)")
    if rank == 0:
        hbm, peak_kind = _peaks()
        step_gbs = (alg_enc + alg_dec) / (st_ms * 1e-3) / 1e9
        kernels = {}
        prof_ms = sum(v["ms_total"] for v in kprof.values()) or 1.0
        for name, v in kprof.items():
            per = v["ms_total"] / v["launches"]
            alg = _alg_bytes(name, raw_bytes, payload_total, dense_out)
            kernels[name] = dict(us_per_launch=round(per * 1e3, 2), launches_per_step=v["launches"] // args.steps,
                                 share=round(v["ms_total"] / prof_ms, 4), alg_bytes_per_launch=alg,
                                 alg_gbs=round(alg / (per * 1e-3) / 1e9, 1) if alg else 0.0)
        cand = [k for k, v in kernels.items() if v["alg_bytes_per_launch"]]
        dom = max(cand, key=lambda k: (kernels[k]["alg_bytes_per_launch"], kernels[k]["us_per_launch"])) \
            if cand else None
        roof = None
        if dom:
            kd = kernels[dom]
            roof = dict(bound="hbm", kernel=dom, achieved=kd["alg_gbs"], peak=hbm, unit="GB/s",
                        frac=round(kd["alg_gbs"] / hbm, 4), traffic=(_ncu_traffic("c5") or {}).get(dom),
                        peak_source=peak_kind, algorithmic_bytes_per_launch=kd["alg_bytes_per_launch"],
                        us_per_launch=kd["us_per_launch"], share_of_step=kd["share"],
                        note="per-launch duration from CUDA events around each library kernel")
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
                        parallelism=f"dp{world} (streams sharded by LPT on bytes, no collectives)",
                        launch=("CUDA graph per step" if args.graph else "direct launches") +
                               f", {args.depth} pipeline slot(s) on separate streams",
                        l2="per-step inputs %.0f MB/GPU exceed the 126 MB L2; no flush" % (raw_bytes / 1e6)),
            roofline=roof,
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
            cpu_baseline=cpu,
        )
        print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


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
    ap.add_argument("--depth", type=int, default=None,
                    help="pipeline slots: consecutive steps overlap on this many streams (1 = sequential); "
                         "default per config (c2 4, c3 8, c4 4, c5 2: measured, tools/sweep_depth*.sh)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    conf = CONFIGS[args.config]
    if args.depth is None:
        args.depth = conf.get("depth", 3)
    if args.impl == "reference":
        run_reference(args, conf, rank)
        return
    if conf.get("mixed"):
        run_ours_mixed(args, conf, rank, world, local_rank)
        return
    run_ours(args, conf, rank, world, local_rank)


if __name__ == "__main__":
    main()
