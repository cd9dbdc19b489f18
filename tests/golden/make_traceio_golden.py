"""Golden fixtures for the native trace / manifest I/O,
made by running the REAL reference in this container:

    python tests/golden/make_traceio_golden.py [--ref /root/reference/pkg]

* traceio/<job>/      save_job() output of the reference for a few generated
                      jobs (manifest + rank_<r>.trace), byte for byte;
* traceio_jobs.npz    rawtrace.from_reference(load_job(manifest, cluster)) of
                      each, i.e. what the native loader must produce;
* traceio_errors.json parse / validation / collation failures: the input
                      (a trace text, or a manifest plus trace texts) and the
                      reference's exception class and message.
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

JOBS = [
    # name, model (name, L, h, s, vocab), cluster (hosts, dph), config, schedule
    ("c1_gpt2_2r", ("gpt2-small", 12, 768, 1024, 50304), (1, 2), (1, 1, 1, 1, 0, 0, 0, 8), None),
    ("tp2pp2_8r", ("t", 8, 128, 64, 512), (1, 8), (2, 2, 2, 1, 1, 1, 1, 16), None),
    ("pp4vs2_16r_2h", ("t", 8, 128, 64, 512), (2, 8), (2, 4, 1, 2, 0, 1, 0, 32), "interleaved"),
    ("tp1pp2dp4_8r_gpipe", ("t", 8, 128, 64, 512), (1, 8), (1, 2, 2, 1, 1, 0, 1, 32), "gpipe"),
]


def header(rank=0, host=0, device=0):
    return f"dltsim-trace v1 rank={rank} host={host} device={device}\n"


def trace_cases():
    """(text) inputs for parse_trace: every TraceParseError path and every
    validate_trace rule (trace.py:333-495)."""
    H = header()
    ok_kernel = "0 KernelLaunch stream=0 op=gemm dtype=bf16 flops=10 bytes=20 a.k=1 a.m=2\n"
    cases = [
        "", "\n", "garbage\n", "dltsim-trace v2 rank=0 host=0 device=0\n",
        "dltsim-trace v1 rank=0 host=0\n", "dltsim-trace v1 rank=x host=0 device=0\n",
        "  dltsim-trace v1 rank=0 host=0 device=0\n",
        "dltsim-trace v1 rank=3 host=0 device=3   \n",
        H + "0\n", H + "x HostGap dur=1\n", H + "1 HostGap dur=1\n",
        H + "0 HostGap dur\n", H + "0 Bogus dur=1\n", H + "0 HostGap len=1\n",
        H + "0 HostGap\n", H + "0 HostGap dur=1 extra=2\n", H + "0 HostGap dur=1.5\n",
        H + "0 HostGap dur=1_000\n", H + "0 HostGap dur=+7\n", H + "0 HostGap dur=-7\n",
        H + "0 HostGap dur=1__0\n", H + "0 HostGap dur=_1\n", H + "0 HostGap dur=1\r\n1 HostGap dur=2\n",
        H + "0 KernelLaunch stream=0 op=gemm dtype=bf16 flops=1 bytes=2 b.m=1\n",
        H + "0 KernelLaunch stream=0 op=gemm dtype=bf16 flops=1 bytes=2 a.M=1\n",
        H + "0 KernelLaunch stream=0 op=gemm dtype=bf16 flops=1 bytes=2 a.=1\n",
        H + "0 KernelLaunch stream=0 op=gemm dtype=bf16 flops=1 bytes=2 a.m=2 a.k=1\n",
        H + "0 KernelLaunch stream=0 op=gemm dtype=bf16 flops=1 bytes=2 a.m=x\n",
        H + "0 KernelLaunch stream=s op=gemm dtype=bf16 flops=f bytes=2\n",
        H + "0 KernelLaunch stream=0 op=gemm dtype=bf16 flops=f bytes=2\n",
        H + "0 KernelLaunch stream=0 op=gemm dtype=int8 flops=-1 bytes=-2\n",
        H + "0 KernelLaunch stream=-1 op=gemm dtype=\"it's\" flops=1 bytes=2\n",
        H + "0 HostGap dur=-5\n",
        H + "0 MemAlloc id=1 bytes=0\n1 MemAlloc id=1 bytes=5\n2 MemFree id=1\n3 MemFree id=1\n"
            "4 MemFree id=9\n",
        H + "0 Memcpy stream=0 dir=X2Y bytes=0\n1 Memset stream=0 bytes=-1\n",
        H + "0 EventRecord stream=0 event=1 ver=1\n1 EventRecord stream=0 event=1 ver=0\n"
            "2 StreamWaitEvent stream=1 event=2 ver=0\n3 EventSynchronize event=1 ver=5\n",
        H + "0 CommInit comm=a.b nranks=0 rank=3\n1 CommInit comm=bad/id nranks=2 rank=0\n"
            "2 CommInit comm=c nranks=2 rank=1\n3 CommInit comm=c nranks=2 rank=0\n",
        H + "0 Collective stream=0 comm=zz idx=0 kind=AllReduce bytes=8 nranks=2\n"
            "1 CommInit comm=c nranks=2 rank=1\n"
            "2 Collective stream=0 comm=c idx=1 kind=AllToAll bytes=0 nranks=3\n"
            "3 Collective stream=0 comm=c idx=1 kind=SendRecv bytes=8 nranks=2\n",
        H + "".join(f"{i} HostGap dur=-{i + 1}\n" for i in range(8)),
        H + ok_kernel + "\n\n1 StreamSynchronize stream=-3\n2 DeviceSynchronize\n",
        H + "0 DeviceSynchronize x=1\n",
        H + "0 KernelLaunch stream=0 op=gemm dtype=bf16\n",
        H + "0 HostGap dur=99999999999999999999\n",
    ]
    return cases


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    args = ap.parse_args()
    sys.path.insert(0, os.path.join(args.ref, "src"))
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.collate import CollationError, collate, load_job, save_job
    from dltsim.trace import TraceParseError, TraceValidationError, loads_trace
    from dltsim.workload import (ConfigPoint, ModelSpec, ScheduleKind, default_schedule,
                                 generate_representatives)
    from paper_2503_20191_b200.rawtrace import from_reference, raw_digest, save_jobs

    fast = load_device_preset("fast")
    out_root = os.path.join(HERE, "traceio")
    shutil.rmtree(out_root, ignore_errors=True)
    os.makedirs(out_root)
    raws, meta = [], []
    for name, mspec, (nh, dph), cfg, sched in JOBS:
        model = ModelSpec(*mspec)
        cluster = ClusterSpec(nh, dph, 80 * 2 ** 30, fast)
        c = ConfigPoint(*[bool(x) if 4 <= i <= 6 else x for i, x in enumerate(cfg)])
        sk = ScheduleKind(sched) if sched else default_schedule(c)
        tr, ex = generate_representatives(model, c, cluster, sk, dispatch_overhead_ns=5000)
        job = collate(tr, ex, cluster)
        d = os.path.join(out_root, name)
        save_job(job, d)
        back = load_job(os.path.join(d, "job.manifest"), cluster)
        raw = from_reference(back, name=name)
        raws.append(raw)
        meta.append({"name": name, "num_hosts": nh, "devices_per_host": dph,
                     "digest": raw_digest(raw), "reps": len(job.reps), "dups": len(job.dup_of)})
    save_jobs(os.path.join(HERE, "traceio_jobs.npz"), raws,
              {"meta": __import__("numpy").array([json.dumps(meta)])})

    errors = []
    for text in trace_cases():
        try:
            loads_trace(text)
            errors.append({"text": text, "kind": "ok", "message": ""})
        except TraceParseError as e:
            errors.append({"text": text, "kind": "parse", "message": str(e)})
        except TraceValidationError as e:
            errors.append({"text": text, "kind": "validation", "message": str(e)})
        except Exception as e:   # int64 overflow etc.: the reference accepts or raises otherwise
            errors.append({"text": text, "kind": type(e).__name__, "message": str(e)})

    # manifest-level collation failures: mutate the saved 8-rank job
    base = os.path.join(out_root, "tp2pp2_8r")
    files = {f: open(os.path.join(base, f)).read() for f in os.listdir(base)}
    man = files["job.manifest"]
    lines = man.splitlines()
    first_dup = next(l for l in lines if l.startswith("dup "))
    dup_rank = first_dup.split()[1].split("=")[1]
    first_worker = next(l for l in lines if l.startswith("worker "))
    w_rank = first_worker.split()[1].split("=")[1]
    first_dc = next(l for l in lines if l.startswith("dupcomm "))
    muts = {
        "bad_header": man.replace("dltsim-job v1", "dltsim-job v0", 1),
        "unknown_kind": man + "bogus rank=1\n",
        "rep_and_dup": man + f"dup rank={w_rank} rep={w_rank}\n",
        "missing_rep": man.replace(first_dup, f"dup rank={dup_rank} rep=77"),
        "coverage": man.replace(first_dup + "\n", ""),
        "missing_translation": man.replace(first_dc + "\n", ""),
        "position_clash": man.replace(first_dc, " ".join(
            first_dc.split()[:-1]) + " myrank=" + ("1" if first_dc.endswith("=0") else "0")),
        "unresolved": man.replace(first_dc, " ".join(first_dc.split()[:-1]) + " myrank=7"),
        "renamed_comm": man.replace(first_dc, first_dc.replace(" to=", " to=zz")),
    }
    # placement: a trace claiming another slot
    tf = f"rank_{w_rank}.trace"
    t0 = files[tf]
    hdr_line = t0.splitlines()[0]
    muts_traces = {"placement": {tf: t0.replace(hdr_line, hdr_line.replace("device=", "device=9"), 1)}}
    # inconsistent collective bytes on one rep
    import re
    coll = re.search(r"^(\d+) Collective stream=(\d+) comm=(\S+) idx=0 kind=(SendRecv) bytes=(\d+)",
                     t0, re.M)
    if coll:
        muts_traces["inconsistent"] = {tf: t0.replace(coll.group(0), coll.group(0)[:-len(coll.group(5))]
                                                      + str(int(coll.group(5)) + 1), 1)}
    cluster = ClusterSpec(1, 8, 80 * 2 ** 30, fast)
    cases = [(k, v, {}) for k, v in muts.items()] + [(k, man, v) for k, v in muts_traces.items()]
    for key, manifest, tmods in cases:
        with tempfile.TemporaryDirectory() as td:
            for f, body in files.items():
                with open(os.path.join(td, f), "w") as fh:
                    fh.write(tmods.get(f, body) if f != "job.manifest" else manifest)
            try:
                load_job(os.path.join(td, "job.manifest"), cluster)
                kind, msg = "ok", ""
            except CollationError as e:
                kind, msg = "collation", str(e)
            except TraceParseError as e:
                kind, msg = "parse", str(e)
            except TraceValidationError as e:
                kind, msg = "validation", str(e)
            except Exception as e:
                kind, msg = type(e).__name__, str(e)
        errors.append({"case": key, "manifest": manifest, "traces": tmods, "kind": kind,
                       "message": msg, "base": "tp2pp2_8r", "num_hosts": 1,
                       "devices_per_host": 8})
    with open(os.path.join(HERE, "traceio_errors.json"), "w") as f:
        json.dump(errors, f, indent=0)
    print(len(raws), "jobs,", len(errors), "error cases")
    for e in errors:
        print(e.get("case", ""), e["kind"], e["message"][:120])


if __name__ == "__main__":
    main()
