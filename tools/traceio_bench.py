"""Native vs reference load_job on a saved job (container only: imports the
reference from /root/reference to write the job and to time its loader)."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")
from dltsim.cluster import ClusterSpec, load_device_preset
from dltsim.collate import collate, load_job, save_job
from dltsim.workload import ConfigPoint, ModelSpec, default_schedule, generate_representatives
from paper_2503_20191_b200 import traceio
from paper_2503_20191_b200.rawtrace import from_reference, raw_digest

model = ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cl = ClusterSpec(1, 8, 80 * 2 ** 30, load_device_preset("fast"))
cfg = ConfigPoint(1, 8, 8, 1, True, False, False, 512)
tr, ex = generate_representatives(model, cfg, cl, default_schedule(cfg), dispatch_overhead_ns=5000)
with tempfile.TemporaryDirectory() as d:
    save_job(collate(tr, ex, cl), d)
    nbytes = sum(os.path.getsize(os.path.join(d, f)) for f in os.listdir(d))
    t0 = time.perf_counter(); ref = from_reference(load_job(os.path.join(d, "job.manifest"), cl)); t1 = time.perf_counter()
    nat = traceio.load_raw_job(os.path.join(d, "job.manifest"), cl); t2 = time.perf_counter()
    assert raw_digest(ref) == raw_digest(nat)
    print(f"{cfg.label()}: {nbytes / 1e6:.1f} MB text, {ref.n_events} events; reference load_job + "
          f"from_reference {t1 - t0:.2f} s, native {t2 - t1:.3f} s ({(t1 - t0) / (t2 - t1):.0f}x), "
          f"native {nbytes / 1e6 / (t2 - t1):.0f} MB/s")
