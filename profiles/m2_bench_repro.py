"""Reproduce bench.py's M2 hot number in isolation: measure_config('M2') alone, after the 2^4
chain, after M1."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1612_07873_b200 as cd  # noqa: E402

pm = bench._perfmodel()
peak = bench.measured_peak()[0]
sampler = bench.ClockSampler(0)
mode = sys.argv[1]
if mode == "chain":
    bench.measure_chain(cd, torch, pm, sampler)
if mode == "m1":
    bench.measure_config(cd, torch, pm, sampler, "M1", "fp32", peak)
if mode == "eager":
    os.environ["CD_TUNE_EAGER"] = "1"
r = bench.measure_config(cd, torch, pm, sampler, "M2", "fp32", peak)
print(mode, r["variant"], r["hot"]["us"], r["cold"]["us"])
r = bench.measure_config(cd, torch, pm, sampler, "M2", "fp32", peak)
print(mode, "again", r["variant"], r["hot"]["us"], r["cold"]["us"])
