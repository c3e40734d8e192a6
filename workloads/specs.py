"""GPU hardware-spec table S (paper Table II / Table VI) as raw input records.

This module holds *data only*: the Table II parameter vector for each GPU the
paper evaluates, plus the hypothetical-hardware grid of BASELINE config 5.  It
contains none of the method's arithmetic (no cycles, no reciprocals, no
occupancy); both the CUDA path and the CPU oracle consume these records.

Sources
-------
* PAPER.md Table II ("Hardware specifications required by SynPerf")
  fixes the field list and value ranges.
* PAPER.md Table VI prints, per GPU, only: SMs, Mem BW (GB/s),
  Tensor BF16 (ops/clk/SM) and Freq (MHz).  Those four values are used
  verbatim, including the printed oddities (L20 Tensor = 516 next to L40's 512,
  P:452/P:458; H200 BW = 4917 > Table II's max 4916).
* Every other field is a fill (listed in DESIGN.md):
  compute capability, FMA lanes/SM (64 on sm_80, else 128), XU = 16 (Table II),
  shared-memory bytes/clk/SM = 128 (Table II), shared memory per SM, register
  file = 256 KB (Table II), max warps / CTAs per SM — all from public CUDA
  compute-capability data.  L2 bandwidth is absent from Table VI; we use the
  placeholder clamp(2.5 * BW_glob, 2430, 10400) GB/s (Table II's L2 range),
  flagged "parity unpinned" in DESIGN.md.  fp16 tensor throughput = bf16;
  fp8 = 2 * bf16 on sm_89+ and 0 (absent) on sm_80/86.

The record layout (`SPEC_DTYPE`) is byte-identical to `sp_gpu_spec` in
include/synperf.h (112 bytes, natural alignment).
"""
from __future__ import annotations

import numpy as np

KB = 1024

SPEC_DTYPE = np.dtype(
    [
        ("name", "S32"),
        ("cc_major", "<i4"),
        ("cc_minor", "<i4"),
        ("num_sms", "<i4"),
        ("th_tensor_bf16", "<i4"),
        ("th_tensor_fp16", "<i4"),
        ("th_tensor_fp8", "<i4"),
        ("th_fma", "<i4"),
        ("th_xu", "<i4"),
        ("smem_bw_bytes_per_clk", "<i4"),
        ("smem_per_sm_bytes", "<i4"),
        ("regfile_per_sm_bytes", "<i4"),
        ("max_warps_per_sm", "<i4"),
        ("max_ctas_per_sm", "<i4"),
        ("_pad", "<i4"),
        ("sm_clock_mhz", "<f8"),
        ("bw_global_gbps", "<f8"),
        ("bw_l2_gbps", "<f8"),
    ],
    align=True,
)
assert SPEC_DTYPE.itemsize == 112, SPEC_DTYPE.itemsize


def l2_placeholder_gbps(bw_glob: float) -> float:
    """R19 fill: L2 bandwidth is not printed in Table VI."""
    return float(min(max(2.5 * bw_glob, 2430.0), 10400.0))


# name, arch, CC, SMs, MemBW, TensorBF16, MHz  -- Table VI rows
# followed by fills: smem/SM (KB), max warps/SM, max CTAs/SM
_TABLE_VI = [
    # ---- training GPUs (Table VI top half) ----
    ("A40", (8, 6), 84, 696.0, 1024, 1740.0, 100, 48, 16),
    ("A100", (8, 0), 108, 2039.0, 2048, 1410.0, 164, 64, 32),
    ("RTX 6000 Ada", (8, 9), 142, 960.0, 1024, 2505.0, 100, 48, 24),
    ("L20", (8, 9), 92, 864.0, 516, 2520.0, 100, 48, 24),
    ("H20", (9, 0), 78, 4023.0, 1024, 1830.0, 228, 64, 32),
    ("H800", (9, 0), 132, 3352.0, 4096, 1830.0, 228, 64, 32),
    # ---- unseen GPUs (Table VI bottom half) ----
    ("RTX A6000", (8, 6), 84, 768.0, 1024, 1800.0, 100, 48, 16),
    ("L40", (8, 9), 142, 864.0, 512, 2490.0, 100, 48, 24),
    ("H100", (9, 0), 132, 3352.0, 4096, 1830.0, 228, 64, 32),
    ("H200", (9, 0), 132, 4917.0, 4096, 1830.0, 228, 64, 32),
    ("RTX PRO 6000 S", (12, 0), 188, 1792.0, 1024, 2340.0, 100, 48, 24),
]

GPU_NAMES = [row[0] for row in _TABLE_VI]


def paper_gpu_specs() -> np.ndarray:
    """The 11 GPUs of Table VI as SPEC_DTYPE records, in table order."""
    out = np.zeros(len(_TABLE_VI), dtype=SPEC_DTYPE)
    for i, (name, cc, sms, bw, tbf16, mhz, smem_kb, mw, mc) in enumerate(_TABLE_VI):
        r = out[i]
        r["name"] = name.encode()
        r["cc_major"], r["cc_minor"] = cc
        r["num_sms"] = sms
        r["th_tensor_bf16"] = tbf16
        r["th_tensor_fp16"] = tbf16
        r["th_tensor_fp8"] = 2 * tbf16 if cc >= (8, 9) else 0
        r["th_fma"] = 64 if cc == (8, 0) else 128
        r["th_xu"] = 16
        r["smem_bw_bytes_per_clk"] = 128
        r["smem_per_sm_bytes"] = smem_kb * KB
        r["regfile_per_sm_bytes"] = 256 * KB
        r["max_warps_per_sm"] = mw
        r["max_ctas_per_sm"] = mc
        r["sm_clock_mhz"] = mhz
        r["bw_global_gbps"] = bw
        r["bw_l2_gbps"] = l2_placeholder_gbps(bw)
    return out


def spec_by_name(name: str) -> np.ndarray:
    s = paper_gpu_specs()
    idx = GPU_NAMES.index(name)
    return s[idx : idx + 1].copy()


def hypothetical_sweep_specs(n: int | None = None) -> np.ndarray:
    """BASELINE config 5: the 100,000-point hypothetical-hardware grid.

    SMs {64,68,...,260} (50) x HBM BW log-spaced 500..16000 GB/s (40) x clock
    {1200,1400,...,3000} MHz (10) x SMEM/SM {100,164,228,256,320} KB (5).
    Fixed: Tensor 8192 ops/clk/SM (B200-like, beyond Table II's 4096), FMA 128,
    XU 16, L2 = 2.5*BW (no clamp: beyond Table II), 128 B/clk, 256 KB RF,
    64 warps, 32 CTAs.  Spec-major order: SMs slowest, SMEM fastest.
    If `n` is given, the first n grid points are returned.
    """
    sms = np.arange(64, 261, 4)
    bws = np.geomspace(500.0, 16000.0, 40)
    mhz = np.arange(1200.0, 3000.0 + 1, 200.0)
    smem = np.array([100, 164, 228, 256, 320])
    assert len(sms) == 50 and len(bws) == 40 and len(mhz) == 10
    grid = np.stack(np.meshgrid(sms, bws, mhz, smem, indexing="ij"), -1).reshape(-1, 4)
    if n is not None:
        grid = grid[:n]
    out = np.zeros(len(grid), dtype=SPEC_DTYPE)
    out["name"] = [f"hyp-{i}".encode() for i in range(len(grid))]
    out["cc_major"] = 10
    out["cc_minor"] = 0
    out["num_sms"] = grid[:, 0].astype(np.int32)
    out["th_tensor_bf16"] = 8192
    out["th_tensor_fp16"] = 8192
    out["th_tensor_fp8"] = 16384
    out["th_fma"] = 128
    out["th_xu"] = 16
    out["smem_bw_bytes_per_clk"] = 128
    out["smem_per_sm_bytes"] = (grid[:, 3] * KB).astype(np.int32)
    out["regfile_per_sm_bytes"] = 256 * KB
    out["max_warps_per_sm"] = 64
    out["max_ctas_per_sm"] = 32
    out["sm_clock_mhz"] = grid[:, 2]
    out["bw_global_gbps"] = grid[:, 1]
    out["bw_l2_gbps"] = 2.5 * grid[:, 1]
    return out


# ---- communication calibration tables (inputs of the E2E composition) ----
# The paper profiles All-Reduce / Send-Recv per topology and regresses latency on
# volume; no profile is published.  These are synthetic alpha-beta tables
# ("a synthetic alpha-beta generator produces desk-scale tables"):
# latency = alpha + algorithmic bytes / link GB/s at 2^10 .. 2^30 bytes.
# Link bandwidths are public interconnect figures (NVLink for the SXM parts,
# PCIe otherwise): realism "parity unpinned".
LINK_GBPS = {"A40": 56.0, "A100": 300.0, "RTX 6000 Ada": 25.0, "L20": 25.0, "H20": 450.0,
             "H800": 200.0, "RTX A6000": 56.0, "L40": 25.0, "H100": 450.0, "H200": 450.0,
             "RTX PRO 6000 S": 50.0}
COMM_POINTS = np.array([2.0 ** k for k in range(10, 31)])


def synthetic_comm_tables(spec_arr: np.ndarray, tp: int, alpha_us: float = 8.0) -> dict:
    """{"bytes": [P], "allreduce_us": [G][P], "sendrecv_us": [G][P]} (fp64).
    Ring all-reduce moves 2(tp-1)/tp of the buffer per GPU; send/recv moves it once."""
    names = [n.decode() if isinstance(n, bytes) else str(n) for n in spec_arr["name"]]
    bw = np.array([LINK_GBPS.get(n, 450.0) for n in names]) * 1e3  # bytes per us
    ar_factor = 2.0 * (tp - 1) / tp if tp > 1 else 0.0
    b = COMM_POINTS
    ar = alpha_us + ar_factor * b[None, :] / bw[:, None]
    sr = 0.5 * alpha_us + b[None, :] / bw[:, None]
    return {"bytes": b.copy(), "allreduce_us": ar, "sendrecv_us": sr}
