"""The paper's unfused-ABFT overhead model (§V.A), used only to report the
prediction next to measured overheads:

    T_ovhd = (6 + 2K/Kc) t_mv,    T_ovhd / T_GEMM = (6 + 2K/Kc) P_mm / (n P_mv)
"""


def predict_unfused_overhead(n: int, K: int, Kc: int, P_mm: float, P_mv: float) -> float:
    if min(n, K, Kc) <= 0 or P_mm <= 0 or P_mv <= 0 or Kc > K:
        raise ValueError("need positive n, K, Kc <= K and throughputs")
    return (6.0 + 2.0 * K / Kc) * P_mm / (n * P_mv)
