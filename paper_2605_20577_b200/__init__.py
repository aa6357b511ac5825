"""B200-native batched Riichi-Mahjong environment step (Pgx-style API).

Drop-in for the reference `mjsim` env path (init / step / observe, the
legal mask, rewards and the random-policy rollout), computed by
hand-written sm_100a CUDA kernels behind the C ABI in include/rinshan.h.
"""
