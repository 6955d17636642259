"""paper_2602_21203_b200 -- B200-native (sm_100a) hot path of Squint's visual SAC update
(arXiv 2602.21203): libsquint (C ABI, include/squint.h) + this thin ctypes binding."""
from . import squint  # noqa: F401  (fails loudly when libsquint.so is missing)
from .squint import (FP32, BF16, Dims, HParams, Learner, Replay, State, act_workspace_bytes,  # noqa: F401
                     make_dims, make_hparams, param_layout, replay_from_tensors, squint_act, squint_insert, squint_insert2, squint_insert_ex,
                     squint_soft_update, squint_stage_pinned, squint_update, workspace_bytes, workspace_region)
