"""Hot-path hyperparameters (the fields of ref/config.py:14-86 that the
epipolar adjustment and the global translation read).

The drop-in functions accept any config object with these attributes -- in
particular the reference's own ``fastmap.config.PipelineConfig`` -- so no new
required keys are introduced.
"""

from dataclasses import dataclass


@dataclass
class HotPathConfig:
    # translation (ref/config.py:37-39)
    translation_lr: float = 1e-3
    translation_steps: int = 6000
    translation_inits: int = 3
    # epipolar adjustment (ref/config.py:43-50)
    epipolar_lr: float = 1e-4
    lr_decay: float = 2.0
    prune_rounds: int = 3
    prune_threshold_start: float = 0.01
    prune_threshold_end: float = 0.005
    irls_iters_between_prunes: int = 3
    epipolar_epoch_steps: int = 100
    refine_focal: bool = True
    # optimizer (ref/config.py:52-54)
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8

    def __post_init__(self):
        for name in ("translation_steps", "translation_inits", "prune_rounds",
                     "irls_iters_between_prunes", "epipolar_epoch_steps"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        for name in ("translation_lr", "epipolar_lr"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.prune_threshold_start < self.prune_threshold_end:
            raise ValueError("prune thresholds must be non-increasing")
        if self.prune_threshold_end <= 0:
            raise ValueError("prune thresholds must be positive")


PipelineConfig = HotPathConfig
