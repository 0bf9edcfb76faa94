// Meta-gradient path (BASELINE config 4) -- see lrnr_gpu.cu meta_step.
#pragma once
