// Force-included (-include) into the reference's own test sources so every
// plan_workload call they make — directly, or through cli.hpp's commands —
// runs the B200 planner (wavesched_gpu::plan_workload over libwsgpu.so).
// The reference planner header is included first so its definition keeps its
// name; everything included after the #define calls the GPU.
#pragma once
#include "wavesched/planner.hpp"
#include "wsgpu/wavesched_compat.hpp"
#define plan_workload wavesched_gpu::plan_workload
#include "wavesched/baselines.hpp"
#include "wavesched/cli.hpp"
#include "wavesched/scenarios.hpp"
#include "wavesched/simulate.hpp"
#include "wavesched/validate.hpp"
