// Ready-queue schedule of a planned phase (host side; executed by k_exec_rq in
// exec.cu).  The phase's task DAG (XTask + xdeps, plan.h) is turned into
//   * successor lists (CSR) and per-task predecessor counts,
//   * a priority level per schedulable node from its bottom level (estimated
//     cost of the longest path from the node to the end of the phase),
//   * RQ_NQ FIFO queues scanned in priority order.
// A schedulable node is a single task or a whole cooperative truncation group
// (XTask.sub == 0 .. nsub-1, consecutive in xt): a group is pushed as nsub
// consecutive slots of one queue, so at most one group per queue is ever
// partially claimed and the CTAs spinning in group barriers never exceed
// RQ_NCOOP * (TR_COOP_MAX - 1) < grid (deadlock freedom, see exec.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "plan.h"

namespace hm {

constexpr int RQ_NSINGLE = 28;                 // priority levels for single tasks
constexpr int RQ_NCOOP = 4;                    // priority levels for cooperative groups
constexpr int RQ_NQ = RQ_NSINGLE + RQ_NCOOP;   // queues, scanned 0 (highest) .. RQ_NQ-1
static_assert(RQ_NQ <= 32, "one queue per lane of the scheduling warp");

struct Sched {
    std::vector<int32_t> succ_begin;   // nx + 1
    std::vector<int32_t> succ;         // successor task positions (group leaders or single tasks)
    std::vector<int32_t> need;         // nx: predecessors a node waits for (0 for roots and non-leader subs)
    std::vector<int32_t> queue;        // nx: queue id of the node (leaders/singles), -1 for non-leader subs
    std::vector<int32_t> qbase;        // RQ_NQ + 1: first slot of each queue
    std::vector<int32_t> slot_init;    // nx: task id in the slot (roots pre-filled) or -1
    std::vector<int32_t> ctl_init;     // 2 * RQ_NQ + 2: {head, tail} per queue, finished, pad
    int32_t max_nsub = 1;              // largest cooperative group of the phase
    std::vector<int32_t> succ2;        // 2 |succ|: {successor, need << 11 | nsub << 5 | queue} (device form)
};

constexpr int RQ_NEED_SHIFT = 11, RQ_NSUB_SHIFT = 5;
inline int rq_pack(int need, int nsub, int queue) { return (need << RQ_NEED_SHIFT) | (nsub << RQ_NSUB_SHIFT) | queue; }

// Queue id of priority level `lvl` in [0, RQ_NSINGLE) for a single task / a group.
int rq_queue_of(int lvl, bool coop);

// Build the schedule of phase `p` (throws ApiError on a malformed DAG).
void build_sched(const Phase& p, Sched& s);

}  // namespace hm
