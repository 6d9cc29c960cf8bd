#pragma once
// GPU Manager + Cache Manager state of the function-execution path.
//
// Public API mirrors proj/include/gpufaas/cluster.hpp:19-140 (ClusterState is
// concrete, GpuState getters return the same container types) so the
// reference's own callers — the naive ReferenceScheduler oracle and the
// reference test suites — compile unchanged against it.
//
// Differences under the hood (B200 build):
//   * model ids are interned to dense integers (catalog rows when a catalog is
//     bound), so the scheduler's hot loops never hash strings;
//   * residency, pins and model locations are vectors indexed by that integer;
//   * an ExecutionListener (extension) receives every begin/complete — this is
//     where the per-GPU daemon with the HBM arena (paper_2303_05601_b200/csrc/
//     device) attaches, at exactly the points where the reference charges the
//     profiled load/infer constants (proj/src/cluster.cpp:159-168, 176-187).

#include <cstdint>
#include <deque>
#include <list>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "gpufaas/catalog.hpp"
#include "gpufaas/sim_time.hpp"
#include "gpufaas/workload.hpp"

namespace gpufaas {

struct CachedModel {
    std::string model_id;
    double occupation_mb = 0.0;
    std::uint64_t last_use_tick = 0;  // cluster-wide counter; larger = more recent
    std::int64_t uses = 0;            // insert counts as one use
};

struct LocalEntry {
    int request_id = -1;
    std::string model_id;
    SimTime infer_time_us = 0;
};

struct RunningTask {
    int request_id = -1;
    std::string model_id;
};

struct ExecutionStart {
    SimTime completion_us = 0;
    bool cache_hit = false;
    std::vector<std::string> evicted;  // LRU-first
};

// Extension: dense model-id interning shared by a cluster and its GPUs.
class ModelTable {
public:
    int find(const std::string& id) const {
        auto it = ids_.find(id);
        return it == ids_.end() ? -1 : it->second;
    }
    int intern(const std::string& id) {
        auto [it, fresh] = ids_.emplace(id, static_cast<int>(names_.size()));
        if (fresh) names_.push_back(id);
        return it->second;
    }
    const std::string& name(int idx) const { return names_.at(static_cast<std::size_t>(idx)); }
    int size() const { return static_cast<int>(names_.size()); }

private:
    std::unordered_map<std::string, int> ids_;
    std::vector<std::string> names_;
};

// Extension: data-plane hook. Called after the cache bookkeeping of
// begin_execution (model = interned index, evicted = interned LRU-first list,
// source_gpu = lowest-id *other* GPU that held the model just before this
// start, -1 if none — the NVLink peer for a false miss), and from complete().
class ExecutionListener {
public:
    virtual ~ExecutionListener() = default;
    virtual void on_begin_execution(int gpu_id, const Request& request, int model, bool cache_hit,
                                    const std::vector<int>& evicted, int source_gpu, SimTime now,
                                    SimTime completion_us) = 0;
    virtual void on_complete(int gpu_id, int request_id, SimTime now) = 0;
};

class ClusterState;

class GpuState {
public:
    GpuState() = default;
    GpuState(const GpuState& other) { *this = other; }
    GpuState& operator=(const GpuState& other);  // re-binds the index into the copied list
    GpuState(GpuState&&) noexcept = default;
    GpuState& operator=(GpuState&&) noexcept = default;

    int gpu_id() const { return id_; }
    double capacity_mb() const { return capacity_mb_; }
    double cached_mb() const { return used_mb_; }
    double free_mb() const { return capacity_mb_ - used_mb_; }

    bool is_busy() const { return running_.has_value(); }
    SimTime busy_until_us() const;  // logic_error when idle
    const std::optional<RunningTask>& running() const { return running_; }
    // Extension (pipelined GPUs, SchedulerConfig::pipeline): can a dispatch
    // start here now? Reference mode: when idle. Pipelined: while nothing is
    // staged behind the running task.
    // A running GPU stages only while its unpinned memory could take any
    // catalog model (so the staged load's victim selection cannot fail).
    bool accepting() const {
        if (!pipeline_) return !running_.has_value();
        if (staged_) return false;
        return !running_ || capacity_mb_ - pinned_mb() >= stage_headroom_mb_;
    }
    double pinned_mb() const;  // occupation of models with pins, summed MRU -> LRU
    const std::optional<RunningTask>& staged() const { return staged_; }
    SimTime staged_until_us() const { return staged_until_us_; }

    // Resident models, most recently used first.
    const std::list<CachedModel>& cache() const { return lru_; }
    std::vector<std::string> cached_model_ids() const;
    bool is_cached(const std::string& model_id) const;
    const CachedModel* cached_entry(const std::string& model_id) const;

    // Sum of `uses` over residents: the idle-GPU service order key.
    std::int64_t hotness() const { return hotness_; }

    const std::deque<LocalEntry>& local_queue() const { return local_; }
    SimTime local_queue_infer_us() const { return local_infer_us_; }
    int pin_count(const std::string& model_id) const;

    // Extension: integer-keyed fast paths used by the B200 scheduler.
    bool holds(int model) const {
        return model >= 0 && static_cast<std::size_t>(model) < slot_.size() && slot_[model].live;
    }
    const CachedModel* entry(int model) const { return holds(model) ? &*slot_[model].it : nullptr; }
    int pins(int model) const {
        return model >= 0 && static_cast<std::size_t>(model) < slot_.size() ? slot_[model].pins : 0;
    }
    int running_model() const { return running_model_; }

private:
    friend class ClusterState;
    struct Slot {
        std::list<CachedModel>::iterator it{};
        bool live = false;
        int pins = 0;  // running + locally queued references
    };
    Slot& slot(int model) {
        if (static_cast<std::size_t>(model) >= slot_.size()) slot_.resize(static_cast<std::size_t>(model) + 1);
        return slot_[static_cast<std::size_t>(model)];
    }

    int id_ = -1;
    double capacity_mb_ = 0.0;
    double used_mb_ = 0.0;          // maintained with += / -= like the reference
    std::int64_t hotness_ = 0;
    std::list<CachedModel> lru_;    // front = MRU
    std::vector<Slot> slot_;        // by interned model
    std::deque<LocalEntry> local_;
    SimTime local_infer_us_ = 0;
    std::optional<RunningTask> running_;
    int running_model_ = -1;
    SimTime busy_until_us_ = 0;
    std::optional<RunningTask> staged_;  // pipelined mode: next task, behind running_
    int staged_model_ = -1;
    SimTime staged_until_us_ = 0;
    SimTime copy_free_us_ = 0;           // end of the last model load started here
    bool pipeline_ = false;
    double stage_headroom_mb_ = 0.0;     // largest catalog model
    int pinned_models_ = 0;         // models with pins > 0
    std::shared_ptr<ModelTable> table_;
};

class ClusterState {
public:
    ClusterState(int gpu_count, double capacity_mb);

    int gpu_count() const { return static_cast<int>(gpus_.size()); }
    const GpuState& gpu(int gpu_id) const;

    bool is_cached(int gpu_id, const std::string& model_id) const;
    const std::set<int>& locations(const std::string& model_id) const;  // ascending ids
    int location_count(const std::string& model_id) const;
    bool cached_anywhere_except(const std::string& model_id, int gpu_id) const;

    // Remaining run time plus summed inference of the local queue.
    SimTime estimate_finish_time(int gpu_id, SimTime now) const;

    // LRU-first victims freeing `needed_mb`, skipping pinned models (pure query).
    std::vector<std::string> select_victims(int gpu_id, double needed_mb) const;

    ExecutionStart begin_execution(int gpu_id, const Request& request, SimTime now,
                                   const Catalog& catalog);
    int complete(int gpu_id, SimTime now);

    void push_local(int gpu_id, const Request& request, const Catalog& catalog);
    LocalEntry pop_local(int gpu_id);

    bool fully_drained() const;
    void check_consistency() const;  // logic_error on any drift

    // ---- extensions -------------------------------------------------------
    // Intern the catalog first so interned index == catalog row.
    void bind_catalog(const Catalog& catalog);
    int model_index(const std::string& model_id) const { return table_->find(model_id); }
    int intern(const std::string& model_id) { return table_->intern(model_id); }
    const std::string& model_name(int model) const { return table_->name(model); }
    const std::set<int>& locations_of(int model) const;
    bool held_elsewhere(int model, int gpu_id) const;
    void set_listener(ExecutionListener* listener) { listener_ = listener; }
    ExecutionListener* listener() const { return listener_; }
    // Live (closed-loop) mode, run_live(): completions come from the device at
    // real times, so complete() accepts any time and estimate_finish_time()
    // treats a task running past its predicted end as finishing now. The
    // default (replay) mode keeps the reference's exact checks.
    void set_live(bool live) { live_ = live; }
    bool live() const { return live_; }
    // Pipelined GPUs (SchedulerConfig::pipeline); set before the first dispatch.
    void set_pipeline(bool on, double stage_headroom_mb);
    bool pipeline() const { return !gpus_.empty() && gpus_.front().pipeline_; }

private:
    GpuState& gpu_mut(int gpu_id);
    void touch(GpuState& g, int model);
    void evict(GpuState& g, int model);
    void insert(GpuState& g, int model, const ModelProfile& profile);
    void pin(GpuState& g, int model);
    void unpin(GpuState& g, int model);
    std::set<int>& holders(int model);
    void select_victims_idx(const GpuState& g, double needed_mb, std::vector<int>& out) const;

    std::vector<GpuState> gpus_;
    std::shared_ptr<ModelTable> table_;
    std::vector<std::set<int>> holders_;  // by interned model
    std::uint64_t tick_ = 0;
    ExecutionListener* listener_ = nullptr;
    std::vector<int> scratch_victims_;
    bool live_ = false;
};

}  // namespace gpufaas
