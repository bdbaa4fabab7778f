/*
 * citywalk_b200.h -- C ABI of the B200 env-side hot path (libcitywalk_b200.so).
 *
 * Drop-in boundary for the reference's Python entry points (paths relative to
 * /root/reference/pkg/src/citywalk):
 *
 *   cw_sample_scenes   replaces, per env, urbangen/scene.py:38 generate_scene
 *                      (minus route anchors, scene.py:87/102-158), occupancy.py:28
 *                      rasterize_occupancy, crowd/field.py:60-67 _prepare_env
 *                      (walk cells + _nearest_obstacle_map :571) and
 *                      crowd/step.py:37 spawn_agents (+ routes.py:35 sample_routes),
 *                      as driven by envcore/batch.py:117-122 / 170-181 / 326-339.
 *   cw_spawn_agents    replaces crowd/step.py:37 spawn_agents for host-built grids.
 *   cw_prepare_envs    replaces crowd/field.py:60-67 _prepare_env for host-built grids.
 *   cw_crowd_step      replaces crowd/field.py:90 CrowdField.step (workers ignored:
 *                      results are split-invariant by construction): three
 *                      stream-ordered kernels k_guide -> k_astar -> k_orca.
 *   cw_seed_streams    replaces np.random.Generator(np.random.PCG64(seed)) for
 *                      field.py:36 (per-env goal-resample streams).
 *   cw_child_seeds     replaces rng.py:15 child_seed for the batch seed tree
 *                      (batch.py:85, 165, 179, 332).
 *
 * Conventions: every pointer inside the structs and every array argument is a
 * DEVICE pointer; `stream` is a cudaStream_t (NULL = legacy default stream).
 * Calls are stream-ordered, never synchronise the host and create no threads.
 * The return value is 0 or a cudaError_t; per-env sampling failures are
 * reported in buffers->status (cw_status), guidance capacity errors in
 * state->flags[1].  Results are independent of launch configuration.
 */
#ifndef CITYWALK_B200_H
#define CITYWALK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CW_MAX_TILES 44
#define CW_MAX_CATALOG 32
#define CW_MAX_BLOCKS 64
#define CW_ZONE_PARAMS 8

enum cw_status {
  CW_OK = 0,
  CW_E_CONTRADICTION = 1, /* errors.ContradictionAfterRetries (wfc.py:51)   */
  CW_E_NOROUTE = 2,       /* errors.NoRouteAvailable (routes.py:58, 84)     */
  CW_E_EXTENT = 3,        /* errors.ExtentTooSmall (zones.py:60-61)         */
  CW_E_PATHCAP = 4,       /* guidance path longer than state path_cap       */
  CW_E_HEAPCAP = 5        /* A* open list exceeded heap_cap                 */
};

/* SceneSpec shape shared by a batch (urbangen/types.py:88-115). */
typedef struct cw_scene_params {
  int32_t nx, ny;
  double res;
  double w, l;
  int32_t task;   /* 0 NavClear, 1 NavStatic, 2 NavDynamic, 3 Traverse */
  int32_t split;  /* 0 Train, 1 Test */
  double mix[4];  /* Flat, Slope, Stair, Rough */
  int32_t layout; /* 0 courtyard, 1 blocks, 2 strip */
  int32_t brows, bcols;
  double quad_cdf[3];
  int32_t trows, tcols, cpt;
  int32_t nonflat_split_col;
  int32_t n_cat;
  double cat_w[CW_MAX_CATALOG], cat_l[CW_MAX_CATALOG];
  double cat_reach[CW_MAX_CATALOG];
  uint32_t cat_zones[CW_MAX_CATALOG];
  int32_t small_first[CW_MAX_CATALOG];
  int32_t obj_count, obj_max, attempts;
  int32_t region;
  int32_t peds;
  int32_t spawn_region;   /* 1: Traverse strip columns (batch.py:174-177) */
  int32_t route_roadway;  /* cw_sample_routes: 1 = Walkable | Roadway (vehicle kinds, routes.py:52-55) */
  double route_max_radius; /* cw_sample_routes: separation radius (routes.py:62-63) */
} cw_scene_params;

/* Output rows (E envs, written at slots[e]) + scratch. */
typedef struct cw_scene_buffers {
  uint8_t* zones; uint8_t* labels; float* elev;
  int32_t* assign; int32_t* n_tiles; int8_t* tile_code; int8_t* tile_kind;
  double* tile_param; double* tile_p; double* tile_w; uint64_t* allowed;
  uint64_t* noise_seed; int32_t* wfc_attempts;
  int32_t* obj_cat; double* obj_pose; int32_t* obj_n; uint8_t* overflow;
  int32_t* nearest; uint8_t* has_obs;
  int32_t* walk; int32_t* walk_n;
  int32_t* reach;       /* (E, ny*nx) 4-connected component of passable cells, -1 = obstacle */
  uint8_t* moves;       /* (E, ny*nx) A* move table: bit d set iff move d (N S W E NW NE SW SE)
                           from the cell is legal (paths.py:70-72: in bounds, passable,
                           diagonals need both orthogonal cells passable) */
  double* sp_pos; double* sp_goal; int8_t* sp_kind; double* sp_pref;
  int32_t* status;
  int32_t* scratch_i32; /* (E, 10*ny*nx) */
  double* scratch_f64;  /* (E, max(obj_max*8, ny*nx)) */
  double* zone_params;  /* (E, CW_ZONE_PARAMS) ZoneMap.params (zones.py:69-122):
                           courtyard [blob_half x, y, extra_rects, trail, buildings],
                           blocks [sidewalk_width, road_width], strip [border_m] */
  uint8_t* block_var;   /* (E, CW_MAX_BLOCKS) block variant kind*4 + orientation of
                           connect_blocks (blocks.py:34-77), row-major; layout 1 only */
  const uint8_t* region; /* (E, ny*nx) optional route region mask (step.py:37 region_mask); NULL = none */
  int32_t* epoch;       /* (E) optional grid generation: +1 for every row a sampling call writes
                           (validates the crowd's next-tick search prefetch, cw_spec_create) */
} cw_scene_buffers;

size_t cw_scene_seed_scratch_bytes(int E);

int cw_sample_scenes(const cw_scene_params* params, int E, const uint64_t* scene_seeds,
                     const uint64_t* crowd_seeds, const int32_t* slots, void* seed_scratch,
                     const cw_scene_buffers* buffers, void* stream);

/* cw_sample_scenes + cw_route_anchors (below) as one pipeline: the route anchors read
 * only the labels, so they run on a side stream beside the nearest-obstacle BFS, walk
 * list and spawn.  Same outputs as the two calls in sequence. */
int cw_sample_scenes_routes(const cw_scene_params* params, int E, const uint64_t* scene_seeds,
                            const uint64_t* crowd_seeds, const int32_t* slots, void* seed_scratch,
                            const cw_scene_buffers* buffers, double* routes, int32_t* n_routes,
                            void* route_scratch, int chunk, void* stream);

/* Run-length coding of the sampled grids for scene_to_dict (urbangen/scene.py:163-178,
 * jsonio.rle_encode jsonio.py:42-54): rows rows[e] (NULL = e) of buffers->zones (ny*nx u8)
 * and buffers->assign (trows*tcols int32).  Count pass (offsets = pairs = NULL):
 * runs[2e] = zone runs, runs[2e+1] = assignment runs.  Fill pass: int32
 * [value, run, ...] lists at pairs + offsets[2e] (zones) and pairs + offsets[2e+1]
 * (assignment), offsets in int32 elements (2 per run). */
int cw_scene_rle(const cw_scene_params* params, int E, const int32_t* rows,
                 const cw_scene_buffers* buffers, int32_t* runs, const int64_t* offsets,
                 int32_t* pairs, void* stream);

/* Route anchors (urbangen/scene.py:102-178) for rows slots[e] of buffers->labels
 * (scene seeds as for cw_sample_scenes): routes (E, 8, 2, 2) float64
 * [[start x, y], [goal x, y]], n_routes (E); NoRouteAvailable in buffers->status.
 * scratch: cw_route_scratch_bytes(nx, ny, chunk) (chunk envs per launch). */
size_t cw_route_scratch_bytes(int nx, int ny, int chunk);
int cw_route_anchors(const cw_scene_params* params, int E, const uint64_t* scene_seeds,
                     const int32_t* slots, const cw_scene_buffers* buffers, double* routes,
                     int32_t* n_routes, void* scratch, int chunk, void* stream);

/* spawn_agents for caller-supplied labels (crowd/step.py:37-63): fills sp_* and
 * status of rows slots[e] from buffers->labels; seed_scratch as for sampling. */
int cw_spawn_agents(const cw_scene_params* params, int E, const uint64_t* crowd_seeds,
                    const int32_t* slots, void* seed_scratch, const cw_scene_buffers* buffers,
                    void* stream);

/* sample_routes(occupancy, count, seed, kind, region_mask, max_radius) (crowd/routes.py:35-87)
 * for rows slots[e] of buffers->labels: params->peds routes seeded PCG64(route_seeds[e]),
 * params->route_roadway / route_max_radius, optional buffers->region; starts in sp_pos,
 * goals in sp_goal, NoRouteAvailable in status.  spawn_agents(region_mask=) is
 * cw_spawn_agents with buffers->region set. */
int cw_sample_routes(const cw_scene_params* params, int E, const uint64_t* route_seeds,
                     const int32_t* slots, void* seed_scratch, const cw_scene_buffers* buffers,
                     void* stream);

/* connected_components (crowd/routes.py:14-32): 8-connected component ids numbered in
 * row-major order of first cell, -1 elsewhere; ok / comp / rank_scratch (E, ny*nx). */
int cw_connected_components(int nx, int ny, int E, const uint8_t* ok, int32_t* comp,
                            int32_t* rank_scratch, void* stream);

/* rasterize_occupancy(scene, resolution) (urbangen/occupancy.py:28-57) at params->res,
 * nx, ny: buffers->zones rows are (zone_ny, zone_nx) grids at zone_res; assign,
 * tile_code, tile_p, noise_seed, obj_cat, obj_pose, obj_n, status (zero) are inputs;
 * labels and elev ((ny, nx) rows) are written. */
int cw_rasterize(const cw_scene_params* params, int E, const int32_t* slots, int zone_nx,
                 int zone_ny, double zone_res, const cw_scene_buffers* buffers, void* stream);

/* Parity tooling: sin / cos of n doubles as the device computes them (mode 0: CUDA
 * sincos, 1: the correctly rounded cr_sincos of common.cuh). */
int cw_trig_probe(int n, const double* x, double* s, double* c, int mode, void* stream);

/* _prepare_env for caller-supplied labels (field.py:60-67): fills nearest,
 * has_obs, walk, walk_n, reach, moves of rows slots[e] from buffers->labels; needs status
 * (zeroed) and scratch_i32.  Only params->nx/ny are read. */
int cw_prepare_envs(const cw_scene_params* params, int E, const int32_t* slots,
                    const cw_scene_buffers* buffers, void* stream);

/* CrowdConfig + batch shape (crowd/types.py:60-79, field.py:29-58). */
typedef struct cw_crowd_params {
  int32_t E, A;
  int32_t nx, ny;
  double res, res0;
  double time_horizon, obstacle_time_horizon, neighbor_distance, nd2;
  float nd2_f32;
  int32_t max_neighbors;
  double dt, safety_margin, goal_reach2, stall_c, stall_s;
  int32_t resample_goals, use_static, path_cap;
  int32_t heap_cap;     /* A* far-pool entries (16 B) per search warp */
  int32_t astar_ctas;   /* persistent k_astar CTAs (one per SM) */
  int32_t astar_warps;  /* search warps per CTA: 1 = latency shape, else cw_astar_warps() */
  int32_t run_server_warps; /* cw_crowd_run search-server warps per CTA: 0 = 2, or 1 / 2 / 4 */
} cw_crowd_params;

/* Device-resident CrowdField state (field.py:47-58) + guidance/A* scratch. */
typedef struct cw_crowd_state {
  double* pos; double* vel; double* goal; double* waypoint;
  const double* radius; const double* pref_speed; const double* max_speed;
  const uint8_t* active;
  int32_t* path_cells; int32_t* path_head; int32_t* path_n;
  const uint8_t* labels; const int32_t* nearest; const uint8_t* has_obs;
  const int32_t* walk; const int32_t* walk_n;
  const int32_t* reach; const uint8_t* moves;
  void* rng;
  double* last_gap; double* gap_tmp; int32_t* flags;
  void* astar_rec;      /* astar_ctas * cw_astar_warps() x cw_astar_slot_bytes(nx, ny): all-global
                           g/move tiles, parent per cell, tile log (no initialisation needed) */
  void* astar_heap;     /* (astar_ctas * cw_astar_warps(), heap_cap, 16 B) A* far pools */
  void* astar_req;      /* (E*A, 16 B) replanning queue {env, agent, start, goal} */
  int64_t* counters;
  uint8_t* env_req;     /* (E) scratch: env queued a replan this tick (k_guide -> k_orca) */
  void* spec;           /* optional host handle from cw_spec_create: next-tick search prefetch
                           for cw_crowd_step (NULL = off; results are identical either way) */
  const int32_t* env_epoch; /* (E) grid generation of each env; required with `spec`: must change
                           whenever the env's labels / moves / reach change */
} cw_crowd_state;

size_t cw_crowd_step_smem_bytes(int A, int threads);

/* Next-tick search prefetch for cw_crowd_step (no reference counterpart: it changes no
 * result).  While a tick's longest A* searches run, the envs that already committed
 * predict their next tick's replans (the guidance pass, read-only) and search them on a
 * side stream into a per-agent cache; the next tick's k_astar takes a cached result
 * whose (start, goal, grid generation) equals its request, waits for one in flight,
 * and searches everything else as usual.  The context owns its device memory
 * (cw_spec_bytes); destroy synchronises the side streams before freeing it. */
size_t cw_spec_bytes(const cw_crowd_params* params);
int cw_spec_create(const cw_crowd_params* params, void** handle);
int cw_spec_destroy(void* handle);
/* counters: [0] batches launched, plus per-context device totals read back on demand:
 * [1] cache hits, [2] waits on a running prediction, [3] claims of a queued one */
int cw_spec_stats(void* handle, long long* out4);
/* Asynchronous scene sampling (envcore.SceneStandby): predict and search, into `handle`,
 * the first-tick replans of freshly spawned rows `rows` (state S as set_from_spawn leaves
 * it, grids of the standby batch); then, when those scenes are installed into another
 * batch, copy the finished predictions into that batch's context (generations remapped). */
int cw_spec_predict(const cw_crowd_params* params, const cw_crowd_state* state, void* handle,
                    const int32_t* rows, int n_rows, int threads, void* stream);
int cw_spec_install(void* dst, void* src, const int32_t* dst_epoch, const int32_t* src_epoch,
                    const int32_t* rows, int n_rows, void* stream);

int cw_crowd_step(const cw_crowd_params* params, const cw_crowd_state* state,
                  const double* robot_pos, const double* robot_vel, double robot_radius,
                  const uint8_t* env_mask, int threads, void* stream);

/* The same tick as cw_crowd_step, one phase at a time (bit 0 k_guide, bit 1
 * k_astar, bit 2 k_orca); running 1, 2, 4 in order equals one cw_crowd_step.
 * Lets a caller time each kernel with events on its stream.  phases == 7 (what
 * cw_crowd_step runs) overlaps the k_orca of envs without replans with k_astar on
 * two internal streams that are joined back into `stream` before returning. */
int cw_crowd_step_phases(const cw_crowd_params* params, const cw_crowd_state* state,
                         const double* robot_pos, const double* robot_vel, double robot_radius,
                         const uint8_t* env_mask, int threads, int phases, void* stream);

/* `ticks` consecutive cw_crowd_step calls with the same robot inputs and env mask,
 * run without a per-tick barrier: every env advances on its own (envs share no
 * state), its searches served by a persistent A* kernel through a device queue.
 * The final state is bit-identical to the synchronous ticks (last_gap included).
 * Blocks the calling host thread until the run is done (it polls the device to
 * stop launching rounds); device work is ordered after prior work on `stream`.
 * Correct with or without concurrent kernel execution.
 * scratch: cw_crowd_run_scratch_bytes(E, A, ticks) bytes of device memory.
 * Returns 0, a CUDA error, 9001 (device queue error) or 9002 (no env-tick completed for
 * 120 s: the host watchdog ended the run). */
size_t cw_crowd_run_scratch_bytes(int E, int A, int ticks);
/* One segment of a tick window [0, ticks): env e runs its ticks start_tick[e] ..
 * stop_tick[e] - 1 (NULL: 0 / ticks).  flags bit 0: first segment of the window
 * (resets the per-(env, tick) gap history kept in scratch), bit 1: last segment
 * (publishes last_gap_by_env from it).  Between segments the caller may replace
 * env state (e.g. re-sample the scenes of the envs stopped at a re-sampling
 * tick); per env the result equals the same ticks run synchronously.
 * cw_crowd_run == one segment with NULL, NULL, flags 3. */
int cw_crowd_run_window(const cw_crowd_params* params, const cw_crowd_state* state,
                        const double* robot_pos, const double* robot_vel, double robot_radius,
                        const uint8_t* env_mask, int threads, int ticks, const int32_t* start_tick,
                        const int32_t* stop_tick, int flags, void* scratch, void* stream);
/* Round kernels the last cw_crowd_run launched (host-only query; the run also
 * launches one init, one search-server and one finish kernel). */
long long cw_crowd_run_rounds(void);
/* Search-server launches of the last cw_crowd_run (host-only query): the server exits
 * when the run goes quiet and is relaunched when searches are queued, so it never
 * waits on kernels that cannot run beside it (serialised launches, profilers). */
long long cw_crowd_run_servers(void);
int cw_crowd_run(const cw_crowd_params* params, const cw_crowd_state* state,
                 const double* robot_pos, const double* robot_vel, double robot_radius,
                 const uint8_t* env_mask, int threads, int ticks, void* scratch, void* stream);

/* Search warps per k_astar CTA (host-only query). */
int cw_astar_warps(void);
/* Bytes of astar_rec per k_astar search warp for an nx x ny grid (host-only query). */
size_t cw_astar_slot_bytes(int nx, int ny);


/* ---------------------------------------------------------------- ORCA building blocks
 * The tick's pieces as standalone batched calls (device pointers, stream-ordered):
 *
 *   cw_orca_lp            replaces crowd/field.py:500 _batched_lp (and orca.py:130
 *                         solve_velocity as one row): points/normals (N, L, 2) f64,
 *                         valid (N, L) u8, pref (N, 2), max_speed (N), lane_active (N) u8
 *                         (NULL = all) -> out (N, 2); fell_back (N) i32 or NULL.  L <= 64.
 *   cw_orca_halfplanes    replaces field.py:448 _vo_halfplane / orca.py:23 orca_halfplane,
 *                         elementwise over n rows (horizon, share per row).
 *   cw_crowd_constraints  replaces field.py:214 _preferred_velocities + :229
 *                         _build_constraints for envs [e0, e1) of a crowd state: act
 *                         ((e1-e0), A) u8; outputs pref (rows, 2), points / normals
 *                         (rows, lmax, 2), valid (rows, lmax) u8 with lmax = kmax +
 *                         (robot_pos != NULL) + use_static (kmax = min(max_neighbors,
 *                         A-1)), inr (rows) in-range neighbour counts, gap (rows). */
int cw_orca_lp(int N, int L, const double* points, const double* normals, const uint8_t* valid,
               const double* pref, const double* max_speed, const uint8_t* lane_active, double* out,
               int32_t* fell_back, void* stream);
int cw_orca_halfplanes(int n, const double* rel_pos, const double* rel_vel, const double* combined_radius,
                       const double* horizon, double dt, const double* v_self, const double* share,
                       double* point, double* normal, void* stream);
int cw_crowd_constraints(const cw_crowd_params* params, const cw_crowd_state* state, int e0, int e1,
                         const uint8_t* act, const double* robot_pos, const double* robot_vel,
                         double robot_radius, int use_static, int lmax, double* pref, double* points,
                         double* normals, uint8_t* valid, int32_t* inr, double* gap, void* stream);

/* ---------------------------------------------------------------- robot */

/* Robot embodiment (envcore/robot.py:31-80). */
typedef struct cw_robot_model {
  double body_radius, max_speed;
  int32_t holonomic;   /* 1 holonomic velocity command, 0 Ackermann bicycle */
  double wheelbase, max_steer;
  double max_step_rise, max_grade, max_roughness;
} cw_robot_model;

/* EnvConfig + RewardConfig of a batch (envcore/batch.py:39-49, bench/reward.py:15-24). */
typedef struct cw_robot_params {
  int32_t E, A, nx, ny;
  double res, dt, reach_threshold;
  int32_t horizon;
  double terminal_reach, terminal_oob, c1, c2, c3;
  double track_far, track_near, track_near_weight;
  cw_robot_model model;
} cw_robot_params;

/* Device robot state of E envs (batch.py:98-110) + per-tick outputs. */
typedef struct cw_robot_state {
  double* x; double* y; double* yaw; double* vx; double* vy; double* elev;
  double* goal;                 /* (E, 2) */
  int64_t* tick; uint8_t* terminated; uint8_t* truncated;
  const uint8_t* labels;        /* (E, ny, nx) */
  const float* grid_elev;       /* (E, ny, nx) */
  const uint8_t* passable;      /* (E, ny, nx) from cw_traversability */
  const double* crowd_pos;      /* (E, A, 2) after the crowd step; NULL when A == 0 */
  const double* crowd_radius;   /* (E, A) */
  const uint8_t* crowd_active;  /* (E, A) */
  double* reward;               /* (E) */
  uint8_t* events;              /* (E, 6): collision, collision_static, collision_dynamic,
                                   on_walkable, reached, out_of_bounds */
  double* distance; double* path_inc;
  float* depth;                 /* (E, 128) ray-fan depth */
  double* goal_vector;          /* (E, 2) ego frame */
  double* proj_vel;             /* (E) */
  float* height_map;            /* (E, 16, 10) */
  uint8_t* semantics;           /* (E, 128) label of the cell each ray stopped in, 0 when it
                                   reached the cap or left the grid (observe.py:84-85,
                                   include_semantics); NULL = not written */
} cw_robot_state;

/* traversability_maps (robot.py:127-179): passable[e] for rows slots[e] (NULL =
 * identity) from labels / elevation; exact float64 emulation (column-then-row
 * cumulative sums of the edge-padded grid in the reference's order). */
size_t cw_traversability_scratch_bytes(int nx, int ny, int chunk);
int cw_traversability(const cw_robot_params* params, int E, const int32_t* slots,
                      const uint8_t* labels, const float* grid_elev, uint8_t* passable,
                      void* scratch, int chunk, void* stream);

/* Robot part of BatchedEnv.step_batch (batch.py:223-302) after the crowd step:
 * actions (E, 2) clipped to [-1, 1], integrate_motion, traversability gating,
 * crowd contact, elevation / walkable lookup, reward_batch, termination, then
 * observe_batch (observe.py:39-129) into the state's observation outputs. */
int cw_robot_step(const cw_robot_params* params, const cw_robot_state* state,
                  const double* actions, void* stream);

/* observe_batch only (reset / observe(i)). */
int cw_robot_observe(const cw_robot_params* params, const cw_robot_state* state, void* stream);

int cw_seed_streams(int n, const uint64_t* seeds, void* out_states, void* stream);

int cw_child_seeds(int n, const uint64_t* parent, int label_id, const uint64_t* k,
                   uint64_t* out, void* stream);

/* Host-only: sizeof of the four ABI structs (scene params/buffers, crowd params/state). */
int cw_abi_sizes(size_t* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* CITYWALK_B200_H */
