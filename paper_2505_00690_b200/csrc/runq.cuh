// Multi-tick asynchronous run (cw_crowd_run): device queues and per-env state.
//
// Envs never read each other's state (SPEC: no cross-env sharing), so a run of
// T ticks needs no global barrier per tick.  Each env advances through
//   guide -> [its A* searches] -> ORCA + commit -> guide of the next tick ...
// on its own: short "round" kernels (one CTA per env) advance every env as far
// as it can go without waiting, and a persistent k_astar server drains a
// bounded MPMC ring of search requests concurrently on another stream.  An env
// whose tick needs searches parks in WAIT with a pending count; the server
// decrements it and the next round that sees zero resumes the env.  Per env the
// operations, their order and their inputs are exactly those of T synchronous
// cw_crowd_step calls, so the final state is bit-identical; the only
// cross-env quantity, last_gap_by_env (field.py:268-271: published on ticks
// where any env had a neighbour), is rebuilt from a per-(env, tick) history.
#pragma once

namespace cw {

enum { kRunGuide = 0, kRunWait = 1, kRunDone = 3, kRunBusy = 1 << 30 };
constexpr int kPendingGuard = 1 << 24;   // > any per-env request count
constexpr long long kSpinCycles = 8ll << 30;    // ~4.5 s: a full ring slot is an error, not a hang
constexpr long long kIdleCycles = 64ll << 30;   // ~35 s backstop for a server warp that saw no
                                                // env-tick complete anywhere for that long (the
                                                // host normally ends the run via q->shutdown)
constexpr long long kGraceCycles = 1ll << 19;   // ~0.27 ms: a server warp with an empty ring and
                                                // no resident round CTA for this long exits (the
                                                // host relaunches the server when searches queue)

struct RunQueue {                 // device-resident control words
  unsigned long long head, tail;  // search ring positions claimed by consumers / producers
  int n_done, shutdown, error, progress;   // progress: env-ticks completed (wraps; host watchdog)
  int active_rounds;              // round CTAs currently resident (the server's exit test)
  int pad_;
  unsigned long long rhead, rtail;  // ready-env ring (start, yields)
  unsigned long long uhead, utail;  // urgent ring: envs the server released (their chain waits)
};

struct RunArgs {                  // kernel parameter (pointers into cw_crowd_run scratch)
  RunQueue* q;
  int* env_state;                 // tick << 2 | phase
  int* pending;                   // outstanding searches of the env's current tick
  unsigned long long* seq;        // ring slot sequence numbers (Vyukov bounded MPMC)
  AstarReq* items;
  unsigned long long* rseq;       // ready-env ring (each env is in it at most once)
  int* ritems;
  unsigned long long* useq;       // urgent ring, same capacity
  int* uitems;
  unsigned long long rmask;
  double* gap_hist;               // (E, T) per-tick gap of every env
  int* anynb;                     // (T) some env had K > 0 at tick t
  int T, E;                       // T: length of the tick window (history), E: envs
  const int* start;               // per env first tick of this call (nullptr: 0)
  const int* stop;                // per env tick to stop at, exclusive (nullptr: T)
  int init_hist;                  // reset the (env, tick) gap history (first call of a window)
  int burst;                      // ticks one round CTA may run back to back (bounds round length)
  unsigned long long mask;        // ring capacity - 1 (power of two)
  long long* trace;               // debug (CW_RUN_TRACE): per env 8 x i64, see kTr*
};

// debug trace slots per env (ns from %globaltimer)
enum { kTrMark = 0, kTrBusy, kTrSearchWait, kTrQueueWait, kTrWaits, kTrDone, kTrTicksBusy, kTrPad };
CW_DEV long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}



CW_DEV unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
CW_DEV void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
CW_DEV void st_release_i32(int* p, int v) {
  asm volatile("st.release.gpu.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
CW_DEV int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// producer (one thread): blocks only while the slot's previous item is unread
CW_DEV void ring_push(const RunArgs& ra, const AstarReq& R) {
  const unsigned long long pos = atomicAdd(&ra.q->tail, 1ull);
  unsigned long long* sq = ra.seq + (pos & ra.mask);
  const long long t0 = clock64();
  while (ld_acquire_u64(sq) != pos) {
    if (clock64() - t0 > kSpinCycles) { atomicCAS(&ra.q->error, 0, 1); return; }
  }
  ra.items[pos & ra.mask] = R;
  st_release_u64(sq, pos + 1);
}

// ready ring: push (blocking, never full: capacity >= E) / non-blocking pop
CW_DEV void env_push(const RunArgs& ra, unsigned long long* tail, unsigned long long* seq, int* items,
                     int e) {
  const unsigned long long pos = atomicAdd(tail, 1ull);
  unsigned long long* sq = seq + (pos & ra.rmask);
  const long long t0 = clock64();
  while (ld_acquire_u64(sq) != pos) {
    if (clock64() - t0 > kSpinCycles) { atomicCAS(&ra.q->error, 0, 3); return; }
  }
  items[pos & ra.rmask] = e;
  st_release_u64(sq, pos + 1);
}

CW_DEV int env_pop(const RunArgs& ra, unsigned long long* head, unsigned long long* seq, int* items) {
  unsigned long long pos = *(volatile unsigned long long*)head;   // -1: empty right now
  while (true) {
    unsigned long long* sq = seq + (pos & ra.rmask);
    const long long dif = (long long)(ld_acquire_u64(sq) - (pos + 1));
    if (dif == 0) {
      const unsigned long long old = atomicCAS(head, pos, pos + 1);
      if (old == pos) {
        const int e = *(volatile int*)&items[pos & ra.rmask];
        st_release_u64(sq, pos + ra.rmask + 1);
        return e;
      }
      pos = old;
    } else if (dif < 0) {
      return -1;
    } else {
      pos = *(volatile unsigned long long*)head;
    }
  }
}

CW_DEV void ready_push(const RunArgs& ra, int e) { env_push(ra, &ra.q->rtail, ra.rseq, ra.ritems, e); }
CW_DEV void urgent_push(const RunArgs& ra, int e) { env_push(ra, &ra.q->utail, ra.useq, ra.uitems, e); }
// urgent envs first: their searches are done and their chain is the run's critical path
CW_DEV int ready_pop(const RunArgs& ra) {
  const int e = env_pop(ra, &ra.q->uhead, ra.useq, ra.uitems);
  return e >= 0 ? e : env_pop(ra, &ra.q->rhead, ra.rseq, ra.ritems);
}

// consumer (lane 0 of a server warp): false on shutdown / error, or when the run
// has gone quiet -- the ring empty and no round CTA resident for kGraceCycles.
// A position is claimed only once its item is there (Vyukov try-pop), so a warp
// that leaves never strands a request.  The server therefore never waits on
// kernels that cannot run beside it: when launches are serialised (e.g. under a
// profiler) the server drains the queue and exits, the host launches the rounds
// queued behind it and relaunches the server when searches are queued again.
CW_DEV bool ring_pop(const RunArgs& ra, AstarReq& R) {
  long long t0 = clock64(), tq = t0;
  int seen = *(volatile int*)&ra.q->progress;
  unsigned long long pos = *(volatile unsigned long long*)&ra.q->head;
  while (true) {
    unsigned long long* sq = ra.seq + (pos & ra.mask);
    const long long dif = (long long)(ld_acquire_u64(sq) - (pos + 1));
    if (dif == 0) {
      const unsigned long long old = atomicCAS(&ra.q->head, pos, pos + 1);
      if (old == pos) {
        R = ra.items[pos & ra.mask];
        st_release_u64(sq, pos + ra.mask + 1);
        return true;
      }
      pos = old;
      continue;
    }
    if (dif > 0) {   // another consumer took it
      pos = *(volatile unsigned long long*)&ra.q->head;
      continue;
    }
    if (*(volatile int*)&ra.q->shutdown) return false;
    const long long now = clock64();
    const int prog = *(volatile int*)&ra.q->progress;
    if (prog != seen) { seen = prog; t0 = now; }
    if (now - t0 > kIdleCycles) { atomicCAS(&ra.q->error, 0, 2); return false; }
    if (*(volatile int*)&ra.q->active_rounds > 0) tq = now;
    else if (now - tq > kGraceCycles) return false;
    __nanosleep(64);
    pos = *(volatile unsigned long long*)&ra.q->head;
  }
}

}  // namespace cw
