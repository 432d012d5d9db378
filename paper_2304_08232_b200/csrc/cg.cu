// cg.cu — preconditioned conjugate gradients (cg.hpp:77-142) driving the device kernels.
//
// The three scalars per iteration (rho, p'Ap, r'r) never leave the device in fixed-iteration
// runs: the dot kernels write them into ctx->d_scalars, the vector updates divide them on the
// device with IEEE division (bit-identical to the host's), and one CUDA graph per iteration is
// replayed without host synchronisation. The residual history and the breakdown test
// (cg.hpp:124-126) are evaluated on the host from the recorded scalars.
#include <algorithm>
#include <cmath>

#include "common.hpp"
#include "kernels.cuh"

namespace slabgpu {

	CgWorkspace::~CgWorkspace() {
		if( d_hist_rr ) cudaFree( d_hist_rr );
		if( d_hist_pq ) cudaFree( d_hist_pq );
		if( d_iter ) cudaFree( d_iter );
		if( iter_exec ) cudaGraphExecDestroy( iter_exec );
	}

	namespace {

		CgWorkspace * workspace( slab_level_s * H, uint64_t iterations ) {
			slab_ctx_s * ctx = H->ctx;
			if( !H->cg ) {
				H->cg.reset( new CgWorkspace );
				H->cg->r.reset( vec_new( ctx, H->n, 0.0 ) );
				H->cg->z.reset( vec_new( ctx, H->n, 0.0 ) );
				H->cg->p.reset( vec_new( ctx, H->n, 0.0 ) );
				H->cg->q.reset( vec_new( ctx, H->n, 0.0 ) );
				SLAB_CUDA( cudaMalloc( &H->cg->d_iter, sizeof( unsigned int ) ) );
			}
			CgWorkspace * ws = H->cg.get();
			if( iterations + 1 > ws->hist_cap ) {
				SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
				if( ws->d_hist_rr ) cudaFree( ws->d_hist_rr );
				if( ws->d_hist_pq ) cudaFree( ws->d_hist_pq );
				ws->d_hist_rr = ws->d_hist_pq = nullptr;
				ws->hist_cap = std::max< uint64_t >( iterations + 1, 64 );
				SLAB_CUDA( cudaMalloc( &ws->d_hist_rr, ws->hist_cap * sizeof( double ) ) );
				SLAB_CUDA( cudaMalloc( &ws->d_hist_pq, ws->hist_cap * sizeof( double ) ) );
				if( ws->iter_exec ) { // the graph holds the old history pointers
					cudaGraphExecDestroy( ws->iter_exec );
					ws->iter_exec = nullptr;
				}
			}
			return ws;
		}

		// one CG iteration, cg.hpp:110-132, enqueue only
		// deferred (fixed-iteration solves on a communicator): r'r of an iteration is not reduced where it is computed
		// but travels with the next iteration's r'z in one allreduce of two doubles — one collective less per iteration,
		// no change to any rank's arithmetic; the history entry of iteration k-1 is written inside iteration k
		// side_rr (fixed-iteration solves in exact-dot mode on one process): r'r is only needed for the history, and an exact
		// dot is a chain of dependent additions that leaves the GPU almost idle — so the r'r of the PREVIOUS iteration runs
		// on a side stream beside this iteration's V-cycle (both only read r) and is recorded one iteration late, like
		// the deferred reduction above
		// lazy_x (fixed-iteration solves on one process): nothing inside an iteration reads x, and p keeps its value until
		// the next p update — so cg.hpp:128 of iteration k-1 runs inside iteration k, on a low-priority stream that the
		// V-cycle forks after the finest level's pre-smoother: the pass (24 n bytes) streams under the coarse levels, which
		// are latency-bound and leave HBM idle. The r update leaves alpha in S_ALPHA; the last iteration's x update
		// follows the loop. Same operations on the same operands: x has the same bits.
		void iteration_enqueue( slab_level_s * H, CgWorkspace * ws, slab_vec_s * x, const slab_cg_config * cfg, bool deferred, bool side_rr,
			bool lazy_x, bool inline_record ) {
			slab_ctx_s * ctx = H->ctx;
			cudaStream_t st = ctx->stream;
			slab_vec_s * r = ws->r.get();
			slab_vec_s * z = ws->z.get();
			slab_vec_s * p = ws->p.get();
			slab_vec_s * q = ws->q.get();
			bool fused_rz = false;
			if( side_rr ) {
				SLAB_CUDA( cudaEventRecord( ctx->side_fork, st ) );
				SLAB_CUDA( cudaStreamWaitEvent( ctx->side_stream, ctx->side_fork, 0 ) );
				kern::dot_exact( ctx->side_stream, r->d, r->d, H->n, ctx->d_partials_side, ctx->d_counter + 1, ctx->d_scalars + S_RR );
				SLAB_CUDA( cudaEventRecord( ctx->side_join, ctx->side_stream ) );
			}
			const auto fork_x = [ ctx, st, x, p, ws, H ]() {
				SLAB_CUDA( cudaEventRecord( ctx->lazy_fork, st ) );
				SLAB_CUDA( cudaStreamWaitEvent( ctx->lazy_stream, ctx->lazy_fork, 0 ) );
				kern::cg_update_x( ctx->lazy_stream, x->d, p->d, ctx->d_scalars, ws->d_iter, H->n, ctx->sm_count );
				SLAB_CUDA( cudaEventRecord( ctx->lazy_join, ctx->lazy_stream ) );
			};
			ctx->after_presmooth = nullptr;
			if( lazy_x ) {
				ctx->after_presmooth = fork_x;
			}
			if( cfg->use_preconditioner ) {
				// cg.hpp:111: the V-cycle starts from z = 0. Levels that run the plane phases take that as a flag of their
				// first phase (nothing is read, every slab is zeros) instead of a pass that writes the zeros
				const bool hint = mg_vcycle_accepts_zero_guess( H );
				if( !hint ) {
					op_set_all( z, 0.0 );
				}
				// tree-dot mode: r'z (cg.hpp:116) rides on the last two plane phases of the V-cycle, which hold r_i and the
				// final z_i of every row in registers: one pass over r and z less
				fused_rz = hint && ctx->dot_mode == SLAB_DOT_TREE && g_fuse_rz != 0 && g_plane_rows != 2
					&& ( g_fuse_rz >= 2 || H->n >= ( uint64_t( 1 ) << 19 ) ); // below that the fold's own launch costs more than the dot
				mg_vcycle_enqueue( H, z, r, cfg->sweeps, false, hint, fused_rz );
			} else {
				op_waxpby( z, 1.0, r, 0.0, r ); // cg.hpp:114
			}
			if( lazy_x ) {
				if( ctx->after_presmooth ) { // no level took it (no preconditioner, a one-level hierarchy, unfused transfers)
					ctx->after_presmooth = nullptr;
					fork_x();
				}
			}
			if( fused_rz ) {
				kern::sum_partials( st, ctx->d_partials, mg_vcycle_rz_partials( H ), ctx->d_scalars + S_RHO );
			} else {
				op_dot_to_slot( r, z, S_RHO, !deferred );                             // cg.hpp:116
			}
			if( deferred ) {
				allreduce_slots( ctx, S_RHO, 2 ); // r'z of this iteration, r'r of the one before (0 in front of the first)
			}
			if( side_rr ) {
				SLAB_CUDA( cudaStreamWaitEvent( st, ctx->side_join, 0 ) ); // long done: the V-cycle is ten times the dot
			}
			if( lazy_x ) {
				SLAB_CUDA( cudaStreamWaitEvent( st, ctx->lazy_join, 0 ) ); // the pending x update read p
			}
			// inline bookkeeping (fixed-iteration solves on one process): the p update writes the previous iteration's
			// history entry, the r update bumps the iteration counter — no launch of its own for either; the last
			// entry follows the loop
			kern::cg_update_p( st, p->d, z->d, ctx->d_scalars, ws->d_iter, H->n, inline_record ? ws->d_hist_rr : nullptr,
				ws->d_hist_pq );                                                      // cg.hpp:117-121
			if( ( deferred || side_rr ) && !inline_record ) {
				kern::cg_record_deferred( st, ctx->d_scalars, ws->d_hist_rr, ws->d_hist_pq, ws->d_iter, false );
			}
			if( ctx->dot_mode == SLAB_DOT_TREE ) {
				// tree-dot mode: p'Ap rides on the product's epilogue and r'r on the x/r update — two
				// passes over the vectors and two launches fewer per iteration
				halo_exchange( H, p, -1 );
				if( H->A->plan == nullptr && kern::spmv_planes_usable( H->A->tile, static_cast< int64_t >( H->n ), ctx->sm_count ) ) {
					kern::spmv_planes( st, ctx->sm_count, H->A->tile, p->d, q->d, ctx->d_partials, ctx->d_scalars + S_PQ ); // cg.hpp:122-123
				} else {
					kern::spmv( st, H->A->sell, p->d, q->d,
						static_cast< int64_t >( H->n ), ctx->d_partials, ctx->d_counter, ctx->d_scalars + S_PQ ); // cg.hpp:122-123
				}
				allreduce_slot( ctx, S_PQ );
				kern::cg_update_xr_dot( st, lazy_x ? nullptr : x->d, r->d, p->d, q->d, ctx->d_scalars, H->n, ctx->sm_count, ctx->d_partials,
					ctx->d_counter, inline_record ? ws->d_iter : nullptr );           // cg.hpp:127-132
				if( !deferred ) {
					allreduce_slot( ctx, S_RR );
				}
			} else {
				op_mxv( q, nullptr, H->A.get(), p, SLAB_DESC_NONE );                  // cg.hpp:122
				op_dot_to_slot( p, q, S_PQ );                                         // cg.hpp:123
				kern::cg_update_xr( st, lazy_x ? nullptr : x->d, r->d, p->d, q->d, ctx->d_scalars, H->n, inline_record ? ws->d_iter : nullptr ); // cg.hpp:127-130
				if( !side_rr ) {
					op_dot_to_slot( r, r, S_RR, !deferred );                          // cg.hpp:132
				}
			}
			if( !deferred && !side_rr && !inline_record ) {
				kern::cg_record( st, ctx->d_scalars, ws->d_hist_rr, ws->d_hist_pq, ws->d_iter );
			}
		}

		void vcycle_stats_all( slab_level_s * L, uint64_t sweeps ) {
			for( ; L != nullptr; L = L->coarser.get() ) {
				if( L->coarser ) {
					L->stats.nnz_visited += 4 * sweeps * L->nnz + L->nnz + 2 * L->R->nnz;
				} else {
					L->stats.nnz_visited += 2 * sweeps * L->nnz;
				}
			}
		}

	} // namespace

	void cg_solve( slab_level_s * H, slab_vec_s * b, slab_vec_s * x0, const slab_cg_config * cfg, slab_vec_s * x,
		double * history, slab_cg_result * result ) {
		if( !( cfg->rtol > 0.0 ) ) { // cg.hpp:79-81
			fail( SLAB_ERR_INVALID_ARGUMENT, "CGConfig: rtol must be positive" );
		}
		if( cfg->max_iters < 1 ) { // cg.hpp:82-84
			fail( SLAB_ERR_INVALID_ARGUMENT, "CGConfig: max_iters must be at least 1" );
		}
		if( cfg->use_preconditioner && cfg->sweeps < 1 ) { // smoother.hpp:105-107, reached through mg_vcycle
			fail( SLAB_ERR_INVALID_ARGUMENT, "SmootherConfig: sweeps must be at least 1" );
		}
		const uint64_t n = H->n;
		if( b->n != n || x0->n != n || x->n != n ) { // cg.hpp:86-88
			fail( SLAB_ERR_DIMENSION_MISMATCH, "cg_solve: vector lengths differ from the system size" );
		}
		if( x == b || x->d == b->d ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "cg_solve: the solution vector must not alias b" );
		}
		slab_ctx_s * ctx = H->ctx;
		cudaStream_t st = ctx->stream;
		const bool fixed = cfg->has_fixed_iterations != 0;
		const uint64_t planned = fixed ? std::min( cfg->fixed_iterations, cfg->max_iters ) : cfg->max_iters;
		CgWorkspace * ws = workspace( H, planned );
		slab_vec_s * r = ws->r.get();

		SLAB_CUDA( cudaEventRecord( ctx->solve_start, st ) );
		if( x->d != x0->d ) { // out.solution = x0, cg.hpp:91
			SLAB_CUDA( cudaMemcpyAsync( x->d, x0->d, n * sizeof( double ), cudaMemcpyDeviceToDevice, st ) );
		}
		op_mxv( r, nullptr, H->A.get(), x, SLAB_DESC_NONE ); // cg.hpp:95
		op_waxpby( r, 1.0, b, -1.0, r );                     // cg.hpp:96
		op_dot_to_slot( b, b, S_BB );                        // cg.hpp:98
		op_dot_to_slot( r, r, S_RR );                        // cg.hpp:100
		SLAB_CUDA( cudaMemsetAsync( ws->d_iter, 0, sizeof( unsigned int ), st ) );
		ensure_pinned( ctx, 2 * ( planned + 1 ) + 2 );
		// the two initial norms land behind the history's staging area. A tolerance-driven solve needs them on the host
		// before its first iteration (cg.hpp:103); a fixed-iteration solve reads them with the history at the end, so
		// that nothing waits between the prologue and the iterations: the host enqueues the iteration graph while the
		// prologue (or, from host buffers, the upload) is still running
		double * const h_init = ctx->h_pinned + 2 * ( planned + 1 );
		SLAB_CUDA( cudaMemcpyAsync( h_init, ctx->d_scalars + S_RR, sizeof( double ), cudaMemcpyDeviceToHost, st ) );
		SLAB_CUDA( cudaMemcpyAsync( h_init + 1, ctx->d_scalars + S_BB, sizeof( double ), cudaMemcpyDeviceToHost, st ) );
		const bool early_sync = !fixed || halo_has_comm( ctx );
		double denom = 1.0, r_norm = 0.0;
		uint64_t count = 0;
		const auto take_initial_norms = [ & ]() {
			const double b_norm = std::sqrt( h_init[ 1 ] );
			denom = b_norm > 0.0 ? b_norm : 1.0;
			r_norm = std::sqrt( h_init[ 0 ] );
			history[ count++ ] = r_norm;
		};
		if( early_sync ) {
			SLAB_CUDA( cudaStreamSynchronize( st ) );
			take_initial_norms();
		}

		const bool already_converged = !fixed && r_norm / denom < cfg->rtol; // cg.hpp:103
		const uint64_t limit = already_converged ? 0 : planned;

		// on a communicator, fixed-iteration solves combine r'r with the next r'z (iteration_enqueue)
		const bool deferred = fixed && halo_has_comm( ctx );
		if( deferred && limit > 0 ) {
			SLAB_CUDA( cudaMemsetAsync( ctx->d_scalars + S_RR, 0, sizeof( double ), st ) ); // nothing to add in front of the first iteration
		}
		const bool side_rr = fixed && !deferred && ctx->dot_mode == SLAB_DOT_EXACT && g_side_rr != 0 && !ctx->profiling && limit > 0;
		if( side_rr ) { // scratch of the side stream's dot (never shared with the main stream's dots)
			const uint64_t need = ( n + kDotChunk - 1 ) / kDotChunk;
			if( need > ctx->partials_side_cap ) {
				SLAB_CUDA( cudaStreamSynchronize( st ) );
				SLAB_CUDA( cudaStreamSynchronize( ctx->side_stream ) );
				cudaFree( ctx->d_partials_side );
				ctx->d_partials_side = nullptr;
				SLAB_CUDA( cudaMalloc( &ctx->d_partials_side, std::max< uint64_t >( need, 1024 ) * sizeof( double ) ) );
				ctx->partials_side_cap = std::max< uint64_t >( need, 1024 );
				++ctx->scratch_gen;
			}
		}
		const bool inline_record = fixed && !deferred && !halo_has_comm( ctx ) && g_inline_record != 0 && limit > 0;
		const bool lazy_x = fixed && !halo_has_comm( ctx ) && g_lazy_x != 0 && !ctx->profiling && limit > 0
			&& ( g_lazy_x >= 2 || n >= ( uint64_t( 1 ) << 20 ) ); // below that the extra launch and the fork/join cost more than the pass
		// several iterations per graph launch (fixed-iteration solves on one process): the hand-over from one
		// iteration's last kernel to the next one's first is then a programmatic edge inside a graph instead of the gap
		// between two graph launches. The largest divisor of the iteration count up to the knob.
		uint64_t batch = 1;
		if( fixed && !halo_has_comm( ctx ) && g_iter_batch > 1 ) {
			for( uint64_t k = std::min< uint64_t >( limit, static_cast< uint64_t >( g_iter_batch ) ); k > 1; --k ) {
				if( limit % k == 0 ) {
					batch = k;
					break;
				}
			}
		}
		// iteration graph, cached per (x, config)
		bool graphs = ctx->use_graphs != 0 && !ctx->profiling; // timing instrumentation needs plain launches
		if( cfg->use_preconditioner && limit > 0 ) {
			mg_vcycle_prepare( H, ws->z.get(), ws->r.get(), cfg->sweeps ); // before any capture
		}
		// reduction scratch for every dot shape used below (allocation is illegal while capturing)
		ensure_partials( ctx, std::max< uint64_t >( std::max< uint64_t >( ( n + kDotChunk - 1 ) / kDotChunk,
			kern::dot_tree_blocks( n, ctx->sm_count ) ), std::max< uint64_t >( kern::spmv_dot_blocks( static_cast< int64_t >( n ) ), 4096 ) ) );
		if( graphs && limit > 0 ) {
			const bool stale = ws->iter_exec == nullptr || ws->key_x != x->d || ws->key_sweeps != cfg->sweeps
				|| ws->key_precond != cfg->use_preconditioner || ws->key_dot != ctx->dot_mode
				|| ws->key_fused != ctx->fused_transfers || ws->key_epoch != g_tuning_epoch
				|| ws->key_scratch != ctx->scratch_gen || ws->key_deferred != ( deferred ? 1 : 0 ) + ( side_rr ? 2 : 0 ) + ( lazy_x ? 4 : 0 ) + ( inline_record ? 8 : 0 ) || ws->key_batch != batch;
			if( stale ) {
				if( ws->iter_exec ) {
					cudaGraphExecDestroy( ws->iter_exec );
					ws->iter_exec = nullptr;
				}
				// reduction scratch must exist before capture (allocation is illegal while capturing)
				ensure_partials( ctx, std::max< uint64_t >( std::max< uint64_t >( ( n + kDotChunk - 1 ) / kDotChunk,
					kern::dot_tree_blocks( n, ctx->sm_count ) ), std::max< uint64_t >( kern::spmv_dot_blocks( static_cast< int64_t >( n ) ), 4096 ) ) );
				cudaGraph_t graph = nullptr;
				const uint64_t before = thread_launches();
				bool captured = false;
				try {
					SLAB_CUDA( cudaStreamBeginCapture( st, halo_has_comm( ctx ) ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal ) );
					try {
						for( uint64_t k = 0; k < batch; ++k ) {
							iteration_enqueue( H, ws, x, cfg, deferred, side_rr, lazy_x, inline_record );
						}
					} catch( ... ) {
						cudaStreamEndCapture( st, &graph );
						if( graph ) {
							cudaGraphDestroy( graph );
							graph = nullptr;
						}
						throw;
					}
					SLAB_CUDA( cudaStreamEndCapture( st, &graph ) );
					ws->iter_launches = thread_launches() - before;
					const cudaError_t err = cudaGraphInstantiate( &ws->iter_exec, graph,
						lazy_x && g_lazy_x_prio != 0 ? cudaGraphInstantiateFlagUseNodePriority : 0 ); // the x pass yields to the V-cycle
					cudaGraphDestroy( graph );
					SLAB_CUDA( err );
					captured = true;
				} catch( const Error & ) {
					// With a communicator attached the iteration contains NCCL operations on two streams; if
					// this driver/NCCL pair refuses to capture them, the same operations are enqueued launch by
					// launch instead — on EVERY rank: the ranks agree on that below.
					if( !halo_has_comm( ctx ) ) {
						throw;
					}
					cudaGetLastError();
					if( ws->iter_exec ) {
						cudaGraphExecDestroy( ws->iter_exec );
					}
					ws->iter_exec = nullptr;
					captured = false;
				}
				g_launch_count -= thread_launches() - before; // enqueued into the graph, not launched
				thread_launches() = before;
				if( halo_has_comm( ctx ) ) {
					// every rank must run the same mode (a graph replay and launch-by-launch enqueueing issue their
					// collectives from different streams' points of view): the ranks agree on the number of failures
					ensure_pinned( ctx, 1 );
					ctx->h_pinned[ 0 ] = captured ? 0.0 : 1.0;
					SLAB_CUDA( cudaMemcpyAsync( ctx->d_scalars + S_TMP, ctx->h_pinned, sizeof( double ), cudaMemcpyHostToDevice, st ) );
					allreduce_slot( ctx, S_TMP );
					if( read_scalar( ctx, S_TMP ) != 0.0 ) {
						if( ws->iter_exec ) {
							cudaGraphExecDestroy( ws->iter_exec );
							ws->iter_exec = nullptr;
						}
						captured = false;
						ctx->use_graphs = 0;
						graphs = false;
					}
				}
				if( captured ) {
					ws->key_x = x->d;
					ws->key_sweeps = cfg->sweeps;
					ws->key_precond = cfg->use_preconditioner;
					ws->key_dot = ctx->dot_mode;
					ws->key_fused = ctx->fused_transfers;
					ws->key_epoch = g_tuning_epoch;
					ws->key_scratch = ctx->scratch_gen;
					ws->key_deferred = ( deferred ? 1 : 0 ) + ( side_rr ? 2 : 0 ) + ( lazy_x ? 4 : 0 ) + ( inline_record ? 8 : 0 );
					ws->key_batch = batch;
				}
			}
		}

		// `count` iterations: the graph holds `batch` of them
		const auto run_iterations = [ & ]( uint64_t count ) {
			if( graphs ) {
				SLAB_CUDA( cudaGraphLaunch( ws->iter_exec, st ) );
				count_launch( ws->iter_launches );
			} else {
				for( uint64_t k = 0; k < count; ++k ) {
					iteration_enqueue( H, ws, x, cfg, deferred, side_rr, lazy_x, inline_record );
				}
			}
			if( cfg->use_preconditioner ) {
				for( uint64_t k = 0; k < count; ++k ) {
					vcycle_stats_all( H, cfg->sweeps );
				}
			}
		};

		int breakdown = 0;
		if( fixed ) {
			for( uint64_t iter = 0; iter < limit; iter += batch ) {
				run_iterations( batch );
			}
			if( deferred && limit > 0 ) { // the last iteration's r'r is still this rank's part
				allreduce_slot( ctx, S_RR );
				kern::cg_record_deferred( st, ctx->d_scalars, ws->d_hist_rr, ws->d_hist_pq, ws->d_iter, true );
			}
			if( side_rr ) { // the last iteration's r'r has not been taken yet
				op_dot_to_slot( ws->r.get(), ws->r.get(), S_RR );
			}
			if( side_rr || inline_record ) { // ... and its history entry has not been written
				kern::cg_record_deferred( st, ctx->d_scalars, ws->d_hist_rr, ws->d_hist_pq, ws->d_iter, true );
			}
			if( lazy_x ) { // the last iteration's x update is still pending (the iteration counter is past 0 here)
				kern::cg_update_x( st, x->d, ws->p->d, ctx->d_scalars, ws->d_iter, n, 0 );
			}
			if( limit > 0 ) {
				SLAB_CUDA( cudaMemcpyAsync( ctx->h_pinned, ws->d_hist_rr, limit * sizeof( double ), cudaMemcpyDeviceToHost,
					st ) );
				SLAB_CUDA( cudaMemcpyAsync( ctx->h_pinned + limit, ws->d_hist_pq, limit * sizeof( double ),
					cudaMemcpyDeviceToHost, st ) );
			}
			SLAB_CUDA( cudaEventRecord( ctx->solve_stop, st ) );
			SLAB_CUDA( cudaStreamSynchronize( st ) );
			if( !early_sync ) {
				take_initial_norms();
			}
			for( uint64_t k = 0; k < limit; ++k ) {
				if( ctx->h_pinned[ limit + k ] <= 0.0 ) { // cg.hpp:124-126
					breakdown = 1;
					break;
				}
				r_norm = std::sqrt( ctx->h_pinned[ k ] );
				history[ count++ ] = r_norm;
			}
		} else {
			for( uint64_t iter = 1; iter <= limit; ++iter ) {
				run_iterations( 1 );
				SLAB_CUDA( cudaMemcpyAsync( ctx->h_pinned, ctx->d_scalars + S_RR, sizeof( double ), cudaMemcpyDeviceToHost,
					st ) );
				SLAB_CUDA( cudaMemcpyAsync( ctx->h_pinned + 1, ctx->d_scalars + S_PQ, sizeof( double ),
					cudaMemcpyDeviceToHost, st ) );
				SLAB_CUDA( cudaStreamSynchronize( st ) );
				if( ctx->h_pinned[ 1 ] <= 0.0 ) {
					breakdown = 1;
					break;
				}
				r_norm = std::sqrt( ctx->h_pinned[ 0 ] );
				history[ count++ ] = r_norm;
				if( r_norm / denom < cfg->rtol ) { // cg.hpp:134-136
					break;
				}
			}
			SLAB_CUDA( cudaEventRecord( ctx->solve_stop, st ) );
			SLAB_CUDA( cudaStreamSynchronize( st ) );
		}
		float ms = 0.0f;
		SLAB_CUDA( cudaEventElapsedTime( &ms, ctx->solve_start, ctx->solve_stop ) );
		if( result ) {
			result->iterations = count - 1;
			result->converged = r_norm / denom < cfg->rtol ? 1 : 0;
			result->solve_ms = ms;
		}
		if( breakdown ) {
			fail( SLAB_ERR_SOLVER_BREAKDOWN, "cg_solve: p'Ap <= 0, operator is not SPD" );
		}
	}

	// cg_solve with host buffers: the staging vectors live in the workspace so that the iteration
	// graph (keyed by the solution vector) is captured once and replayed across calls.
	void cg_solve_host( slab_level_s * H, const double * b, const double * x0, const slab_cg_config * cfg, double * x,
		double * history, slab_cg_result * result ) {
		slab_ctx_s * ctx = H->ctx;
		const uint64_t n = H->n;
		CgWorkspace * ws = workspace( H, 1 );
		if( !ws->host_b ) {
			ws->host_b.reset( vec_new( ctx, n, 0.0 ) );
			ws->host_x.reset( vec_new( ctx, n, 0.0 ) );
		}
		if( n > 0 ) {
			SLAB_CUDA( cudaMemcpyAsync( ws->host_b->d, b, n * sizeof( double ), cudaMemcpyHostToDevice, ctx->stream ) );
			SLAB_CUDA( cudaMemcpyAsync( ws->host_x->d, x0, n * sizeof( double ), cudaMemcpyHostToDevice, ctx->stream ) );
		}
		cg_solve( H, ws->host_b.get(), ws->host_x.get(), cfg, ws->host_x.get(), history, result );
		if( n > 0 ) {
			SLAB_CUDA( cudaMemcpyAsync( x, ws->host_x->d, n * sizeof( double ), cudaMemcpyDeviceToHost, ctx->stream ) );
			SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
		}
	}

	// cg.hpp:59-67
	double residual_norm( slab_mat_s * A, slab_vec_s * x, slab_vec_s * b ) {
		if( A->nrows != b->n || A->ncols != x->n ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "residual_norm: operand sizes do not match the matrix" );
		}
		std::unique_ptr< slab_vec_s > r( vec_new( A->ctx, b->n, 0.0 ) );
		op_mxv( r.get(), nullptr, A, x, SLAB_DESC_NONE );
		op_waxpby( r.get(), 1.0, b, -1.0, r.get() );
		const double rr = op_dot( r.get(), r.get() );
		return std::sqrt( rr );
	}

} // namespace slabgpu
